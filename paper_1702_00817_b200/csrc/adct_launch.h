// adct_launch.h — internal host-side interface between the C ABI (capi.cu)
// and the template instantiation units (k_retain_tab*.cu).
#pragma once

#include "adct_kernels.cuh"

namespace adct {

typedef void (*RetainKernel)(PlaneSetDev, u64*);

// Pruned retain-r kernels (two blocks per thread), r in [16q+1, 16q+16].
RetainKernel retain_kernel_q0(int r);
RetainKernel retain_kernel_q1(int r);
RetainKernel retain_kernel_q2(int r);
RetainKernel retain_kernel_q3(int r);

inline RetainKernel retain_kernel(int r) {
  if (r <= 16) return retain_kernel_q0(r);
  if (r <= 32) return retain_kernel_q1(r);
  if (r <= 48) return retain_kernel_q2(r);
  return retain_kernel_q3(r);
}

}  // namespace adct
