// Instantiates the compile-time-pruned retain-r kernels for r = 1..16.
#include "adct_launch.h"

namespace adct {

#define ADCT_RK(R) &k_retain<R, true>
RetainKernel retain_kernel_q0(int r) {
  static const RetainKernel table[16] = {
      ADCT_RK(1),
      ADCT_RK(2),
      ADCT_RK(3),
      ADCT_RK(4),
      ADCT_RK(5),
      ADCT_RK(6),
      ADCT_RK(7),
      ADCT_RK(8),
      ADCT_RK(9),
      ADCT_RK(10),
      ADCT_RK(11),
      ADCT_RK(12),
      ADCT_RK(13),
      ADCT_RK(14),
      ADCT_RK(15),
      ADCT_RK(16),
  };
  return table[r - 1];
}
#undef ADCT_RK

}  // namespace adct
