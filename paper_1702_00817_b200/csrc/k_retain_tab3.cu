// Instantiates the compile-time-pruned retain-r kernels for r = 49..64.
#include "adct_launch.h"

namespace adct {

#define ADCT_RK(R) &k_retain<R, true>
RetainKernel retain_kernel_q3(int r) {
  static const RetainKernel table[16] = {
      ADCT_RK(49),
      ADCT_RK(50),
      ADCT_RK(51),
      ADCT_RK(52),
      ADCT_RK(53),
      ADCT_RK(54),
      ADCT_RK(55),
      ADCT_RK(56),
      ADCT_RK(57),
      ADCT_RK(58),
      ADCT_RK(59),
      ADCT_RK(60),
      ADCT_RK(61),
      ADCT_RK(62),
      ADCT_RK(63),
      ADCT_RK(64),
  };
  return table[r - 49];
}
#undef ADCT_RK

}  // namespace adct
