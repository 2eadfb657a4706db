// Instantiates the compile-time-pruned retain-r kernels for r = 17..32.
#include "adct_launch.h"

namespace adct {

#define ADCT_RK(R) &k_retain<R, true>
RetainKernel retain_kernel_q1(int r) {
  static const RetainKernel table[16] = {
      ADCT_RK(17),
      ADCT_RK(18),
      ADCT_RK(19),
      ADCT_RK(20),
      ADCT_RK(21),
      ADCT_RK(22),
      ADCT_RK(23),
      ADCT_RK(24),
      ADCT_RK(25),
      ADCT_RK(26),
      ADCT_RK(27),
      ADCT_RK(28),
      ADCT_RK(29),
      ADCT_RK(30),
      ADCT_RK(31),
      ADCT_RK(32),
  };
  return table[r - 17];
}
#undef ADCT_RK

}  // namespace adct
