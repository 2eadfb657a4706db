// Instantiates the compile-time-pruned retain-r kernels for r = 33..48.
#include "adct_launch.h"

namespace adct {

#define ADCT_RK(R) &k_retain<R, true>
RetainKernel retain_kernel_q2(int r) {
  static const RetainKernel table[16] = {
      ADCT_RK(33),
      ADCT_RK(34),
      ADCT_RK(35),
      ADCT_RK(36),
      ADCT_RK(37),
      ADCT_RK(38),
      ADCT_RK(39),
      ADCT_RK(40),
      ADCT_RK(41),
      ADCT_RK(42),
      ADCT_RK(43),
      ADCT_RK(44),
      ADCT_RK(45),
      ADCT_RK(46),
      ADCT_RK(47),
      ADCT_RK(48),
  };
  return table[r - 33];
}
#undef ADCT_RK

}  // namespace adct
