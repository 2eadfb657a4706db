// adct_jit.h — host-side interface of quant_jit.cu (run-time specialisation of
// the quantised kernels for one quantiser table; internal, not part of the C ABI).
#pragma once

#include "adct_kernels.cuh"

namespace adct {
namespace jit {

enum Kind { kQuantPairAligned = 0, kQuantPairFlip = 1, kQuantSingleAligned = 2, kQuantSingleFlip = 3, kHybrid = 4,
            kFloatOffset = 5,  // + kind: the float-quantiser (QF) variant
            kHybridF = kHybrid + kFloatOffset };

// The specialised kernel for (kind, table) once the table has been used often
// enough and compiled; nullptr while the generic kernel should run.
void* quant_function(int kind, const QParamsDev& q, cudaStream_t stream);
// cuLaunchKernel on `fn` with the same parameters as the generic kernel; the CUresult (0 on success).
int launch(void* fn, dim3 grid, dim3 block, size_t smem, cudaStream_t stream, void** args);
void stats(long long* compiled, long long* launches, long long* failures);

}  // namespace jit
}  // namespace adct
