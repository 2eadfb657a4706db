// Copy-bandwidth probe: (a) 16-byte ld.global.nc / st.global.cs per thread (the
// retain kernel's access style), (b) TMA bulk copies global->smem->global with
// an mbarrier, one 16 KiB chunk per stage, persistent CTAs, (c) cudaMemcpy D2D.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_vec(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n16) {
  size_t i = (size_t)blockIdx.x * blockDim.x * 8 + threadIdx.x;
  uint4 v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    size_t j = i + (size_t)k * blockDim.x;
    if (j < n16) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                              : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(in + j));
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    size_t j = i + (size_t)k * blockDim.x;
    if (j < n16) asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(out + j), "r"(v[k].x), "r"(v[k].y), "r"(v[k].z), "r"(v[k].w) : "memory");
  }
}

constexpr int CHUNK = 16384, STAGES = 4;
__global__ void __launch_bounds__(32) k_tma(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, size_t nchunks) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(a));
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase[STAGES] = {0, 0, 0, 0};
  size_t c0 = blockIdx.x;
  // prologue: issue STAGES loads
  for (int s = 0; s < STAGES; ++s) {
    size_t c = c0 + (size_t)s * gridDim.x;
    if (c >= nchunks) break;
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    uint32_t d = (uint32_t)__cvta_generic_to_shared(sm + s * CHUNK);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(a), "r"(CHUNK));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(d), "l"(in + c * CHUNK), "r"(CHUNK), "r"(a) : "memory");
  }
  for (size_t it = 0;; ++it) {
    int s = (int)(it % STAGES);
    size_t c = c0 + it * gridDim.x;
    if (c >= nchunks) break;
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    uint32_t d = (uint32_t)__cvta_generic_to_shared(sm + s * CHUNK);
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(a), "r"(phase[s]));
    phase[s] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(out + c * CHUNK), "r"(d), "r"(CHUNK) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // before refilling this stage, its store must have read the smem
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    size_t cn = c + (size_t)STAGES * gridDim.x;
    if (cn < nchunks) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(a), "r"(CHUNK));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(d), "l"(in + cn * CHUNK), "r"(CHUNK), "r"(a) : "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t bytes = (size_t)8 << 30;  // 8 GiB each way
  uint8_t *a, *b;
  cudaMalloc(&a, bytes); cudaMalloc(&b, bytes);
  cudaMemset(a, 1, bytes); cudaMemset(b, 0, bytes);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto time = [&](auto f, const char* name) {
    f(); cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("%-28s %8.3f ms  %7.1f GB/s  %s\n", name, best, 2.0 * bytes / best / 1e6, cudaGetErrorString(err));
  };
  size_t n16 = bytes / 16;
  time([&] { k_vec<<<(unsigned)((n16 + 128 * 8 - 1) / (128 * 8)), 128>>>((const uint4*)a, (uint4*)b, n16); }, "vec16 ld.nc/st.cs");
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * CHUNK);
  for (int per : {2, 4, 6}) {
    char nm[64]; snprintf(nm, 64, "tma bulk %dKiB x%d, %d/SM", CHUNK / 1024, STAGES, per);
    time([&] { k_tma<<<sms * per, 32, STAGES * CHUNK>>>(a, b, bytes / CHUNK); }, nm);
  }
  time([&] { cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice); }, "cudaMemcpy D2D");
  // correctness of the tma copy
  uint8_t h = 0; cudaMemset(b, 0, bytes);
  k_tma<<<sms * 4, 32, STAGES * CHUNK>>>(a, b, bytes / CHUNK); cudaDeviceSynchronize();
  cudaMemcpy(&h, b + bytes - 1, 1, cudaMemcpyDeviceToHost);
  printf("tma last byte = %d (want 1)\n", h);
  return 0;
}
