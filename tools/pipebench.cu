// Pipe throughput microbenchmark: ops per SMSP per clock for integer/fp mixes on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define N_ITER 4096
typedef unsigned long long u64;

template <int MODE>
__global__ void __launch_bounds__(256) kb(unsigned* out, unsigned seed, float fr, long long* cyc) {
  long long c0 = clock64();
  unsigned a[8]; u64 f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = seed * (threadIdx.x + i); f[i] = ((u64)__float_as_uint(fr * i) << 32) | __float_as_uint(fr + i); }
  u64 rr = ((u64)__float_as_uint(fr) << 32) | __float_as_uint(fr);
#pragma unroll 1
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) { asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(a[(i+3)&7])); }                 // IADD
      if (MODE == 1) { asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(a[(i+5)&7]), "r"(seed)); } // IMAD
      if (MODE == 2) { asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(f[i]) : "l"(rr)); }         // FFMA2
      if (MODE == 3) { asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(f[i]) : "l"(rr)); }             // FADD2
      if (MODE == 4) { asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+r"(a[i]) : "r"(seed)); }          // FFMA reg
      if (MODE == 5) { // IADD + FFMA2 alternating
        if (i & 1) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(a[(i+3)&7]));
        else asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(f[i]) : "l"(rr)); }
      if (MODE == 6) { // IMAD + FFMA2 alternating
        if (i & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(a[(i+5)&7]), "r"(seed));
        else asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(f[i]) : "l"(rr)); }
      if (MODE == 7) { // IADD + IMAD alternating
        if (i & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(a[(i+5)&7]), "r"(seed));
        else asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(a[(i+3)&7])); }
      if (MODE == 8) { // IADD, IMAD, FFMA2 in thirds (i%3)
        if (i % 3 == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(a[(i+5)&7]), "r"(seed));
        else if (i % 3 == 1) asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(a[(i+3)&7]));
        else asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(f[i]) : "l"(rr)); }
      if (MODE == 9) { // PRMT
        asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(a[i]) : "r"(a[(i+3)&7])); }
      if (MODE == 10) { // mul.hi
        asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(a[(i+3)&7])); }
      if (MODE == 11) { // FFMA2 + FADD2 alt
        if (i & 1) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(f[i]) : "l"(rr));
        else asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(f[i]) : "l"(rr)); }
      if (MODE == 12) { // IADD IADD IMAD FFMA2 (quarters)
        if (i % 4 == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(a[(i+5)&7]), "r"(seed));
        else if (i % 4 == 3) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(f[i]) : "l"(rr));
        else asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(a[(i+3)&7])); }
    }
  }
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] + (unsigned)f[i] + (unsigned)(f[i] >> 32);
  out[blockIdx.x * 256 + threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - c0;
}

template <int MODE>
void run(const char* name, unsigned* d, int sms) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * 8;  // 8 x 256 threads per SM = 64 warps
  static long long* cyc = nullptr; if (!cyc) cudaMallocManaged(&cyc, blocks * 8);
  kb<MODE><<<blocks, 256>>>(d, 3, 1.0001f, cyc);
  cudaEventRecord(e0);
  kb<MODE><<<blocks, 256>>>(d, 3, 1.0001f, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double warp_insts = (double)blocks * 8 * N_ITER * 8;  // per SM: blocks/sms*8 warps
  double per_smsp_clk = warp_insts / (sms * 4) / (ms * 1e-3 * clk * 1e3);
  cudaDeviceSynchronize(); double mc = 0; for (int b = 0; b < blocks; ++b) mc += cyc[b]; mc /= blocks;
  // each SMSP runs 16 warps x N_ITER x 8 instructions (all blocks resident at once)
  double ipc = 16.0 * N_ITER * 8 / mc;
  printf("%-28s %8.3f ms  eff clk %.0f MHz  warp-inst/SMSP/cycle = %.3f\n", name, ms, mc / (ms * 1e3), ipc);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* d; cudaMalloc(&d, sms * 8 * 256 * 4);
  run<0>("IADD", d, sms); run<1>("IMAD", d, sms); run<2>("FFMA2", d, sms); run<3>("FADD2", d, sms);
  run<4>("FFMA(reg)", d, sms); run<5>("IADD+FFMA2", d, sms); run<6>("IMAD+FFMA2", d, sms);
  run<7>("IADD+IMAD", d, sms); run<8>("IMAD+IADD+FFMA2", d, sms); run<9>("PRMT", d, sms);
  run<10>("IMAD.HI", d, sms); run<11>("FFMA2+FADD2", d, sms); run<12>("2IADD+IMAD+FFMA2", d, sms);
  return 0;
}
