// adct_kernels.cuh — sm_100a kernels of the approximate-DCT hot path.
// See adct_device.cuh for the arithmetic model and DESIGN.md for rooflines.
//
//   K2  k_retain<R,PAIR>      compress_image + mse, r pruned at compile time
//                             (reference codec.py:144-155, metrics.py:49-56)
//   K2' k_retain_rt<PAIR,F>   same, runtime r; optional unrounded SSE
//   K3  k_quant_p / k_quant   quantised pipeline, two blocks per thread
//                             (forward_2d_unscaled + folded Q' + inverse_2d,
//                             codec.py:74-104)
//   K3" k_quant_hybrid        coarse tables: packed forward/quantiser, 32-bit inverse
//   K3' k_quant_wide          remaining coarse tables, one block per thread
//   K7  k_sweep_inc / k_sweep SSE for every r from one read (cli.py:101-113)
//   K1  k_forward<PAIR,T>     T X T^T coefficients in _tile order (codec.py:74-81,107-131)
//   f64 / dense kernels       real-valued and non-proposed transforms (codec.py:68-71,84-87;
//                             kernels.py:166-178)
//   k_synth                   BASELINE's blob generator (input only, never timed)
#pragma once

#include "adct_device.cuh"

namespace adct {

// ---------------------------------------------------------------------------
// Quantiser constants in kernel-parameter (constant bank) space, 1280 bytes.
// Filled from adct_qtab_t by the host (capi.cu).
// ---------------------------------------------------------------------------
struct QParamsDev {
  // One 16-byte record per coefficient position: sm_100 ptxas stages every
  // kernel-parameter operand through LDC/LDCU, and records load as LDC.64
  // pairs (the SoA layout cost 5 loads per position; measured 2.6 % slower).
  uint4 pos[64];  // x: magic (umulhi(U, magic) == floor(U / divisor), verified exhaustively)
                  // y: mult  (2: odd Q', divisor 2Q'; 1: even Q', divisor Q')
                  // z: bm    (bias times mult, both lanes: B * mult * 65537)
                  // w: qe    (Q' * E[u][v])
  u32 wadd[64];   // -kq*qe*65537 (+ (O+32)*65537 at DC: rounding, output offset)
};

struct QParamsWide {  // scalar quantiser of k_quant_wide
  uint4 pos[64];  // x: magic, y: cadd, z: qe, w: wadd = -kw*qe (+ 32 + 8192 at DC)
};

// Quantise + dequantise one coefficient position of both blocks, returning
// W = E o (q Q') in linear form.  z = T(X-128)T^T in linear form (lanes
// |Z| <= 8192).  Lane signs are bits 15 and 31 of z: bit 15 is exactly the
// sign of lane A; bit 31 is the sign of lane B minus A's borrow, which only
// errs when Z_B == 0, where both tie-breaks give q = 0 (host-verified).
//   U = (Z + B) * mult + [Z >= 0]   (both 16-bit fields, no carry)
//   q + kq = umulhi(U, magic)       (exact, adct_qtab_build)
// Where the quantiser constants come from: the kernel parameters (any
// table), or — in kernels specialised at run time for one table (capi.cu,
// NVRTC) — compile-time constants that become instruction immediates
// (removes the 2 LDC.64 + 1 LDCU per position: +5.5 % on config 4).
struct ParamTab {
  static constexpr bool kBaked = false;  // constants unknown at compile time
  static __device__ __forceinline__ uint4 pos(const QParamsDev& q, int p) { return q.pos[p]; }
  static __device__ __forceinline__ u32 wadd(const QParamsDev& q, int p) { return q.wadd[p]; }
};

template <class TAB = ParamTab>
__device__ __forceinline__ u32 quant_pair(u32 z, int p, const QParamsDev& q) {
  const uint4 c = TAB::pos(q, p);
  // mult == 2 <=> odd Q': no ties, so the sign term never matters (the host
  // check verifies both values); a specialised kernel drops it there
  const u32 s = (TAB::kBaked && c.y == 2u) ? 0u : ((z >> 15) & 0x10001u) ^ 0x10001u;
  const u32 U = z * c.y + c.z + s;
  const u32 qa = __umulhi(U & 0xFFFFu, c.x);
  const u32 qb = __umulhi(U >> 16, c.x);
  return (qa + (qb << 16)) * c.w + TAB::wadd(q, p);
}

// Float quantiser (QF kernels): both lanes at once on the FP32x2 pipe.
// `zb` is the linear form biased by 0x80008000, i.e. two unsigned 16-bit
// fields Z + 32768 (|Z| <= 8192, no borrow).  PRMT places each field under
// the exponent of 2^23, so the two floats are 2^23 + 32768 + Z exactly; one
// FADD2 removes the offset (exact), one FFMA2 computes RN(M + Z r) with r the
// float just above 1/Q' chosen by adct_qtab_build: r - 1/Q' < 1/(2 Q' 8192)
// pushes exact ties away from zero and never moves a non-tie across a
// rounding boundary, so the result is M + round_half_away(Z/Q') (verified
// exhaustively over |Z| <= 8192 per position by the host).  M is an even
// integer in [2^23 + 8192, 2^24 - 8192], where the float grid is the
// integers, so the result's bits are bits(M) + q.
// Lane magics: M_A = 1.5 * 2^23 (bits 0x4B400000) and M_B = M_A + 0xB4C0
// (bits 0x4B40B4C0).  Packing the lanes as qa + (qb << 16) then gives
//   0x4B400000 + qA + ((0xB4C0 + qB) << 16) = 2^32 + qA + (qB << 16),
// i.e. exactly the linear form of (qA, qB) mod 2^32: the dequantising IMAD
// needs no additive constant (no per-position constant register).  This
// replaces the SHF/LOP3 sign logic, the lane split and two IMAD.HI per
// position of the integer quantiser (quant_pair below).
constexpr u32 kQfMagicA = 0x4B400000u;   // 12582912.0f
constexpr u32 kQfMagicB = 0x4B40B4C0u;   // 12629184.0f
constexpr unsigned long long kQfOffset = 0x4B0080004B008000ull;  // (2^23 + 32768) in both halves
constexpr u32 kQfBias = 0x80008000u;                      // +32768 in both 16-bit fields

// The lane magics as run-time values (`small` is a kernel parameter < 256, so
// the adds are 0): ptxas cannot fold them, keeps the pair in two registers
// and gives FFMA2's immediate slot to r (else every position's r costs a MOV).
// SAME_LANES: both lanes use M_A (the hybrid kernel dequantises each lane on
// its own, with the 0x4B400000 * qe offset folded into its scalar wadd).
template <bool SAME_LANES = false>
__device__ __forceinline__ unsigned long long qf_magic(int32_t small) {
  const u32 a = kQfMagicA + ((u32)small >> 8);
  const u32 b = (SAME_LANES ? kQfMagicA : kQfMagicB) + ((u32)small >> 8);
  unsigned long long m;
  asm("mov.b64 %0, {%1, %2};" : "=l"(m) : "r"(a), "r"(b));
  return m;
}

__device__ __forceinline__ void quant_lanes_f(u32 zb, float r, u32& qa, u32& qb, unsigned long long magic) {
  const u32 fa = __byte_perm(zb, 0x4B000000u, 0x7610);  // 2^23 + field A
  const u32 fb = __byte_perm(zb, 0x4B000000u, 0x7632);  // 2^23 + field B
  unsigned long long F, Zf, Q, R;
  asm("mov.b64 %0, {%1, %2};" : "=l"(F) : "r"(fa), "r"(fb));
  asm("mov.b64 %0, {%1, %1};" : "=l"(R) : "f"(r));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(Zf) : "l"(F), "l"(kQfOffset));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(Q) : "l"(Zf), "l"(R), "l"(magic));
  asm("mov.b64 {%0, %1}, %2;" : "=r"(qa), "=r"(qb) : "l"(Q));
}

template <class TAB = ParamTab>
__device__ __forceinline__ u32 quant_pair_f(u32 zb, int p, const QParamsDev& q, unsigned long long magic) {
  const uint4 c = TAB::pos(q, p);  // x: r (float bits), w: qe
  u32 qa, qb;
  quant_lanes_f(zb, __uint_as_float(c.x), qa, qb, magic);
  return (qa + (qb << 16)) * c.w + TAB::wadd(q, p);  // wadd: 0 except the DC rounding/offset term
}

// ---------------------------------------------------------------------------
// K2: fused retain-r, r a template parameter (pruned at compile time).
// ---------------------------------------------------------------------------
// Retain tiles are 128 units (4 warps): measured faster than 256 for this
// memory-bound kernel (more, smaller CTAs per SM).
constexpr int kRetainThreads = 128;

template <int R, bool PAIR>
__global__ void __launch_bounds__(kRetainThreads) k_retain(PlaneSetDev ps, u64* __restrict__ sse) {
  __shared__ CtaSum cta;
  cta_sum_init(cta);
  UnitLoc L;
  u32 acc = 0;
  if (locate_unit<PAIR, kRetainThreads>(ps, L)) {
    uint4 w[8];
    load_unit<PAIR>(L.src, L.width, w);
    u32 x[8][8], Z[8][8], W[8][8], U[8][8];
    unpack_unit(w, x);
    fwd2d(x, Z);
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int v = 0; v < 8; ++v)
        W[u][v] = zz_kept(u, v, R) ? (Z[u][v] << (e_log2(u) + e_log2(v))) : 0u;
    W[0][0] += kDcRound;
    inv2d(W, U);
    acc = emit_unit<PAIR>(U, w, L.dst, L.width);
  }
  if (sse != nullptr)
    cta_sum_add<kRetainThreads>(cta, acc, sse, L.frame * ps.n_planes + L.plane, ps.x, ps.p[L.plane].units);
}

// Runtime-r variant: ragged widths (PAIR=false) and the exact "unrounded"
// SSE of the reference's float convention (FSSE).
template <bool PAIR, bool FSSE>
__global__ void __launch_bounds__(kThreads)
    k_retain_rt(PlaneSetDev ps, int r, u64* __restrict__ sse, u64* __restrict__ ssef) {
  __shared__ CtaSum cta;
  cta_sum_init(cta);
  UnitLoc L;
  u32 acc = 0;
  u64 accf = 0;
  if (locate_unit<PAIR>(ps, L)) {
    uint4 w[8];
    load_unit<PAIR>(L.src, L.width, w);
    u32 x[8][8], Z[8][8], W[8][8], U[8][8];
    unpack_unit(w, x);
    fwd2d(x, Z);
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int v = 0; v < 8; ++v)
        W[u][v] = (zz_rank(u, v) < r) ? (Z[u][v] << (e_log2(u) + e_log2(v))) : 0u;
    W[0][0] += kDcRound;
    inv2d(W, U);
    acc = emit_unit<PAIR>(U, w, L.dst, L.width);
    if (FSSE) {
      // sum (64 x - clamp(64 x_hat, 0, 16320))^2 with 64 x_hat = U - 24608.
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const u32 c = __vmaxu2(__vminu2(U[i][j], 0x9FE09FE0u), 0x60206020u);
          const u32 d = (x[i][j] << 6) + 0x60206020u - c;
          const int da = (int)(d << 16) >> 16;
          const int db = (int)(d - (u32)da) >> 16;
          accf += (u64)(da * da) + (PAIR ? (u64)(db * db) : 0ull);
        }
    }
  }
  if (sse != nullptr) cta_sum_add(cta, acc, sse, L.frame * ps.n_planes + L.plane, ps.x, ps.p[L.plane].units);
  if (FSSE) block_add_u64(accf, ssef + L.frame * ps.n_planes + L.plane);
}

// ---------------------------------------------------------------------------
// K3: fused quantised pipeline, 16-bit lanes end to end (exact when the host
// proved |64(x_hat-128)+32| <= 32767 for the table, adct_qtab_t.wide == 0).
// ---------------------------------------------------------------------------
template <bool PAIR, bool FLIP>
__global__ void __launch_bounds__(kThreads, 2)
    k_quant(PlaneSetDev ps, const __grid_constant__ QParamsDev q, u64* __restrict__ sse) {
  // Original pixel words wait in shared memory for the SSE (frees 32
  // registers); each thread only reads back its own slots, so no barrier.
  __shared__ uint4 s_orig[8][kThreads];
  UnitLoc L;
  u32 acc = 0;
  if (locate_unit<PAIR>(ps, L)) {
    uint4 w[8];
    load_unit<PAIR>(L.src, L.width, w);
    u32 x[8][8], U[8][8];
    unpack_unit(w, x);
#pragma unroll
    for (int i = 0; i < 8; ++i) s_orig[i][threadIdx.x] = w[i];
    {
      // Streamed 2-D transform: row pass, then per column v: forward column,
      // quantise/dequantise its 8 coefficients, inverse column; then rows.
      u32 t[8][8], c[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i) fwd8(x[i], t[i]);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        u32 col[8], Zc[8], Wc[8], cc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) col[i] = t[i][v];
        fwd8(col, Zc);
        if (v == 0) Zc[0] -= 8192u * 65537u;  // level shift: T(X-128)T^T = Z - 8192 e0 e0^T
#pragma unroll
        for (int u = 0; u < 8; ++u) Wc[u] = quant_pair(Zc[u], u * 8 + v, q);
        inv8(Wc, cc);
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i][v] = cc[i];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) inv8(c[i], U[i]);
    }
    uint4 wo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) wo[i] = s_orig[i][threadIdx.x];
    acc = emit_unit<PAIR, FLIP>(U, wo, L.dst, L.width);
  }
  // Per-warp atomics: measured 8% faster than the per-CTA accumulator for
  // this issue-bound kernel (the memory-bound retain kernels prefer per-CTA).
  if (sse != nullptr) block_add_u32(acc, sse + L.frame * ps.n_planes + L.plane);
}

// ---------------------------------------------------------------------------
// K3, persistent + cp.async pipelined: a fixed grid (2 CTAs per SM) walks the
// tiles of all frames; while a tile is transformed, the next tile's rows are
// already in flight into a 2-stage shared-memory ring (cp.async, no register
// cost).  Each thread only touches its own smem slots, so the ring needs no
// CTA barrier; cp.async.wait_group is per thread.
// ---------------------------------------------------------------------------
#ifndef ADCT_QP_MINB
#define ADCT_QP_MINB 2  // resident CTAs per SM for k_quant_p (register budget 128)
#endif
struct TileCursor {
  int plane;
  int64_t frame;
  bool active;
  const uint8_t* src;
  uint8_t* dst;
  int32_t width;
};

template <bool PAIR, int NT = kThreads>
__device__ __forceinline__ TileCursor tile_unit(const PlaneSetDev& ps, int64_t tile, u32 tiles_per_frame) {
  TileCursor c;
  c.frame = tile / tiles_per_frame;
  const u32 tb = (u32)(tile - c.frame * tiles_per_frame);
  int p = 0;
  if (ps.n_planes > 1 && tb >= ps.p[1].cta_begin) p = 1;
  if (ps.n_planes > 2 && tb >= ps.p[2].cta_begin) p = 2;
  const PlaneDev& P = ps.p[p];
  const u32 unit = (tb - P.cta_begin) * NT + threadIdx.x;
  c.plane = p;
  c.width = P.width;
  c.active = unit < P.units;
  if (c.active) {
    // a plain division measured ~2 % faster here than the multiply-high form
    // (register allocation of the persistent loop), so it stays
    const u32 brow = unit / P.upr;
    const u32 ucol = unit - brow * P.upr;
    const int64_t off = (int64_t)brow * 8 * P.width + (int64_t)ucol * (PAIR ? 16 : 8);
    c.src = P.src + c.frame * P.src_fs + off;
    c.dst = P.dst ? P.dst + c.frame * P.dst_fs + off : nullptr;
  } else {
    c.src = nullptr;
    c.dst = nullptr;
  }
  return c;
}

template <bool PAIR, int NT = kThreads>
__device__ __forceinline__ void cp_async_rows(uint4* slot_base, const TileCursor& c) {
  if (!c.active) return;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const u32 sa = (u32)__cvta_generic_to_shared(slot_base + i * NT);
    const uint8_t* g = c.src + (int64_t)i * c.width;
    if (PAIR)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
    else
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(g) : "memory");
  }
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <bool PAIR, bool FLIP, class TAB = ParamTab, bool QF = false>
__global__ void __launch_bounds__(kThreads, ADCT_QP_MINB)
    k_quant_p(PlaneSetDev ps, const __grid_constant__ QParamsDev q, u64* __restrict__ sse,
              int64_t n_tiles, u32 tiles_per_frame) {
  extern __shared__ uint4 s_ring[];  // [2][8][kThreads]
  const unsigned long long magic = qf_magic(ps.n_planes);
  const int64_t stride = gridDim.x;
  int64_t tile = blockIdx.x;
  if (tile >= n_tiles) return;
  TileCursor cur = tile_unit<PAIR>(ps, tile, tiles_per_frame);
  cp_async_rows<PAIR>(s_ring + threadIdx.x, cur);
  cp_async_commit();
  for (int stage = 0; tile < n_tiles; tile += stride, stage ^= 1) {
    const int64_t nt = tile + stride;
    TileCursor nxt;
    nxt.active = false;
    if (nt < n_tiles) {
      nxt = tile_unit<PAIR>(ps, nt, tiles_per_frame);
      cp_async_rows<PAIR>(s_ring + (stage ^ 1) * 8 * kThreads + threadIdx.x, nxt);
    }
    cp_async_commit();
    cp_async_wait1();
    const uint4* rows = s_ring + stage * 8 * kThreads + threadIdx.x;
    u32 acc = 0;
    if (cur.active) {
      uint4 w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        w[i] = rows[i * kThreads];
        if (!PAIR) w[i].z = w[i].w = 0u;
      }
      u32 x[8][8], U[8][8];
      unpack_unit(w, x);
      u32 t[8][8], c[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i) fwd8(x[i], t[i]);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        u32 col[8], Zc[8], Wc[8], cc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) col[i] = t[i][v];
        fwd8(col, Zc);
        if (QF) {
#pragma unroll
          for (int u = 0; u < 8; ++u) Zc[u] += kQfBias;  // folds into the butterfly's last IADD3
        }
        if (v == 0) Zc[0] -= 8192u * 65537u;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          Wc[u] = QF ? quant_pair_f<TAB>(Zc[u], u * 8 + v, q, magic) : quant_pair<TAB>(Zc[u], u * 8 + v, q);
        inv8(Wc, cc);
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i][v] = cc[i];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) inv8(c[i], U[i]);
      uint4 wo[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        wo[i] = rows[i * kThreads];
        if (!PAIR) wo[i].z = wo[i].w = 0u;
      }
      acc = emit_unit<PAIR, FLIP>(U, wo, cur.dst, cur.width);
    }
    if (sse != nullptr) block_add_u32(acc, sse + cur.frame * ps.n_planes + cur.plane);
    cur = nxt;
    if (nt >= n_tiles) break;
  }
}

// K3 for coarse tables whose quantiser still fits 16-bit lanes (every
// Q' <= 8191, e.g. q = 10): the forward transform and the two-lane quantiser
// run packed for two blocks (exact: |Z| <= 8192), dequantisation goes to
// int32 per block, and only the inverse — the part whose range needs more
// than 16 bits — runs per block in 32 bits.  Block A's column inverse
// streams in registers; block B's dequantised coefficients wait in shared
// memory.  `q.wadd` holds the scalar offsets here (-kq*qe, + 32 + 8192 at DC).
__device__ __forceinline__ u32 pack_px8(const int (&V)[8], int half) {
  u32 h2[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int a = V[4 * half + 2 * j] >> 6, b = V[4 * half + 2 * j + 1] >> 6;  // |.| < 2^15
    h2[j] = __vimin_s16x2_relu(__byte_perm((u32)a, (u32)b, 0x5410), 0x00FF00FFu);
  }
  return __byte_perm(h2[0], h2[1], 0x6420);
}

constexpr unsigned long long kHybridSmem = 64ull * kThreads * sizeof(int) + 8ull * kThreads * sizeof(uint4);

template <class TAB = ParamTab, bool QF = false>
__global__ void __launch_bounds__(kThreads, 2)
    k_quant_hybrid(PlaneSetDev ps, const __grid_constant__ QParamsDev q, u64* __restrict__ sse) {
  extern __shared__ uint4 s_dyn[];
  uint4* s_orig = s_dyn;                                          // [8][kThreads]
  int* s_wb = reinterpret_cast<int*>(s_dyn + 8 * kThreads);       // [64][kThreads]
  const unsigned long long magic = qf_magic<true>(ps.n_planes);
  UnitLoc L;
  u32 acc = 0;
  if (locate_unit<true>(ps, L)) {
    uint4 w[8];
    load_unit<true>(L.src, L.width, w);
    u32 x[8][8];
    unpack_unit(w, x);
#pragma unroll
    for (int i = 0; i < 8; ++i) s_orig[i * kThreads + threadIdx.x] = w[i];
    int cA[8][8];
    {
      u32 t[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i) fwd8(x[i], t[i]);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        u32 col[8], Zc[8];
        int wa[8], cc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) col[i] = t[i][v];
        fwd8(col, Zc);
        if (QF) {
#pragma unroll
          for (int u = 0; u < 8; ++u) Zc[u] += kQfBias;
        }
        if (v == 0) Zc[0] -= 8192u * 65537u;  // level shift
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int p = u * 8 + v;
          const uint4 c = TAB::pos(q, p);
          const u32 z = Zc[u];
          u32 qa, qb;
          if (QF) {
            quant_lanes_f(z, __uint_as_float(c.x), qa, qb, magic);  // 0x4B400000 + q per lane
          } else {
            const u32 sg = (TAB::kBaked && c.y == 2u) ? 0u : ((z >> 15) & 0x10001u) ^ 0x10001u;
            const u32 U = z * c.y + c.z + sg;
            qa = __umulhi(U & 0xFFFFu, c.x);  // q + kq, lane A
            qb = __umulhi(U >> 16, c.x);      // lane B
          }
          wa[u] = (int)(qa * c.w) + (int)TAB::wadd(q, p);
          s_wb[p * kThreads + threadIdx.x] = (int)(qb * c.w) + (int)TAB::wadd(q, p);
        }
        inv8(wa, cc);
#pragma unroll
        for (int i = 0; i < 8; ++i) cA[i][v] = cc[i];
      }
    }
    // block A rows go out now (8-byte stores; L2 merges them with B's halves)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int V[8];
      inv8(cA[i], V);
      const uint2 o = make_uint2(pack_px8(V, 0), pack_px8(V, 1));
      if (L.dst != nullptr) st_stream8(L.dst + (int64_t)i * L.width, o);
      const uint4 wi = s_orig[i * kThreads + threadIdx.x];
      acc = sse4(wi.x, o.x, acc);
      acc = sse4(wi.y, o.y, acc);
    }
    int cB[8][8];
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      int col[8], cc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) col[u] = s_wb[(u * 8 + v) * kThreads + threadIdx.x];
      inv8(col, cc);
#pragma unroll
      for (int i = 0; i < 8; ++i) cB[i][v] = cc[i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int V[8];
      inv8(cB[i], V);
      const uint2 o = make_uint2(pack_px8(V, 0), pack_px8(V, 1));
      if (L.dst != nullptr) st_stream8(L.dst + (int64_t)i * L.width + 8, o);
      const uint4 wi = s_orig[i * kThreads + threadIdx.x];
      acc = sse4(wi.z, o.x, acc);
      acc = sse4(wi.w, o.y, acc);
    }
  }
  if (sse != nullptr) block_add_u32(acc, sse + L.frame * ps.n_planes + L.plane);
}

// ---------------------------------------------------------------------------
// K3f k_quant_fi: the float-pair inverse.  Any table (q = 10's reconstruction
// needs 17 bits, beyond the packed kernels' 16-bit lanes).  Same pipeline as
// K3: forward_2d_unscaled of the level-shifted block, the D^2-folded
// quantiser, inverse_2d (reference codec.py:74-104, 84-87), round, clamp, SSE.  The forward and
// the float quantiser run packed as in k_quant_p; from the quantised integers
// on, the two blocks travel as fp32 pairs (A, B) in 64-bit register pairs, so
// every step of the inverse is one FP32x2 instruction for both blocks on the
// FMA pipe (the packed integer kernels keep the ALU pipe the busier one).
// Exact: every value is a multiple of 1/64 below 2^18 in magnitude (the host
// checks the table's bound, fi_exact in capi.cu), i.e. fits the 24-bit
// significand, so no add or fused multiply-add ever rounds.
//   * dequantisation folds into the column inverse: each butterfly add
//     X_a +- X_b becomes FFMA2(q_b, +-k_b, X_a) with k = Q' E / 64 (the
//     column's DC term is one FMUL2/FFMA2), so the inverse yields x_hat - 128
//     directly; + 128.5 rides on W[0][0] (the all-ones basis image).
//   * output: add.rm.f32x2 with 1.5 * 2^23 + 32768 floors to the integer grid,
//     so the low 16 bits of each lane are 32768 + floor(x_hat + 0.5); PRMT
//     pairs two lanes, VIADDMNMX.S16x2.RELU clamps both to [0, 255], PRMT
//     gathers the bytes.
// Rows 0-3 of the column pass stay in registers, rows 4-7 wait in shared
// memory (as 64-bit pairs); the original pixels wait there too for the SSE.
// pos[p].x = r (float bits), pos[p].y = k = Q' E / 64 (float bits).
// ---------------------------------------------------------------------------
struct F2 {  // two fp32 lanes (block A, block B) in one 64-bit register pair
  unsigned long long v;
};
__device__ __forceinline__ F2 f2_splat(float a) {
  F2 r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(r.v) : "f"(a));
  return r;
}
__device__ __forceinline__ F2 operator+(F2 a, F2 b) {
  F2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ F2 operator-(F2 a, F2 b) {
  F2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ F2 f2_fma(F2 a, float k, F2 c) {  // a * k + c, k shared by both lanes
  F2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(f2_splat(k).v), "l"(c.v));
  return r;
}
__device__ __forceinline__ F2 f2_mul(F2 a, float k) {
  F2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(f2_splat(k).v));
  return r;
}

// q (exact, as floats) of one coefficient position for both blocks from the
// biased linear form zb (see quant_lanes_f); `magic` = {M, M}.
__device__ __forceinline__ F2 quant_q2(u32 zb, float r, F2 magic) {
  F2 F, Zf, Q;
  const u32 fa = __byte_perm(zb, 0x4B000000u, 0x7610);
  const u32 fb = __byte_perm(zb, 0x4B000000u, 0x7632);
  asm("mov.b64 %0, {%1, %2};" : "=l"(F.v) : "r"(fa), "r"(fb));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(Zf.v) : "l"(F.v), "l"(kQfOffset));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(Q.v) : "l"(Zf.v), "l"(f2_splat(r).v), "l"(magic.v));
  return Q - magic;
}

// Column inverse x = T^T (k o q) with the dequantisation folded into the
// butterfly (inv8's graph; each X_u, u > 0, enters one add and one subtract).
template <bool DC>
__device__ __forceinline__ void inv8_dq(const F2 (&q)[8], const float (&k)[8], F2 dc, F2 (&x)[8]) {
  const F2 X0 = DC ? f2_fma(q[0], k[0], dc) : f2_mul(q[0], k[0]);
  const F2 b0 = f2_fma(q[4], k[4], X0), b1 = f2_fma(q[4], -k[4], X0);
  const F2 a0 = f2_fma(q[2], k[2], b0), a3 = f2_fma(q[2], -k[2], b0);
  const F2 a1 = f2_fma(q[6], -k[6], b1), a2 = f2_fma(q[6], k[6], b1);
  x[0] = f2_fma(q[1], k[1], a0);
  x[7] = f2_fma(q[1], -k[1], a0);
  x[1] = f2_fma(q[5], -k[5], a1);
  x[6] = f2_fma(q[5], k[5], a1);
  x[2] = f2_fma(q[3], -k[3], a2);
  x[5] = f2_fma(q[3], k[3], a2);
  x[3] = f2_fma(q[7], -k[7], a3);
  x[4] = f2_fma(q[7], k[7], a3);
}

// One reconstructed row of both blocks (y = x_hat + 0.5 per lane) -> bytes.
constexpr u32 kFiFloorMagic = 0x4B408000u;  // 1.5 * 2^23 + 32768
__device__ __forceinline__ uint4 pack_row_f(const F2 (&y)[8]) {
  u32 lo[8], hi[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    unsigned long long t;
    asm("add.rm.f32x2 %0, %1, %2;" : "=l"(t) : "l"(y[j].v), "l"(f2_splat(__uint_as_float(kFiFloorMagic)).v));
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo[j]), "=r"(hi[j]) : "l"(t));
  }
  u32 ha[4], hb[4];  // 16-bit fields 32768 + floor -> clamped pixels
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    ha[j] = __viaddmin_s16x2_relu(__byte_perm(lo[2 * j], lo[2 * j + 1], 0x5410), 0x80008000u, 0x00FF00FFu);
    hb[j] = __viaddmin_s16x2_relu(__byte_perm(hi[2 * j], hi[2 * j + 1], 0x5410), 0x80008000u, 0x00FF00FFu);
  }
  return make_uint4(__byte_perm(ha[0], ha[1], 0x6420), __byte_perm(ha[2], ha[3], 0x6420),
                    __byte_perm(hb[0], hb[1], 0x6420), __byte_perm(hb[2], hb[3], 0x6420));
}

__device__ __forceinline__ u32 f2_lo(F2 a) { return (u32)a.v; }
__device__ __forceinline__ u32 f2_hi(F2 a) { return (u32)(a.v >> 32); }
__device__ __forceinline__ F2 f2_make(u32 lo, u32 hi) {
  F2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "r"(lo), "r"(hi));
  return r;
}

// Forward, quantiser and column inverse of one unit (rows w).  Rows 0-3 of the
// column-pass result stay in c; rows 4-7 go to the park, two columns per
// 16-byte slot: park(r, j) is this thread's slot for row 4 + r, columns 2j, 2j+1.
template <class TAB, class PARK>
__device__ __forceinline__ void fi_columns(const uint4 (&w)[8], const QParamsDev& q, F2 magic, F2 (&c)[4][8],
                                           PARK park) {
  u32 x[8][8], t[8][8];
  unpack_unit(w, x);
#pragma unroll
  for (int i = 0; i < 8; ++i) fwd8(x[i], t[i]);
  const F2 dc = f2_splat(128.5f);
#pragma unroll
  for (int v = 0; v < 8; v += 2) {
    F2 hold[4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int vv = v + h;
      u32 col[8], Zc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) col[i] = t[i][vv];
      fwd8(col, Zc);
#pragma unroll
      for (int u = 0; u < 8; ++u) Zc[u] += kQfBias;
      if (vv == 0) Zc[0] -= 8192u * 65537u;  // level shift
      F2 qv[8], cc[8];
      float k[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint4 cst = TAB::pos(q, u * 8 + vv);
        qv[u] = quant_q2(Zc[u], __uint_as_float(cst.x), magic);
        k[u] = __uint_as_float(cst.y);
      }
      if (vv == 0)
        inv8_dq<true>(qv, k, dc, cc);
      else
        inv8_dq<false>(qv, k, dc, cc);
#pragma unroll
      for (int i = 0; i < 4; ++i) c[i][vv] = cc[i];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (h == 0)
          hold[i] = cc[4 + i];
        else
          park(i, v >> 1) = make_uint4(f2_lo(hold[i]), f2_hi(hold[i]), f2_lo(cc[4 + i]), f2_hi(cc[4 + i]));
      }
    }
  }
}

// Row pass of row i -> packed bytes; `c` rows 0-3, park for rows 4-7.
template <class PARK>
__device__ __forceinline__ uint4 fi_row(int i, const F2 (&c)[4][8], PARK park) {
  F2 row[8], y[8];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (i < 4) {
      row[2 * j] = c[i & 3][2 * j];
      row[2 * j + 1] = c[i & 3][2 * j + 1];
    } else {
      const uint4 s = park(i - 4, j);
      row[2 * j] = f2_make(s.x, s.y);
      row[2 * j + 1] = f2_make(s.z, s.w);
    }
  }
  inv8(row, y);
  return pack_row_f(y);
}

// Shared memory per thread: 8 slots of original rows + 16 park slots.  CTAs
// of kFiThreads units (128: 4 CTAs per SM at 48 KB each, so one CTA's load
// phase overlaps the others' arithmetic).
constexpr int kFiThreads = 128;
__host__ __device__ constexpr unsigned long long fi_smem(int nt) { return 24ull * nt * sizeof(uint4); }
constexpr unsigned long long kFiSmem = fi_smem(kFiThreads);

template <class TAB = ParamTab, int NT = kFiThreads>
__global__ void __launch_bounds__(NT, 512 / NT)
    k_quant_fi(PlaneSetDev ps, const __grid_constant__ QParamsDev q, u64* __restrict__ sse) {
  extern __shared__ uint4 s_dyn[];
  uint4* const sm = s_dyn + threadIdx.x;  // slot k of this thread: sm[k * NT]
  auto park = [sm](int r, int j) -> uint4& { return sm[(8 + r * 4 + j) * NT]; };
  const F2 magic{qf_magic<true>(ps.n_planes)};
  UnitLoc L;
  u32 acc = 0;
  if (locate_unit<true, NT>(ps, L)) {
    F2 c[4][8];
    {
      uint4 w[8];
      load_unit<true>(L.src, L.width, w);
#pragma unroll
      for (int i = 0; i < 8; ++i) sm[i * NT] = w[i];
      fi_columns<TAB>(w, q, magic, c, park);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 o = fi_row(i, c, park);
      if (L.dst != nullptr) st_stream16(L.dst + (int64_t)i * L.width, o);
      const uint4 wi = sm[i * NT];
      acc = sse4(wi.x, o.x, acc);
      acc = sse4(wi.y, o.y, acc);
      acc = sse4(wi.z, o.z, acc);
      acc = sse4(wi.w, o.w, acc);
    }
  }
  if (sse != nullptr) block_add_u32(acc, sse + L.frame * ps.n_planes + L.plane);
}

// ---------------------------------------------------------------------------
// K7: retain-r sweep — one read and one forward per unit, then for every r in
// [r_min, r_max] the masked inverse, rounding and SSE, all from registers
// (replaces the per-r reconstruct_image + mse loop, cli.py:105-113).
// Reconstructions are not stored.
// ---------------------------------------------------------------------------
template <bool PAIR>
__global__ void __launch_bounds__(kThreads)
    k_sweep(PlaneSetDev ps, int r_min, int r_max, u64* __restrict__ sse, u64* __restrict__ ssef) {
  UnitLoc L;
  const bool active = locate_unit<PAIR>(ps, L);
  uint4 w[8];
  u32 Z[8][8];
  if (active) {
    u32 x[8][8];
    load_unit<PAIR>(L.src, L.width, w);
    unpack_unit(w, x);
    fwd2d(x, Z);
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int v = 0; v < 8; ++v) Z[u][v] <<= (e_log2(u) + e_log2(v));
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      w[i] = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int j = 0; j < 8; ++j) Z[i][j] = 0;
    }
  }
  const int nr = r_max - r_min + 1;
  u64* out = sse + L.frame * nr;
#pragma unroll 1
  for (int r = r_min; r <= r_max; ++r) {
    u32 acc = 0;
    u64 accf = 0;
    if (active) {
      u32 W[8][8], U[8][8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) W[u][v] = (zz_rank(u, v) < r) ? Z[u][v] : 0u;
      W[0][0] += kDcRound;
      inv2d(W, U);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint4 o;
        pack_row(U[i], o);
        acc = sse4(w[i].x, o.x, acc);
        acc = sse4(w[i].y, o.y, acc);
        if (PAIR) {
          acc = sse4(w[i].z, o.z, acc);
          acc = sse4(w[i].w, o.w, acc);
        }
      }
      if (ssef != nullptr) {
        // the reference's unrounded convention: sum (64 x - clamp(64 x_hat, 0, 16320))^2
        u32 x[8][8];
        unpack_unit(w, x);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const u32 c = __vmaxu2(__vminu2(U[i][j], 0x9FE09FE0u), 0x60206020u);
            const u32 d = (x[i][j] << 6) + 0x60206020u - c;
            const int da = (int)(d << 16) >> 16;
            const int db = (int)(d - (u32)da) >> 16;
            accf += (u64)(da * da) + (PAIR ? (u64)(db * db) : 0ull);
          }
      }
    }
    block_add_u32(acc, out + (r - r_min));
    if (ssef != nullptr) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) accf += __shfl_xor_sync(0xffffffffu, accf, o);
      if ((threadIdx.x & 31) == 0 && accf != 0) atomicAdd(ssef + L.frame * nr + (r - r_min), accf);
    }
  }
}

// ---------------------------------------------------------------------------
// K7, incremental form (rounded SSE only): the inverse is linear, so going
// from r-1 to r kept coefficients adds one basis image,
//   64 X += E_uv Z_uv T[u]^T T[v]      ((u, v) = zigzag position r-1),
// i.e. 8 + 64 multiply-adds with factors in {-1, 0, 1} from a uniform table
// instead of 64 masks + a full 224-add inverse.  The E-scaled coefficients
// wait in shared memory (their index is the runtime zigzag position).
// ---------------------------------------------------------------------------
#ifdef ADCT_DEFINE_PLAIN_KERNELS  // one __constant__ copy: defined in capi.cu only
constexpr int kSweepThreads = 128;

struct SweepTables {
  int4 t[8][2];   // rows of T, t[u][h] = T[u][4h .. 4h+3]
  int zz[64];     // zigzag rank -> u*8+v
};
__host__ __device__ constexpr SweepTables make_sweep_tables() {
  SweepTables s{};
  for (int u = 0; u < 8; ++u)
    for (int h = 0; h < 2; ++h) {
      s.t[u][h].x = t_entry(u, 4 * h);
      s.t[u][h].y = t_entry(u, 4 * h + 1);
      s.t[u][h].z = t_entry(u, 4 * h + 2);
      s.t[u][h].w = t_entry(u, 4 * h + 3);
    }
  for (int k = 0; k < 64; ++k) s.zz[k] = zz_pos(k);
  return s;
}
__constant__ SweepTables c_sweep = make_sweep_tables();

// PRMT with sign replication (selector nibble msb set: the byte's sign fills
// it); the __byte_perm intrinsic ignores that bit, so this is inline PTX.
__device__ __forceinline__ u32 prmt_sext(u32 a, u32 sel) {
  u32 r;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(a), "r"(sel));
  return r;
}

template <bool PAIR, bool FSSE = false>
__global__ void __launch_bounds__(kSweepThreads)
    k_sweep_inc(PlaneSetDev ps, int r_min, int r_max, u64* __restrict__ sse, u64* __restrict__ ssef = nullptr) {
  __shared__ u32 zs[64][kSweepThreads];
  UnitLoc L;
  const bool active = locate_unit<PAIR, kSweepThreads>(ps, L);
  uint4 w[8];
  if (active) {
    u32 x[8][8], Z[8][8];
    load_unit<PAIR>(L.src, L.width, w);
    unpack_unit(w, x);
    fwd2d(x, Z);
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int v = 0; v < 8; ++v) zs[u * 8 + v][threadIdx.x] = Z[u][v] << (e_log2(u) + e_log2(v));
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int p = 0; p < 64; ++p) zs[p][threadIdx.x] = 0u;
  }
  u32 U[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) U[i][j] = kDcRound;  // T^T (kDcRound e0 e0^T) T = kDcRound everywhere
  // Rounded SSE without the output byte order: the original pixels are
  // regrouped once per unit into the order of pack_row's first PRMT level
  // (a_j b_j a_j+1 b_j+1) and flipped by 0x80 like the packed pixels, so
  // per r a row costs one PRMT level and a signed |a - b| per byte (the 0x80
  // flip is x - 128 read as a signed byte): no second PRMT level, no XOR.
  // Unpaired units: B's inputs are 0, so its lanes reconstruct to 0 and its
  // flipped bytes cancel against the flipped zero bytes of the original.
  if (!FSSE) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 v = w[i];
      w[i] = make_uint4(__byte_perm(v.x, v.z, 0x5140) ^ 0x80808080u, __byte_perm(v.x, v.z, 0x7362) ^ 0x80808080u,
                        __byte_perm(v.y, v.w, 0x5140) ^ 0x80808080u, __byte_perm(v.y, v.w, 0x7362) ^ 0x80808080u);
    }
  }
  const int nr = r_max - r_min + 1;
  const u32 four = 4u | ((u32)r_min >> 8);  // 4 (r_min <= 64), opaque to the compiler: stays an IMAD
  u64* out = sse != nullptr ? sse + L.frame * nr : nullptr;
#pragma unroll 1
  for (int r = 1; r <= r_max; ++r) {
    const int p = c_sweep.zz[r - 1];
    const u32 z = zs[p][threadIdx.x];
    const int u = p >> 3, v = p & 7;
    const int4 a0 = c_sweep.t[u][0], a1 = c_sweep.t[u][1];
    const int4 b0 = c_sweep.t[v][0], b1 = c_sweep.t[v][1];
    const int a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const int b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    u32 bz[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) bz[j] = z * (u32)b[j];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) U[i][j] += (u32)a[i] * bz[j];
    if (r >= r_min) {
      u32 acc = 0;
      u64 accf = 0;
      if (active) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (!FSSE) {
            // clamp on the ALU, the x4 (moving bits 6..13 to bytes 1/3) as a
            // multiply by a run-time 4 on the otherwise idle FMA pipe
            u32 cs[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) cs[j] = __vmaxu2(__vminu2(U[i][j], 0x9FFF9FFFu), 0x60006000u) * four;
            const u32 q[4] = {__byte_perm(cs[0], cs[1], 0x7531), __byte_perm(cs[2], cs[3], 0x7531),
                              __byte_perm(cs[4], cs[5], 0x7531), __byte_perm(cs[6], cs[7], 0x7531)};
            const u32 ow[4] = {w[i].x, w[i].y, w[i].z, w[i].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const u32 d = __vabsdiffs4(q[k], ow[k]);
              acc = __dp4a(d, d, acc);
            }
            continue;
          }
          if (sse != nullptr) {  // (FSSE callers may want only the unrounded SSE)
            uint4 o;
            pack_row(U[i], o);
            acc = sse4(w[i].x, o.x, acc);
            acc = sse4(w[i].y, o.y, acc);
            if (PAIR) {
              acc = sse4(w[i].z, o.z, acc);
              acc = sse4(w[i].w, o.w, acc);
            }
          }
          if (FSSE) {
            // the reference's unrounded convention, row by row from the input
            // words: sum (64 x - clamp(64 x_hat, 0, 16320))^2, 64 x_hat = U - 24608
            const u32 p01 = __byte_perm(w[i].x, w[i].z, 0x5410), p23 = __byte_perm(w[i].x, w[i].z, 0x7632);
            const u32 p45 = __byte_perm(w[i].y, w[i].w, 0x5410), p67 = __byte_perm(w[i].y, w[i].w, 0x7632);
            const u32 xr[8] = {__byte_perm(p01, 0u, 0x4240), __byte_perm(p01, 0u, 0x4341),
                               __byte_perm(p23, 0u, 0x4240), __byte_perm(p23, 0u, 0x4341),
                               __byte_perm(p45, 0u, 0x4240), __byte_perm(p45, 0u, 0x4341),
                               __byte_perm(p67, 0u, 0x4240), __byte_perm(p67, 0u, 0x4341)};
            // per lane d = 64 x - clamp(64 x_hat) (|d| <= 16320, linear form);
            // a row's 16 squares stay below 2^32 (16 * 16320^2), so they add up
            // in 32 bits; lanes split by sign-extending PRMTs
            u32 row = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const u32 c = __vmaxu2(__vminu2(U[i][j], 0x9FE09FE0u), 0x60206020u);
              const u32 d = (xr[j] << 6) + 0x60206020u - c;
              const u32 da = prmt_sext(d, 0x9910);  // lane A, sign-extended
              row += da * da;
              if (PAIR) {
                const u32 db = prmt_sext(d - da, 0xBB32);  // lane B (A's borrow removed)
                row += db * db;
              }
            }
            accf += row;
          }
        }
      }
      if (sse != nullptr) block_add_u32(acc, out + (r - r_min));
      if (FSSE) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) accf += __shfl_xor_sync(0xffffffffu, accf, o);
        if ((threadIdx.x & 31) == 0 && accf != 0) atomicAdd(ssef + L.frame * nr + (r - r_min), accf);
      }
    }
  }
}
#endif  // ADCT_DEFINE_PLAIN_KERNELS

// ---------------------------------------------------------------------------
// K1: forward integer transform, coefficients in _tile order.
// The output block of unit u is 2u (pair) or u, so a warp's output is one
// contiguous run of 32 units x 2 blocks.  Each thread writes one block at a
// time into a swizzled per-warp shared-memory stage (row = lane, 16-byte
// piece k at k ^ lane, conflict-free both ways) and the warp then stores it
// as whole 256/128-byte block runs: 512 contiguous bytes per store
// instruction instead of 16-byte pieces at a 512-byte stride.
// ---------------------------------------------------------------------------
constexpr int kForwardThreads = 128;

template <bool PAIR, typename OutT>
__global__ void __launch_bounds__(kForwardThreads)
    k_forward(PlaneSetDev ps, int level_shift, OutT* __restrict__ coef) {
  constexpr int S = 64 * (int)sizeof(OutT);  // bytes per block
  constexpr int NP = S / 16;                 // 16-byte pieces per block (16 or 8)
  constexpr int OB = (PAIR ? 2 : 1) * S;     // bytes per unit
  __shared__ uint4 stage[kForwardThreads / 32][32 * NP];
  const PlaneDev& P = ps.p[0];
  const int lane = threadIdx.x & 31;
  const u32 unit0 = blockIdx.x * kForwardThreads + (threadIdx.x & ~31u);
  const u32 unit = unit0 + lane;
  const bool active = unit < P.units;
  const int64_t frame = (int64_t)ps.frame_base + blockIdx.y;
  u32 Z[8][8];
  if (active) {
    const u32 brow = unit / P.upr;
    const u32 ucol = unit - brow * P.upr;
    const uint8_t* src =
        P.src + frame * P.src_fs + (int64_t)brow * 8 * P.width + (int64_t)ucol * (PAIR ? 16 : 8);
    uint4 w[8];
    load_unit<PAIR>(src, P.width, w);
    u32 x[8][8];
    unpack_unit(w, x);
    fwd2d(x, Z);
  }
  const u32 dc_shift = level_shift ? 8192u * 65537u : 0u;
  // level shift at DC, then bias both lanes to unsigned fields
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) Z[u][v] += 0x8000u - ((u == 0 && v == 0) ? dc_shift : 0u);
  uint4* st = stage[threadIdx.x >> 5];
  uint8_t* base = reinterpret_cast<uint8_t*>(coef) + (frame * (int64_t)P.units + unit0) * OB;
  const int n_here = (int)min(32u, P.units > unit0 ? P.units - unit0 : 0u);
#pragma unroll
  for (int half = 0; half < (PAIR ? 2 : 1); ++half) {
    if (active) {
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        uint4 piece;
        if (sizeof(OutT) == 4) {  // piece k = coefficients [4k, 4k+4) of the block
          const int u = k >> 1, v0 = (k & 1) * 4;
          u32* e = &piece.x;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const u32 z = Z[u][v0 + j];
            e[j] = half == 0 ? (u32)((int)(z & 0xFFFFu) - 32768) : (u32)((int)z >> 16);
          }
        } else {  // piece k = row k of the block, 8 int16
          const int u = k;
          u32* e = &piece.x;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const u32 z0 = Z[u][2 * j], z1 = Z[u][2 * j + 1];
            e[j] = half == 0 ? (__byte_perm(z0, z1, 0x5410) ^ 0x80008000u) : __byte_perm(z0, z1, 0x7632);
          }
        }
        st[lane * NP + (k ^ (lane & (NP - 1)))] = piece;
      }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const int g = j * 32 + lane;  // piece g of the warp's run: thread t = g / NP, piece k
      const int t = g / NP, k = g % NP;
      if (t < n_here) st_stream16(base + (int64_t)t * OB + half * S + k * 16, st[t * NP + (k ^ (t & (NP - 1)))]);
    }
    __syncwarp();
  }
}

#ifdef ADCT_DEFINE_PLAIN_KERNELS  // non-template kernels: defined once, in capi.cu
// SSE exchange for the quantised planes path (row f3): after the compress
// kernel on the same stream, copy the finished per-(frame, plane) SSE into
// every peer's symmetric vector with P2P stores.  Folding this into the
// issue-bound quant epilogue measured 19-22 % slower.
__global__ void k_push_sse(const u64* __restrict__ sse, int64_t n, u64* const* __restrict__ peers,
                           int n_peers, int64_t offset) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const u64 v = sse[i];
    for (int p = 0; p < n_peers; ++p) peers[p][offset + i] = v;
  }
  __threadfence_system();
}

// K3 for coarse tables (wide == 1, e.g. q < 25): one block per thread.  The
// B lane is empty, so the "linear form" is a plain int32 and every
// intermediate is exact whatever its magnitude.
__global__ void __launch_bounds__(kThreads)
    k_quant_wide(PlaneSetDev ps, const __grid_constant__ QParamsWide q, u64* __restrict__ sse) {
  UnitLoc L;
  u32 acc = 0;
  if (locate_unit<false>(ps, L)) {
    uint4 w[8];
    load_unit<false>(L.src, L.width, w);
    int x[8][8], t[8][8], c[8][8], V[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j)
        x[i][j] = (int)__byte_perm(j < 4 ? w[i].x : w[i].y, 0u, 0x4440 | (j & 3));
#pragma unroll
    for (int i = 0; i < 8; ++i) fwd8(x[i], t[i]);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      int col[8], Zc[8], Wc[8], cc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) col[i] = t[i][v];
      fwd8(col, Zc);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int p = u * 8 + v;
        const uint4 k = q.pos[p];
        const int z = Zc[u] - (p == 0 ? 8192 : 0);  // level shift
        const u32 U = (u32)(2 * z + (z >> 31)) + k.y;
        const u32 h = __umulhi(U, k.x);  // q + kw
        Wc[u] = (int)h * (int)k.z + (int)k.w;  // (h - kw) * qe (+ rounding, +128 back at DC)
      }
      inv8(Wc, cc);
#pragma unroll
      for (int i = 0; i < 8; ++i) c[i][v] = cc[i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) inv8(c[i], V[i]);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      // |V >> 6| < 2^15: clamp two pixels per packed 16x2 min/relu
      u32 h2[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        h2[j] = __vimin_s16x2_relu(__byte_perm((u32)(V[i][2 * j] >> 6), (u32)(V[i][2 * j + 1] >> 6), 0x5410),
                                   0x00FF00FFu);
      const u32 lo = __byte_perm(h2[0], h2[1], 0x6420);
      const u32 hi = __byte_perm(h2[2], h2[3], 0x6420);
      if (L.dst != nullptr) st_stream8(L.dst + (int64_t)i * L.width, make_uint2(lo, hi));
      acc = sse4(w[i].x, lo, acc);
      acc = sse4(w[i].y, hi, acc);
    }
  }
  if (sse != nullptr) block_add_u32(acc, sse + L.frame * ps.n_planes + L.plane);
}

// ---------------------------------------------------------------------------
// Float64 transforms (real-valued inputs; signature parity with the
// reference's float API).  Eight threads per 8x8 block, one block row or
// column each (a warp holds 4 consecutive blocks).  Every global access goes
// through a padded per-warp shared-memory tile [4 blocks][8 rows][9]:
// pixels arrive one image row segment (4 blocks x 8 values, 32 consecutive
// elements) per warp instruction and coefficients as the warp's 256
// contiguous doubles, 32 per instruction, so every load and store is
// coalesced; the 1-D passes read a row or a column of the tile (the 9-value
// pitch keeps both conflict-free).  8 values per thread in registers.
// ---------------------------------------------------------------------------
constexpr int kRowThreads = 256;               // threads per CTA: 32 blocks
constexpr int kRowBlocks = kRowThreads / 8;    // blocks per CTA
constexpr int kXposeWarp = 4 * 8 * 9;          // doubles per warp tile

// zigzag rank -> position u*8+v (ZIGZAG_INDICES, codec.py:24-33)
__constant__ unsigned char kZigzagPos[64] = {
    0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,  12, 19, 26, 33, 40, 48,
    41, 34, 27, 20, 13, 6,  7,  14, 21, 28, 35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23,
    30, 37, 44, 51, 58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

// Bit p set for the first r zigzag positions (a uniform loop: the same for
// every thread, no per-element rank computation).
__device__ __forceinline__ unsigned long long zz_keep_mask(int r) {
  unsigned long long m = 0;
  for (int k = 0; k < r; ++k) m |= 1ull << kZigzagPos[k];
  return m;
}

__device__ __forceinline__ double dscale(int u) {
  // d = (1/sqrt8, 1/sqrt2, 1/2, 1/sqrt2, 1/sqrt8, 1/sqrt2, 1/2, 1/sqrt2), kernels.py:149-157
  return (u & 1) ? 0.70710678118654757 : ((u & 2) ? 0.5 : 0.35355339059327379);
}

struct RowLoc {
  int64_t blk0;  // first block of this warp (within the frame)
  int64_t frame;
  int i;         // row / column of its block this thread owns
  int g;         // the thread's block within the warp (0..3)
  int lane;
  int64_t nblocks;
  double* buf;   // the warp's tile
};

__device__ __forceinline__ RowLoc row_locate(int64_t nblocks, double* tiles) {
  RowLoc L;
  L.lane = threadIdx.x & 31;
  L.blk0 = (int64_t)blockIdx.x * kRowBlocks + (threadIdx.x >> 5) * 4;
  L.frame = blockIdx.y;
  L.i = L.lane & 7;
  L.g = L.lane >> 3;
  L.nblocks = nblocks;
  L.buf = tiles + (threadIdx.x >> 5) * kXposeWarp;
  return L;
}

__device__ __forceinline__ double& tile_at(const RowLoc& L, int g, int row, int col) {
  return L.buf[(g * 8 + row) * 9 + col];
}
__device__ __forceinline__ void tile_get_row(const RowLoc& L, double (&r)[8]) {
#pragma unroll
  for (int v = 0; v < 8; ++v) r[v] = tile_at(L, L.g, L.i, v);
}
__device__ __forceinline__ void tile_put_row(const RowLoc& L, const double (&r)[8]) {
#pragma unroll
  for (int v = 0; v < 8; ++v) tile_at(L, L.g, L.i, v) = r[v];
}
__device__ __forceinline__ void tile_get_col(const RowLoc& L, double (&c)[8]) {
#pragma unroll
  for (int u = 0; u < 8; ++u) c[u] = tile_at(L, L.g, u, L.i);
}
__device__ __forceinline__ void tile_put_col(const RowLoc& L, const double (&c)[8]) {
#pragma unroll
  for (int u = 0; u < 8; ++u) tile_at(L, L.g, u, L.i) = c[u];
}

// Image rows of the warp's 4 blocks -> tile (row k of block g at [g][k][*]).
// Instruction k reads row k of all four blocks: 32 consecutive elements when
// the blocks share a block row.  Blocks past the end read as 0.
template <typename InT>
__device__ __forceinline__ void tile_load_image(const RowLoc& L, const InT* img, int h, int w) {
  const int64_t blk = L.blk0 + L.g, nbc = w / 8;
  const bool on = blk < L.nblocks;
  const int64_t brow = blk / nbc, bcol = blk - brow * nbc;
  const InT* src = img + L.frame * (int64_t)h * w + brow * 8 * w + bcol * 8 + L.i;
#pragma unroll
  for (int k = 0; k < 8; ++k) tile_at(L, L.g, k, L.i) = on ? (double)src[(int64_t)k * w] : 0.0;
  __syncwarp();
}

__device__ __forceinline__ void tile_store_image(const RowLoc& L, double* out, int h, int w, int clamp) {
  __syncwarp();
  const int64_t blk = L.blk0 + L.g, nbc = w / 8;
  if (blk >= L.nblocks) return;
  const int64_t brow = blk / nbc, bcol = blk - brow * nbc;
  double* dst = out + L.frame * (int64_t)h * w + brow * 8 * w + bcol * 8 + L.i;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double v = tile_at(L, L.g, k, L.i);
    dst[(int64_t)k * w] = clamp ? fmin(fmax(v, 0.0), 255.0) : v;
  }
}

// The warp's 4 x 64 contiguous coefficients <-> tile, 32 per instruction.
// Element e = 32 k + lane is block e / 64, row (e % 64) / 8, column e % 8.
__device__ __forceinline__ void tile_store_coef(const RowLoc& L, double* coef) {
  __syncwarp();
  double* dst = coef + (L.frame * L.nblocks + L.blk0) * 64;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int e = 32 * k + L.lane, g = e >> 6;
    if (L.blk0 + g < L.nblocks) dst[e] = tile_at(L, g, (e >> 3) & 7, e & 7);
  }
}

// SCALE: multiply by d_u d_v (the proposed transform's D); r: zigzag mask.
template <bool SCALE>
__device__ __forceinline__ void tile_load_coef(const RowLoc& L, const double* coef, int r) {
  const double* src = coef + (L.frame * L.nblocks + L.blk0) * 64;
  const unsigned long long keep = zz_keep_mask(r);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int e = 32 * k + L.lane, g = e >> 6, u = (e >> 3) & 7, v = e & 7;
    double val = 0.0;
    if (L.blk0 + g < L.nblocks && ((keep >> (e & 63)) & 1)) val = SCALE ? src[e] * (dscale(u) * dscale(v)) : src[e];
    tile_at(L, g, u, v) = val;
  }
  __syncwarp();
}

template <typename InT>
__global__ void __launch_bounds__(kRowThreads)
    k_forward_f64(const InT* __restrict__ img, int h, int w, int64_t nblocks,
                  double* __restrict__ coef) {
  __shared__ double tiles[kRowThreads / 32 * kXposeWarp];
  const RowLoc L = row_locate(nblocks, tiles);
  double a[8], b[8];
  tile_load_image(L, img, h, w);
  tile_get_col(L, a);   // column i of X
  fwd8(a, b);           // (T X)[u][i]
  __syncwarp();
  tile_put_col(L, b);
  __syncwarp();
  tile_get_row(L, a);   // row i of T X
  fwd8(a, b);           // Z[i][v] = (T X T^T)[i][v]
#pragma unroll
  for (int v = 0; v < 8; ++v) b[v] *= dscale(L.i) * dscale(v);
  __syncwarp();
  tile_put_row(L, b);
  tile_store_coef(L, coef);
}

__global__ void __launch_bounds__(kRowThreads)
    k_inverse_f64(const double* __restrict__ coef, int h, int w, int64_t nblocks, int r,
                  int clamp, double* __restrict__ out) {
  __shared__ double tiles[kRowThreads / 32 * kXposeWarp];
  const RowLoc L = row_locate(nblocks, tiles);
  double a[8], b[8];
  tile_load_coef<true>(L, coef, r);
  tile_get_row(L, a);   // row u = i of W
  inv8(a, b);           // (W T)[i][j]
  __syncwarp();
  tile_put_row(L, b);
  __syncwarp();
  tile_get_col(L, a);   // column j = i of W T
  inv8(a, b);           // x[i'][j] = (T^T W T)[i'][j]
  __syncwarp();
  tile_put_col(L, b);
  tile_store_image(L, out, h, w, clamp);
}

// ---------------------------------------------------------------------------
// SSE of two uint8 batches (numerator of metrics.mse).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
    k_sse_u8(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, int64_t numel,
             int64_t sa, int64_t sb, int vec, u64* __restrict__ sse) {
  const int64_t frame = blockIdx.y;
  const uint8_t* pa = a + frame * sa;
  const uint8_t* pb = b + frame * sb;
  u32 acc = 0;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  if (vec) {
    const int64_t nv = numel / 16;
    for (int64_t k = (int64_t)blockIdx.x * kThreads + threadIdx.x; k < nv; k += stride) {
      const uint4 va = ld_stream16(pa + k * 16), vb = ld_stream16(pb + k * 16);
      acc = sse4(va.x, vb.x, acc);
      acc = sse4(va.y, vb.y, acc);
      acc = sse4(va.z, vb.z, acc);
      acc = sse4(va.w, vb.w, acc);
    }
    for (int64_t k = nv * 16 + (int64_t)blockIdx.x * kThreads + threadIdx.x; k < numel;
         k += stride) {
      const int d = (int)pa[k] - (int)pb[k];
      acc += (u32)(d * d);
    }
  } else {
    for (int64_t k = (int64_t)blockIdx.x * kThreads + threadIdx.x; k < numel; k += stride) {
      const int d = (int)pa[k] - (int)pb[k];
      acc += (u32)(d * d);
    }
  }
  // per-thread partial may exceed 2^24 for huge frames: reduce in 64 bits
  block_add_u64((u64)acc, sse + frame);
}

// ---------------------------------------------------------------------------
// Dense 8x8 transforms in float64 for any matrix C (the exact DCT and the
// reference's registry kernels): forward Y = C X C^T,
// inverse X = C^T mask_r(Y) C (the reference's transpose inverse,
// codec.py:84-87, also used for flagged non-orthogonal kernels), and an
// r-sweep that reconstructs incrementally:
//   x_hat_r = x_hat_{r-1} + Y[u][v] * C[u]^T C[v]   ((u,v) = zigzag position r-1)
// with the clamped float64 SSE of the reference's convention per r
// (cli.py:105-113: reconstruct_image + mse).  Same row-per-thread layout as
// the float64 flow-graph kernels above.
// ---------------------------------------------------------------------------
struct DenseMat {
  double c[64];  // row-major C[u][k]
};

__device__ __forceinline__ void dense8(const DenseMat& M, const double (&x)[8], double (&y)[8]) {
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) a = fma(M.c[u * 8 + k], x[k], a);
    y[u] = a;
  }
}

__device__ __forceinline__ void dense8t(const DenseMat& M, const double (&y)[8], double (&x)[8]) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    double a = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) a = fma(M.c[u * 8 + k], y[u], a);
    x[k] = a;
  }
}

template <typename InT>
__global__ void __launch_bounds__(kRowThreads)
    k_dense_forward(const InT* __restrict__ img, int h, int w, int64_t nblocks, const DenseMat M,
                    double* __restrict__ coef) {
  __shared__ double tiles[kRowThreads / 32 * kXposeWarp];
  const RowLoc L = row_locate(nblocks, tiles);
  double a[8], b[8];
  tile_load_image(L, img, h, w);
  tile_get_col(L, a);   // column i of X
  dense8(M, a, b);      // (C X)[u][i]
  __syncwarp();
  tile_put_col(L, b);
  __syncwarp();
  tile_get_row(L, a);   // row i of C X
  dense8(M, a, b);      // Y[i][v] = (C X C^T)[i][v]
  __syncwarp();
  tile_put_row(L, b);
  tile_store_coef(L, coef);
}

__global__ void __launch_bounds__(kRowThreads)
    k_dense_inverse(const double* __restrict__ coef, int h, int w, int64_t nblocks, int r, int clamp,
                    const DenseMat M, double* __restrict__ out) {
  __shared__ double tiles[kRowThreads / 32 * kXposeWarp];
  const RowLoc L = row_locate(nblocks, tiles);
  double a[8], b[8];
  tile_load_coef<false>(L, coef, r);
  tile_get_row(L, a);   // row u = i of Y
  dense8t(M, a, b);     // (Y C)[i][j]
  __syncwarp();
  tile_put_row(L, b);
  __syncwarp();
  tile_get_col(L, a);   // column j = i of Y C
  dense8t(M, a, b);     // x[i'][j] = (C^T Y C)[i'][j]
  __syncwarp();
  tile_put_col(L, b);
  tile_store_image(L, out, h, w, clamp);
}

// r-sweep: the block's Y waits in shared memory (read once per r at the
// zigzag position, a broadcast within each block's 8 threads); each thread
// updates its reconstruction row (8 FMAs per r) and adds its clamped squared
// errors; per r a warp reduction into a per-warp shared partial, one atomic
// per (CTA, r) at the end.  kZigzagPos (zigzag rank -> u*8+v) is above.

template <typename InT>
__global__ void __launch_bounds__(kRowThreads)
    k_dense_sweep(const InT* __restrict__ img, int h, int w, int64_t nblocks, const DenseMat M, int r_min,
                  int r_max, double* __restrict__ sse) {
  __shared__ double tiles[kRowThreads / 32 * kXposeWarp];
  __shared__ double ys[kRowBlocks * 64];             // [block][u*8+v]
  __shared__ double cs[64];                          // C
  __shared__ double part[64][kRowThreads / 32];      // [r - r_min][warp]
  const RowLoc L = row_locate(nblocks, tiles);
  const bool active = L.blk0 + L.g < nblocks;
  const int nr = r_max - r_min + 1;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x < 64) cs[threadIdx.x] = M.c[threadIdx.x];
  double x[8], a[8], b[8], V[8];
  tile_load_image(L, img, h, w);
  tile_get_row(L, x);   // row i of X, kept for the SSE
  tile_get_col(L, a);
  dense8(M, a, b);      // (C X)[u][i]
  __syncwarp();
  tile_put_col(L, b);
  __syncwarp();
  tile_get_row(L, a);
  dense8(M, a, b);      // Y[i][v]
  double* yb = ys + (threadIdx.x >> 3) * 64;
#pragma unroll
  for (int v = 0; v < 8; ++v) yb[L.i * 8 + v] = b[v];
#pragma unroll
  for (int j = 0; j < 8; ++j) V[j] = 0.0;
  __syncthreads();  // cs, ys
#pragma unroll 1
  for (int k = 0; k < r_max; ++k) {
    const int pos = kZigzagPos[k], u = pos >> 3, v = pos & 7;
    const double c = yb[pos] * cs[u * 8 + L.i];
#pragma unroll
    for (int j = 0; j < 8; ++j) V[j] = fma(c, cs[v * 8 + j], V[j]);
    if (k + 1 < r_min) continue;
    double acc = 0.0;
    if (active) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double d = x[j] - fmin(fmax(V[j], 0.0), 255.0);
        acc = fma(d, d, acc);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (L.lane == 0) part[k + 1 - r_min][warp] = acc;
  }
  __syncthreads();
  if (threadIdx.x < nr) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < kRowThreads / 32; ++q) t += part[threadIdx.x][q];
    atomicAdd(sse + L.frame * nr + threadIdx.x, t);
  }
}

#endif  // ADCT_DEFINE_PLAIN_KERNELS

// ---------------------------------------------------------------------------
// Synthetic blob images (BASELINE.json generator).  Not on the timed path.
// ---------------------------------------------------------------------------
__device__ __forceinline__ u64 mix64(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Standard normal from the counter (seed, pixel index): Box-Muller on two
// 24-bit uniforms.  The host generator (synth.py) evaluates the same formula.
__device__ __forceinline__ float hash_normal(u64 seed, u64 idx) {
  const u64 h = mix64(seed * 0x9E3779B97F4A7C15ull + idx + 1ull);
  const float u1 = ((float)(h >> 40) + 0.5f) * (1.0f / 16777216.0f);
  const float u2 = ((float)((h >> 8) & 0xFFFFFFull) + 0.5f) * (1.0f / 16777216.0f);
  return sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
}

constexpr int kSynthRows = 16;

template <int NB>
__global__ void __launch_bounds__(kThreads)
    k_synth(uint8_t* __restrict__ out, int h, int w, int64_t stride,
            const float* __restrict__ blobs, const u64* __restrict__ seeds, int64_t frame_base) {
  __shared__ float gy[NB][kSynthRows];
  const int64_t frame = frame_base + blockIdx.z;
  const float* B = blobs + frame * NB * 4;
  const int row0 = blockIdx.y * kSynthRows;
  for (int idx = threadIdx.x; idx < NB * kSynthRows; idx += kThreads) {
    const int k = idx / kSynthRows, r = idx % kSynthRows;
    const float dy = (float)(row0 + r) - B[k * 4 + 0];
    const float s = B[k * 4 + 2];
    gy[k][r] = expf(-(dy * dy) / (2.0f * s * s));
  }
  __syncthreads();
  const int col = blockIdx.x * kThreads + threadIdx.x;
  if (col >= w) return;
  float gx[NB];
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    const float dx = (float)col - B[k * 4 + 1];
    const float s = B[k * 4 + 2];
    gx[k] = B[k * 4 + 3] * expf(-(dx * dx) / (2.0f * s * s));
  }
  const u64 seed = seeds[frame];
  uint8_t* dst = out + frame * stride;
  for (int r = 0; r < kSynthRows; ++r) {
    const int y = row0 + r;
    if (y >= h) break;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < NB; ++k) s = fmaf(gx[k], gy[k][r], s);
    const float v = 128.0f + s + 4.0f * hash_normal(seed, (u64)y * (u64)w + (u64)col);
    dst[(int64_t)y * w + col] = (uint8_t)fminf(fmaxf(rintf(v), 0.0f), 255.0f);
  }
}

}  // namespace adct
