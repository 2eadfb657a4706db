// capi.cu — extern "C" entry points of libadct_cuda.so (declared in
// include/adct_cuda.h).  Validation mirrors the reference's contract errors
// (errors.py:21-33) and happens before anything is enqueued.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "host_copy.h"

#include "adct_cuda.h"
#define ADCT_DEFINE_PLAIN_KERNELS
#include "adct_jit.h"
#include "adct_launch.h"

using namespace adct;

namespace {

thread_local int g_last_cuda = 0;

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int cuda_fail(cudaError_t e) {
  g_last_cuda = (int)e;
  return ADCT_ERR_CUDA;
}

#define ADCT_CUDA_TRY(expr)                         \
  do {                                              \
    cudaError_t _e = (expr);                        \
    if (_e != cudaSuccess) return cuda_fail(_e);    \
  } while (0)

inline bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// Host view of a plane set ready to launch.
struct PlaneSetHost {
  PlaneSetDev dev;
  uint32_t grid_x = 0;
  bool pair = true;
};

// Validate planes and lay out the tile grid.  `force_single` selects one
// block per thread (used by k_quant_wide).
int build_planes(const adct_plane_t* planes, int n_planes, int64_t n_frames, PlaneSetHost& out,
                 bool force_single = false, int tile = kThreads) {
  // frames are indexed as int32 inside a launch (frame_base + blockIdx.y)
  if (planes == nullptr || n_planes < 1 || n_planes > 3 || n_frames < 0 || n_frames > 0x7FFFFFFF)
    return ADCT_ERR_INVALID_ARGUMENT;
  std::memset(&out.dev, 0, sizeof(out.dev));
  bool pair = !force_single;
  for (int k = 0; k < n_planes; ++k) {
    const adct_plane_t& p = planes[k];
    if (p.height < 0 || p.width < 0 || (p.height % 8) != 0 || (p.width % 8) != 0)
      return ADCT_ERR_BAD_DIMENSIONS;
    const int64_t plane_px = (int64_t)p.height * p.width;
    if (n_frames > 0 && plane_px > 0 && p.src == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
    if (n_frames > 1 && p.src_frame_stride < plane_px) return ADCT_ERR_INVALID_ARGUMENT;
    if (n_frames > 1 && p.dst != nullptr && p.dst_frame_stride < plane_px)
      return ADCT_ERR_INVALID_ARGUMENT;
    if (plane_px / 64 > (int64_t)0x7FFFFFFF) return ADCT_ERR_INVALID_ARGUMENT;
    if (!aligned(p.src, 8) || (p.dst && !aligned(p.dst, 8)) || (p.src_frame_stride % 8) ||
        (p.dst && (p.dst_frame_stride % 8)))
      return ADCT_ERR_MISALIGNED;
    if ((p.width % 16) || !aligned(p.src, 16) || (p.dst && !aligned(p.dst, 16)) ||
        (p.src_frame_stride % 16) || (p.dst && (p.dst_frame_stride % 16)))
      pair = false;
  }
  uint32_t cta = 0;
  for (int k = 0; k < n_planes; ++k) {
    const adct_plane_t& p = planes[k];
    PlaneDev& d = out.dev.p[k];
    d.src = p.src;
    d.dst = p.dst;
    d.src_fs = p.src_frame_stride;
    d.dst_fs = p.dst_frame_stride;
    d.width = p.width;
    d.upr = (uint32_t)(p.width / (pair ? 16 : 8));
    d.units = d.upr * (uint32_t)(p.height / 8);
    d.upr_magic = 0;  // 0 encodes upr == 1 (brow = unit)
    if (d.units > 0 && d.upr > 1) {
      // unit / upr as one multiply-high, verified at every block-row start and
      // the unit before it (both sides are monotone step functions of unit)
      const uint64_t m = (0x100000000ull + d.upr - 1) / d.upr;
      if (m > 0xFFFFFFFFull) return ADCT_ERR_INVALID_ARGUMENT;
      d.upr_magic = (uint32_t)m;
      for (uint32_t u = 0; u < d.units; u += (d.units > 4096 ? d.upr : 1)) {
        // check every row start and the unit before it (where floor() changes)
        const uint32_t cand[2] = {u, u ? u - 1 : 0};
        for (uint32_t c : cand)
          if ((uint32_t)(((uint64_t)c * m) >> 32) != c / d.upr) return ADCT_ERR_INVALID_ARGUMENT;
      }
      const uint32_t last = d.units - 1;
      if ((uint32_t)(((uint64_t)last * m) >> 32) != last / d.upr) return ADCT_ERR_INVALID_ARGUMENT;
    }
    d.cta_begin = cta;
    cta += (d.units + tile - 1) / tile;
  }
  for (int k = n_planes; k < 3; ++k) out.dev.p[k].cta_begin = 0xFFFFFFFFu;
  out.dev.n_planes = n_planes;
  out.grid_x = cta;
  out.pair = pair;
  return ADCT_OK;
}

adct_plane_t single_plane(const uint8_t* img, uint8_t* rec, int32_t h, int32_t w,
                          int64_t img_stride, int64_t rec_stride) {
  adct_plane_t p;
  p.src = img;
  p.dst = rec;
  p.height = h;
  p.width = w;
  p.src_frame_stride = img_stride;
  p.dst_frame_stride = rec_stride;
  return p;
}

constexpr int64_t kMaxGridY = 65535;

// Launch f(ps) once per chunk of <= 65535 frames.
template <class F>
int for_frame_chunks(PlaneSetHost& ps, int64_t n_frames, F&& launch) {
  if (ps.grid_x == 0 || n_frames == 0) return ADCT_OK;
  for (int64_t f0 = 0; f0 < n_frames; f0 += kMaxGridY) {
    const int64_t nf = (n_frames - f0) < kMaxGridY ? (n_frames - f0) : kMaxGridY;
    ps.dev.frame_base = (int32_t)f0;
    launch(dim3(ps.grid_x, (unsigned)nf, 1));
    ADCT_CUDA_TRY(cudaGetLastError());
  }
  return ADCT_OK;
}

// Persistent kernels: ADCT_QP_MINB (2) CTAs of 256 threads per SM.
int persistent_grid(int* grid) {
  int dev = 0, sms = 0;
  ADCT_CUDA_TRY(cudaGetDevice(&dev));
  ADCT_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  *grid = ADCT_QP_MINB * sms;
  return ADCT_OK;
}

// ADCT_QUANT_KERNEL = pipe (default) | grid selects the quant kernel (A/B).
int quant_kernel_choice() {
  static const int v = [] {
    const char* e = std::getenv("ADCT_QUANT_KERNEL");
    return (e && std::strcmp(e, "grid") == 0) ? 0 : 1;
  }();
  return v;
}

// ADCT_SWEEP_KERNEL = inc (default) | full selects the rounded-SSE sweep kernel (A/B).
int sweep_kernel_choice() {
  static const int v = [] {
    const char* e = std::getenv("ADCT_SWEEP_KERNEL");
    return (e && std::strcmp(e, "full") == 0) ? 0 : 1;
  }();
  return v;
}

QParamsDev to_qparams(const adct_qtab_t& t) {
  QParamsDev q;
  const uint32_t dc_out = t.aligned ? 24576u : 32768u;  // output-field offset (see pack_row)
  for (int p = 0; p < 64; ++p) {
    q.pos[p].x = t.magic[p];
    q.pos[p].y = (uint32_t)t.mult[p];
    q.pos[p].z = (uint32_t)t.bias[p] * (uint32_t)t.mult[p] * 65537u;
    q.pos[p].w = (uint32_t)t.qe[p];
    q.wadd[p] = (uint32_t)0 - (uint32_t)t.kq[p] * (uint32_t)t.qe[p] * 65537u;
  }
  q.wadd[0] += (dc_out + 32u) * 65537u;
  return q;
}

// Packed quantiser + scalar dequantiser (k_quant_hybrid); false when some
// position's Q' is beyond the two-lane quantiser (mult == 0).
bool to_qparams_hybrid(const adct_qtab_t& t, QParamsDev* q) {
  for (int p = 0; p < 64; ++p) {
    if (t.mult[p] == 0) return false;
    q->pos[p].x = t.magic[p];
    q->pos[p].y = (uint32_t)t.mult[p];
    q->pos[p].z = (uint32_t)t.bias[p] * (uint32_t)t.mult[p] * 65537u;
    q->pos[p].w = (uint32_t)t.qe[p];
    q->wadd[p] = (uint32_t)0 - (uint32_t)t.kq[p] * (uint32_t)t.qe[p];
  }
  q->wadd[0] += 32u + 8192u;  // rounding, +128 back (64 * 128)
  return true;
}

// Float-quantiser constants (QF kernels): pos.x = r (float bits), pos.w = qe.
// Packed kernels: the lane magics make the packed result exactly the linear
// form (adct_kernels.cuh), so wadd is only the DC rounding/output offset.
// `scalar` (hybrid kernel, each lane dequantised alone): a lane carries
// 0x4B400000 + q, whose 0x4B400000 * qe is cancelled in wadd.
QParamsDev to_qparams_f(const adct_qtab_t& t, bool scalar) {
  QParamsDev q;
  std::memset(&q, 0, sizeof q);
  const uint32_t dc_out = t.aligned ? 24576u : 32768u;
  for (int p = 0; p < 64; ++p) {
    q.pos[p].x = t.recip_f[p];
    q.pos[p].w = (uint32_t)t.qe[p];
    q.wadd[p] = scalar ? (uint32_t)0 - 0x4B400000u * (uint32_t)t.qe[p] : 0u;
  }
  q.wadd[0] += scalar ? 32u + 8192u : (dc_out + 32u) * 65537u;
  return q;
}

// Float-pair inverse (k_quant_fi): pos.x = r (float bits), pos.y = Q' E / 64
// (float bits; exact: Q' E < 2^24).
QParamsDev to_qparams_fi(const adct_qtab_t& t) {
  QParamsDev q;
  std::memset(&q, 0, sizeof q);
  for (int p = 0; p < 64; ++p) {
    const float k = (float)t.qe[p] / 64.0f;
    uint32_t kb;
    std::memcpy(&kb, &k, sizeof kb);
    q.pos[p].x = t.recip_f[p];
    q.pos[p].y = kb;
  }
  return q;
}

// k_quant_fi is exact when every partial sum of the inverse, in units of
// 1/64, stays below 2^24: they are bounded by sum_uv |W_uv| + 64 * 128.5
// (the DC offset) <= sum_uv (|Z_uv| + Q'_uv / 2) E_uv + 8224
// <= 64 * 8192 + 8224 + sum_uv qe_uv / 2
// (|Z_uv| E_uv <= 128 n_u n_v * 64 / (n_u n_v) = 8192).
bool fi_exact(const adct_qtab_t& t) {
  double s = 64.0 * 8192.0 + 8224.0;
  for (int p = 0; p < 64; ++p) s += 0.5 * (double)t.qe[p];
  return s < 16777216.0;
}

// ADCT_FI_KERNEL: "wide" (default) runs k_quant_fi for coarse tables (the
// 16-bit-lane kernels cannot hold their reconstruction), "all" for every
// paired table, "off" keeps k_quant_hybrid (A/B).
int fi_kernel_choice() {
  static const int v = [] {
    const char* e = std::getenv("ADCT_FI_KERNEL");
    if (e && std::strcmp(e, "off") == 0) return 0;
    if (e && std::strcmp(e, "all") == 0) return 2;
    return 1;
  }();
  return v;
}

// ADCT_FI_THREADS = 256 runs k_quant_fi with 256-unit tiles (A/B; default 128).
int fi_threads_choice() {
  static const int v = [] {
    const char* e = std::getenv("ADCT_FI_THREADS");
    return (e && std::strcmp(e, "256") == 0) ? 256 : kFiThreads;
  }();
  return v;
}

// ADCT_QUANT_FLOAT = 0 selects the integer (multiply-high) quantiser (A/B).
int quant_float_choice() {
  static const int v = [] {
    const char* e = std::getenv("ADCT_QUANT_FLOAT");
    return (e && std::strcmp(e, "0") == 0) ? 0 : 1;
  }();
  return v;
}

// ADCT_WIDE_KERNEL = scalar forces k_quant_wide for every coarse table (A/B).
int wide_kernel_choice() {
  static const int v = [] {
    const char* e = std::getenv("ADCT_WIDE_KERNEL");
    return (e && std::strcmp(e, "scalar") == 0) ? 0 : 1;
  }();
  return v;
}

QParamsWide to_qparams_wide(const adct_qtab_t& t) {
  QParamsWide q;
  for (int p = 0; p < 64; ++p) {
    q.pos[p].x = t.magic_w[p];
    q.pos[p].y = (uint32_t)t.cadd_w[p];
    q.pos[p].z = (uint32_t)t.qe[p];
    q.pos[p].w = (uint32_t)0 - (uint32_t)t.kw[p] * (uint32_t)t.qe[p];
  }
  q.pos[0].w += 32u + 8192u;  // rounding, +128 back (64 * 128)
  return q;
}

// --- quantiser table -------------------------------------------------------

// Row L1 norms of T: n = (8,2,4,2,8,2,4,2); E[u][v] = 64/(n_u n_v).
inline int row_nnz(int u) { return (u & 1) ? 2 : ((u & 2) ? 4 : 8); }

// Reference scaling diag d (kernels.py:149-157), float64, evaluated exactly
// as the reference does so Q' rounds identically.
inline double ref_d(int u) {
  const double s8 = 1.0 / std::sqrt(8.0), s2 = 1.0 / std::sqrt(2.0);
  return (u & 1) ? s2 : ((u & 2) ? 0.5 : s8);
}

// round half away from zero of z / q, exact integer arithmetic
inline int64_t rha_div(int64_t z, int64_t q) {
  const int64_t a = (2 * (z < 0 ? -z : z) + q) / (2 * q);
  return z < 0 ? -a : a;
}

// Float quantiser constant: the float r just above 1/Q such that
// RN(M + Z r) - M == round_half_away(Z / Q) for every |Z| <= zmax, M = 1.5 * 2^23
// (the device FFMA2 computes M + Z r exactly and rounds once, ties to even).
// Verified in exact integer arithmetic: r = mant * 2^-sh, so M + Z r rounds to
// M + round_half_even(Z mant / 2^sh) (M is even).
bool float_recip(int64_t Q, int64_t zmax, uint32_t* bits) {
  float r = (float)(1.0 / (double)Q);
  for (int attempt = 0; attempt < 64; ++attempt, r = std::nextafter(r, 2.0f)) {
    int e = 0;
    const float fr = std::frexp(r, &e);  // r = fr * 2^e, fr in [0.5, 1)
    const int64_t mant = (int64_t)std::ldexp((double)fr, 24);  // exact 24-bit integer
    const int sh = 24 - e;  // r = mant * 2^-sh
    if (sh < 1 || sh > 62) return false;
    // r must exceed 1/Q strictly (mant * Q > 2^sh) and by less than 1/(2 Q zmax)
    bool ok = true;
    for (int64_t Z = -zmax; ok && Z <= zmax; ++Z) {
      const int64_t num = Z * mant;
      int64_t fl = num >> sh;  // floor (arithmetic shift)
      const int64_t rem = num - (fl << sh), half = (int64_t)1 << (sh - 1);
      if (rem > half || (rem == half && (fl & 1))) ++fl;
      if (fl != rha_div(Z, Q)) ok = false;
    }
    if (ok) {
      std::memcpy(bits, &r, sizeof r);
      return true;
    }
  }
  return false;
}

int build_qtab_from_rounded(const int32_t* qp, int32_t quality, adct_qtab_t* out) {
  std::memset(out, 0, sizeof(*out));
  constexpr int64_t kZmax = 8192;  // |T (X-128) T^T| <= 128 n_u n_v <= 8192
  bool packed_ok = true;
  for (int p = 0; p < 64; ++p) {
    const int u = p >> 3, v = p & 7;
    const int64_t Q = qp[p];
    if (Q < 1) return ADCT_ERR_NON_POSITIVE_QUANTIZER;
    if (Q > (1 << 20)) return ADCT_ERR_UNSUPPORTED;
    const int64_t E = 64 / (row_nnz(u) * row_nnz(v));
    if (Q * E > 0x7FFFFFFF / 4) return ADCT_ERR_UNSUPPORTED;
    out->qprime[p] = (int32_t)Q;
    out->qe[p] = (int32_t)(Q * E);

    // Two-lane quantiser: U = (Z + B) * mult + [Z >= 0] must fit 16 bits.
    // Odd Q': U = 2Z + Q' - [Z<0] + 2Q' K, divisor 2Q'.  Even Q': ties of
    // (2Z + Q' - [Z<0]) / 2Q' cannot hit the odd numerator, so
    // floor((Z + Q'/2 - [Z<0]) / Q') is the same quotient, divisor Q'.
    if (Q <= 8191) {
      const bool odd = (Q & 1) != 0;
      const int64_t mult = odd ? 2 : 1, D = odd ? 2 * Q : Q;
      const int64_t b0 = odd ? (Q - 1) / 2 : Q / 2 - 1;
      int64_t K1 = (kZmax - b0 + Q - 1) / Q;
      if (K1 < 0) K1 = 0;
      const int64_t B = b0 + Q * K1;
      const uint64_t m = ((1ull << 32) + (uint64_t)D - 1) / (uint64_t)D;
      bool ok = m <= 0xFFFFFFFFull;
      for (int64_t Z = -kZmax; ok && Z <= kZmax; ++Z) {
        // s = [Z >= 0]; at Z == 0 the kernel's lane-B sign bit may read 1
        // (borrow from a negative lane A), so both values must agree there.
        // odd Q': both s values for every Z (2Z + Q' is odd, so no tie exists
        // and s never matters) — specialised kernels drop s there
        const int s_lo = odd ? 0 : (Z == 0 ? 0 : (Z > 0 ? 1 : 0));
        const int s_hi = odd ? 1 : (Z >= 0 ? 1 : 0);
        for (int s = s_lo; s <= s_hi; ++s) {
          const int64_t U = (Z + B) * mult + s;
          if (U < 0 || U > 0xFFFF) { ok = false; break; }
          const int64_t got = (int64_t)(((uint64_t)U * m) >> 32) - K1;
          if (got != rha_div(Z, Q)) { ok = false; break; }
        }
      }
      if (ok) {
        out->magic[p] = (uint32_t)m;
        out->bias[p] = (int32_t)B;
        out->mult[p] = (int32_t)mult;
        out->kq[p] = (int32_t)K1;
      } else {
        packed_ok = false;
      }
    } else {
      packed_ok = false;
    }

    if (!float_recip(Q, kZmax, &out->recip_f[p])) return ADCT_ERR_UNSUPPORTED;

    // Scalar quantiser: U = 2Z - [Z<0] + C, C = Q'(2K+1), divisor 2Q'.
    {
      const int64_t D = 2 * Q;
      int64_t K = (2 * kZmax + 1 - Q + D - 1) / D;
      if (K < 0) K = 0;
      const int64_t C = Q * (2 * K + 1);
      if (C + 2 * kZmax >= (1ll << 32)) return ADCT_ERR_UNSUPPORTED;
      // umulhi alone is exact over the reachable window (for Q' > 16384 the
      // quotient is identically 0); shift_w stays 0 (field kept for layout).
      const uint64_t mw = ((1ull << 32) + (uint64_t)D - 1) / (uint64_t)D;
      bool ok = mw <= 0xFFFFFFFFull;
      for (int64_t Z = -kZmax; ok && Z <= kZmax; ++Z) {
        const int64_t U = 2 * Z - (Z < 0 ? 1 : 0) + C;
        const int64_t got = (int64_t)(((uint64_t)U * mw) >> 32) - K;
        if (U < 0 || got != rha_div(Z, Q)) ok = false;
      }
      if (!ok) return ADCT_ERR_UNSUPPORTED;
      out->magic_w[p] = (uint32_t)mw;
      out->cadd_w[p] = (int32_t)C;
      out->kw[p] = (int32_t)K;
      out->shift_w[p] = 0;
    }
  }
  // |64 (x_hat - 128)| <= 8192 + max_ij sum_uv |T_ui T_vj| E_uv Q'_uv / 2
  // (exact reconstruction of the level-shifted block is within [-8192, 8128];
  // dequantisation moves each coefficient by at most Q'/2).
  double worst = 0.0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double s = 0.0;
      for (int u = 0; u < 8; ++u)
        for (int v = 0; v < 8; ++v)
          if (t_entry(u, i) * t_entry(v, j) != 0) s += 0.5 * (double)out->qe[u * 8 + v];
      if (s > worst) worst = s;
    }
  const double bound = 8192.0 + worst;
  if (bound > 1.0e9) return ADCT_ERR_UNSUPPORTED;  // keeps the 32-bit path far from overflow
  out->max_abs_v = (int32_t)std::ceil(bound);
  out->wide = (!packed_ok || bound + 32.0 > 32767.0) ? 1 : 0;
  out->aligned = (!out->wide && bound + 32.0 <= 24575.0) ? 1 : 0;
  out->quality = quality;
  return ADCT_OK;
}

inline int32_t round_half_away_pos(double x) { return (int32_t)std::floor(x + 0.5); }

}  // namespace

// ===========================================================================
static int f64_geometry(int64_t n, int32_t h, int32_t w, int64_t& nblocks) {
  if (n < 0) return ADCT_ERR_INVALID_ARGUMENT;
  if (h < 0 || w < 0 || (h % 8) || (w % 8)) return ADCT_ERR_BAD_DIMENSIONS;
  nblocks = (int64_t)(h / 8) * (w / 8);
  if (nblocks > (int64_t)kThreads * 0x7FFFFFFF) return ADCT_ERR_INVALID_ARGUMENT;
  return ADCT_OK;
}

template <typename InT>
static int forward_f64_impl(const InT* img, int64_t n, int32_t h, int32_t w, double* coef, void* stream) {
  int64_t nb;
  int rc = f64_geometry(n, h, w, nb);
  if (rc != ADCT_OK) return rc;
  if (n == 0 || nb == 0) return ADCT_OK;
  if (img == nullptr || coef == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  cudaStream_t s = as_stream(stream);
  const unsigned gx = (unsigned)((nb + kRowBlocks - 1) / kRowBlocks);
  for (int64_t f0 = 0; f0 < n; f0 += kMaxGridY) {
    const int64_t nf = (n - f0) < kMaxGridY ? (n - f0) : kMaxGridY;
    k_forward_f64<InT><<<dim3(gx, (unsigned)nf), kRowThreads, 0, s>>>(img + f0 * (int64_t)h * w, h, w, nb,
                                                                     coef + f0 * nb * 64);
    ADCT_CUDA_TRY(cudaGetLastError());
  }
  return ADCT_OK;
}

extern "C" {

int adct_version(void) { return 1 * 10000 + 0 * 100 + 0; }

const char* adct_strerror(int code) {
  switch (code) {
    case ADCT_OK: return "ok";
    case ADCT_ERR_BAD_DIMENSIONS: return "image dimensions must be divisible by 8";
    case ADCT_ERR_INVALID_RETENTION: return "retention count must be in [1, 64]";
    case ADCT_ERR_NON_POSITIVE_QUANTIZER: return "quantization steps must be strictly positive";
    case ADCT_ERR_DIMENSION_MISMATCH: return "shape mismatch";
    case ADCT_ERR_INVALID_ARGUMENT: return "invalid argument";
    case ADCT_ERR_MISALIGNED: return "pointer or stride not 8-byte aligned";
    case ADCT_ERR_CUDA: return "CUDA runtime error";
    case ADCT_ERR_UNSUPPORTED: return "quantiser table outside the exactly supported range";
    default: return "unknown error";
  }
}

int adct_last_cuda_error(void) { return g_last_cuda; }

int adct_qtab_build(const double* qpu, adct_qtab_t* out) {
  if (qpu == nullptr || out == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  int32_t qp[64];
  for (int p = 0; p < 64; ++p) {
    if (!(qpu[p] > 0.0) || !std::isfinite(qpu[p])) return ADCT_ERR_NON_POSITIVE_QUANTIZER;
    if (qpu[p] > (double)(1 << 20)) return ADCT_ERR_UNSUPPORTED;
    const int32_t r = round_half_away_pos(qpu[p]);
    qp[p] = r < 1 ? 1 : r;
  }
  return build_qtab_from_rounded(qp, -1, out);
}

int adct_qtab_from_quality(const int32_t* base, int32_t quality, adct_qtab_t* out) {
  if (base == nullptr || out == nullptr || quality < 1 || quality > 100)
    return ADCT_ERR_INVALID_ARGUMENT;
  // IJG quality scale as a float64 factor: s(q) = (5000/q)/100 or (200-2q)/100.
  const double s = (quality < 50 ? 5000.0 / quality : 200.0 - 2.0 * quality) / 100.0;
  double qpu[64];
  for (int p = 0; p < 64; ++p) {
    if (base[p] <= 0) return ADCT_ERR_NON_POSITIVE_QUANTIZER;
    const double scaled = (double)base[p] * s;
    qpu[p] = scaled / (ref_d(p >> 3) * ref_d(p & 7));
  }
  int32_t qp[64];
  for (int p = 0; p < 64; ++p) {
    const int32_t r = round_half_away_pos(qpu[p]);
    qp[p] = r < 1 ? 1 : r;
  }
  return build_qtab_from_rounded(qp, quality, out);
}

// --- K1 forward ------------------------------------------------------------
static int forward_common(const uint8_t* img, int64_t n, int32_t h, int32_t w, int64_t img_stride,
                          int32_t level_shift, void* coef, bool out16, void* stream) {
  if (n < 0) return ADCT_ERR_INVALID_ARGUMENT;
  adct_plane_t pl = single_plane(img, nullptr, h, w, img_stride, 0);
  PlaneSetHost ps;
  int rc = build_planes(&pl, 1, n, ps, false, kForwardThreads);
  if (rc != ADCT_OK) return rc;
  if (ps.grid_x == 0 || n == 0) return ADCT_OK;
  if (coef == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  if (!aligned(coef, 16)) return ADCT_ERR_MISALIGNED;
  cudaStream_t s = as_stream(stream);
  const int T = kForwardThreads;
  return for_frame_chunks(ps, n, [&](dim3 g) {
    if (out16) {
      if (ps.pair)
        k_forward<true, int16_t><<<g, T, 0, s>>>(ps.dev, level_shift, (int16_t*)coef);
      else
        k_forward<false, int16_t><<<g, T, 0, s>>>(ps.dev, level_shift, (int16_t*)coef);
    } else {
      if (ps.pair)
        k_forward<true, int32_t><<<g, T, 0, s>>>(ps.dev, level_shift, (int32_t*)coef);
      else
        k_forward<false, int32_t><<<g, T, 0, s>>>(ps.dev, level_shift, (int32_t*)coef);
    }
  });
}

int adct_forward_int32(const uint8_t* img, int64_t n, int32_t h, int32_t w, int64_t img_stride,
                       int32_t level_shift, int32_t* coef, void* stream) {
  return forward_common(img, n, h, w, img_stride, level_shift, coef, false, stream);
}

int adct_forward_int16(const uint8_t* img, int64_t n, int32_t h, int32_t w, int64_t img_stride,
                       int32_t level_shift, int16_t* coef, void* stream) {
  return forward_common(img, n, h, w, img_stride, level_shift, coef, true, stream);
}

// --- K2 retain ---------------------------------------------------------------
static int retain_planes(const adct_plane_t* planes, int32_t n_planes, int64_t n_frames, int32_t r,
                         uint64_t* sse, uint64_t* ssef, void* stream, const XchgDev* xchg = nullptr) {
  if (r < 1 || r > 64) return ADCT_ERR_INVALID_RETENTION;
  PlaneSetHost ps;
  int rc = build_planes(planes, n_planes, n_frames, ps);
  if (rc != ADCT_OK) return rc;
  if (xchg != nullptr) ps.dev.x = *xchg;  // no unrounded SSE with an exchange (checked by the caller)
  cudaStream_t s = as_stream(stream);
  const size_t nsse = (size_t)n_frames * n_planes;
  if (sse && nsse) ADCT_CUDA_TRY(cudaMemsetAsync(sse, 0, nsse * sizeof(uint64_t), s));
  if (ssef && nsse) ADCT_CUDA_TRY(cudaMemsetAsync(ssef, 0, nsse * sizeof(uint64_t), s));
  u64* d_sse = reinterpret_cast<u64*>(sse);
  u64* d_ssef = reinterpret_cast<u64*>(ssef);
  if (ssef == nullptr && ps.pair) {
    PlaneSetHost ps128;  // the pruned retain kernels run 128-unit tiles
    rc = build_planes(planes, n_planes, n_frames, ps128, false, kRetainThreads);
    if (rc != ADCT_OK) return rc;
    if (xchg != nullptr) ps128.dev.x = *xchg;
    RetainKernel k = retain_kernel(r);
    return for_frame_chunks(ps128, n_frames, [&](dim3 g) { k<<<g, kRetainThreads, 0, s>>>(ps128.dev, d_sse); });
  }
  return for_frame_chunks(ps, n_frames, [&](dim3 g) {
    if (ps.pair) {
      if (ssef) k_retain_rt<true, true><<<g, kThreads, 0, s>>>(ps.dev, r, d_sse, d_ssef);
      else k_retain_rt<true, false><<<g, kThreads, 0, s>>>(ps.dev, r, d_sse, d_ssef);
    } else {
      if (ssef) k_retain_rt<false, true><<<g, kThreads, 0, s>>>(ps.dev, r, d_sse, d_ssef);
      else k_retain_rt<false, false><<<g, kThreads, 0, s>>>(ps.dev, r, d_sse, d_ssef);
    }
  });
}

int adct_compress_retain(const uint8_t* img, uint8_t* rec, int64_t n, int32_t h, int32_t w,
                         int64_t img_stride, int64_t rec_stride, int32_t r, uint64_t* sse,
                         uint64_t* sse_unrounded, void* stream) {
  if (n < 0) return ADCT_ERR_INVALID_ARGUMENT;
  adct_plane_t pl = single_plane(img, rec, h, w, img_stride, rec_stride);
  return retain_planes(&pl, 1, n, r, sse, sse_unrounded, stream);
}

int adct_compress_retain_exchange(const uint8_t* img, uint8_t* rec, int64_t n, int32_t h, int32_t w,
                                  int64_t img_stride, int64_t rec_stride, int32_t r, uint64_t* sse,
                                  uint64_t* const* peer_sse, int32_t n_peers, int64_t peer_offset,
                                  uint32_t* arrivals, void* stream) {
  if (n < 0 || n_peers < 1 || n_peers > 1024 || peer_offset < 0) return ADCT_ERR_INVALID_ARGUMENT;
  if (r < 1 || r > 64) return ADCT_ERR_INVALID_RETENTION;
  if (n == 0) return ADCT_OK;  // nothing to compute or exchange
  if (sse == nullptr || peer_sse == nullptr || arrivals == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  if (!aligned(sse, 8) || !aligned(peer_sse, 8) || !aligned(arrivals, 4)) return ADCT_ERR_MISALIGNED;
  XchgDev x;
  x.peers = reinterpret_cast<u64* const*>(peer_sse);
  x.arrivals = arrivals;
  x.offset = peer_offset;
  x.n_peers = n_peers;
  // packed CTA counting needs < 2^16 CTAs (128- or 256-unit tiles) per image;
  // ADCT_XCHG_PACKED=0 forces the fenced arrival-counter form (tests)
  const char* fp = std::getenv("ADCT_XCHG_PACKED");
  x.packed = (fp && std::strcmp(fp, "0") == 0) ? 0 : (((int64_t)h / 8 * (w / 8) + 127) / 128 <= 65535 ? 1 : 0);
  adct_plane_t pl = single_plane(img, rec, h, w, img_stride, rec_stride);
  return retain_planes(&pl, 1, n, r, sse, nullptr, stream, &x);
}

int adct_compress_retain_planes(const adct_plane_t* planes, int32_t n_planes, int64_t n_frames,
                                int32_t r, uint64_t* sse, void* stream) {
  return retain_planes(planes, n_planes, n_frames, r, sse, nullptr, stream);
}

// --- K3/K6 quant -------------------------------------------------------------
static int quant_planes(const adct_plane_t* planes, int32_t n_planes, int64_t n_frames, const adct_qtab_t* qtab,
                        uint64_t* sse, void* stream, const void* unused);

int adct_compress_quant_planes(const adct_plane_t* planes, int32_t n_planes, int64_t n_frames,
                               const adct_qtab_t* qtab, uint64_t* sse, void* stream) {
  return quant_planes(planes, n_planes, n_frames, qtab, sse, stream, nullptr);
}

int adct_compress_quant_planes_exchange(const adct_plane_t* planes, int32_t n_planes, int64_t n_frames,
                                        const adct_qtab_t* qtab, uint64_t* sse, uint64_t* const* peer_sse,
                                        int32_t n_peers, int64_t peer_offset, uint32_t* arrivals,
                                        void* stream) {
  (void)arrivals;  // not needed by the push form (kept for symmetry with the retain entry point)
  if (n_frames < 0 || n_peers < 1 || n_peers > 1024 || peer_offset < 0) return ADCT_ERR_INVALID_ARGUMENT;
  if (n_frames == 0) return quant_planes(planes, n_planes, 0, qtab, sse, stream, nullptr);
  if (sse == nullptr || peer_sse == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  if (!aligned(sse, 8) || !aligned(peer_sse, 8)) return ADCT_ERR_MISALIGNED;
  int rc = quant_planes(planes, n_planes, n_frames, qtab, sse, stream, nullptr);
  if (rc != ADCT_OK) return rc;
  const int64_t n = n_frames * n_planes;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 1024);
  k_push_sse<<<blocks, 256, 0, as_stream(stream)>>>(reinterpret_cast<const u64*>(sse), n,
                                                    reinterpret_cast<u64* const*>(peer_sse), n_peers, peer_offset);
  ADCT_CUDA_TRY(cudaGetLastError());
  return ADCT_OK;
}

static int quant_planes(const adct_plane_t* planes, int32_t n_planes, int64_t n_frames, const adct_qtab_t* qtab,
                        uint64_t* sse, void* stream, const void* /*unused*/) {
  if (qtab == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  for (int p = 0; p < 64; ++p)
    if (qtab->qprime[p] < 1) return ADCT_ERR_NON_POSITIVE_QUANTIZER;
  if (!qtab->wide && qtab->mult[0] == 0) return ADCT_ERR_INVALID_ARGUMENT;  // not built by adct_qtab_*
  // float quantiser: any Q' fits, so only the inverse's range decides "wide"
  const bool qf = quant_float_choice() == 1 && qtab->recip_f[0] != 0u;
  const bool wide = (qf && quant_kernel_choice() == 1) ? (qtab->max_abs_v + 32 > 32767) : qtab->wide != 0;
  PlaneSetHost ps;
  int rc = build_planes(planes, n_planes, n_frames, ps, wide);
  if (rc != ADCT_OK) return rc;
  cudaStream_t s = as_stream(stream);
  const size_t nsse = (size_t)n_frames * n_planes;
  if (sse && nsse) ADCT_CUDA_TRY(cudaMemsetAsync(sse, 0, nsse * sizeof(uint64_t), s));
  u64* d_sse = reinterpret_cast<u64*>(sse);
  if (qf && quant_kernel_choice() == 1 && fi_exact(*qtab) &&
      (fi_kernel_choice() == 2 || (wide && fi_kernel_choice() == 1))) {
    const int nt = fi_threads_choice();  // units per tile = threads per CTA
    PlaneSetHost pf;  // two blocks per thread where every plane pairs
    rc = build_planes(planes, n_planes, n_frames, pf, false, nt);
    if (rc != ADCT_OK) return rc;
    if (pf.pair) {
      QParamsDev qi = to_qparams_fi(*qtab);
      const size_t smem = fi_smem(nt);
      // no run-time table specialisation here: with the constants as
      // immediates this kernel measured 2.3 % slower (ptxas already feeds them
      // to the FP32x2 instructions from the constant bank)
      if (nt == 256) {
        ADCT_CUDA_TRY(cudaFuncSetAttribute(k_quant_fi<ParamTab, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
        return for_frame_chunks(pf, n_frames, [&](dim3 g) {
          k_quant_fi<ParamTab, 256><<<g, 256, smem, s>>>(pf.dev, qi, d_sse);
        });
      }
      ADCT_CUDA_TRY(
          cudaFuncSetAttribute(k_quant_fi<ParamTab>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      return for_frame_chunks(pf, n_frames, [&](dim3 g) {
        k_quant_fi<ParamTab><<<g, kFiThreads, smem, s>>>(pf.dev, qi, d_sse);
      });
    }
  }
  if (wide) {
    QParamsDev qh;
    if (wide_kernel_choice() == 1 && (qf ? (qh = to_qparams_f(*qtab, true), true) : to_qparams_hybrid(*qtab, &qh))) {
      PlaneSetHost ph;  // two blocks per thread where every plane pairs
      rc = build_planes(planes, n_planes, n_frames, ph, false);
      if (rc != ADCT_OK) return rc;
      if (ph.pair) {
        if (void* jf = jit::quant_function(qf ? jit::kHybridF : jit::kHybrid, qh, s)) {  // table-specialised build
          void* args[] = {&ph.dev, &qh, &d_sse};
          int rcj = ADCT_OK;
          const int rcc = for_frame_chunks(ph, n_frames, [&](dim3 g) {
            if (const int cr = jit::launch(jf, g, dim3(kThreads), kHybridSmem, s, args)) {
              g_last_cuda = cr;  // CUresult of the driver launch
              rcj = ADCT_ERR_CUDA;
            }
          });
          return rcj != ADCT_OK ? rcj : rcc;
        }
        if (qf) {
          ADCT_CUDA_TRY(cudaFuncSetAttribute(k_quant_hybrid<ParamTab, true>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kHybridSmem));
          return for_frame_chunks(ph, n_frames, [&](dim3 g) {
            k_quant_hybrid<ParamTab, true><<<g, kThreads, kHybridSmem, s>>>(ph.dev, qh, d_sse);
          });
        }
        ADCT_CUDA_TRY(cudaFuncSetAttribute(k_quant_hybrid<>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)kHybridSmem));
        return for_frame_chunks(ph, n_frames, [&](dim3 g) {
          k_quant_hybrid<><<<g, kThreads, kHybridSmem, s>>>(ph.dev, qh, d_sse);
        });
      }
    }
    const QParamsWide qw = to_qparams_wide(*qtab);
    return for_frame_chunks(ps, n_frames, [&](dim3 g) { k_quant_wide<<<g, kThreads, 0, s>>>(ps.dev, qw, d_sse); });
  }
  // the one-tile-per-CTA A/B kernel (ADCT_QUANT_KERNEL=grid) keeps the integer quantiser
  const QParamsDev q = (qf && quant_kernel_choice() == 1) ? to_qparams_f(*qtab, false) : to_qparams(*qtab);
  const bool al = qtab->aligned != 0;
  if (quant_kernel_choice() == 1 && ps.grid_x > 0 && n_frames > 0) {
    const int64_t n_tiles = (int64_t)ps.grid_x * n_frames;
    int grid = 0;
    int rc2 = persistent_grid(&grid);
    if (rc2 != ADCT_OK) return rc2;
    if ((int64_t)grid > n_tiles) grid = (int)n_tiles;
    ps.dev.frame_base = 0;
    const size_t smem = 2 * 8 * kThreads * sizeof(uint4);
    const int kind = (ps.pair ? (al ? jit::kQuantPairAligned : jit::kQuantPairFlip)
                              : (al ? jit::kQuantSingleAligned : jit::kQuantSingleFlip)) +
                     (qf ? jit::kFloatOffset : 0);
    if (void* jf = jit::quant_function(kind, q, s)) {  // table-specialised build
      QParamsDev qa = q;
      uint32_t tpf = ps.grid_x;
      void* args[] = {&ps.dev, &qa, &d_sse, const_cast<int64_t*>(&n_tiles), &tpf};
      if (const int cr = jit::launch(jf, dim3(grid), dim3(kThreads), smem, s, args)) {
        g_last_cuda = cr;  // CUresult of the driver launch
        return ADCT_ERR_CUDA;
      }
      return ADCT_OK;
    }
#define ADCT_QP(PA, FL, QF)                                                                    \
  do {                                                                                             \
    ADCT_CUDA_TRY(cudaFuncSetAttribute(k_quant_p<PA, FL, ParamTab, QF>,                            \
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));     \
    k_quant_p<PA, FL, ParamTab, QF><<<grid, kThreads, smem, s>>>(ps.dev, q, d_sse, n_tiles, ps.grid_x); \
  } while (0)
    if (qf) {
      if (ps.pair) {
        if (al) ADCT_QP(true, false, true); else ADCT_QP(true, true, true);
      } else {
        if (al) ADCT_QP(false, false, true); else ADCT_QP(false, true, true);
      }
    } else if (ps.pair) {
      if (al) ADCT_QP(true, false, false); else ADCT_QP(true, true, false);
    } else {
      if (al) ADCT_QP(false, false, false); else ADCT_QP(false, true, false);
    }
#undef ADCT_QP
    ADCT_CUDA_TRY(cudaGetLastError());
    return ADCT_OK;
  }
  return for_frame_chunks(ps, n_frames, [&](dim3 g) {
    if (ps.pair) {
      if (al) k_quant<true, false><<<g, kThreads, 0, s>>>(ps.dev, q, d_sse);
      else k_quant<true, true><<<g, kThreads, 0, s>>>(ps.dev, q, d_sse);
    } else {
      if (al) k_quant<false, false><<<g, kThreads, 0, s>>>(ps.dev, q, d_sse);
      else k_quant<false, true><<<g, kThreads, 0, s>>>(ps.dev, q, d_sse);
    }
  });
}

int adct_compress_quant(const uint8_t* img, uint8_t* rec, int64_t n, int32_t h, int32_t w,
                        int64_t img_stride, int64_t rec_stride, const adct_qtab_t* qtab,
                        uint64_t* sse, void* stream) {
  if (n < 0) return ADCT_ERR_INVALID_ARGUMENT;
  adct_plane_t pl = single_plane(img, rec, h, w, img_stride, rec_stride);
  return adct_compress_quant_planes(&pl, 1, n, qtab, sse, stream);
}

// --- K7 sweep ----------------------------------------------------------------
int adct_sweep_retain_sse(const uint8_t* img, int64_t n, int32_t h, int32_t w, int64_t img_stride,
                          int32_t r_min, int32_t r_max, uint64_t* sse, uint64_t* sse_unrounded,
                          void* stream) {
  if (n < 0) return ADCT_ERR_INVALID_ARGUMENT;
  if (r_min < 1 || r_max > 64 || r_min > r_max) return ADCT_ERR_INVALID_RETENTION;
  adct_plane_t pl = single_plane(img, nullptr, h, w, img_stride, 0);
  PlaneSetHost ps;
  int rc = build_planes(&pl, 1, n, ps);
  if (rc != ADCT_OK) return rc;
  // at least one output; the rounded one may be skipped when the unrounded is
  // wanted (incremental kernel only)
  if (sse == nullptr && (sse_unrounded == nullptr || sweep_kernel_choice() != 1)) return ADCT_ERR_INVALID_ARGUMENT;
  cudaStream_t s = as_stream(stream);
  const size_t nsse = (size_t)n * (size_t)(r_max - r_min + 1);
  if (nsse && sse) ADCT_CUDA_TRY(cudaMemsetAsync(sse, 0, nsse * sizeof(uint64_t), s));
  if (nsse && sse_unrounded) ADCT_CUDA_TRY(cudaMemsetAsync(sse_unrounded, 0, nsse * sizeof(uint64_t), s));
  u64* d_sse = reinterpret_cast<u64*>(sse);
  u64* d_ssef = reinterpret_cast<u64*>(sse_unrounded);
  if (sweep_kernel_choice() == 1) {  // incremental form
    PlaneSetHost ps2;
    rc = build_planes(&pl, 1, n, ps2, false, kSweepThreads);
    if (rc != ADCT_OK) return rc;
    return for_frame_chunks(ps2, n, [&](dim3 g) {
      if (d_ssef != nullptr) {
        if (ps2.pair) k_sweep_inc<true, true><<<g, kSweepThreads, 0, s>>>(ps2.dev, r_min, r_max, d_sse, d_ssef);
        else k_sweep_inc<false, true><<<g, kSweepThreads, 0, s>>>(ps2.dev, r_min, r_max, d_sse, d_ssef);
      } else {
        if (ps2.pair) k_sweep_inc<true><<<g, kSweepThreads, 0, s>>>(ps2.dev, r_min, r_max, d_sse);
        else k_sweep_inc<false><<<g, kSweepThreads, 0, s>>>(ps2.dev, r_min, r_max, d_sse);
      }
    });
  }
  return for_frame_chunks(ps, n, [&](dim3 g) {
    if (ps.pair) k_sweep<true><<<g, kThreads, 0, s>>>(ps.dev, r_min, r_max, d_sse, d_ssef);
    else k_sweep<false><<<g, kThreads, 0, s>>>(ps.dev, r_min, r_max, d_sse, d_ssef);
  });
}

// --- float64 -----------------------------------------------------------------

int adct_forward_f64(const double* img, int64_t n, int32_t h, int32_t w, double* coef, void* stream) {
  return forward_f64_impl(img, n, h, w, coef, stream);
}

int adct_forward_f64_u8(const uint8_t* img, int64_t n, int32_t h, int32_t w, double* coef, void* stream) {
  return forward_f64_impl(img, n, h, w, coef, stream);
}

int adct_inverse_f64(const double* coef, int64_t n, int32_t h, int32_t w, int32_t r, int32_t clamp,
                     double* out, void* stream) {
  if (r < 1 || r > 64) return ADCT_ERR_INVALID_RETENTION;
  int64_t nb;
  int rc = f64_geometry(n, h, w, nb);
  if (rc != ADCT_OK) return rc;
  if (n == 0 || nb == 0) return ADCT_OK;
  if (out == nullptr || coef == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  cudaStream_t s = as_stream(stream);
  const unsigned gx = (unsigned)((nb + kRowBlocks - 1) / kRowBlocks);
  for (int64_t f0 = 0; f0 < n; f0 += kMaxGridY) {
    const int64_t nf = (n - f0) < kMaxGridY ? (n - f0) : kMaxGridY;
    k_inverse_f64<<<dim3(gx, (unsigned)nf), kRowThreads, 0, s>>>(coef + f0 * nb * 64, h, w, nb, r,
                                                               clamp, out + f0 * (int64_t)h * w);
    ADCT_CUDA_TRY(cudaGetLastError());
  }
  return ADCT_OK;
}

// --- dense float64 transforms (exact DCT, registry kernels) -----------------
static int dense_setup(const double* C, DenseMat& M) {
  if (C == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  for (int k = 0; k < 64; ++k) {
    if (!std::isfinite(C[k])) return ADCT_ERR_INVALID_ARGUMENT;
    M.c[k] = C[k];
  }
  return ADCT_OK;
}

int adct_forward_dense(const void* img, int32_t img_is_f64, int64_t n, int32_t h, int32_t w,
                       const double* C, double* coef, void* stream) {
  int64_t nb;
  int rc = f64_geometry(n, h, w, nb);
  if (rc != ADCT_OK) return rc;
  DenseMat M;
  if ((rc = dense_setup(C, M)) != ADCT_OK) return rc;
  if (n == 0 || nb == 0) return ADCT_OK;
  if (img == nullptr || coef == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  cudaStream_t s = as_stream(stream);
  const unsigned gx = (unsigned)((nb + kRowBlocks - 1) / kRowBlocks);
  for (int64_t f0 = 0; f0 < n; f0 += kMaxGridY) {
    const int64_t nf = (n - f0) < kMaxGridY ? (n - f0) : kMaxGridY;
    const dim3 g(gx, (unsigned)nf);
    if (img_is_f64)
      k_dense_forward<double><<<g, kRowThreads, 0, s>>>((const double*)img + f0 * (int64_t)h * w, h, w, nb, M,
                                                      coef + f0 * nb * 64);
    else
      k_dense_forward<uint8_t><<<g, kRowThreads, 0, s>>>((const uint8_t*)img + f0 * (int64_t)h * w, h, w, nb, M,
                                                       coef + f0 * nb * 64);
    ADCT_CUDA_TRY(cudaGetLastError());
  }
  return ADCT_OK;
}

int adct_inverse_dense(const double* coef, int64_t n, int32_t h, int32_t w, const double* C, int32_t r,
                       int32_t clamp, double* out, void* stream) {
  if (r < 1 || r > 64) return ADCT_ERR_INVALID_RETENTION;
  int64_t nb;
  int rc = f64_geometry(n, h, w, nb);
  if (rc != ADCT_OK) return rc;
  DenseMat M;
  if ((rc = dense_setup(C, M)) != ADCT_OK) return rc;
  if (n == 0 || nb == 0) return ADCT_OK;
  if (coef == nullptr || out == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  cudaStream_t s = as_stream(stream);
  const unsigned gx = (unsigned)((nb + kRowBlocks - 1) / kRowBlocks);
  for (int64_t f0 = 0; f0 < n; f0 += kMaxGridY) {
    const int64_t nf = (n - f0) < kMaxGridY ? (n - f0) : kMaxGridY;
    k_dense_inverse<<<dim3(gx, (unsigned)nf), kRowThreads, 0, s>>>(coef + f0 * nb * 64, h, w, nb, r, clamp, M,
                                                               out + f0 * (int64_t)h * w);
    ADCT_CUDA_TRY(cudaGetLastError());
  }
  return ADCT_OK;
}

int adct_sweep_dense(const void* img, int32_t img_is_f64, int64_t n, int32_t h, int32_t w, const double* C,
                     int32_t r_min, int32_t r_max, double* sse, void* stream) {
  if (r_min < 1 || r_max > 64 || r_min > r_max) return ADCT_ERR_INVALID_RETENTION;
  int64_t nb;
  int rc = f64_geometry(n, h, w, nb);
  if (rc != ADCT_OK) return rc;
  DenseMat M;
  if ((rc = dense_setup(C, M)) != ADCT_OK) return rc;
  if (n == 0) return ADCT_OK;
  if (sse == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  cudaStream_t s = as_stream(stream);
  const int nr = r_max - r_min + 1;
  ADCT_CUDA_TRY(cudaMemsetAsync(sse, 0, (size_t)n * nr * sizeof(double), s));
  if (nb == 0) return ADCT_OK;
  if (img == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  const unsigned gx = (unsigned)((nb + kRowBlocks - 1) / kRowBlocks);
  for (int64_t f0 = 0; f0 < n; f0 += kMaxGridY) {
    const int64_t nf = (n - f0) < kMaxGridY ? (n - f0) : kMaxGridY;
    const dim3 g(gx, (unsigned)nf);
    if (img_is_f64)
      k_dense_sweep<double><<<g, kRowThreads, 0, s>>>((const double*)img + f0 * (int64_t)h * w, h, w, nb, M, r_min,
                                                    r_max, sse + f0 * nr);
    else
      k_dense_sweep<uint8_t><<<g, kRowThreads, 0, s>>>((const uint8_t*)img + f0 * (int64_t)h * w, h, w, nb, M,
                                                     r_min, r_max, sse + f0 * nr);
    ADCT_CUDA_TRY(cudaGetLastError());
  }
  return ADCT_OK;
}

int adct_sse_u8(const uint8_t* a, const uint8_t* b, int64_t n, int64_t numel, int64_t stride_a,
                int64_t stride_b, uint64_t* sse, void* stream) {
  if (n < 0 || numel < 0) return ADCT_ERR_INVALID_ARGUMENT;
  if (n == 0) return ADCT_OK;
  if (sse == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  cudaStream_t s = as_stream(stream);
  ADCT_CUDA_TRY(cudaMemsetAsync(sse, 0, (size_t)n * sizeof(uint64_t), s));
  if (numel == 0) return ADCT_OK;
  if (a == nullptr || b == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  const int vec = aligned(a, 16) && aligned(b, 16) && (stride_a % 16 == 0) && (stride_b % 16 == 0);
  int64_t per = vec ? numel / 16 : numel;
  int64_t gx = (per + kThreads - 1) / kThreads;
  if (gx > 1184) gx = 1184;  // 8 CTAs per SM on 148 SMs, grid-stride beyond
  if (gx < 1) gx = 1;
  for (int64_t f0 = 0; f0 < n; f0 += kMaxGridY) {
    const int64_t nf = (n - f0) < kMaxGridY ? (n - f0) : kMaxGridY;
    k_sse_u8<<<dim3((unsigned)gx, (unsigned)nf), kThreads, 0, s>>>(
        a + f0 * stride_a, b + f0 * stride_b, numel, stride_a, stride_b, vec,
        reinterpret_cast<u64*>(sse) + f0);
    ADCT_CUDA_TRY(cudaGetLastError());
  }
  return ADCT_OK;
}

// --- synthetic generator ----------------------------------------------------
int adct_synth_blobs(uint8_t* out, int64_t n, int32_t h, int32_t w, int64_t img_stride,
                     const float* blobs, int32_t n_blobs, const uint64_t* noise_seed,
                     void* stream) {
  if (n < 0 || h < 0 || w < 0) return ADCT_ERR_INVALID_ARGUMENT;
  if (n == 0 || h == 0 || w == 0) return ADCT_OK;
  if (out == nullptr || blobs == nullptr || noise_seed == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  if (n_blobs != 16 && n_blobs != 32 && n_blobs != 64) return ADCT_ERR_UNSUPPORTED;
  cudaStream_t s = as_stream(stream);
  const dim3 g((unsigned)((w + kThreads - 1) / kThreads), (unsigned)((h + kSynthRows - 1) / kSynthRows));
  for (int64_t f0 = 0; f0 < n; f0 += kMaxGridY) {
    const int64_t nf = (n - f0) < kMaxGridY ? (n - f0) : kMaxGridY;
    const dim3 gg(g.x, g.y, (unsigned)nf);
    const u64* seeds = reinterpret_cast<const u64*>(noise_seed);
    if (n_blobs == 16) k_synth<16><<<gg, kThreads, 0, s>>>(out, h, w, img_stride, blobs, seeds, f0);
    else if (n_blobs == 32) k_synth<32><<<gg, kThreads, 0, s>>>(out, h, w, img_stride, blobs, seeds, f0);
    else k_synth<64><<<gg, kThreads, 0, s>>>(out, h, w, img_stride, blobs, seeds, f0);
    ADCT_CUDA_TRY(cudaGetLastError());
  }
  return ADCT_OK;
}

// --- host pipeline -------------------------------------------------------------
}  // extern "C"

struct adct_pipeline {
  int device = 0;
  size_t chunk_bytes = 0;
  static constexpr int kMaxDepth = 8;
  int depth = 3;  // streams / staging slots in flight (ADCT_PIPELINE_DEPTH, 2..8)
  cudaStream_t stream[kMaxDepth] = {};
  cudaEvent_t done[kMaxDepth] = {};  // slot b's last chunk finished (staged path)
  uint8_t* d_in[kMaxDepth] = {};
  uint8_t* d_out[kMaxDepth] = {};
  uint8_t* h_in[kMaxDepth] = {};   // page-locked staging ring for pageable callers
  uint8_t* h_out[kMaxDepth] = {};
  size_t h_bytes = 0;              // size of each h_in / h_out slot (0: not allocated yet)
  uint64_t* d_sse = nullptr;  // SSE of a whole call, copied to the host once at the end
  int64_t sse_cap = 0;
  adct::HostCopyPool* pool = nullptr;  // host threads for the staging memcpys
  std::mutex mu;  // calls on one pipeline are serialised (one set of streams and staging slots)
};

namespace {

void pipeline_free(adct_pipeline* p) {
  for (int k = 0; k < p->depth; ++k) {
    if (p->stream[k]) cudaStreamSynchronize(p->stream[k]);
  }
  for (int k = 0; k < p->depth; ++k) {
    if (p->stream[k]) cudaStreamDestroy(p->stream[k]);
    if (p->done[k]) cudaEventDestroy(p->done[k]);
    if (p->d_in[k]) cudaFree(p->d_in[k]);
    if (p->d_out[k]) cudaFree(p->d_out[k]);
    if (p->h_in[k]) cudaFreeHost(p->h_in[k]);
    if (p->h_out[k]) cudaFreeHost(p->h_out[k]);
  }
  if (p->d_sse) cudaFree(p->d_sse);
  delete p->pool;
  delete p;
}

// Drain every stream before an error return: no copy may still be queued on
// host or staging memory the caller is about to reuse or free.
int pipeline_fail(adct_pipeline* p, int rc) {
  for (int k = 0; k < p->depth; ++k)
    if (p->stream[k]) cudaStreamSynchronize(p->stream[k]);
  return rc;
}

#define ADCT_PIPE_TRY(expr)                                    \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return pipeline_fail(p, cuda_fail(_e)); \
  } while (0)

// Staging slots of at least `unit_bytes` (one image / one frame of planes)
// and a device SSE vector of at least `n_sse` entries; with `staged`, also
// the page-locked host ring of the same slot size.
int pipeline_reserve(adct_pipeline* p, size_t unit_bytes, int64_t n_sse, bool staged) {
  if (unit_bytes > p->chunk_bytes) {  // one unit larger than a chunk: grow the staging buffers
    for (int k = 0; k < p->depth; ++k) ADCT_CUDA_TRY(cudaStreamSynchronize(p->stream[k]));
    const size_t nb = (unit_bytes + 15) / 16 * 16;
    p->chunk_bytes = 0;  // invalid until every slot is reallocated (a failed grow retries next call)
    for (int k = 0; k < p->depth; ++k) {
      ADCT_CUDA_TRY(cudaFree(p->d_in[k]));
      ADCT_CUDA_TRY(cudaFree(p->d_out[k]));
      p->d_in[k] = p->d_out[k] = nullptr;
    }
    for (int k = 0; k < p->depth; ++k) {
      ADCT_CUDA_TRY(cudaMalloc(&p->d_in[k], nb));
      ADCT_CUDA_TRY(cudaMalloc(&p->d_out[k], nb));
    }
    p->chunk_bytes = nb;
  }
  if (staged && p->h_bytes < p->chunk_bytes) {  // page-locked ring, allocated on first pageable use
    for (int k = 0; k < p->depth; ++k) ADCT_CUDA_TRY(cudaStreamSynchronize(p->stream[k]));
    p->h_bytes = 0;
    for (int k = 0; k < p->depth; ++k) {
      if (p->h_in[k]) ADCT_CUDA_TRY(cudaFreeHost(p->h_in[k]));
      if (p->h_out[k]) ADCT_CUDA_TRY(cudaFreeHost(p->h_out[k]));
      p->h_in[k] = p->h_out[k] = nullptr;
    }
    for (int k = 0; k < p->depth; ++k) {
      ADCT_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&p->h_in[k]), p->chunk_bytes, cudaHostAllocPortable));
      ADCT_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&p->h_out[k]), p->chunk_bytes, cudaHostAllocPortable));
      if (p->done[k] == nullptr) ADCT_CUDA_TRY(cudaEventCreateWithFlags(&p->done[k], cudaEventDisableTiming));
    }
    p->h_bytes = p->chunk_bytes;
    if (p->pool == nullptr) p->pool = new adct::HostCopyPool(adct::HostCopyPool::default_threads());
  }
  if (n_sse > p->sse_cap) {  // grow the per-call device SSE vector
    if (p->d_sse) ADCT_CUDA_TRY(cudaFree(p->d_sse));
    p->d_sse = nullptr;
    p->sse_cap = 0;
    ADCT_CUDA_TRY(cudaMalloc(&p->d_sse, (size_t)n_sse * sizeof(uint64_t)));
    p->sse_cap = n_sse;
  }
  return ADCT_OK;
}

// Page-locked (cudaHostAlloc'ed or cudaHostRegister'ed) host memory?
bool is_pinned(const void* ptr) {
  if (ptr == nullptr) return true;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();  // clear the sticky-free error of an unknown pointer
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// One chunk of host frames of 1..3 planes: how its bytes map between the
// caller's arrays and a frame-interleaved slot [plane 0 | plane 1 | plane 2]
// per frame (a single-image batch is one plane).
struct ChunkMap {
  const adct_plane_t* hp;
  int n_planes;
  size_t off[3];
  size_t frame_bytes;
};

// Host segments (slot <- caller for inputs, caller <- slot for outputs) of frames [f0, f0+m).
void chunk_segments(const ChunkMap& cm, int64_t f0, int64_t m, uint8_t* slot, bool out,
                    std::vector<adct::HostCopyPool::Seg>& segs) {
  segs.clear();
  for (int k = 0; k < cm.n_planes; ++k) {
    const adct_plane_t& q = cm.hp[k];
    const size_t row = (size_t)q.height * q.width;
    if (row == 0 || (out && q.dst == nullptr)) continue;
    const int64_t fs = out ? q.dst_frame_stride : q.src_frame_stride;
    if (cm.n_planes == 1 && (m == 1 || fs == (int64_t)row) && cm.frame_bytes == row) {
      // contiguous frames map onto a contiguous slot: one segment
      if (out) segs.push_back({q.dst + f0 * fs, slot, (size_t)m * row});
      else segs.push_back({slot, q.src + f0 * fs, (size_t)m * row});
      continue;
    }
    for (int64_t f = 0; f < m; ++f) {
      uint8_t* s = slot + (size_t)f * cm.frame_bytes + cm.off[k];
      if (out) segs.push_back({q.dst + (f0 + f) * fs, s, row});
      else segs.push_back({s, q.src + (f0 + f) * fs, row});
    }
  }
}

// The compress launch of one chunk on the device slot.
using ChunkLaunch = int (*)(const adct_plane_t* dev, int n_planes, int64_t m, int kind, int32_t r,
                            const adct_qtab_t* qtab, uint64_t* sse, cudaStream_t s);

int launch_chunk(const adct_plane_t* dev, int n_planes, int64_t m, int kind, int32_t r, const adct_qtab_t* qtab,
                 uint64_t* sse, cudaStream_t s) {
  if (kind == 0) {
    if (n_planes == 1)  // single images: the retain entry point (128-unit pruned kernels)
      return adct_compress_retain(dev[0].src, dev[0].dst, m, dev[0].height, dev[0].width, dev[0].src_frame_stride,
                                  dev[0].dst_frame_stride, r, sse, nullptr, s);
    return adct_compress_retain_planes(dev, n_planes, m, r, sse, s);
  }
  return adct_compress_quant_planes(dev, n_planes, m, qtab, sse, s);
}

// Frames of 1..3 host planes through the device in chunks of whole frames.
// Pinned callers: each chunk is copied straight from/to their arrays (2-D
// copies per plane), chunk i on stream i % depth so the copy engines overlap
// chunk i's D2H with chunk i+1's H2D.  Pageable callers (ordinary numpy
// arrays, never registered per call): the library's own page-locked ring is
// filled and drained by host threads (HostCopyPool) while the previous
// chunks' H2D / kernel / D2H run, one cudaMemcpyAsync per chunk each way.
int pipeline_frames_run(adct_pipeline* p, const adct_plane_t* hp, int32_t n_planes, int64_t n_frames, int kind,
                        int32_t r, const adct_qtab_t* qtab, uint64_t* host_sse) {
  if (p == nullptr || hp == nullptr || n_planes < 1 || n_planes > 3 || n_frames < 0)
    return ADCT_ERR_INVALID_ARGUMENT;
  if (kind == 0 && (r < 1 || r > 64)) return ADCT_ERR_INVALID_RETENTION;
  if (kind == 1 && qtab == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  ChunkMap cm{hp, n_planes, {0, 0, 0}, 0};
  bool any_dst = false, pinned = true;
  for (int k = 0; k < n_planes; ++k) {
    const adct_plane_t& q = hp[k];
    if (q.height < 0 || q.width < 0 || (q.height % 8) || (q.width % 8)) return ADCT_ERR_BAD_DIMENSIONS;
    const int64_t px = (int64_t)q.height * q.width;
    if (n_frames > 0 && px > 0 && q.src == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
    if (n_frames > 1 && (q.src_frame_stride < px || (q.dst && q.dst_frame_stride < px)))
      return ADCT_ERR_INVALID_ARGUMENT;
    cm.off[k] = cm.frame_bytes;
    cm.frame_bytes += n_planes == 1 ? (size_t)px : ((size_t)px + 15) / 16 * 16;
    any_dst = any_dst || q.dst != nullptr;
  }
  if (n_frames == 0) return ADCT_OK;
  if (host_sse == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  if (cm.frame_bytes == 0) {
    std::memset(host_sse, 0, (size_t)n_frames * n_planes * sizeof(uint64_t));
    return ADCT_OK;
  }
  ADCT_CUDA_TRY(cudaSetDevice(p->device));
  for (int k = 0; k < n_planes; ++k)
    pinned = pinned && is_pinned(hp[k].src) && is_pinned(hp[k].dst);
  const bool staged = !pinned;
  int rc0 = pipeline_reserve(p, cm.frame_bytes, n_frames * n_planes, staged);
  if (rc0 != ADCT_OK) return pipeline_fail(p, rc0);
  const int64_t per = (int64_t)(p->chunk_bytes / cm.frame_bytes);
  const int64_t n_chunks = (n_frames + per - 1) / per;
  std::vector<adct::HostCopyPool::Seg> segs;
  auto chunk_frames = [&](int64_t c) { return std::min<int64_t>(per, n_frames - c * per); };
  std::vector<adct::HostCopyPool::Seg> segs_out;
  // staged path: results of chunk c leave the ring once its slot's event
  // fired; their segments join the next input fill in one pool batch
  auto drain = [&](int64_t c, bool run_now) -> int {
    const int b = (int)(c % p->depth);
    ADCT_PIPE_TRY(cudaEventSynchronize(p->done[b]));
    segs_out.clear();
    if (any_dst) chunk_segments(cm, c * per, chunk_frames(c), p->h_out[b], true, segs_out);
    if (run_now) p->pool->run(segs_out);
    return ADCT_OK;
  };
  for (int64_t c = 0; c < n_chunks; ++c) {
    const int b = (int)(c % p->depth);
    const int64_t f0 = c * per, m = chunk_frames(c);
    cudaStream_t s = p->stream[b];
    adct_plane_t dev[3];
    for (int k = 0; k < n_planes; ++k) {
      dev[k].src = p->d_in[b] + cm.off[k];
      dev[k].dst = any_dst ? p->d_out[b] + cm.off[k] : nullptr;
      dev[k].height = hp[k].height;
      dev[k].width = hp[k].width;
      dev[k].src_frame_stride = (int64_t)cm.frame_bytes;
      dev[k].dst_frame_stride = (int64_t)cm.frame_bytes;
    }
    if (staged) {
      segs_out.clear();
      if (c >= p->depth) {  // slot b still holds chunk c - depth
        int rc = drain(c - p->depth, false);
        if (rc != ADCT_OK) return rc;
      }
      chunk_segments(cm, f0, m, p->h_in[b], false, segs);
      segs.insert(segs.end(), segs_out.begin(), segs_out.end());
      p->pool->run(segs);
      ADCT_PIPE_TRY(cudaMemcpyAsync(p->d_in[b], p->h_in[b], (size_t)m * cm.frame_bytes, cudaMemcpyHostToDevice, s));
    } else {
      for (int k = 0; k < n_planes; ++k) {
        const adct_plane_t& q = hp[k];
        const size_t row = (size_t)q.height * q.width;
        const size_t sfs = m > 1 ? (size_t)q.src_frame_stride : row;
        if (row)
          ADCT_PIPE_TRY(cudaMemcpy2DAsync(p->d_in[b] + cm.off[k], cm.frame_bytes, q.src + f0 * q.src_frame_stride,
                                          sfs, row, (size_t)m, cudaMemcpyHostToDevice, s));
      }
    }
    int rc = launch_chunk(dev, n_planes, m, kind, r, qtab, p->d_sse + f0 * n_planes, s);
    if (rc != ADCT_OK) return pipeline_fail(p, rc);
    if (staged) {
      if (any_dst)
        ADCT_PIPE_TRY(cudaMemcpyAsync(p->h_out[b], p->d_out[b], (size_t)m * cm.frame_bytes, cudaMemcpyDeviceToHost, s));
      ADCT_PIPE_TRY(cudaEventRecord(p->done[b], s));
    } else {
      for (int k = 0; k < n_planes; ++k) {
        const adct_plane_t& q = hp[k];
        const size_t row = (size_t)q.height * q.width;
        if (q.dst == nullptr || row == 0) continue;
        const size_t dfs = m > 1 ? (size_t)q.dst_frame_stride : row;
        ADCT_PIPE_TRY(cudaMemcpy2DAsync(q.dst + f0 * q.dst_frame_stride, dfs, p->d_out[b] + cm.off[k],
                                        cm.frame_bytes, row, (size_t)m, cudaMemcpyDeviceToHost, s));
      }
    }
  }
  if (staged)
    for (int64_t c = std::max<int64_t>(0, n_chunks - p->depth); c < n_chunks; ++c) {
      int rc = drain(c, true);
      if (rc != ADCT_OK) return rc;
    }
  for (int k = 0; k < p->depth; ++k) ADCT_PIPE_TRY(cudaStreamSynchronize(p->stream[k]));
  ADCT_PIPE_TRY(cudaMemcpy(host_sse, p->d_sse, (size_t)n_frames * n_planes * sizeof(uint64_t),
                           cudaMemcpyDeviceToHost));
  return ADCT_OK;
}

// kind: 0 retain (r), 1 quant (qtab) — a batch of single images is one plane.
int pipeline_run(adct_pipeline* p, const uint8_t* host_img, uint8_t* host_rec, int64_t n, int32_t h,
                 int32_t w, int kind, int32_t r, const adct_qtab_t* qtab, uint64_t* host_sse) {
  if (p == nullptr || n < 0) return ADCT_ERR_INVALID_ARGUMENT;
  if (h < 0 || w < 0 || (h % 8) || (w % 8)) return ADCT_ERR_BAD_DIMENSIONS;
  if (kind == 0 && (r < 1 || r > 64)) return ADCT_ERR_INVALID_RETENTION;
  if (kind == 1 && qtab == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  if (n == 0) return ADCT_OK;
  if (host_img == nullptr || host_sse == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  adct_plane_t pl = single_plane(host_img, host_rec, h, w, (int64_t)h * w, (int64_t)h * w);
  return pipeline_frames_run(p, &pl, 1, n, kind, r, qtab, host_sse);
}

}  // namespace

extern "C" {

int adct_pipeline_create(int32_t device, size_t chunk_bytes, adct_pipeline_t** out) {
  if (out == nullptr || chunk_bytes < 64) return ADCT_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  adct_pipeline* p = new (std::nothrow) adct_pipeline();
  if (p == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  p->device = device;
  p->chunk_bytes = (chunk_bytes + 15) / 16 * 16;
  if (const char* d = std::getenv("ADCT_PIPELINE_DEPTH")) {
    const int v = std::atoi(d);
    if (v >= 2 && v <= adct_pipeline::kMaxDepth) p->depth = v;
  }
  cudaError_t e = cudaSetDevice(device);
  for (int k = 0; e == cudaSuccess && k < p->depth; ++k) {
    e = cudaStreamCreateWithFlags(&p->stream[k], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_in[k], p->chunk_bytes);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_out[k], p->chunk_bytes);
  }
  if (e != cudaSuccess) {
    pipeline_free(p);
    return cuda_fail(e);
  }
  *out = p;
  return ADCT_OK;
}

int adct_pipeline_destroy(adct_pipeline_t* p) {
  if (p == nullptr) return ADCT_OK;
  pipeline_free(p);
  return ADCT_OK;
}

int adct_pipeline_compress_retain(adct_pipeline_t* p, const uint8_t* host_img, uint8_t* host_rec,
                                  int64_t n, int32_t h, int32_t w, int32_t r, uint64_t* host_sse) {
  if (p == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lk(p->mu);
  return pipeline_run(p, host_img, host_rec, n, h, w, 0, r, nullptr, host_sse);
}

int adct_pipeline_compress_quant(adct_pipeline_t* p, const uint8_t* host_img, uint8_t* host_rec,
                                 int64_t n, int32_t h, int32_t w, const adct_qtab_t* qtab,
                                 uint64_t* host_sse) {
  if (p == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lk(p->mu);
  return pipeline_run(p, host_img, host_rec, n, h, w, 1, 0, qtab, host_sse);
}

int adct_pipeline_compress_quant_planes(adct_pipeline_t* p, const adct_plane_t* host_planes,
                                        int32_t n_planes, int64_t n_frames, const adct_qtab_t* qtab,
                                        uint64_t* host_sse) {
  if (p == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  std::lock_guard<std::mutex> lk(p->mu);
  return pipeline_frames_run(p, host_planes, n_planes, n_frames, 1, 0, qtab, host_sse);
}

int adct_quant_jit_stats(int64_t* compiled, int64_t* launches, int64_t* failures) {
  long long c = 0, l = 0, f = 0;
  jit::stats(&c, &l, &f);
  if (compiled) *compiled = c;
  if (launches) *launches = l;
  if (failures) *failures = f;
  return ADCT_OK;
}

int adct_host_register(void* ptr, size_t bytes) {
  if (ptr == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  if (bytes == 0) return ADCT_OK;
  ADCT_CUDA_TRY(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable));
  return ADCT_OK;
}

int adct_host_is_pinned(const void* ptr) {
  if (ptr == nullptr) return 0;
  return is_pinned(ptr) ? 1 : 0;
}

int adct_host_unregister(void* ptr) {
  if (ptr == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  ADCT_CUDA_TRY(cudaHostUnregister(ptr));
  return ADCT_OK;
}

int adct_host_alloc(size_t bytes, void** out) {
  if (out == nullptr) return ADCT_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (bytes == 0) return ADCT_OK;
  ADCT_CUDA_TRY(cudaHostAlloc(out, bytes, cudaHostAllocPortable));
  return ADCT_OK;
}

int adct_host_free(void* ptr) {
  if (ptr == nullptr) return ADCT_OK;
  ADCT_CUDA_TRY(cudaFreeHost(ptr));
  return ADCT_OK;
}

}  // extern "C"
