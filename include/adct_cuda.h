/*
 * adct_cuda.h — C ABI of libadct_cuda.so, the B200 (sm_100a) implementation of
 * the blockwise 8x8 approximate-DCT hot path of arxiv 1702.00817
 * (reference package `adct`, /root/reference/pkg/src/adct).
 *
 * The reference has no FFI: its boundary is the Python codec/metrics API
 * (codec.py:53-155, metrics.py:49-65).  Each entry point below names the
 * reference function(s) it replaces.  A maintainer binds them with ctypes
 * (INTEGRATION.md); the in-tree binding is paper_1702_00817_b200/_lib.py.
 *
 * Conventions (all entry points):
 *   - Plain C types only.  Pointers documented "device" must be CUDA device
 *     (or managed) memory owned by the caller; "host" pointers are CPU memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Device entry points are asynchronous on that stream, never allocate,
 *     never synchronise, keep no global mutable state and are reentrant.
 *   - Images are 8-bit, row-major with row pitch == width; image k of a batch
 *     starts at base + k*image_stride (elements).  height and width must be
 *     multiples of 8 (reference: BadDimensions, codec.py:128-129).
 *   - Block order of coefficient outputs is the reference's `_tile` order
 *     (codec.py:107-109): raster over block rows, then block columns.
 *   - Return value: ADCT_OK or one of the error codes; validation happens
 *     before anything is enqueued (reference raises before compute).
 *   - SSE outputs are zeroed by the call (on the stream) and then accumulated
 *     with integer atomics, so they are exact and order independent.
 */
#ifndef ADCT_CUDA_H
#define ADCT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes.  The first four mirror the reference's contract errors. */
enum {
  ADCT_OK = 0,
  ADCT_ERR_BAD_DIMENSIONS = 1,         /* adct.errors.BadDimensions      (errors.py:29) */
  ADCT_ERR_INVALID_RETENTION = 2,      /* adct.errors.InvalidRetention   (errors.py:21) */
  ADCT_ERR_NON_POSITIVE_QUANTIZER = 3, /* adct.errors.NonPositiveQuantizer (errors.py:25) */
  ADCT_ERR_DIMENSION_MISMATCH = 4,     /* adct.errors.DimensionMismatch  (errors.py:33) */
  ADCT_ERR_INVALID_ARGUMENT = 5,       /* null pointer, negative count, bad plane count */
  ADCT_ERR_MISALIGNED = 6,             /* base pointer or stride not 8-byte aligned */
  ADCT_ERR_CUDA = 7,                   /* a CUDA runtime call failed (see adct_last_cuda_error) */
  ADCT_ERR_UNSUPPORTED = 8             /* quantiser table outside the exactly-provable range */
};

/* Library version (major*10000 + minor*100 + patch) and error strings. */
int adct_version(void);
const char* adct_strerror(int code);
/* cudaError_t of the most recent ADCT_ERR_CUDA on the calling thread. */
int adct_last_cuda_error(void);

/* ---------------------------------------------------------------------------
 * Quantiser table (BASELINE configs 2 and 4).
 *
 * Q'[u][v] = max(1, round_half_away(Q[u][v] / (d[u] d[v]))), the reference's
 * fold_scaling_into_quantization (codec.py:90-104) followed by the rounding
 * BASELINE.json specifies.  The device quantiser computes
 *   q = sign(Z) * floor((2|Z| + Q') / (2 Q'))      (round half away from zero)
 *   Z' = q * Q'
 * exactly with one multiply-high per coefficient; the constants below make
 * it exact and are verified exhaustively over every reachable coefficient
 * (|Z| <= 8192) by adct_qtab_build.  Treat the struct as opaque except for
 * `qprime`, `qe`, `wide`, `max_abs_v` and `aligned`.
 * ------------------------------------------------------------------------- */
typedef struct adct_qtab {
  int32_t qprime[64];   /* rounded Q', row-major (u*8+v) */
  int32_t qe[64];       /* Q' * E[u][v], E = 64 d[u]^2 d[v]^2 in {1,2,4,8,16} */
  /* Two-lane quantiser (wide == 0): for each 16-bit lane Z,
   *   U = (Z + bias) * mult + [Z >= 0],  q = umulhi(U, magic) - kq,
   * mult = 2 and divisor 2Q' for odd Q', mult = 1 and divisor Q' for even Q'. */
  uint32_t magic[64];
  int32_t bias[64];
  int32_t mult[64];
  int32_t kq[64];
  /* Scalar quantiser (any table): U = 2Z - [Z<0] + cadd,
   *   q = umulhi(U, magic_w) - kw  (divisor 2Q'; shift_w is always 0 and is
   *   kept for layout: for Q' > 16384 the quotient window is identically 0). */
  uint32_t magic_w[64];
  int32_t cadd_w[64];
  int32_t kw[64];
  int32_t shift_w[64];
  int32_t wide;         /* 1: 16-bit-lane inverse not provably exact -> one block per thread */
  int32_t max_abs_v;    /* proven bound of |64*(x_hat-128)| before clamping */
  int32_t quality;      /* JPEG quality used to build it, or -1 for an explicit table */
  int32_t aligned;      /* 1: max_abs_v + 32 <= 24575: fused one-op output clamp, no bit flip */
  /* Float quantiser (default device path): q = RN(1.5*2^23 + Z * r) - 1.5*2^23
   * in fp32 (one FFMA2 per lane pair), r = the float bits below, chosen just
   * above 1/Q' so exact ties round away from zero; verified exhaustively over
   * |Z| <= 8192 like the integer constants above. */
  uint32_t recip_f[64];
} adct_qtab_t;

/* Build from an unrounded Q' table (64 float64, row-major), i.e. the output of
 * the reference's fold_scaling_into_quantization.  Host-only, no CUDA.
 * Errors: NON_POSITIVE_QUANTIZER if any entry <= 0 or not finite;
 * UNSUPPORTED if the table cannot be handled exactly. */
int adct_qtab_build(const double* qprime_unrounded, adct_qtab_t* out);

/* Convenience: Q' from the standard JPEG luminance table Q50 (`base`, 64
 * int32, row-major) and JPEG quality q in [1,100] with the IJG scale
 * s(q) = 50/q (q<50) or 2 - q/50 (q>=50):
 *   Q'[u][v] = max(1, round_half_away(Q50[u][v] * s(q) / (d[u] d[v]))).
 * Errors: INVALID_ARGUMENT for q outside [1,100] or null pointers. */
int adct_qtab_from_quality(const int32_t* base, int32_t quality, adct_qtab_t* out);

/* ---------------------------------------------------------------------------
 * K1 — forward integer transform.
 * Replaces forward_2d_unscaled (codec.py:74-81) batched like
 * coefficient_blocks (codec.py:120-131): coef = T * X * T^T per 8x8 block,
 * exact.  level_shift != 0 transforms X-128 instead (DC - 8192).
 * coef: device int32 [n][h/8*w/8][8][8]. */
int adct_forward_int32(const uint8_t* img, int64_t n, int32_t h, int32_t w,
                       int64_t img_stride, int32_t level_shift, int32_t* coef,
                       void* stream);
/* Same, int16 output (|coef| <= 16320 always fits). */
int adct_forward_int16(const uint8_t* img, int64_t n, int32_t h, int32_t w,
                       int64_t img_stride, int32_t level_shift, int16_t* coef,
                       void* stream);

/* ---------------------------------------------------------------------------
 * K2 + K4 — fused retain-r compression.
 * Replaces compress_image (codec.py:144-155) + mse (metrics.py:49-56) for a
 * batch: forward, keep the first r zigzag coefficients (codec.py:24-50),
 * orthonormal inverse, round (half away from zero) and clamp to [0,255].
 * Reads each pixel once and writes each reconstructed pixel once.
 *   rec           device uint8 [n][h][w] (rec_stride apart), nullable
 *   sse           device uint64 [n]: sum over pixels of (x - rec)^2, nullable
 *   sse_unrounded device uint64 [n], nullable: sum of (64 x - clamp(64 x_hat,
 *                 0, 16320))^2, i.e. 4096 * the reference's own unrounded
 *                 clamped SSE (codec.py:141, metrics.py:56), exactly.
 * Errors: INVALID_RETENTION unless 1 <= r <= 64. */
int adct_compress_retain(const uint8_t* img, uint8_t* rec, int64_t n, int32_t h,
                         int32_t w, int64_t img_stride, int64_t rec_stride,
                         int32_t r, uint64_t* sse, uint64_t* sse_unrounded,
                         void* stream);

/* adct_compress_retain with the cross-GPU SSE exchange fused into the kernel
 * epilogue (replaces the separate all-reduce of the SSE
 * vector).  When the last CTA of image i finishes, it stores the image's
 * exact SSE into peer_sse[p][peer_offset + i] for every p < n_peers.
 *   sse        device uint64 [n]: local accumulator (zeroed by the call)
 *   peer_sse   DEVICE array of n_peers device pointers (symmetric / peer-
 *              mapped memory, e.g. torch symmetric memory buffer_ptrs_dev),
 *              each to a uint64 vector with >= peer_offset + n entries
 *   arrivals   device uint32 [n], zero before the first call; every call
 *              leaves it zero again
 * The caller orders peers' reads after every rank's launch (e.g. a stream-
 * ordered symmetric-memory barrier).  Single plane, rounded SSE only. */
int adct_compress_retain_exchange(const uint8_t* img, uint8_t* rec, int64_t n, int32_t h,
                                  int32_t w, int64_t img_stride, int64_t rec_stride, int32_t r,
                                  uint64_t* sse, uint64_t* const* peer_sse, int32_t n_peers,
                                  int64_t peer_offset, uint32_t* arrivals, void* stream);

/* ---------------------------------------------------------------------------
 * K3 + K4 — fused quantised compression (single plane batch).
 * Level shift -128, forward T X T^T, quantise by Q' (round half away),
 * dequantise, inverse T^T D Y D T, +128, round, clamp; per-image SSE.
 * New (the reference has no quantised pipeline; BASELINE config 2).
 * Kernel choice is internal: tables whose reconstruction fits 16-bit lanes
 * run the packed kernel; coarser ones (e.g. q = 10) the float-pair inverse;
 * tables beyond both exactness bounds the 32-bit scalar kernel.  Results
 * are identical (exact) either way. */
int adct_compress_quant(const uint8_t* img, uint8_t* rec, int64_t n, int32_t h,
                        int32_t w, int64_t img_stride, int64_t rec_stride,
                        const adct_qtab_t* qtab, uint64_t* sse, void* stream);

/* K6 — several planes (e.g. Y, Cb, Cr of 4:2:0 frames) in ONE launch. */
typedef struct adct_plane {
  const uint8_t* src;       /* device, frame f at src + f*src_frame_stride */
  uint8_t* dst;             /* device, nullable */
  int32_t height, width;    /* multiples of 8 */
  int64_t src_frame_stride; /* elements */
  int64_t dst_frame_stride; /* elements */
} adct_plane_t;

/* sse: device uint64 [n_frames][n_planes]; 1 <= n_planes <= 3. */
int adct_compress_quant_planes(const adct_plane_t* planes, int32_t n_planes,
                               int64_t n_frames, const adct_qtab_t* qtab,
                               uint64_t* sse, void* stream);
/* adct_compress_quant_planes plus the SSE exchange: stream-ordered after the
 * compress kernel, a small push kernel stores the exact SSE of (frame f,
 * plane k) into peer_sse[p][peer_offset + f*n_planes + k] for every peer
 * (P2P stores; no collective).  Unlike the memory-bound retain kernel, the
 * issue-bound quant kernels lose 19-22 % with the exchange inside their
 * epilogue, hence the separate push.  `arrivals` is unused (may be NULL). */
int adct_compress_quant_planes_exchange(const adct_plane_t* planes, int32_t n_planes,
                                        int64_t n_frames, const adct_qtab_t* qtab, uint64_t* sse,
                                        uint64_t* const* peer_sse, int32_t n_peers,
                                        int64_t peer_offset, uint32_t* arrivals, void* stream);
/* Retain-r over planes in one launch (sse as above). */
int adct_compress_retain_planes(const adct_plane_t* planes, int32_t n_planes,
                                int64_t n_frames, int32_t r, uint64_t* sse,
                                void* stream);

/* ---------------------------------------------------------------------------
 * K7 — retain-r sweep: one read of each image, SSE for every r in
 * [r_min, r_max].  Replaces the per-r loop of cli.run_sweep
 * (cli.py:101-113: reconstruct_image + mse per r).
 * sse:           device uint64 [n][r_max - r_min + 1], rounded reconstructions;
 *                nullable when sse_unrounded is given (then only that is computed)
 * sse_unrounded: device uint64 [n][r_max - r_min + 1], nullable; 4096 x the
 *                reference's own unrounded clamped SSE (exact). */
int adct_sweep_retain_sse(const uint8_t* img, int64_t n, int32_t h, int32_t w,
                          int64_t img_stride, int32_t r_min, int32_t r_max,
                          uint64_t* sse, uint64_t* sse_unrounded, void* stream);

/* ---------------------------------------------------------------------------
 * Dense 8x8 transforms in float64 for any 8x8 matrix C (SURVEY §8f row f1:
 * the exact DCT, kernels.py:166-178, and the registry's comparison kernels,
 * kernels.py:228-327).  `C` is a HOST pointer to 64 float64 (row-major, the
 * transform's .matrix), passed to the kernel by value.  Images are uint8
 * (img_is_f64 == 0) or float64 (img_is_f64 != 0), like the reference's
 * float64 samples.
 *   adct_forward_dense:  coef = C X C^T per block (coefficient_blocks, codec.py:120-131)
 *   adct_inverse_dense:  out = clamp?(untile(C^T mask_r(coef) C))  (reconstruct_image, codec.py:134-141)
 *   adct_sweep_dense:    sse[n][r] = sum (x - clamp(C^T mask_r(C X C^T) C, 0, 255))^2,
 *                        float64, every r in [r_min, r_max] (cli.py:105-113). */
int adct_forward_dense(const void* img, int32_t img_is_f64, int64_t n, int32_t h, int32_t w,
                       const double* C, double* coef, void* stream);
int adct_inverse_dense(const double* coef, int64_t n, int32_t h, int32_t w, const double* C,
                       int32_t r, int32_t clamp, double* out, void* stream);
int adct_sweep_dense(const void* img, int32_t img_is_f64, int64_t n, int32_t h, int32_t w,
                     const double* C, int32_t r_min, int32_t r_max, double* sse, void* stream);

/* ---------------------------------------------------------------------------
 * Real-valued (float64) transforms, for the reference's float API on
 * non-integral data (the reference accepts any real image, codec.py:127).
 *   adct_forward_f64:  coef = C X C^T per block, C = D T  (forward_2d /
 *                      coefficient_blocks, codec.py:68-71, 120-131)
 *   adct_inverse_f64:  out = clamp?(untile(C^T mask_r(coef) C))
 *                      (inverse_2d / reconstruct_image, codec.py:84-87,
 *                      134-141); r in [1,64] (64 = no truncation),
 *                      clamp != 0 clamps to [0,255] like codec.py:141.
 * img/out: device float64 [n][h][w]; coef: device float64 [n][h*w/64][8][8]. */
int adct_forward_f64(const double* img, int64_t n, int32_t h, int32_t w,
                     double* coef, void* stream);
/* Same for uint8 images (the reference converts them to float64 first,
 * codec.py:127; here the kernel reads the bytes: 1 B per pixel in). */
int adct_forward_f64_u8(const uint8_t* img, int64_t n, int32_t h, int32_t w,
                        double* coef, void* stream);
int adct_inverse_f64(const double* coef, int64_t n, int32_t h, int32_t w,
                     int32_t r, int32_t clamp, double* out, void* stream);

/* Device SSE between two uint8 batches (metrics.mse numerator,
 * metrics.py:49-56).  sse: device uint64 [n]. */
int adct_sse_u8(const uint8_t* a, const uint8_t* b, int64_t n, int64_t numel,
                int64_t stride_a, int64_t stride_b, uint64_t* sse, void* stream);

/* ---------------------------------------------------------------------------
 * Synthetic image generator (BASELINE.json configs; not a reference API).
 * pixel = clip(rint(128 + sum_k amp_k exp(-((y-cy_k)^2+(x-cx_k)^2)/(2 sig_k^2))
 *                   + 4 * N(0,1)), 0, 255)
 * blobs: device float32 [n][n_blobs][4] = (cy, cx, sigma, amp) per image;
 * noise_seed: device uint64 [n]; N(0,1) comes from a counter-based hash of
 * (noise_seed, y, x), identical on every GPU count. */
int adct_synth_blobs(uint8_t* out, int64_t n, int32_t h, int32_t w,
                     int64_t img_stride, const float* blobs, int32_t n_blobs,
                     const uint64_t* noise_seed, void* stream);

/* ---------------------------------------------------------------------------
 * Host-buffer pipeline (the end-to-end entry point).  Replaces the host-side
 * per-image loop of the reference (numpy images from corpus.read_pgm,
 * corpus.py:65-111, each through compress_image + mse, cli.py:101-113) for
 * whole batches: H2D copy of chunk i+1, fused compress of chunk i and D2H
 * copy of chunk i-1 overlap on separate streams.
 * Host buffers may be ordinary pageable memory (e.g. numpy arrays): the
 * pipeline then stages every chunk through its own page-locked ring (host
 * threads fill and drain it while the previous chunks' copies and kernels
 * run; nothing is registered per call; ADCT_PIPELINE_THREADS sets the
 * thread count).  Page-locked buffers (adct_host_alloc, cudaHostAlloc, or
 * adct_host_register'd) skip the staging and are copied directly — the
 * fastest case.  Errors drain every pipeline stream before returning.
 * ------------------------------------------------------------------------- */
typedef struct adct_pipeline adct_pipeline_t;

int adct_pipeline_create(int32_t device, size_t chunk_bytes, adct_pipeline_t** out);
int adct_pipeline_destroy(adct_pipeline_t* p);
/* host_rec nullable; host_sse: host uint64 [n].  Blocks until done.
 * Calls on one pipeline from several threads are serialised (a pipeline is
 * one set of streams and staging slots); use one pipeline per thread for
 * concurrent transfers. */
int adct_pipeline_compress_retain(adct_pipeline_t* p, const uint8_t* host_img,
                                  uint8_t* host_rec, int64_t n, int32_t h, int32_t w,
                                  int32_t r, uint64_t* host_sse);
int adct_pipeline_compress_quant(adct_pipeline_t* p, const uint8_t* host_img,
                                 uint8_t* host_rec, int64_t n, int32_t h, int32_t w,
                                 const adct_qtab_t* qtab, uint64_t* host_sse);
/* Frames of 1..3 planes in HOST memory (adct_plane_t with host src/dst;
 * dst nullable): the quantised pipeline of adct_compress_quant_planes,
 * streamed in chunks of frames.  host_sse: uint64 [n_frames][n_planes]. */
int adct_pipeline_compress_quant_planes(adct_pipeline_t* p, const adct_plane_t* host_planes,
                                        int32_t n_planes, int64_t n_frames, const adct_qtab_t* qtab,
                                        uint64_t* host_sse);
/* Run-time specialisation of the quantised kernels (adct_compress_quant*):
 * once a quantiser table has been used ADCT_QUANT_JIT_AFTER times (env,
 * default 3, 0 = never), the kernel is rebuilt with NVRTC with that table as
 * compile-time constants and cached for the process (same results, ~5 % faster;
 * without NVRTC the generic kernel keeps running).  Counters since load. */
int adct_quant_jit_stats(int64_t* compiled, int64_t* launches, int64_t* failures);
/* Page-lock / unlock caller memory (cudaHostRegister). */
int adct_host_register(void* ptr, size_t bytes);
int adct_host_unregister(void* ptr);
/* 1 if ptr is page-locked host memory (cudaHostAlloc'ed or registered), else 0. */
int adct_host_is_pinned(const void* ptr);
/* Page-locked host allocation (cudaHostAlloc, portable); *out = NULL for 0 bytes. */
int adct_host_alloc(size_t bytes, void** out);
int adct_host_free(void* ptr);

#ifdef __cplusplus
}
#endif

#endif /* ADCT_CUDA_H */
