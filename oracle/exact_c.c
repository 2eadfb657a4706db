/* exact_c.c — plain-C exact oracle (TEST INFRASTRUCTURE ONLY, see
 * oracle/__init__.py).  Built by oracle/Makefile into oracle/_build/; loaded
 * only by tests/ (as the checker for full-size parity runs) and never by the
 * product library.
 *
 * A second, independent restatement of the reference's hot path next to the
 * numpy oracle (oracle/exact.py), written as straight matrix products with
 * the kernel T (not the 14-add flow graph the CUDA kernels use), so the two
 * share no arithmetic structure:
 *   forward   Z = T X T^T            codec.py:74-81 (forward_2d_unscaled), per
 *                                    _tile block (codec.py:107-131)
 *   retain    keep the first r zigzag positions (codec.py:24-58)
 *   inverse   64 X = T^T (E o Z') T  codec.py:84-87 (inverse_2d with C = D T,
 *                                    D^2 = 1/n folded into E = 64 d^2 d^2^T)
 *   quantise  q = sign(Z) floor((2|Z| + Q') / 2Q'), Z' = q Q'   (BASELINE
 *             configs 2/4 on top of fold_scaling_into_quantization, codec.py:90-104)
 *   round     x = clip(floor((64 x_hat + 32) / 64), 0, 255)     (BASELINE
 *             "round and clamp"; reference keeps floats, codec.py:141)
 *   SSE       sum (x - rec)^2 (metrics.py:49-56 numerator), and the
 *             reference's unrounded convention sum (64 x - clip(64 x_hat, 0, 16320))^2.
 * Everything is exact integer arithmetic (int64 accumulators).
 */
#include <stdint.h>
#include <string.h>

/* The proposed kernel T (kernels.py:35-47, the paper's matrix T). */
static const int T[8][8] = {
    {1, 1, 1, 1, 1, 1, 1, 1},     {1, 0, 0, 0, 0, 0, 0, -1}, {1, 0, 0, -1, -1, 0, 0, 1},
    {0, 0, -1, 0, 0, 1, 0, 0},    {1, -1, -1, 1, 1, -1, -1, 1}, {0, -1, 0, 0, 0, 0, 1, 0},
    {0, -1, 1, 0, 0, 1, -1, 0},   {0, 0, 0, -1, 1, 0, 0, 0},
};

/* E[u][v] = 64 d_u^2 d_v^2 = 64 / (n_u n_v), n = row L1 norms of T
 * (kernels.py:149-157: d = 1/sqrt(n)). */
static int E[8][8];
/* zigzag rank of position u*8+v (codec.py:24-33, JPEG order). */
static int ZZ_RANK[64];
static int g_init = 0;

static void init_tables(void) {
  if (g_init) return;
  int n[8];
  for (int u = 0; u < 8; ++u) {
    n[u] = 0;
    for (int i = 0; i < 8; ++i) n[u] += T[u][i] < 0 ? -T[u][i] : T[u][i];
  }
  for (int u = 0; u < 8; ++u)
    for (int v = 0; v < 8; ++v) E[u][v] = 64 / (n[u] * n[v]);
  int k = 0;
  for (int s = 0; s < 15; ++s) {
    const int lo = s < 8 ? 0 : s - 7, hi = s < 8 ? s : 7;
    if (s % 2 == 0)
      for (int u = hi; u >= lo; --u) ZZ_RANK[u * 8 + (s - u)] = k++;
    else
      for (int u = lo; u <= hi; ++u) ZZ_RANK[u * 8 + (s - u)] = k++;
  }
  g_init = 1;
}

/* tables are built once at load time (the entry points run on many threads) */
__attribute__((constructor)) static void oracle_init(void) { init_tables(); }

/* Z = T X T^T (X given as int64 8x8). */
static void forward_block(const int64_t X[8][8], int64_t Z[8][8]) {
  int64_t t[8][8];
  for (int i = 0; i < 8; ++i)
    for (int v = 0; v < 8; ++v) {
      int64_t a = 0;
      for (int j = 0; j < 8; ++j) a += X[i][j] * T[v][j];
      t[i][v] = a; /* (X T^T)[i][v] */
    }
  for (int u = 0; u < 8; ++u)
    for (int v = 0; v < 8; ++v) {
      int64_t a = 0;
      for (int i = 0; i < 8; ++i) a += T[u][i] * t[i][v];
      Z[u][v] = a;
    }
}

/* V = T^T W T. */
static void inverse_block(const int64_t W[8][8], int64_t V[8][8]) {
  int64_t t[8][8];
  for (int i = 0; i < 8; ++i)
    for (int v = 0; v < 8; ++v) {
      int64_t a = 0;
      for (int u = 0; u < 8; ++u) a += T[u][i] * W[u][v];
      t[i][v] = a; /* (T^T W)[i][v] */
    }
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      int64_t a = 0;
      for (int v = 0; v < 8; ++v) a += t[i][v] * T[v][j];
      V[i][j] = a;
    }
}

static inline int64_t floor_div64(int64_t a) { return a >= 0 ? a / 64 : -((-a + 63) / 64); }

static inline int clamp255(int64_t x) { return x < 0 ? 0 : (x > 255 ? 255 : (int)x); }

static void load_block(const uint8_t* img, int64_t w, int64_t by, int64_t bx, int64_t X[8][8]) {
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) X[i][j] = img[(by * 8 + i) * w + bx * 8 + j];
}

/* Forward coefficients in _tile order: coef[img][block][8][8] (int32). */
int oracle_forward(const uint8_t* img, int64_t n, int32_t h, int32_t w, int64_t stride, int32_t level_shift,
                   int32_t* coef) {
  init_tables();
  const int64_t nbr = h / 8, nbc = w / 8;
  for (int64_t f = 0; f < n; ++f)
    for (int64_t by = 0; by < nbr; ++by)
      for (int64_t bx = 0; bx < nbc; ++bx) {
        int64_t X[8][8], Z[8][8];
        load_block(img + f * stride, w, by, bx, X);
        if (level_shift)
          for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 8; ++j) X[i][j] -= 128;
        forward_block(X, Z);
        int32_t* out = coef + ((f * nbr + by) * nbc + bx) * 64;
        for (int u = 0; u < 8; ++u)
          for (int v = 0; v < 8; ++v) out[u * 8 + v] = (int32_t)Z[u][v];
      }
  return 0;
}

/* Retain-r round trip over block rows [row0, row1) of each of n images.
 * rec (nullable) gets the rounded reconstruction; sse[f] and ssef[f]
 * (nullable) are ACCUMULATED (callers zero them). */
int oracle_compress_retain(const uint8_t* img, int64_t n, int32_t h, int32_t w, int64_t stride, int32_t r,
                           int32_t row0, int32_t row1, uint8_t* rec, int64_t rec_stride, int64_t* sse,
                           int64_t* ssef) {
  init_tables();
  (void)h;
  if (r < 1 || r > 64) return 2;
  const int64_t nbc = w / 8;
  for (int64_t f = 0; f < n; ++f) {
    int64_t acc = 0, accf = 0;
    for (int64_t by = row0; by < row1; ++by)
      for (int64_t bx = 0; bx < nbc; ++bx) {
        int64_t X[8][8], Z[8][8], W[8][8], V[8][8];
        load_block(img + f * stride, w, by, bx, X);
        forward_block(X, Z);
        for (int u = 0; u < 8; ++u)
          for (int v = 0; v < 8; ++v) W[u][v] = ZZ_RANK[u * 8 + v] < r ? E[u][v] * Z[u][v] : 0;
        inverse_block(W, V); /* 64 x_hat, exact */
        for (int i = 0; i < 8; ++i)
          for (int j = 0; j < 8; ++j) {
            const int px = clamp255(floor_div64(V[i][j] + 32));
            if (rec) rec[f * rec_stride + (by * 8 + i) * w + bx * 8 + j] = (uint8_t)px;
            const int64_t d = X[i][j] - px;
            acc += d * d;
            const int64_t vf = V[i][j] < 0 ? 0 : (V[i][j] > 16320 ? 16320 : V[i][j]);
            const int64_t df = 64 * X[i][j] - vf;
            accf += df * df;
          }
      }
    if (sse) sse[f] += acc;
    if (ssef) ssef[f] += accf;
  }
  return 0;
}

/* SSE for every r in [r_min, r_max] (the run_sweep loop, cli.py:101-113),
 * block rows [row0, row1); sse[f][k] and ssef[f][k] (nullable) ACCUMULATED. */
int oracle_sweep_sse(const uint8_t* img, int64_t n, int32_t h, int32_t w, int64_t stride, int32_t r_min,
                     int32_t r_max, int32_t row0, int32_t row1, int64_t* sse, int64_t* ssef) {
  init_tables();
  (void)h;
  if (r_min < 1 || r_max > 64 || r_min > r_max) return 2;
  const int nr = r_max - r_min + 1;
  const int64_t nbc = w / 8;
  for (int64_t f = 0; f < n; ++f)
    for (int64_t by = row0; by < row1; ++by)
      for (int64_t bx = 0; bx < nbc; ++bx) {
        int64_t X[8][8], Z[8][8], W[8][8], V[8][8];
        load_block(img + f * stride, w, by, bx, X);
        forward_block(X, Z);
        for (int k = 0; k < nr; ++k) {
          const int r = r_min + k;
          for (int u = 0; u < 8; ++u)
            for (int v = 0; v < 8; ++v) W[u][v] = ZZ_RANK[u * 8 + v] < r ? E[u][v] * Z[u][v] : 0;
          inverse_block(W, V);
          int64_t acc = 0, accf = 0;
          for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 8; ++j) {
              const int64_t d = X[i][j] - clamp255(floor_div64(V[i][j] + 32));
              acc += d * d;
              const int64_t vf = V[i][j] < 0 ? 0 : (V[i][j] > 16320 ? 16320 : V[i][j]);
              const int64_t df = 64 * X[i][j] - vf;
              accf += df * df;
            }
          sse[f * nr + k] += acc;
          if (ssef) ssef[f * nr + k] += accf;
        }
      }
  return 0;
}

/* Quantised pipeline (BASELINE configs 2/4) over block rows [row0, row1):
 * level shift, Z = T (X-128) T^T, q = round_half_away(Z / Q'), Z' = q Q',
 * 64 (x_hat - 128) = T^T (E o Z') T, +128, round, clamp.  qp: 64 rounded Q'
 * (row-major).  sse[f] ACCUMULATED. */
int oracle_compress_quant(const uint8_t* img, int64_t n, int32_t h, int32_t w, int64_t stride,
                          const int32_t* qp, int32_t row0, int32_t row1, uint8_t* rec, int64_t rec_stride,
                          int64_t* sse) {
  init_tables();
  (void)h;
  for (int p = 0; p < 64; ++p)
    if (qp[p] < 1) return 3;
  const int64_t nbc = w / 8;
  for (int64_t f = 0; f < n; ++f) {
    int64_t acc = 0;
    for (int64_t by = row0; by < row1; ++by)
      for (int64_t bx = 0; bx < nbc; ++bx) {
        int64_t X[8][8], Z[8][8], W[8][8], V[8][8], Xs[8][8];
        load_block(img + f * stride, w, by, bx, X);
        for (int i = 0; i < 8; ++i)
          for (int j = 0; j < 8; ++j) Xs[i][j] = X[i][j] - 128;
        forward_block(Xs, Z);
        for (int u = 0; u < 8; ++u)
          for (int v = 0; v < 8; ++v) {
            const int64_t Q = qp[u * 8 + v], z = Z[u][v];
            const int64_t a = (2 * (z < 0 ? -z : z) + Q) / (2 * Q);
            W[u][v] = E[u][v] * (z < 0 ? -a : a) * Q;
          }
        inverse_block(W, V); /* 64 (x_hat - 128) */
        for (int i = 0; i < 8; ++i)
          for (int j = 0; j < 8; ++j) {
            const int px = clamp255(floor_div64(V[i][j] + 32) + 128);
            if (rec) rec[f * rec_stride + (by * 8 + i) * w + bx * 8 + j] = (uint8_t)px;
            const int64_t d = X[i][j] - px;
            acc += d * d;
          }
      }
    if (sse) sse[f] += acc;
  }
  return 0;
}
