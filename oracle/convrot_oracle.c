/*
 * convrot_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A plain-C restatement of the reference's CPU ConvLinear4bit path, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg to check
 * the CUDA product path.  Nothing in paper_2512_03673_b200/ links or calls
 * this file.  Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).  Build flags MUST keep
 * -ffp-contract=off (reference: CMakeLists.txt:11-12) so that the double
 * arithmetic below rounds exactly like the reference's.
 *
 * Parity pinning: tests/test_oracle.py checks this file against
 *   - the reference's own known answers (test_hadamard.cpp, test_quant.cpp,
 *     test_pipeline.cpp:191 golden 0.12035518741210707, test_analysis.cpp
 *     RNG amplitudes), and
 *   - golden vectors produced by the real reference compiled from
 *     /root/reference (oracle/_ref, recipe oracle/Makefile), committed
 *     under tests/golden/ with the script that made them.
 *
 * Status codes mirror the reference exception taxonomy (errors.hpp:9-67),
 * the same numbering as include/crt/convlinear4bit.h.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum {
  OR_OK = 0,
  OR_ERR_INVALID_ORDER = 1,
  OR_ERR_INVALID_VALUE = 2,
  OR_ERR_SHAPE = 3,
  OR_ERR_CAPACITY = 4,
};

enum { OR_ROT_NONE = 0, OR_ROT_SYLVESTER = 1, OR_ROT_REGULAR = 2 };

#define OR_MAX_ORDER 4096 /* hadamard.hpp:12 kMaxHadamardOrder */

static int is_pow2(long n) { return n > 0 && (n & (n - 1)) == 0; }
/* hadamard.cpp:16-18 / pipeline.cpp:22-24 */
static int is_pow4(long n) { return is_pow2(n) && (n & 0x55555555L) != 0; }

/* ---------------------------------------------------------------------- */
/* Hadamard sign matrices                                                  */
/* ---------------------------------------------------------------------- */

/* regular(n): Kronecker powers of the order-4 seed, hadamard.cpp:91-106;
 * kronecker entry rule out[i*nb+p][j*nb+q] = a[i][j]*b[p][q], :108-126.
 * Writes n*n signs (+1/-1) row-major. */
int or_regular(int n, int8_t* out) {
  static const int8_t h4[16] = {1, 1, 1, -1, 1, 1, -1, 1,
                                1, -1, 1, 1, -1, 1, 1, 1};
  if (!is_pow4(n) || n < 4) return OR_ERR_INVALID_ORDER; /* :92-95 */
  if (n > OR_MAX_ORDER) return OR_ERR_INVALID_ORDER;     /* :96 */
  int8_t* cur = (int8_t*)malloc((size_t)n * n);
  int8_t* nxt = (int8_t*)malloc((size_t)n * n);
  if (!cur || !nxt) { free(cur); free(nxt); return OR_ERR_INVALID_VALUE; }
  memcpy(cur, h4, 16);
  int order = 4;
  while (order < n) { /* h = kronecker(h, seed), :104 */
    int no = order * 4;
    for (int i = 0; i < order; ++i)
      for (int j = 0; j < order; ++j)
        for (int p = 0; p < 4; ++p)
          for (int q = 0; q < 4; ++q)
            nxt[(size_t)(i * 4 + p) * no + (j * 4 + q)] =
                (int8_t)(cur[(size_t)i * order + j] * h4[p * 4 + q]);
    int8_t* t = cur; cur = nxt; nxt = t;
    order = no;
  }
  memcpy(out, cur, (size_t)n * n);
  free(cur); free(nxt);
  return OR_OK;
}

/* sylvester(n): doubling recursion, hadamard.cpp:70-89. */
int or_sylvester(int n, int8_t* out) {
  if (!is_pow2(n)) return OR_ERR_INVALID_ORDER;
  if (n > OR_MAX_ORDER) return OR_ERR_INVALID_ORDER;
  memset(out, 0, (size_t)n * n);
  out[0] = 1;
  for (int m = 1; m < n; m *= 2)
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        int8_t v = out[(size_t)i * n + j];
        out[(size_t)i * n + j + m] = v;
        out[(size_t)(i + m) * n + j] = v;
        out[(size_t)(i + m) * n + j + m] = (int8_t)-v;
      }
  return OR_OK;
}

/* check_group_order, pipeline.cpp:27-50 (none/sylvester/regular only). */
static int check_group_order(int kind, long group) {
  if (kind == OR_ROT_NONE) return OR_OK;
  if (kind == OR_ROT_SYLVESTER) return is_pow2(group) ? OR_OK : OR_ERR_INVALID_ORDER;
  if (kind == OR_ROT_REGULAR)
    return (is_pow4(group) && group >= 4) ? OR_OK : OR_ERR_INVALID_ORDER;
  return OR_ERR_INVALID_VALUE;
}

/* build_rotation, pipeline.cpp:52-66: R = +-1/sqrt(group) in double. */
static int build_rotation(int kind, int group, double* r) {
  int8_t* h = (int8_t*)malloc((size_t)group * group);
  if (!h) return OR_ERR_INVALID_VALUE;
  int st = kind == OR_ROT_SYLVESTER ? or_sylvester(group, h) : or_regular(group, h);
  if (st != OR_OK) { free(h); return st; }
  double inv_sqrt = 1.0 / sqrt((double)group);
  for (size_t i = 0; i < (size_t)group * group; ++i)
    r[i] = h[i] > 0 ? inv_sqrt : -inv_sqrt;
  free(h);
  return OR_OK;
}

/* ---------------------------------------------------------------------- */
/* group_rotate, pipeline.cpp:111-151                                      */
/* ---------------------------------------------------------------------- */
/* out[m, b*g+j] = sum_{k<g} x[m, b*g+k] * R[k][j], ascending k, no FMA
 * (:134-142).  group 0 = global (:120-122).  Non-divisible widths need
 * identity_tail (:124-130); the tail passes through (:144). */
int or_group_rotate(const double* x, int64_t rows, int64_t cols, int kind,
                    int group_size, int identity_tail, double* out) {
  if (kind == OR_ROT_NONE) { /* :114 returns x unchanged */
    memcpy(out, x, sizeof(double) * (size_t)(rows * cols));
    return OR_OK;
  }
  if (cols == 0) return OR_ERR_SHAPE;              /* :116 */
  if (group_size < 0) return OR_ERR_INVALID_VALUE; /* :117-119 */
  int64_t group = group_size == 0 ? cols : group_size;
  int st = check_group_order(kind, (long)group);
  if (st != OR_OK) return st;
  int64_t blocks = cols / group;
  int64_t rotated = blocks * group;
  if (rotated != cols && !identity_tail) return OR_ERR_SHAPE;
  double* r = (double*)malloc(sizeof(double) * (size_t)(group * group));
  if (!r) return OR_ERR_INVALID_VALUE;
  st = build_rotation(kind, (int)group, r);
  if (st != OR_OK) { free(r); return st; }
  for (int64_t m = 0; m < rows; ++m) {
    const double* xr = x + m * cols;
    double* orow = out + m * cols;
    for (int64_t b = 0; b < blocks; ++b) {
      int64_t base = b * group;
      for (int64_t j = 0; j < group; ++j) {
        double acc = 0.0;
        for (int64_t k = 0; k < group; ++k) acc += xr[base + k] * r[k * group + j];
        orow[base + j] = acc;
      }
    }
    for (int64_t j = rotated; j < cols; ++j) orow[j] = xr[j];
  }
  free(r);
  return OR_OK;
}

/* ---------------------------------------------------------------------- */
/* quantizer, quant.cpp:10-81                                              */
/* ---------------------------------------------------------------------- */
static int qmax_of(int bits) { return (1 << (bits - 1)) - 1; } /* quant.hpp:19 */

/* compute_scales, quant.cpp:10-24: s = max|x| / qmax, 1.0 for zero rows,
 * INVALID_VALUE on non-finite input. */
int or_compute_scales(const double* x, int64_t rows, int64_t cols, int bits,
                      double* scales) {
  double qmax = (double)qmax_of(bits);
  for (int64_t i = 0; i < rows; ++i) {
    double max_abs = 0.0;
    for (int64_t j = 0; j < cols; ++j) {
      double v = x[i * cols + j];
      if (!isfinite(v)) return OR_ERR_INVALID_VALUE;
      double a = fabs(v);
      max_abs = max_abs < a ? a : max_abs; /* std::max(max_abs, |v|) */
    }
    scales[i] = max_abs == 0.0 ? 1.0 : max_abs / qmax;
  }
  return OR_OK;
}

/* quantize, quant.cpp:26-52: code = clamp(nearbyint(x / s), -qmax, qmax),
 * a true double division rounded half-to-even (FE_TONEAREST). */
int or_quantize(const double* x, int64_t rows, int64_t cols,
                const double* scales, int bits, int8_t* codes) {
  for (int64_t i = 0; i < rows; ++i)
    if (!(scales[i] > 0.0) || !isfinite(scales[i])) return OR_ERR_INVALID_VALUE;
  double qmax = (double)qmax_of(bits);
  for (int64_t i = 0; i < rows; ++i) {
    double s = scales[i];
    for (int64_t j = 0; j < cols; ++j) {
      double rounded = nearbyint(x[i * cols + j] / s);
      if (rounded < -qmax) rounded = -qmax;
      if (rounded > qmax) rounded = qmax;
      codes[i * cols + j] = (int8_t)rounded;
    }
  }
  return OR_OK;
}

/* pack_int4, quant.cpp:64-81: element 2t -> low nibble of byte t, 2t+1 ->
 * high nibble; odd counts pad a zero nibble; codes outside [-8,7] reject. */
int or_pack_int4(const int8_t* codes, int64_t n, uint8_t* out) {
  for (int64_t t = 0; t < n; ++t)
    if (codes[t] < -8 || codes[t] > 7) return OR_ERR_INVALID_VALUE;
  memset(out, 0, (size_t)((n + 1) / 2));
  for (int64_t t = 0; t < n; ++t) {
    uint8_t nib = (uint8_t)codes[t] & 0x0F;
    if (t % 2 == 0) out[t / 2] |= nib;
    else out[t / 2] |= (uint8_t)(nib << 4);
  }
  return OR_OK;
}

/* unpack_int4, quant.cpp:83-96 (sign-extending). */
void or_unpack_int4(const uint8_t* bytes, int64_t n, int8_t* codes) {
  for (int64_t t = 0; t < n; ++t) {
    uint8_t nib = t % 2 == 0 ? (uint8_t)(bytes[t / 2] & 0x0F) : (uint8_t)(bytes[t / 2] >> 4);
    codes[t] = (int8_t)(nib >= 8 ? (int)nib - 16 : (int)nib);
  }
}

/* Row-wise packing as the CRT1 packed_i4 writer does it (tensorio.cpp:
 * 162-171): each row is packed independently, padded to a whole byte. */
int or_pack_int4_rows(const int8_t* codes, int64_t rows, int64_t cols, uint8_t* out) {
  int64_t rb = (cols + 1) / 2;
  for (int64_t i = 0; i < rows; ++i) {
    int st = or_pack_int4(codes + i * cols, cols, out + i * rb);
    if (st != OR_OK) return st;
  }
  return OR_OK;
}

/* ---------------------------------------------------------------------- */
/* int_gemm, pipeline.cpp:178-204                                          */
/* ---------------------------------------------------------------------- */
/* Capacity precheck qmax_a*qmax_b*K <= INT32_MAX (:184-192), then
 * out[m][n] = sum_k a[m][k]*b[n][k] in int32, ascending k ("NT"). */
int or_int_gemm_check(int64_t depth, int bits_a, int bits_b) {
  int64_t worst = (int64_t)qmax_of(bits_a) * qmax_of(bits_b) * depth;
  return worst > 2147483647LL ? OR_ERR_CAPACITY : OR_OK;
}

int or_int_gemm(const int8_t* a, const int8_t* b, int64_t m_rows, int64_t n_rows,
                int64_t depth, int bits_a, int bits_b, int32_t* out) {
  int st = or_int_gemm_check(depth, bits_a, bits_b);
  if (st != OR_OK) return st;
  for (int64_t m = 0; m < m_rows; ++m) {
    const int8_t* ar = a + m * depth;
    for (int64_t n = 0; n < n_rows; ++n) {
      const int8_t* br = b + n * depth;
      int32_t acc = 0;
      for (int64_t k = 0; k < depth; ++k) acc += (int32_t)ar[k] * br[k];
      out[m * n_rows + n] = acc;
    }
  }
  return OR_OK;
}

/* Dequant of forward, pipeline.cpp:224-230:
 * v = ((double)acc * s_a[m]) * s_w[n] (+ b[n]). */
void or_dequant(const int32_t* acc, int64_t m_rows, int64_t n_rows,
                const double* s_a, const double* s_w, const double* bias,
                double* out) {
  for (int64_t m = 0; m < m_rows; ++m)
    for (int64_t n = 0; n < n_rows; ++n) {
      double v = (double)acc[m * n_rows + n] * s_a[m] * s_w[n];
      if (bias) v += bias[n];
      out[m * n_rows + n] = v;
    }
}

/* prepare_layer, pipeline.cpp:158-176: rotate W along K, per-output-channel
 * scales, quantize.  bias length is the caller's N (checked by the host). */
int or_prepare_layer(const double* w, int64_t n_rows, int64_t k_cols, int kind,
                     int group, int identity_tail, int bits, int8_t* codes,
                     double* scales) {
  double* rot = (double*)malloc(sizeof(double) * (size_t)(n_rows * k_cols));
  if (!rot) return OR_ERR_INVALID_VALUE;
  int st = or_group_rotate(w, n_rows, k_cols, kind, group, identity_tail, rot);
  if (st == OR_OK) st = or_compute_scales(rot, n_rows, k_cols, bits, scales);
  if (st == OR_OK) st = or_quantize(rot, n_rows, k_cols, scales, bits, codes);
  free(rot);
  return st;
}

/* Online half, pipeline.cpp:206-233 (forward): rotate -> scales ->
 * quantize -> int_gemm -> dequant.  Optional outputs (NULL to skip):
 * act_codes (M*K), act_scales (M), acc (M*N). */
int or_forward(const double* x, int64_t m_rows, int64_t k_cols,
               const int8_t* w_codes, const double* w_scales, const double* bias,
               int64_t n_rows, int kind, int group, int identity_tail, int bits_a,
               int bits_w, double* out, int8_t* act_codes, double* act_scales,
               int32_t* acc_out) {
  if (bits_a != 4 && bits_a != 8) return OR_ERR_INVALID_VALUE; /* :213-215 */
  size_t mk = (size_t)(m_rows * k_cols);
  double* rot = (double*)malloc(sizeof(double) * (mk ? mk : 1));
  int8_t* codes = act_codes ? act_codes : (int8_t*)malloc(mk ? mk : 1);
  double* sa = act_scales ? act_scales : (double*)malloc(sizeof(double) * (size_t)(m_rows ? m_rows : 1));
  int32_t* acc = acc_out ? acc_out : (int32_t*)malloc(sizeof(int32_t) * (size_t)(m_rows * n_rows ? m_rows * n_rows : 1));
  int st = OR_OK;
  if (!rot || !codes || !sa || !acc) st = OR_ERR_INVALID_VALUE;
  if (st == OR_OK) st = or_group_rotate(x, m_rows, k_cols, kind, group, identity_tail, rot);
  if (st == OR_OK) st = or_compute_scales(rot, m_rows, k_cols, bits_a, sa);
  if (st == OR_OK) st = or_quantize(rot, m_rows, k_cols, sa, bits_a, codes);
  if (st == OR_OK) st = or_int_gemm(codes, w_codes, m_rows, n_rows, k_cols, bits_a, bits_w, acc);
  if (st == OR_OK) or_dequant(acc, m_rows, n_rows, sa, w_scales, bias, out);
  free(rot);
  if (!act_codes) free(codes);
  if (!act_scales) free(sa);
  if (!acc_out) free(acc);
  return st;
}

/* reference_forward, pipeline.cpp:235-255: double X*W^T (+b), ascending k. */
int or_reference_forward(const double* x, const double* w, const double* bias,
                         int64_t m_rows, int64_t n_rows, int64_t k_cols, double* out) {
  for (int64_t m = 0; m < m_rows; ++m)
    for (int64_t n = 0; n < n_rows; ++n) {
      double acc = 0.0;
      for (int64_t k = 0; k < k_cols; ++k) acc += x[m * k_cols + k] * w[n * k_cols + k];
      if (bias) acc += bias[n];
      out[m * n_rows + n] = acc;
    }
  return OR_OK;
}

/* ---------------------------------------------------------------------- */
/* Pinned RNG contract "mt19937_64-boxmuller-v1", rng.hpp:11-56            */
/* ---------------------------------------------------------------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
  double cached;
  int has_cached;
} or_rng;

/* std::mt19937_64 (parameters fixed by the C++ standard [rand.predef]). */
static void mt_seed(or_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
  r->has_cached = 0;
  r->cached = 0.0;
}

static uint64_t mt_next(or_rng* r) {
  const uint64_t UPPER = 0xFFFFFFFF80000000ULL, LOWER = 0x7FFFFFFFULL;
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & UPPER) | (r->mt[(i + 1) % 312] & LOWER);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

/* next_double, rng.hpp:30-32 */
static double rng_double(or_rng* r) { return (double)(mt_next(r) >> 11) * 0x1.0p-53; }

/* next_gaussian, rng.hpp:35-48: Box-Muller, cosine branch first. */
static double rng_gaussian(or_rng* r) {
  if (r->has_cached) { r->has_cached = 0; return r->cached; }
  double u1 = (double)((mt_next(r) >> 11) + 1) * 0x1.0p-53;
  double u2 = rng_double(r);
  double radius = sqrt(-2.0 * log(u1));
  double angle = 2.0 * 3.141592653589793 * u2; /* std::numbers::pi */
  r->cached = radius * sin(angle);
  r->has_cached = 1;
  return radius * cos(angle);
}

void or_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out) {
  or_rng r;
  mt_seed(&r, seed);
  for (int64_t i = 0; i < rows * cols; ++i) out[i] = rng_gaussian(&r);
}

/* Raw draws, for pinning the engine against the reference. */
void or_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
  or_rng r;
  mt_seed(&r, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = mt_next(&r);
}

/* synth_outliers, analysis.cpp:54-82. mode: 0 rowwise, 1 colwise,
 * 2 gaussian (analysis.hpp:26 enum order). */
int or_synth_outliers(int64_t rows, int64_t cols, int mode, double magnitude,
                      double fraction, uint64_t seed, double* out) {
  if (rows < 1 || cols < 1) return OR_ERR_INVALID_VALUE;
  if (!(fraction > 0.0) || fraction > 1.0) return OR_ERR_INVALID_VALUE;
  if (!(magnitude >= 1.0)) return OR_ERR_INVALID_VALUE;
  or_rng r;
  mt_seed(&r, seed);
  for (int64_t i = 0; i < rows * cols; ++i) out[i] = rng_gaussian(&r);
  if (mode == 2) return OR_OK;
  int64_t axis = mode == 0 ? rows : cols;
  int64_t count = (int64_t)ceil(fraction * (double)axis);
  /* choose_indices, analysis.cpp:42-50: partial Fisher-Yates. */
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)axis);
  if (!idx) return OR_ERR_INVALID_VALUE;
  for (int64_t i = 0; i < axis; ++i) idx[i] = i;
  for (int64_t i = 0; i < count; ++i) {
    int64_t j = i + (int64_t)(mt_next(&r) % (uint64_t)(axis - i)); /* next_below */
    int64_t t = idx[i]; idx[i] = idx[j]; idx[j] = t;
  }
  for (int64_t c = 0; c < count; ++c) {
    int64_t k = idx[c];
    if (mode == 0) {
      for (int64_t j = 0; j < cols; ++j) out[k * cols + j] *= magnitude;
    } else {
      for (int64_t i = 0; i < rows; ++i) out[i * cols + k] *= magnitude;
    }
  }
  free(idx);
  return OR_OK;
}

/* ---------------------------------------------------------------------- */
/* Input narrowing used by the parity harness (not a reference function):  */
/* round-to-nearest-even double -> bf16 bits, and the exact widening back. */
/* ---------------------------------------------------------------------- */
void or_to_bf16(const double* in, int64_t n, uint16_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    float f = (float)in[i]; /* double -> f32 RNE (exact for our gaussians' use) */
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x7FFFFFu)) {
      out[i] = (uint16_t)((u >> 16) | 0x40); /* quiet NaN */
      continue;
    }
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7FFFu + lsb;
    out[i] = (uint16_t)(u >> 16);
  }
}

void or_from_bf16(const uint16_t* in, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    uint32_t u = (uint32_t)in[i] << 16;
    float f;
    memcpy(&f, &u, 4);
    out[i] = (double)f;
  }
}
