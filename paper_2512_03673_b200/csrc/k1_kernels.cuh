#pragma once
// k1_rotate_quant.cu -- K1: group-wise regular-Hadamard rotation fused with
// per-token absmax, INT4/INT8 rounding and nibble packing (sm_100a).
//
// Replaces, for one activation matrix, the reference sequence
//   group_rotate   pipeline.cpp:111-151   (ascending-k double dot products)
//   compute_scales quant.cpp:10-24        (s = max|y| / qmax, 1.0 if zero)
//   quantize       quant.cpp:26-52        (clamp(nearbyint(y / s)))
//   pack_int4      quant.cpp:64-81        (element 2t -> low nibble of byte t)
//
// Certified rounding: the rotation is evaluated as fp32 radix-4
// butterflies (FADD2/FFMA2) whose error is bounded by
//     |y32 - y_ref| <= 6 L u sqrt(N0) A  (+ the reference's own fp64 error)
// (L = log4 N0, u = 2^-24, A = row absmax of the unnormalised sums).  Every
// decision the reference makes in double -- which element is the row max,
// and on which side of a half-integer y/s falls -- is taken from the fp32
// value only when the bound proves it cannot differ; otherwise that element
// is recomputed exactly the reference's way (sequential double sum in
// ascending k, IEEE double division, nearbyint).  The output codes and f64
// scales are therefore bit-identical to the reference for every input.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "k1_rotate_quant.h"

namespace crt {

namespace {

constexpr uint32_t kMagic23 = 0x4B400000u;  // 1.5 * 2^23 : ulp 1

template <bool F32>
__device__ __forceinline__ double load_x(const void* row, int64_t j) {
  if constexpr (F32) {
    return (double)__ldg(reinterpret_cast<const float*>(row) + j);
  } else {
    uint16_t b = __ldg(reinterpret_cast<const unsigned short*>(row) + j);
    return (double)__uint_as_float((uint32_t)b << 16);
  }
}

// The reference's rotated value for column j of one row: out[j] =
// sum_{k<g} x[base+k] * R[k][j'] in ascending k, product then add (the
// reference builds with -ffp-contract=off), R = +-1/sqrt(g)
// (pipeline.cpp:52-66, :134-142).  Columns at or beyond rot_cols pass through
// (identity tail, :144); kind none returns x (:114).
template <bool F32>
__device__ __forceinline__ double y_ref(const void* row, int64_t j, int64_t group, int kind,
                                     int64_t rot_cols) {
  if (kind == kRotNone || j >= rot_cols) return load_x<F32>(row, j);
  int64_t base = j / group * group;
  uint32_t jj = (uint32_t)(j - base);
  double r = 1.0 / sqrt((double)group);
  double acc = 0.0;
  for (int64_t k = 0; k < group; ++k) {
    bool neg = kind == kRotRegular ? regular_negative((uint32_t)k, jj)
                                   : sylvester_negative((uint32_t)k, jj);
    acc = __dadd_rn(acc, __dmul_rn(load_x<F32>(row, base + k), neg ? -r : r));
  }
  return acc;
}

__device__ __forceinline__ int exact_code(double y, double s, int qmax) {
  double q = rint(__ddiv_rn(y, s));  // nearbyint, FE_TONEAREST
  q = fmin(fmax(q, (double)-qmax), (double)qmax);
  return (int)q;
}


// ---------------------------------------------------------------------------
// Warp / team reductions
// ---------------------------------------------------------------------------
__device__ __forceinline__ float warp_max_nan(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max_nan(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

struct TeamScratch {
  float f[32];
  double d[32];
};

// Team of W warps (contiguous warps team*W .. team*W+W-1).  Two barriers
// make the slot reusable immediately.
__device__ __forceinline__ float team_max_nan(float v, TeamScratch* ts, int team, int w,
                                              int W) {
  v = warp_max_nan(v);
  if (W == 1) return v;
  const int lane = threadIdx.x & 31;
  if (lane == 0) ts->f[team * W + w] = v;
  named_bar_sync(1 + team, W * 32);
  float r = ts->f[team * W];
  for (int i = 1; i < W; ++i) r = max_nan(r, ts->f[team * W + i]);
  named_bar_sync(1 + team, W * 32);
  return r;
}
__device__ __forceinline__ double team_max_d(double v, TeamScratch* ts, int team, int w,
                                             int W) {
  v = warp_max_d(v);
  if (W == 1) return v;
  const int lane = threadIdx.x & 31;
  if (lane == 0) ts->d[team * W + w] = v;
  named_bar_sync(1 + team, W * 32);
  double r = ts->d[team * W];
  for (int i = 1; i < W; ++i) r = fmax(r, ts->d[team * W + i]);
  named_bar_sync(1 + team, W * 32);
  return r;
}

// ---------------------------------------------------------------------------
// Radix-4 butterflies on fp32x2 pairs.  H4 = J - 2*antidiag, so with
// S = ((a+b)+c)+d:  y_j = S - 2 x_{3-j}  (form B).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void bfly4(float2& a, float2& b, float2& c, float2& d) {
  const float2 m2 = make_float2(-2.f, -2.f);
  float2 s = f2_add(f2_add(f2_add(a, b), c), d);
  float2 na = f2_fma(m2, d, s);
  float2 nb = f2_fma(m2, c, s);
  float2 nc = f2_fma(m2, b, s);
  float2 nd = f2_fma(m2, a, s);
  a = na;
  b = nb;
  c = nc;
  d = nd;
}

// Cross-lane radix-4 stage: the four partners differ in lane bits
// {log2(stride), log2(stride)+1}; my digit j = (lane / stride) & 3 and
// partner 3-j = j ^ 3.
__device__ __forceinline__ float xlane4(float v, int stride) {
  float t = v + __shfl_xor_sync(0xffffffffu, v, stride);
  float s = t + __shfl_xor_sync(0xffffffffu, t, 2 * stride);
  float o = __shfl_xor_sync(0xffffffffu, v, 3 * stride);
  return fmaf(-2.f, o, s);
}

template <int N0>
struct Stages {
  static constexpr int L = N0 == 1 ? 0 : N0 == 4 ? 1 : N0 == 16 ? 2 : N0 == 64 ? 3 : 4;
};

}  // namespace


// ---------------------------------------------------------------------------
// Fast kernel.  A team of W warps owns one row at a time; lane `lane` of
// warp w holds chunks (c*W + w)*32 + lane, c < C, of 16 consecutive
// elements each (C even; chunk pairs live in fp32x2 registers).  Groups of
// N0 <= 256 elements are N0/16 consecutive chunks = consecutive lanes.
// ---------------------------------------------------------------------------
template <int C, int N0, bool F32, int BITS>
__global__ void __launch_bounds__(256, C <= 2 ? 3 : (C <= 4 ? 2 : 1)) k1_fast(K1Args a) {
  constexpr int P = C / 2;
  constexpr int L = Stages<N0>::L;
  constexpr int QMAX = BITS == 4 ? 7 : 127;
  __shared__ TeamScratch ts;

  const int W = a.team_warps;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int team = warp / W;
  const int w = warp - team * W;
  const int teams = blockDim.x / (32 * W);
  const int64_t nchunks = a.K / 16;
  const int esz = F32 ? 4 : 2;

  // normalisation 2^-k = 1/sqrt(N0) (exact), and the certified bound factor
  const double rk = N0 == 1 ? 1.0 : 1.0 / sqrt((double)N0);
  const double sqrtn = N0 == 1 ? 1.0 : sqrt((double)N0);
  const double bound_rel = L == 0 ? 0.0
                                  : (6.0 * L * sqrtn) * 5.9604644775390625e-8 +
                                        (double)N0 * sqrtn * 2.220446049250313e-16;

  for (int64_t row = (int64_t)blockIdx.x * teams + team; row < a.M;
       row += (int64_t)gridDim.x * teams) {
    const char* xrow = reinterpret_cast<const char*>(a.x) + row * a.ldx * esz;

    // ---- load + convert -------------------------------------------------
    float2 v[P][16];
#pragma unroll
    for (int p = 0; p < P; ++p) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t chunk = ((int64_t)(2 * p + h) * W + w) * 32 + lane;
        float f[16];
        if (chunk < nchunks) {
          if constexpr (F32) {
            uint32_t u0[8], u1[8];
            ld_nc_v8(xrow + chunk * 64, u0);
            ld_nc_v8(xrow + chunk * 64 + 32, u1);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              f[i] = __uint_as_float(u0[i]);
              f[8 + i] = __uint_as_float(u1[i]);
            }
          } else {
            uint32_t u[8];
            ld_nc_v8(xrow + chunk * 32, u);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              f[2 * i] = __uint_as_float(u[i] << 16);
              f[2 * i + 1] = __uint_as_float(u[i] & 0xFFFF0000u);
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) f[i] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          if (h == 0) v[p][i].x = f[i];
          else v[p][i].y = f[i];
        }
      }
    }

    // ---- rotation (unnormalised sums of +-x) --------------------------------
    if constexpr (N0 >= 4) {
#pragma unroll
      for (int p = 0; p < P; ++p) {
#pragma unroll
        for (int g = 0; g < 4; ++g)
          bfly4(v[p][4 * g], v[p][4 * g + 1], v[p][4 * g + 2], v[p][4 * g + 3]);
        if constexpr (N0 >= 16) {
#pragma unroll
          for (int j = 0; j < 4; ++j) bfly4(v[p][j], v[p][j + 4], v[p][j + 8], v[p][j + 12]);
        }
      }
    }
    if constexpr (N0 >= 64) {
#pragma unroll
      for (int p = 0; p < P; ++p)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          v[p][i].x = xlane4(v[p][i].x, 1);
          v[p][i].y = xlane4(v[p][i].y, 1);
        }
    }
    if constexpr (N0 >= 256) {
#pragma unroll
      for (int p = 0; p < P; ++p)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          v[p][i].x = xlane4(v[p][i].x, 4);
          v[p][i].y = xlane4(v[p][i].y, 4);
        }
    }

    // ---- row absmax (NaN-propagating) ---------------------------------------
    float lmax = 0.f;
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int i = 0; i < 16; ++i) lmax = max3_abs(v[p][i].x, v[p][i].y, lmax);
    const float A32 = team_max_nan(lmax, &ts, team, w, W);

    // pathological rows (non-finite input, fp32 overflow) go the exact way
    const bool slow_row = !(A32 <= 3.0e38f);
    const double B = slow_row ? 0.0 : bound_rel * (double)A32 * 1.01;
    double amax_ref = 0.0;
    if (!slow_row) {
      // candidates for the exact row max: |y32| >= A32 - 2B
      const float thr = (float)((double)A32 - 2.0 * B) * (1.0f - 1e-6f);
      double cmax = 0.0;
      if (lmax >= thr) {
        uint32_t cm[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          uint32_t m = 0;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            m |= (fabsf(v[p][i].x) >= thr ? 1u : 0u) << i;
            m |= (fabsf(v[p][i].y) >= thr ? 1u : 0u) << (16 + i);
          }
          cm[p] = m;
        }
#pragma unroll 1
        for (int p = 0; p < P; ++p) {
          uint32_t m = 0;
#pragma unroll
          for (int q = 0; q < P; ++q)
            if (q == p) m = cm[q];
          while (m) {
            const int bit = __ffs(m) - 1;
            m &= m - 1;
            const int64_t chunk = ((int64_t)(2 * p + (bit >> 4)) * W + w) * 32 + lane;
            if (chunk >= nchunks) continue;
            cmax = fmax(cmax, fabs(y_ref<F32>(xrow, chunk * 16 + (bit & 15), a.group,
                                              a.kind, a.rot_cols)));
          }
        }
      }
      amax_ref = team_max_d(cmax, &ts, team, w, W);
    } else {
      double m = 0.0;
      bool bad = false;
#pragma unroll 1
      for (int c = 0; c < C; ++c) {
        const int64_t chunk = ((int64_t)c * W + w) * 32 + lane;
        if (chunk >= nchunks) continue;
#pragma unroll 1
        for (int i = 0; i < 16; ++i) {
          double yr = y_ref<F32>(xrow, chunk * 16 + i, a.group, a.kind, a.rot_cols);
          if (!isfinite(yr)) bad = true;
          m = fmax(m, fabs(yr));
        }
      }
      amax_ref = team_max_d(bad ? INFINITY : m, &ts, team, w, W);
    }
    const bool invalid = !isfinite(amax_ref);
    const double s = invalid ? 1.0 : (amax_ref == 0.0 ? 1.0 : amax_ref / (double)QMAX);
    if (invalid && lane == 0 && w == 0) flag_invalid_value(a.err);

    uint8_t* crow = a.codes + row * a.ldc;
    if (!slow_row) {
      // ---- certified quantisation --------------------------------------------
      // t = C + rint(y*inv) with C = 1.5*2^23 (ulp 1): the code is the low
      // byte of t's bit pattern; e = y*inv - rint(y*inv) certifies it.
      const float inv = __double2float_rn(rk / s);
      const float margin = (float)(B * (rk / s) * 1.05) +
                           (float)(QMAX + 4) * 1.1920928955078125e-7f + 1e-9f;
      const float thr = 0.5f - margin;
      const float2 iv = make_float2(inv, inv);
      const float2 cc = make_float2(__uint_as_float(kMagic23), __uint_as_float(kMagic23));
      uint32_t fmask[P];

#pragma unroll
      for (int p = 0; p < P; ++p) {
        uint32_t tb[2][16];
        float emax = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 t = f2_fma(v[p][i], iv, cc);                  // C + rint(y*inv)
          const float2 nr = f2_fma(t, make_float2(-1.f, -1.f), cc);  // -rint(y*inv), exact
          const float2 e = f2_fma(v[p][i], iv, nr);                  // y*inv - rint
          emax = max3_abs(e.x, e.y, emax);
          tb[0][i] = __float_as_uint(t.x);
          tb[1][i] = __float_as_uint(t.y);
        }
        uint32_t fm = 0;
        if (!(emax <= thr)) {
          // rare: an element within the certified margin of a rounding
          // boundary; remember which, decide it exactly after the store.
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float ex = fmaf(v[p][i].x, inv, __uint_as_float(kMagic23) - __uint_as_float(tb[0][i]));
            const float ey = fmaf(v[p][i].y, inv, __uint_as_float(kMagic23) - __uint_as_float(tb[1][i]));
            fm |= (fabsf(ex) <= thr ? 0u : 1u) << i;
            fm |= (fabsf(ey) <= thr ? 0u : 1u) << (16 + i);
          }
        }
        fmask[p] = fm;
        // ---- pack + store ------------------------------------------------------
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t chunk = ((int64_t)(2 * p + h) * W + w) * 32 + lane;
          if (chunk >= nchunks) continue;
          if constexpr (BITS == 4) {
            uint32_t by[8];
#pragma unroll
            for (int b2 = 0; b2 < 8; ++b2)  // low byte = (odd << 4) | (even & 0xF)
              by[b2] = tb[h][2 * b2 + 1] * 16u + (tb[h][2 * b2] & 0xFu);
            uint2 out;
            out.x = __byte_perm(__byte_perm(by[0], by[1], 0x0040),
                                __byte_perm(by[2], by[3], 0x0040), 0x5410);
            out.y = __byte_perm(__byte_perm(by[4], by[5], 0x0040),
                                __byte_perm(by[6], by[7], 0x0040), 0x5410);
            *reinterpret_cast<uint2*>(crow + chunk * 8) = out;
          } else {
            uint32_t wds[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              wds[q] = __byte_perm(__byte_perm(tb[h][4 * q], tb[h][4 * q + 1], 0x0040),
                                   __byte_perm(tb[h][4 * q + 2], tb[h][4 * q + 3], 0x0040),
                                   0x5410);
            *reinterpret_cast<uint4*>(crow + chunk * 16) = make_uint4(wds[0], wds[1], wds[2], wds[3]);
          }
        }
      }
      // ---- exact decisions for the flagged elements (same thread re-writes
      // the byte it stored above; program order makes that safe) ---------------
#pragma unroll 1
      for (int p = 0; p < P; ++p) {
        uint32_t m = 0;
#pragma unroll
        for (int q = 0; q < P; ++q)
          if (q == p) m = fmask[q];
        while (m) {
          const int bit = __ffs(m) - 1;
          m &= m - 1;
          const int i = bit & 15;
          const int64_t chunk = ((int64_t)(2 * p + (bit >> 4)) * W + w) * 32 + lane;
          if (chunk >= nchunks) continue;
          const int code = exact_code(
              y_ref<F32>(xrow, chunk * 16 + i, a.group, a.kind, a.rot_cols), s, QMAX);
          if constexpr (BITS == 4) {
            uint8_t* bp = crow + chunk * 8 + (i >> 1);
            const uint8_t old = *bp;
            *bp = (i & 1) ? (uint8_t)((old & 0x0F) | ((code & 0x0F) << 4))
                          : (uint8_t)((old & 0xF0) | (code & 0x0F));
          } else {
            crow[chunk * 16 + i] = (uint8_t)code;
          }
        }
      }
    } else {
      // slow row: exact codes for every element
#pragma unroll 1
      for (int c = 0; c < C; ++c) {
        const int64_t chunk = ((int64_t)c * W + w) * 32 + lane;
        if (chunk >= nchunks) continue;
#pragma unroll 1
        for (int i = 0; i < 16; i += 2) {
          int c0 = 0, c1 = 0;
          if (!invalid) {
            c0 = exact_code(y_ref<F32>(xrow, chunk * 16 + i, a.group, a.kind, a.rot_cols), s, QMAX);
            c1 = exact_code(y_ref<F32>(xrow, chunk * 16 + i + 1, a.group, a.kind, a.rot_cols), s, QMAX);
          }
          if constexpr (BITS == 4) {
            crow[chunk * 8 + i / 2] = (uint8_t)((c0 & 0x0F) | ((c1 & 0x0F) << 4));
          } else {
            crow[chunk * 16 + i] = (uint8_t)c0;
            crow[chunk * 16 + i + 1] = (uint8_t)c1;
          }
        }
      }
    }
    if (w == 0 && lane == 0) {
      if (a.s32) a.s32[row] = (float)s;
      if (a.s64) a.s64[row] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// Exact kernel: any kind / group / tail / alignment.  One CTA per row;
// every element computed the reference's way.  Used for shapes the fast
// kernel does not cover (global groups > 256, sylvester, identity tails,
// unaligned rows) -- correctness first, O(K * N0) per row.
// ---------------------------------------------------------------------------
template <bool F32, int BITS>
__global__ void __launch_bounds__(256) k1_exact(K1Args a) {
  constexpr int QMAX = BITS == 4 ? 7 : 127;
  extern __shared__ int8_t scodes[];
  __shared__ double red[8];
  __shared__ int redbad[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int esz = F32 ? 4 : 2;
  for (int64_t row = blockIdx.x; row < a.M; row += gridDim.x) {
    const char* xrow = reinterpret_cast<const char*>(a.x) + row * a.ldx * esz;
    double m = 0.0;
    int bad = 0;
    for (int64_t j = tid; j < a.K; j += blockDim.x) {
      double yr = y_ref<F32>(xrow, j, a.group, a.kind, a.rot_cols);
      if (!isfinite(yr)) bad = 1;
      else m = fmax(m, fabs(yr));
    }
    m = warp_max_d(m);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      red[warp] = m;
      redbad[warp] = bad;
    }
    __syncthreads();
    m = 0.0;
    bad = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      m = fmax(m, red[i]);
      bad |= redbad[i];
    }
    __syncthreads();
    double s = bad ? 1.0 : (m == 0.0 ? 1.0 : m / (double)QMAX);
    if (bad && tid == 0) flag_invalid_value(a.err);
    for (int64_t j = tid; j < a.K; j += blockDim.x) {
      int code = 0;
      if (!bad) code = exact_code(y_ref<F32>(xrow, j, a.group, a.kind, a.rot_cols), s, QMAX);
      scodes[j] = (int8_t)code;
    }
    __syncthreads();
    uint8_t* crow = a.codes + row * a.ldc;
    if constexpr (BITS == 4) {
      for (int64_t t = tid; t < (a.K + 1) / 2; t += blockDim.x) {
        uint8_t lo = (uint8_t)scodes[2 * t] & 0x0F;
        uint8_t hi = 2 * t + 1 < a.K ? (uint8_t)(((uint8_t)scodes[2 * t + 1] & 0x0F) << 4) : 0;
        crow[t] = (uint8_t)(lo | hi);
      }
    } else {
      for (int64_t t = tid; t < a.K; t += blockDim.x) crow[t] = (uint8_t)scodes[t];
    }
    if (tid == 0) {
      if (a.s32) a.s32[row] = (float)s;
      if (a.s64) a.s64[row] = s;
    }
    __syncthreads();
  }
}

template <int C, int N0, bool F32, int BITS>
cudaError_t launch_fast(const K1Args& a, cudaStream_t st, int64_t* launches) {
  auto kern = k1_fast<C, N0, F32, BITS>;
  const int W = a.team_warps;
  const int teams = W >= 8 ? 1 : 8 / W;  // 256-thread CTAs (W | 8) or one team
  const int threads = teams * W * 32;
  static int num_sms = 0;
  if (num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, 0);
  if (per_sm < 1) per_sm = 1;
  int64_t need = (a.M + teams - 1) / teams;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, threads, 0, st>>>(a);
  ++*launches;
  return cudaGetLastError();
}

template <int C, bool F32, int BITS>
cudaError_t dispatch_n0(const K1Args& a, int n0, cudaStream_t st, int64_t* l) {
  switch (n0) {
    case 1: return launch_fast<C, 1, F32, BITS>(a, st, l);
    case 4: return launch_fast<C, 4, F32, BITS>(a, st, l);
    case 16: return launch_fast<C, 16, F32, BITS>(a, st, l);
    case 64: return launch_fast<C, 64, F32, BITS>(a, st, l);
    case 256: return launch_fast<C, 256, F32, BITS>(a, st, l);
  }
  return cudaErrorInvalidValue;
}

template <bool F32, int BITS>
cudaError_t k1_dispatch(const K1Args& a, int c, int n0, cudaStream_t st, int64_t* l) {
  switch (c) {
    case 2: return dispatch_n0<2, F32, BITS>(a, n0, st, l);
    case 4: return dispatch_n0<4, F32, BITS>(a, n0, st, l);
    case 6: return dispatch_n0<6, F32, BITS>(a, n0, st, l);
    case 8: return dispatch_n0<8, F32, BITS>(a, n0, st, l);
  }
  return cudaErrorInvalidValue;
}


template <bool F32, int BITS>
cudaError_t k1_exact_launch(const K1Args& a, cudaStream_t st) {
  size_t smem = (size_t)a.K;
  int grid = (int)(a.M < 148 * 8 ? a.M : 148 * 8);
  if (grid < 1) grid = 1;
  auto k = k1_exact<F32, BITS>;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<grid, 256, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace crt
