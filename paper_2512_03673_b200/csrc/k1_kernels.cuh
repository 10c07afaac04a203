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
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "k1_rotate_quant.h"

namespace crt {

namespace {

constexpr uint32_t kMagic23 = 0x4B400000u;  // 1.5 * 2^23 : ulp 1

// Plain (generic-address) loads: `row` may point to global memory or to the
// shared-memory copy of the row.
template <bool F32>
__device__ __forceinline__ float load_xf(const void* row, int64_t j) {
  if constexpr (F32) {
    return reinterpret_cast<const float*>(row)[j];
  } else {
    const uint16_t b = reinterpret_cast<const unsigned short*>(row)[j];
    return __uint_as_float((uint32_t)b << 16);
  }
}
template <bool F32>
__device__ __forceinline__ double load_x(const void* row, int64_t j) {
  return (double)load_xf<F32>(row, j);
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

// y_ref(j) evaluated by a whole warp (all 32 lanes call it with the same j).
// Lanes sum disjoint terms of the group in double and the partial sums are
// combined with shuffles.  The reference's sequential sum (ascending k,
// products +-x*2^-L exact) has no rounding at all whenever
//     log2(group) + (emax - emin) + mantissa_bits <= 53
// over the nonzero inputs of the group (all terms are integer multiples of
// the smallest one's ulp and bounded by group * 2^(emax+1)); then EVERY
// summation order yields the same exact value and the warp sum is returned.
// Otherwise (subnormal / non-finite inputs or a huge exponent span) all
// lanes redo the reference's sequential loop.
template <bool F32>
__device__ __noinline__ double y_exact_warp(const void* row, int64_t j, int64_t group, int kind,
                                            int64_t rot_cols) {
  if (kind == kRotNone || j >= rot_cols) return load_x<F32>(row, j);
  const int lane = threadIdx.x & 31;
  const int64_t base = j / group * group;
  const uint32_t jj = (uint32_t)(j - base);
  double acc = 0.0;
  int emin = 1 << 20, emax = -1;
  int bad = 0;
  for (int k = lane; k < group; k += 32) {
    const float x = load_xf<F32>(row, base + k);
    const int e = (int)((__float_as_uint(x) >> 23) & 0xFFu);
    if (x != 0.f) {
      bad |= (e == 0 || e == 255) ? 1 : 0;
      emin = min(emin, e);
      emax = max(emax, e);
    }
    const bool neg = kind == kRotRegular ? regular_negative((uint32_t)k, jj)
                                         : sylvester_negative((uint32_t)k, jj);
    acc += neg ? -(double)x : (double)x;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, o);
    emin = min(emin, __shfl_xor_sync(0xffffffffu, emin, o));
    emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  const int l2 = __ffsll(group) - 1;
  const bool pow4 = kind == kRotRegular || (l2 % 2 == 0);  // 1/sqrt(group) exact
  if (!bad && pow4 && (emax < 0 || l2 + (emax - emin) + (F32 ? 24 : 8) <= 53))
    return acc * (1.0 / sqrt((double)group));
  return y_ref<F32>(row, j, group, kind, rot_cols);
}

// y_ref(j) for a group that lies in the calling lane's own chunk (N0 <= 16),
// evaluated by that lane alone, given the fp32 butterfly value y32 (the
// unnormalised sum).  If every partial sum of the fp32 butterflies is exact
// -- all inputs of the group are integer multiples of the smallest one's
// ulp and the intermediates (at most 2*group*max|x|) need
//     1 + log2(group) + (emax - emin) + mantissa_bits <= 24 bits --
// then y32 * 2^-L IS the reference's (exact) double value.  Otherwise the
// reference's sequential double loop (at most 16 terms) is run.
template <bool F32>
__device__ __noinline__ double y_exact_lane(const void* row, int64_t j, int64_t group, int kind,
                                            int64_t rot_cols, float y32) {
  if (kind == kRotNone || j >= rot_cols) return load_x<F32>(row, j);
  const int64_t base = j / group * group;
  int emin = 1 << 20, emax = -1;
  bool bad = false;
  for (int64_t k = 0; k < group; ++k) {
    const float x = load_xf<F32>(row, base + k);
    const int e = (int)((__float_as_uint(x) >> 23) & 0xFFu);
    if (x != 0.f) {
      bad |= (e == 0 || e == 255);
      emin = min(emin, e);
      emax = max(emax, e);
    }
  }
  const int l2 = __ffsll(group) - 1;
  if (!bad && kind == kRotRegular && (emax < 0 || 1 + l2 + (emax - emin) + (F32 ? 24 : 8) <= 24))
    return (double)y32 * (1.0 / sqrt((double)group));
  return y_ref<F32>(row, j, group, kind, rot_cols);
}

// y_exact_lane for a group inside one 16-element chunk (N0 <= 16), fully
// unrolled: the chunk is re-read with vector loads and the exponent-span
// certificate is evaluated branch-free.  Falls back to y_exact_lane (the
// reference's sequential loop) only when the certificate fails.
template <bool F32, int N0>
__device__ __noinline__ double y_exact_chunk(const void* row, int64_t chunk, int e, int kind,
                                             int64_t rot_cols, float y32) {
  const int64_t j = chunk * 16 + e;
  if (kind == kRotNone || j >= rot_cols) return load_x<F32>(row, j);
  float x[16];
  if constexpr (F32) {
    const uint4* p = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(row) + chunk * 64);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 v = p[q];
      x[4 * q] = __uint_as_float(v.x);
      x[4 * q + 1] = __uint_as_float(v.y);
      x[4 * q + 2] = __uint_as_float(v.z);
      x[4 * q + 3] = __uint_as_float(v.w);
    }
  } else {
    const uint4* p = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(row) + chunk * 32);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint4 v = p[q];
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        x[8 * q + 2 * i] = __uint_as_float(w[i] << 16);
        x[8 * q + 2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
      }
    }
  }
  // Exponent span of the group's nonzero inputs from two integer reductions
  // on the magnitude bits: |x| bits - 1 (unsigned) sends zeros to the top,
  // so the minimum is the smallest nonzero magnitude; a maximum at or above
  // the inf pattern means inf/NaN, a nonzero minimum below the smallest
  // normal means a subnormal (both: not certified).
  const int g0 = e & ~(N0 - 1);
  uint32_t bmax = 0u, bmin1 = 0xFFFFFFFFu;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if ((i & ~(N0 - 1)) != g0) continue;  // compile-time for N0 == 16
    const uint32_t b = __float_as_uint(x[i]) & 0x7FFFFFFFu;
    bmax = max(bmax, b);
    bmin1 = min(bmin1, b - 1u);
  }
  const bool bad = bmax >= 0x7F800000u || (bmax != 0u && bmin1 + 1u < 0x00800000u);
  const int emax = (int)(bmax >> 23), emin = (int)((bmin1 + 1u) >> 23);
  constexpr int L2 = N0 == 4 ? 2 : 4;
  if (!bad && kind == kRotRegular && (bmax == 0u || 1 + L2 + (emax - emin) + (F32 ? 24 : 8) <= 24))
    return (double)y32 * (N0 == 4 ? 0.5 : 0.25);
  return y_ref<F32>(row, j, N0, kind, rot_cols);
}

__device__ __forceinline__ int exact_code(double y, double s, int qmax) {
  double q = rint(__ddiv_rn(y, s));  // nearbyint, FE_TONEAREST
  q = fmin(fmax(q, (double)-qmax), (double)qmax);
  return (int)q;
}


// ---------------------------------------------------------------------------
// Warp / team reductions
// ---------------------------------------------------------------------------
// Maxima of NON-NEGATIVE values (absolute values, +NaN, +inf): their IEEE
// bit patterns order like unsigned integers (+NaN above +inf), so one REDUX
// replaces a five-step shuffle tree.
__device__ __forceinline__ float warp_max_nan(float v) {
  return __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(v)));
}
__device__ __forceinline__ double warp_max_d(double v) {
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  const uint32_t hi = __reduce_max_sync(0xffffffffu, (uint32_t)(b >> 32));
  const uint32_t lo = __reduce_max_sync(0xffffffffu, (uint32_t)(b >> 32) == hi ? (uint32_t)b : 0u);
  return __longlong_as_double((long long)(((uint64_t)hi << 32) | lo));
}

struct TeamScratch {
  float f[32];
  double d[32];
  int i[32];
  int rs[8][2];  // per team, per row parity: code sum of the row (rowsum_publish)
  int rf[8][2];  // per team, per row parity: "re-sum from memory" flag
};

// Team of W warps (contiguous warps team*W .. team*W+W-1).  ONE barrier per
// reduction: each reduction owns its slot array (f, d), and a slot is written
// again only in the next row, after a later team barrier that every warp
// reaches only once it has read the slot.
__device__ __forceinline__ float team_max_nan(float v, TeamScratch* ts, int team, int w,
                                              int W) {
  v = warp_max_nan(v);
  if (W == 1) return v;
  const int lane = threadIdx.x & 31;
  if (lane == 0) ts->f[team * W + w] = v;
  named_bar_sync(1 + team, W * 32);
  float r = ts->f[team * W];
  for (int i = 1; i < W; ++i) r = max_nan(r, ts->f[team * W + i]);
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
  return r;
}


// Sum of the int8 codes of row `crow` (K bytes) over the team, after the
// team's stores are visible (called past the end-of-row barrier): each lane
// sums 16-byte pieces with DP4A.  The K3 v3 epilogue needs it to remove the
// offset of the decompressed weights (k3_gemm_v3.cu).
__device__ __forceinline__ int team_code_sum(const uint8_t* crow, int64_t K, int W, int w,
                                             TeamScratch* ts, int team) {
  const int lane = threadIdx.x & 31;
  int acc = 0;
  for (int64_t off = ((int64_t)w * 32 + lane) * 16; off < K; off += (int64_t)W * 32 * 16) {
    if (off + 16 <= K) {
      const uint4 v = *reinterpret_cast<const uint4*>(crow + off);
      acc = __dp4a((int)v.x, 0x01010101, acc);
      acc = __dp4a((int)v.y, 0x01010101, acc);
      acc = __dp4a((int)v.z, 0x01010101, acc);
      acc = __dp4a((int)v.w, 0x01010101, acc);
    } else {
      for (int64_t j = off; j < K; ++j) acc += (int)(int8_t)crow[j];
    }
  }
  acc = __reduce_add_sync(0xffffffffu, acc);
  if (W == 1) return acc;
  if (lane == 0) ts->i[team * W + w] = acc;
  named_bar_sync(1 + team, W * 32);
  int r = 0;
  for (int i = 0; i < W; ++i) r += ts->i[team * W + i];
  named_bar_sync(1 + team, W * 32);
  return r;
}

// Row code sum for K3 v3 from the lanes' register sums `csum` (accumulated
// as the codes were stored; a pair re-written by a near-tie redecide is
// re-summed from its own 32 bytes).  Rows whose codes come from elsewhere
// (slow row, partial last chunk) are summed again from memory
// (team_code_sum).
// Called past the end-of-row barrier; two barriers, as team_code_sum.
__device__ __forceinline__ int team_row_sum(int csum, bool resum, const uint8_t* crow, int64_t K,
                                            int W, int w, TeamScratch* ts, int team) {
  const int lane = threadIdx.x & 31;
  csum = __reduce_add_sync(0xffffffffu, csum);
  bool any = __any_sync(0xffffffffu, resum);
  if (W > 1) {
    if (lane == 0) {
      ts->i[team * W + w] = csum;
      ts->f[team * W + w] = any ? 1.f : 0.f;
    }
    named_bar_sync(1 + team, W * 32);
    csum = 0;
    for (int i = 0; i < W; ++i) {
      csum += ts->i[team * W + i];
      any |= ts->f[team * W + i] != 0.f;
    }
    named_bar_sync(1 + team, W * 32);
  }
  return any ? team_code_sum(crow, K, W, w, ts, team) : csum;
}

// Row code sums for teams (W > 1) without extra barriers: before the
// end-of-row barrier each warp adds its sum (and its "re-sum" flag) into the
// team's slot for this row's parity with shared-memory atomics; after the
// barrier every warp reads the flag (uniform decision), the leader the sum.
// The leader clears the slot in the NEXT row after its first team barrier
// (rowsum_clear), when every warp has read it; the row after that reuses it.
__device__ __forceinline__ void rowsum_publish(int csum, bool resum, TeamScratch* ts, int team,
                                               int par) {
  const int sum = __reduce_add_sync(0xffffffffu, csum);
  const bool any = __any_sync(0xffffffffu, resum);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&ts->rs[team][par], sum);
    if (any) atomicOr(&ts->rf[team][par], 1);
  }
}
__device__ __forceinline__ int rowsum_collect(const uint8_t* crow, int64_t K, int W, int w,
                                              TeamScratch* ts, int team, int par) {
  if (ts->rf[team][par]) return team_code_sum(crow, K, W, w, ts, team);
  return ts->rs[team][par];
}
__device__ __forceinline__ void rowsum_clear(TeamScratch* ts, int team, int par) {
  ts->rs[team][par] = 0;
  ts->rf[team][par] = 0;
}

// Code sum of the two int8-code chunks of a pair, re-read after a redecide
// re-wrote some of their bytes (own stores, or the warp's after __syncwarp).
template <bool FULL>
__device__ __forceinline__ int reread_pair_sum(const uint8_t* crow, int64_t c0, int64_t cstride,
                                               int64_t nchunks) {
  int r = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t chunk = c0 + h * cstride;
    if (!FULL && chunk >= nchunks) continue;
    const uint4 v = *reinterpret_cast<const uint4*>(crow + chunk * 16);
    r = __dp4a((int)v.x, 0x01010101, r);
    r = __dp4a((int)v.y, 0x01010101, r);
    r = __dp4a((int)v.z, 0x01010101, r);
    r = __dp4a((int)v.w, 0x01010101, r);
  }
  return r;
}

// ---------------------------------------------------------------------------
// Radix-4 butterflies on fp32x2 pairs.  H4 = J - 2*antidiag, so with
// S = ((a+b)+c)+d:  y_j = S - 2 x_{3-j}  (form B).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void bfly4(float2& a, float2& b, float2& c, float2& d) {
  const float2 m2 = make_float2(-2.f, -2.f);
  float2 s = __fadd2_rn(__fadd2_rn(__fadd2_rn(a, b), c), d);
  float2 na = __ffma2_rn(m2, d, s);
  float2 nb = __ffma2_rn(m2, c, s);
  float2 nc = __ffma2_rn(m2, b, s);
  float2 nd = __ffma2_rn(m2, a, s);
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


// ---------------------------------------------------------------------------
// Per-pair helpers of the fast kernel.  A "pair" is two 16-element chunks
// (2p*W + w)*32 + lane and ((2p+1)*W + w)*32 + lane held as 16 fp32x2
// registers v[i] = (chunk0[i], chunk1[i]).
// ---------------------------------------------------------------------------
template <bool F32, bool SMEM, bool FULL = false>
__device__ __forceinline__ void load_pair(float2 (&v)[16], const void* rowp, int64_t c0,
                                          int64_t cstride, int64_t nchunks) {
  constexpr int CB = F32 ? 64 : 32;  // input bytes per chunk
  // shared row copies are addressed in the 32-bit shared window: one cvta per
  // pair, 32-bit offsets (the row is < 64 KB)
  const uint32_t sbase = SMEM ? smem_u32(rowp) + (uint32_t)c0 * CB : 0u;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t chunk = c0 + h * cstride;
    uint32_t u[CB / 4];
    if (!FULL) {
#pragma unroll
      for (int i = 0; i < CB / 4; ++i) u[i] = 0u;
    }
    if (FULL || chunk < nchunks) {
      const char* src = reinterpret_cast<const char*>(rowp) + chunk * CB;
      if constexpr (SMEM) {
        const uint32_t sa = sbase + (uint32_t)(h * cstride) * CB;
#pragma unroll
        for (int j = 0; j < CB / 16; ++j) {
          const uint4 t = ld_shared_v4(sa + j * 16);
          u[4 * j] = t.x;
          u[4 * j + 1] = t.y;
          u[4 * j + 2] = t.z;
          u[4 * j + 3] = t.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < CB / 32; ++j) {
          uint32_t t[8];
          ld_nc_v8(src + 32 * j, t);
#pragma unroll
          for (int i = 0; i < 8; ++i) u[8 * j + i] = t[i];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float f;
      if constexpr (F32) f = __uint_as_float(u[i]);
      else f = __uint_as_float((i & 1) ? (u[i >> 1] & 0xFFFF0000u) : (u[i >> 1] << 16));
      if (h == 0) v[i].x = f;
      else v[i].y = f;
    }
  }
}

// Unnormalised regular-Hadamard sums of the groups in a pair: radix-4
// stages over the in-chunk digits in registers, outer digits across lanes.
// Warp-uniform (the shuffles need every lane).
template <int N0>
__device__ __forceinline__ void rotate_pair(float2 (&v)[16]) {
  if constexpr (N0 >= 4) {
#pragma unroll
    for (int g = 0; g < 4; ++g) bfly4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
  }
  if constexpr (N0 >= 16) {
#pragma unroll
    for (int j = 0; j < 4; ++j) bfly4(v[j], v[j + 4], v[j + 8], v[j + 12]);
  }
  if constexpr (N0 >= 64) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v[i].x = xlane4(v[i].x, 1);
      v[i].y = xlane4(v[i].y, 1);
    }
  }
  if constexpr (N0 >= 256) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v[i].x = xlane4(v[i].x, 4);
      v[i].y = xlane4(v[i].y, 4);
    }
  }
}

__device__ __forceinline__ float pair_absmax(const float2 (&v)[16]) {
  // four independent chains of depth 4 (not two of depth 8)
  float m[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 16; ++i) m[i & 3] = max3_abs(v[i].x, v[i].y, m[i & 3]);
  return max_nan(max_nan(m[0], m[1]), max_nan(m[2], m[3]));
}

// Per-chunk maxima of a pair: mx over chunk0 (.x), my over chunk1 (.y).
// Same FMNMX3 count as pair_absmax; lets the row-max candidates be tracked
// per chunk instead of per pair.
__device__ __forceinline__ void pair_absmax2(const float2 (&v)[16], float& mx, float& my) {
  float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i & 1] = max3_abs(v[2 * i].x, v[2 * i + 1].x, a[i & 1]);
    a[2 + (i & 1)] = max3_abs(v[2 * i].y, v[2 * i + 1].y, a[2 + (i & 1)]);
  }
  mx = max_nan(a[0], a[1]);
  my = max_nan(a[2], a[3]);
}

// Exponent-span certificate of one bf16 chunk (16 inputs, the same test as
// y_exact_chunk, over the whole chunk, so for N0 = 4 it is conservative):
// true => every fp32 partial sum of the chunk's groups is exact, so each
// y32 * rk IS the reference's double value.  Packed 16-bit SIMD min/max on
// the bf16 magnitudes (zeros sent to 0xFFFF by the -1).
template <int N0, bool SMEM>
__device__ __forceinline__ bool chunk_certified_bf16(const void* rowp, int64_t chunk) {
  uint32_t u[8];
  if constexpr (SMEM) {
    const uint32_t sa = smem_u32(rowp) + (uint32_t)chunk * 32u;
    const uint4 t0 = ld_shared_v4(sa), t1 = ld_shared_v4(sa + 16);
    u[0] = t0.x; u[1] = t0.y; u[2] = t0.z; u[3] = t0.w;
    u[4] = t1.x; u[5] = t1.y; u[6] = t1.z; u[7] = t1.w;
  } else {
    const uint4* q = reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(rowp) + chunk * 32);
    const uint4 t0 = q[0], t1 = q[1];
    u[0] = t0.x; u[1] = t0.y; u[2] = t0.z; u[3] = t0.w;
    u[4] = t1.x; u[5] = t1.y; u[6] = t1.z; u[7] = t1.w;
  }
  uint32_t mx = 0u, mn = 0xFFFFFFFFu;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t m = u[i] & 0x7FFF7FFFu;
    mx = __vmaxu2(mx, m);
    mn = __vminu2(mn, __vsub2(m, 0x00010001u));
  }
  const uint32_t bmax = max(mx & 0xFFFFu, mx >> 16);
  const uint32_t bmin = min(mn & 0xFFFFu, mn >> 16) + 1u;  // 0x10000: all zero
  if (bmax == 0u) return true;                               // all-zero chunk: y = 0
  if (bmax >= 0x7F80u || bmin < 0x0080u) return false;      // inf/NaN or subnormal
  constexpr int L2 = N0 == 4 ? 2 : 4;
  return 1 + L2 + (int)((bmax >> 7) - (bmin >> 7)) + 8 <= 24;
}

// ---- out-of-line cold paths (kept out of the hot loop) ---------------------

// Exact re-decision of flagged elements: bit (h*16 + e) of `m` flags
// element e of chunk c0 + h*cstride.  c0 is the calling lane's own chunk;
// the whole warp participates.
template <bool F32, int BITS>
__device__ __noinline__ void k1_redecide(uint32_t m, const void* rowp, uint8_t* crow,
                                         int64_t c0, int64_t cstride, int64_t nchunks, double s,
                                         int64_t group, int kind, int64_t rot_cols) {
  constexpr int QMAX = BITS == 8 ? 127 : 7;  // BITS 5: 4-bit codes stored as int8
  const int lane = threadIdx.x & 31;
  for (;;) {
    const uint32_t bal = __ballot_sync(0xffffffffu, m != 0);
    if (!bal) break;
    const int src = __ffs(bal) - 1;
    const int bit = __shfl_sync(0xffffffffu, __ffs(m) - 1, src);
    const int i = bit & 15;
    const int64_t chunk = __shfl_sync(0xffffffffu, c0, src) + (bit >> 4) * cstride;
    int code = 0;
    if (chunk < nchunks)
      code = exact_code(y_exact_warp<F32>(rowp, chunk * 16 + i, group, kind, rot_cols), s, QMAX);
    if (lane == src) {
      m &= m - 1;
      if (chunk < nchunks) {
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
  }
}

// Exact row maximum over the candidates |y32| >= thr of every lane that
// has one.  A lane's candidates lie in its best pair `bp` unless its
// second-best pair maximum also reaches thr (then all pairs are scanned).
// Pairs are recomputed from the row copy; the exact values come from
// y_exact_warp.  Whole warp participates.
template <int N0, bool F32, bool SMEM>
__device__ __noinline__ double k1_candidates_max(const void* rowp, int P, int W, int w,
                                                 int64_t nchunks, bool has, int bp, bool all,
                                                 float thr, int64_t group, int kind,
                                                 int64_t rot_cols) {
  const int lane = threadIdx.x & 31;
  double cmax = 0.0;
  for (int p = 0; p < P; ++p) {
    const bool need = has && (all || p == bp);
    if (!__any_sync(0xffffffffu, need)) continue;
    const int64_t c0 = ((int64_t)(2 * p) * W + w) * 32 + lane;
    float2 v[16];
    load_pair<F32, SMEM>(v, rowp, c0, (int64_t)W * 32, nchunks);
    rotate_pair<N0>(v);
    uint32_t m = 0;
    if (need) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        m |= (fabsf(v[i].x) >= thr ? 1u : 0u) << i;
        m |= (fabsf(v[i].y) >= thr ? 1u : 0u) << (16 + i);
      }
    }
    for (;;) {
      const uint32_t bal = __ballot_sync(0xffffffffu, m != 0);
      if (!bal) break;
      const int src = __ffs(bal) - 1;
      const int bit = __shfl_sync(0xffffffffu, __ffs(m) - 1, src);
      const int64_t chunk = __shfl_sync(0xffffffffu, c0, src) + (bit >> 4) * (int64_t)W * 32;
      double y = 0.0;
      if (chunk < nchunks)
        y = y_exact_warp<F32>(rowp, chunk * 16 + (bit & 15), group, kind, rot_cols);
      if (lane == src) {
        cmax = fmax(cmax, fabs(y));
        m &= m - 1;
      }
    }
  }
  return cmax;
}

// Rows the fp32 path cannot certify (non-finite input, fp32 overflow):
// the reference's max and codes element by element.
template <bool F32>
__device__ __noinline__ double k1_slow_row_amax(const void* rowp, int C, int W, int w,
                                                int64_t nchunks, int64_t group, int kind,
                                                int64_t rot_cols) {
  const int lane = threadIdx.x & 31;
  double m = 0.0;
  bool bad = false;
  for (int c = 0; c < C; ++c) {
    const int64_t chunk = ((int64_t)c * W + w) * 32 + lane;
    if (chunk >= nchunks) continue;
    for (int i = 0; i < 16; ++i) {
      const double yr = y_ref<F32>(rowp, chunk * 16 + i, group, kind, rot_cols);
      if (!isfinite(yr)) bad = true;
      m = fmax(m, fabs(yr));
    }
  }
  return bad ? INFINITY : m;
}

template <bool F32, int BITS>
__device__ __noinline__ void k1_slow_row_codes(const void* rowp, uint8_t* crow, int C, int W,
                                               int w, int64_t nchunks, bool invalid, double s,
                                               int64_t group, int kind, int64_t rot_cols) {
  constexpr int QMAX = BITS == 8 ? 127 : 7;  // BITS 5: 4-bit codes stored as int8
  const int lane = threadIdx.x & 31;
  for (int c = 0; c < C; ++c) {
    const int64_t chunk = ((int64_t)c * W + w) * 32 + lane;
    if (chunk >= nchunks) continue;
    for (int i = 0; i < 16; i += 2) {
      int c0 = 0, c1 = 0;
      if (!invalid) {
        c0 = exact_code(y_ref<F32>(rowp, chunk * 16 + i, group, kind, rot_cols), s, QMAX);
        c1 = exact_code(y_ref<F32>(rowp, chunk * 16 + i + 1, group, kind, rot_cols), s, QMAX);
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

}  // namespace

// ---------------------------------------------------------------------------
// Fast kernel.
//
// Layout.  A team of W warps owns one row at a time; lane `lane` of warp w
// handles the chunk pairs p < P = C/2 (chunks (2p*W + w)*32 + lane and
// ((2p+1)*W + w)*32 + lane, 16 elements each).  A group of N0 <= 256
// elements is N0/16 consecutive chunks = consecutive lanes, so in-chunk
// radix-4 digits are in-register butterflies and outer digits are lane
// shuffles.  C is a runtime value: the pair loop is rolled, so the hot loop
// is small (instruction cache) and registers stay at one pair.
//
// Streaming.  Each team streams its rows through a ring of `stages`
// shared-memory row buffers filled by 1-D bulk async copies (TMA engine,
// cp.async.bulk, L2 evict-first) completing on one mbarrier per stage: HBM
// reads of the next rows are in flight while the current row is processed.
// Two passes read the row copy: pass 1 rotates and reduces the row absmax,
// pass 2 rotates again and quantises / packs / stores (recomputing the
// butterflies is cheaper than holding the row in registers).  !BULK reads
// global memory directly (pass 2 then hits L1/L2).
//
// Certified rounding: see the file header and DESIGN.md.
// ---------------------------------------------------------------------------
// Pack + store the codes of one chunk pair from the magic-rounded values
// tb[h][i] (h = chunk of the pair, i = element).  4-bit codes come from the
// biased magic (low nibble = code + 8): one IMAD packs a byte in offset
// binary, one XOR per word turns it into two's-complement nibbles.
template <int BITS, bool FULL>
__device__ __forceinline__ void store_codes_pair(const uint32_t (&tb)[2][16], uint8_t* crow,
                                                 int64_t c0, int64_t cstride, int64_t nchunks,
                                                 int& csum) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t chunk = c0 + h * cstride;
    if (!FULL && chunk >= nchunks) continue;
    if constexpr (BITS == 4) {
      uint32_t by[8];
#pragma unroll
      for (int b2 = 0; b2 < 8; ++b2) by[b2] = tb[h][2 * b2 + 1] * 16u + tb[h][2 * b2];
      uint2 out;
      out.x = __byte_perm(__byte_perm(by[0], by[1], 0x0040), __byte_perm(by[2], by[3], 0x0040),
                          0x5410) ^ 0x88888888u;
      out.y = __byte_perm(__byte_perm(by[4], by[5], 0x0040), __byte_perm(by[6], by[7], 0x0040),
                          0x5410) ^ 0x88888888u;
      *reinterpret_cast<uint2*>(crow + chunk * 8) = out;
    } else {
      uint32_t wds[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        wds[q] = __byte_perm(__byte_perm(tb[h][4 * q], tb[h][4 * q + 1], 0x0040),
                             __byte_perm(tb[h][4 * q + 2], tb[h][4 * q + 3], 0x0040), 0x5410);
      if constexpr (BITS == 5)  // two independent DP4A chains per chunk
        csum += __dp4a((int)wds[0], 0x01010101, __dp4a((int)wds[1], 0x01010101, 0)) +
                __dp4a((int)wds[2], 0x01010101, __dp4a((int)wds[3], 0x01010101, 0));
      *reinterpret_cast<uint4*>(crow + chunk * 16) = make_uint4(wds[0], wds[1], wds[2], wds[3]);
    }
  }
}

// Elements of a pair whose rounding decision is not certified (bit h*16+i).
__device__ __forceinline__ uint32_t near_tie_mask(const float2 (&v)[16], const uint32_t (&tb)[2][16],
                                                  float inv, float mg, float thr) {
  uint32_t fm = 0u;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float ex = fmaf(v[i].x, inv, mg - __uint_as_float(tb[0][i]));
    const float ey = fmaf(v[i].y, inv, mg - __uint_as_float(tb[1][i]));
    fm |= (fabsf(ex) <= thr ? 0u : 1u) << i;
    fm |= (fabsf(ey) <= thr ? 0u : 1u) << (16 + i);
  }
  return fm;
}

// Lane-local exact decisions (N0 <= 16): flagged bits (h*16 + i) of `m`
// index the 32 fp32 sums vl[] of the calling lane's chunk pair.
template <bool F32, int BITS, int N0>
__device__ __noinline__ void k1_redecide_lane(uint32_t m, const float2* vl, const void* rowp,
                                              uint8_t* crow, int64_t c0, int64_t cstride,
                                              int64_t nchunks, double s, int64_t group, int kind,
                                              int64_t rot_cols) {
  constexpr int QMAX = BITS == 8 ? 127 : 7;  // BITS 5: 4-bit codes stored as int8
  while (m) {
    const int bit = __ffs(m) - 1;
    m &= m - 1;
    const int i = bit & 15;
    const int64_t chunk = c0 + (bit >> 4) * cstride;
    if (chunk >= nchunks) continue;
    const float y32 = (bit >> 4) ? vl[i].y : vl[i].x;
    const int code = exact_code(y_exact_chunk<F32, N0>(rowp, chunk, i, kind, rot_cols, y32), s, QMAX);
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

// Lane-local exact |y_ref| maximum over the lane's candidates (N0 <= 16).
template <bool F32, int N0>
__device__ __noinline__ double k1_cands_lane(uint32_t m, const float2* vl, const void* rowp,
                                             int64_t c0, int64_t cstride, int64_t nchunks,
                                             int64_t group, int kind, int64_t rot_cols) {
  double cmax = 0.0;
  while (m) {
    const int bit = __ffs(m) - 1;
    m &= m - 1;
    const int i = bit & 15;
    const int64_t chunk = c0 + (bit >> 4) * cstride;
    if (chunk >= nchunks) continue;
    const float y32 = (bit >> 4) ? vl[i].y : vl[i].x;
    cmax = fmax(cmax, fabs(y_exact_chunk<F32, N0>(rowp, chunk, i, kind, rot_cols, y32)));
  }
  return cmax;
}

// Warp-cooperative versions (N0 >= 64: a group spans lanes).
template <bool F32>
__device__ __noinline__ double k1_cands_warp(uint32_t m, const void* rowp, int64_t c0,
                                             int64_t cstride, int64_t nchunks, int64_t group,
                                             int kind, int64_t rot_cols) {
  const int lane = threadIdx.x & 31;
  double cmax = 0.0;
  for (;;) {
    const uint32_t bal = __ballot_sync(0xffffffffu, m != 0);
    if (!bal) break;
    const int src = __ffs(bal) - 1;
    const int bit = __shfl_sync(0xffffffffu, __ffs(m) - 1, src);
    const int64_t chunk = __shfl_sync(0xffffffffu, c0, src) + (bit >> 4) * cstride;
    double y = 0.0;
    if (chunk < nchunks) y = y_exact_warp<F32>(rowp, chunk * 16 + (bit & 15), group, kind, rot_cols);
    if (lane == src) {
      cmax = fmax(cmax, fabs(y));
      m &= m - 1;
    }
  }
  return cmax;
}

constexpr int kK1MaxTeams = 8;
constexpr int kK1MaxStages = 4;
constexpr int kK1Threads = 256;
constexpr int kK1MinBlocks = 2;  // rolled kernel: <= 128 registers, 16 warps per SM

template <int N0, bool F32, int BITS, bool BULK, bool FULL>
__global__ void __launch_bounds__(kK1Threads, kK1MinBlocks) k1_rolled(K1Args a) {
  constexpr int L = Stages<N0>::L;
  constexpr int QMAX = BITS == 8 ? 127 : 7;  // BITS 5: 4-bit codes stored as int8
  griddep_launch();  // launched with PDL: the successor may queue behind us now
  if constexpr (!BULK) griddep_wait();  // predecessor complete before any global access
  __shared__ TeamScratch ts;
  __shared__ uint64_t full_bar[kK1MaxTeams][kK1MaxStages];
  extern __shared__ __align__(128) uint8_t k1_ring[];

  const int W = a.team_warps;
  const int P = a.chunks / 2;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int team = warp / W;
  const int w = warp - team * W;
  const int teams = blockDim.x / (32 * W);
  const int64_t nchunks = a.K / 16;
  const int64_t cstride = (int64_t)W * 32;
  const int esz = F32 ? 4 : 2;
  const int S = a.stages;
  const uint32_t row_bytes = (uint32_t)(a.K * esz);
  const bool leader = (w == 0 && lane == 0);
  const int64_t row0 = (int64_t)blockIdx.x * teams + team;
  const int64_t row_step = (int64_t)gridDim.x * teams;
  uint8_t* ring = k1_ring + (size_t)team * S * row_bytes;

  if constexpr (BULK) {
    if (threadIdx.x == 0) {
      for (int t = 0; t < teams; ++t)
        for (int s = 0; s < S; ++s) mbar_init(&full_bar[t][s], 1);
      mbar_init_fence();
    }
    if (threadIdx.x < 16) (&ts.rs[0][0])[threadIdx.x] = (&ts.rf[0][0])[threadIdx.x] = 0;
    __syncthreads();
    griddep_wait();  // the shared-memory prologue above overlaps the predecessor's tail
    if (leader) {
      for (int s = 0; s < S; ++s) {
        const int64_t r = row0 + (int64_t)s * row_step;
        if (r >= a.M) break;
        mbar_arrive_expect_tx(&full_bar[team][s], row_bytes);
        bulk_g2s(ring + (size_t)s * row_bytes,
                 reinterpret_cast<const char*>(a.x) + r * a.ldx * esz, row_bytes,
                 &full_bar[team][s]);
      }
    }
  }

  const double rk = N0 == 1 ? 1.0 : 1.0 / sqrt((double)N0);
  const double sqrtn = N0 == 1 ? 1.0 : sqrt((double)N0);
  const double bound_rel = L == 0 ? 0.0
                                  : (6.0 * L * sqrtn) * 5.9604644775390625e-8 +
                                        (double)N0 * sqrtn * 2.220446049250313e-16;

  int it = 0;
  int stage = 0;       // it % S, kept incrementally (no integer division per row)
  uint32_t phase = 0;  // (it / S) & 1
  for (int64_t row = row0; row < a.M;
       row += row_step, ++it, stage = (stage + 1 == S) ? 0 : stage + 1,
               phase ^= (stage == 0) ? 1u : 0u) {
    if constexpr (BULK) mbar_wait(&full_bar[team][stage], phase);
    const void* rowp =
        BULK ? static_cast<const void*>(ring + (size_t)stage * row_bytes)
             : static_cast<const void*>(reinterpret_cast<const char*>(a.x) + row * a.ldx * esz);

    // ---- pass 1: rotate, row absmax (NaN-propagating), best / 2nd pair ----
    // best / second-best CHUNK maxima of this lane (bp = pair, bh = half)
    float lmax = 0.f, lmax_nan = 0.f, m2 = 0.f;
    int bp = 0, bh = 0;
#pragma unroll 1
    for (int p = 0; p < P; ++p) {
      float2 v[16];
      load_pair<F32, BULK, FULL>(v, rowp, ((int64_t)(2 * p) * W + w) * 32 + lane, cstride,
                                 nchunks);
      rotate_pair<N0>(v);
      float mh[2];
      pair_absmax2(v, mh[0], mh[1]);
      lmax_nan = max_nan(lmax_nan, max_nan(mh[0], mh[1]));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (mh[h] > lmax) {
          m2 = lmax;
          lmax = mh[h];
          bp = p;
          bh = h;
        } else {
          m2 = fmaxf(m2, mh[h]);
        }
      }
    }
    const float A32 = team_max_nan(lmax_nan, &ts, team, w, W);
    if (W > 1 && leader && it > 0) rowsum_clear(&ts, team, (it - 1) & 1);  // read by all (barrier)

    // pathological rows (non-finite input, fp32 overflow) go the exact way
    const bool slow_row = !(A32 <= 3.0e38f);
    const double B = slow_row ? 0.0 : bound_rel * (double)A32 * 1.01;
    double amax_ref = 0.0;
    if (!slow_row) {
      if (N0 == 1 || A32 == 0.f) {
        amax_ref = (double)A32;
      } else {
        // candidates |y32| >= A32 - 2B lie in the lane's best pair unless its
        // second-best pair also reaches thr; recompute that pair, settle each
        // candidate exactly (lane-local for N0 <= 16, warp-wide otherwise)
        const float thr = (float)((double)A32 - 2.0 * B) * (1.0f - 1e-6f);
        const bool has = lmax >= thr;
        const bool all = m2 >= thr;
        double cmax = 0.0;
        if constexpr (N0 <= 16) {
          bool settled = false;
          if constexpr (!F32) {
            // common case: every candidate lies in the lane's best chunk and
            // that chunk passes the exponent-span certificate, so its y32 are
            // exact and the candidates' exact maximum is lmax * rk (no
            // re-rotation, no per-element settlement)
            const int64_t bc = ((int64_t)(2 * bp + bh) * W + w) * 32 + lane;
            if (has && !all && a.kind == kRotRegular && a.rot_cols >= a.K && bc < nchunks &&
                chunk_certified_bf16<N0, BULK>(rowp, bc)) {
              cmax = (double)lmax * rk;
              settled = true;
            }
          }
          if (has && !settled) {
#pragma unroll 1
            for (int p = 0; p < P; ++p) {
              if (!(all || p == bp)) continue;
              const int64_t c0 = ((int64_t)(2 * p) * W + w) * 32 + lane;
              float2 vl[16];
              load_pair<F32, BULK, FULL>(vl, rowp, c0, cstride, nchunks);
              rotate_pair<N0>(vl);
              uint32_t m = 0;
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                m |= (fabsf(vl[i].x) >= thr ? 1u : 0u) << i;
                m |= (fabsf(vl[i].y) >= thr ? 1u : 0u) << (16 + i);
              }
              if (m)
                cmax = fmax(cmax, k1_cands_lane<F32, N0>(m, vl, rowp, c0, cstride, nchunks,
                                                         a.group, a.kind, a.rot_cols));
            }
          }
        } else {
          if (__any_sync(0xffffffffu, has))
            cmax = k1_candidates_max<N0, F32, BULK>(rowp, P, W, w, nchunks, has, bp, all, thr,
                                                    a.group, a.kind, a.rot_cols);
        }
        amax_ref = team_max_d(cmax, &ts, team, w, W);
      }
    } else {
      amax_ref = team_max_d(k1_slow_row_amax<F32>(rowp, a.chunks, W, w, nchunks, a.group,
                                                  a.kind, a.rot_cols),
                            &ts, team, w, W);
    }
    if (a.amax_in) amax_ref = a.amax_in[row];  // global row max (row-parallel shard)
    const bool invalid = !isfinite(amax_ref);
    const double s = invalid ? 1.0 : (amax_ref == 0.0 ? 1.0 : amax_ref / (double)QMAX);
    if (invalid && lane == 0 && w == 0) flag_invalid_value(a.err);

    uint8_t* crow = a.codes + row * a.ldc;
    int csum = 0;                       // this lane's code sum (BITS == 5)
    bool resum = (a.K & 15) != 0;       // register sums stale -> re-read the row
    if (!slow_row) {
      // ---- pass 2: certified quantisation + pack + store (see k1_fast) -------
      const float inv = amax_ref == 0.0 ? (float)rk
                                        : (float)(rk * QMAX) * __frcp_rn((float)amax_ref);
      const float margin = (float)B * (inv * 1.05f) +
                           (float)(QMAX + 4) * 2.384185791015625e-7f + 1e-9f;
      const float thr = 0.5f - margin;
      // 4-bit packing wants the +8-biased magic (low nibble = code + 8); int8
      // codes (BITS 5, 8) the plain one: the low byte IS the two's-complement code
      const float mg = __uint_as_float(kMagic23 + (BITS == 4 ? 8u : 0u));
      const float2 iv = make_float2(inv, inv);
      const float2 cc = make_float2(mg, mg);
#pragma unroll 1
      for (int p = 0; p < P; ++p) {
        const int64_t c0 = ((int64_t)(2 * p) * W + w) * 32 + lane;
        float2 v[16];
        load_pair<F32, BULK, FULL>(v, rowp, c0, cstride, nchunks);
        rotate_pair<N0>(v);
        uint32_t tb[2][16];
        float em[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 t = __ffma2_rn(v[i], iv, cc);
          const float2 nr = __ffma2_rn(t, make_float2(-1.f, -1.f), cc);
          const float2 e = __ffma2_rn(v[i], iv, nr);
          em[i & 3] = max3_abs(e.x, e.y, em[i & 3]);
          tb[0][i] = __float_as_uint(t.x);
          tb[1][i] = __float_as_uint(t.y);
        }
        int ps = 0;  // this pair's code sum (BITS == 5)
        store_codes_pair<BITS, FULL>(tb, crow, c0, cstride, nchunks, ps);
        uint32_t fm = 0u;
        if (!(max_nan(max_nan(em[0], em[1]), max_nan(em[2], em[3])) <= thr))
          fm = near_tie_mask(v, tb, inv, mg, thr);
        if constexpr (N0 <= 16) {
          if (fm) {
            float2 vl[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) vl[i] = v[i];
            k1_redecide_lane<F32, BITS, N0>(fm, vl, rowp, crow, c0, cstride, nchunks, s, a.group,
                                            a.kind, a.rot_cols);
            if constexpr (BITS == 5) ps = reread_pair_sum<FULL>(crow, c0, cstride, nchunks);
          }
        } else {
          if (__any_sync(0xffffffffu, fm != 0u)) {
            k1_redecide<F32, BITS>(fm, rowp, crow, c0, cstride, nchunks, s, a.group, a.kind,
                                   a.rot_cols);
            if constexpr (BITS == 5) {
              __syncwarp();
              ps = reread_pair_sum<FULL>(crow, c0, cstride, nchunks);
            }
          }
        }
        csum += ps;
      }
    } else {
      resum = true;
      k1_slow_row_codes<F32, BITS>(rowp, crow, a.chunks, W, w, nchunks, invalid, s, a.group,
                                   a.kind, a.rot_cols);
    }
    if (w == 0 && lane == 0) {
      if (a.s32) a.s32[row] = (float)s;
      if (a.s64) a.s64[row] = s;
      if (a.amax) a.amax[row] = amax_ref;  // exact max|y_ref| (outlier analysis)
    }
    if constexpr (BULK) {
      if (a.rowsum && W > 1) rowsum_publish(csum, resum, &ts, team, it & 1);
      if (W == 1) __syncwarp();
      else named_bar_sync(1 + team, W * 32);
      if (a.rowsum) {
        const int sum = W == 1 ? team_row_sum(csum, resum, crow, a.K, 1, 0, &ts, team)
                               : rowsum_collect(crow, a.K, W, w, &ts, team, it & 1);
        if (leader) a.rowsum[row] = sum;
      }
      if (leader) {
        const int64_t r = row + (int64_t)S * row_step;
        if (r < a.M) {
          fence_proxy_async();
          mbar_arrive_expect_tx(&full_bar[team][stage], row_bytes);
          bulk_g2s(ring + (size_t)stage * row_bytes,
                   reinterpret_cast<const char*>(a.x) + r * a.ldx * esz, row_bytes,
                   &full_bar[team][stage]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Single-pass fast kernel (K <= 24576): the row's C chunks per lane stay in
// registers (fp32x2 pairs, fully unrolled), so each element is loaded once
// from the shared-memory row copy, rotated once and quantised from
// registers.  Per-row work (row absmax, exact max candidates, scale) is
// amortised over 16*C elements per lane.  Layout / streaming / certified
// rounding as in k1_rolled above.
// ---------------------------------------------------------------------------
constexpr int kK1FThreads = 192;  // 6 warps; two CTAs per SM at <= 170 registers
constexpr int kK1FMinBlocks = 2;
// CTAs per SM the single-pass kernel is compiled for: fewer register-resident
// chunks per lane leave room for more warps (C <= 2: 85 registers, 4 CTAs).
constexpr int k1_fast_min_blocks(int C) { return C <= 2 ? 4 : (C <= 4 ? 3 : kK1FMinBlocks); }

template <int C, int N0, bool F32, int BITS, bool BULK, bool FULL>
__global__ void __launch_bounds__(kK1FThreads, k1_fast_min_blocks(C)) k1_fast(K1Args a) {
  constexpr int P = C / 2;
  constexpr int L = Stages<N0>::L;
  constexpr int QMAX = BITS == 8 ? 127 : 7;  // BITS 5: 4-bit codes stored as int8
  __shared__ TeamScratch ts;
  __shared__ uint64_t full_bar[kK1MaxTeams][kK1MaxStages];
  extern __shared__ __align__(128) uint8_t k1_ring[];

  const int W = a.team_warps;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int team = warp / W;
  const int w = warp - team * W;
  const int teams = blockDim.x / (32 * W);
  const int64_t nchunks = a.K / 16;
  const int64_t cstride = (int64_t)W * 32;
  const int esz = F32 ? 4 : 2;
  const int S = a.stages;
  const uint32_t row_bytes = (uint32_t)(a.K * esz);
  const bool leader = (w == 0 && lane == 0);
  const int64_t row0 = (int64_t)blockIdx.x * teams + team;
  const int64_t row_step = (int64_t)gridDim.x * teams;
  uint8_t* ring = k1_ring + (size_t)team * S * row_bytes;

  if constexpr (BULK) {
    if (threadIdx.x == 0) {
      for (int t = 0; t < teams; ++t)
        for (int s = 0; s < S; ++s) mbar_init(&full_bar[t][s], 1);
      mbar_init_fence();
    }
    if (threadIdx.x < 16) (&ts.rs[0][0])[threadIdx.x] = (&ts.rf[0][0])[threadIdx.x] = 0;
    __syncthreads();
    griddep_wait();  // the shared-memory prologue above overlaps the predecessor's tail
    if (leader) {
      for (int s = 0; s < S; ++s) {
        const int64_t r = row0 + (int64_t)s * row_step;
        if (r >= a.M) break;
        mbar_arrive_expect_tx(&full_bar[team][s], row_bytes);
        bulk_g2s(ring + (size_t)s * row_bytes,
                 reinterpret_cast<const char*>(a.x) + r * a.ldx * esz, row_bytes,
                 &full_bar[team][s]);
      }
    }
  }

  const double rk = N0 == 1 ? 1.0 : 1.0 / sqrt((double)N0);
  const double sqrtn = N0 == 1 ? 1.0 : sqrt((double)N0);
  const double bound_rel = L == 0 ? 0.0
                                  : (6.0 * L * sqrtn) * 5.9604644775390625e-8 +
                                        (double)N0 * sqrtn * 2.220446049250313e-16;

  int it = 0;
  int stage = 0;       // it % S, kept incrementally (no integer division per row)
  uint32_t phase = 0;  // (it / S) & 1
  for (int64_t row = row0; row < a.M;
       row += row_step, ++it, stage = (stage + 1 == S) ? 0 : stage + 1,
               phase ^= (stage == 0) ? 1u : 0u) {
    if constexpr (BULK) mbar_wait(&full_bar[team][stage], phase);
    const void* rowp =
        BULK ? static_cast<const void*>(ring + (size_t)stage * row_bytes)
             : static_cast<const void*>(reinterpret_cast<const char*>(a.x) + row * a.ldx * esz);

    // ---- load + rotate (all pairs in registers) ----------------------------
    float2 v[P][16];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      load_pair<F32, BULK, FULL>(v[p], rowp, ((int64_t)(2 * p) * W + w) * 32 + lane, cstride,
                                 nchunks);
      rotate_pair<N0>(v[p]);
    }

    // ---- row absmax (NaN-propagating) with per-quad sub-maxima -------------
    float qmx[P][4];
    float pmx[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float m0 = max3_abs(v[p][4 * q].x, v[p][4 * q].y, 0.f);
        const float m1 = max3_abs(v[p][4 * q + 1].x, v[p][4 * q + 1].y, 0.f);
        const float m2 = max3_abs(v[p][4 * q + 2].x, v[p][4 * q + 2].y, m0);
        const float m3 = max3_abs(v[p][4 * q + 3].x, v[p][4 * q + 3].y, m1);
        qmx[p][q] = max_nan(m2, m3);
      }
      pmx[p] = max_nan(max_nan(qmx[p][0], qmx[p][1]), max_nan(qmx[p][2], qmx[p][3]));
    }
    float lmax = pmx[0];
#pragma unroll
    for (int p = 1; p < P; ++p) lmax = max_nan(lmax, pmx[p]);
    const float A32 = team_max_nan(lmax, &ts, team, w, W);
    if (W > 1 && leader && it > 0) rowsum_clear(&ts, team, (it - 1) & 1);  // read by all (barrier)

    // pathological rows (non-finite input, fp32 overflow) go the exact way
    const bool slow_row = !(A32 <= 3.0e38f);
    const double B = slow_row ? 0.0 : bound_rel * (double)A32 * 1.01;
    double amax_ref = 0.0;
    if (!slow_row) {
      if (N0 == 1 || A32 == 0.f) {
        // no rotation: y32 == x exactly; all-zero fp32 sums <=> all-zero row
        amax_ref = (double)A32;
      } else {
        // candidates for the exact row max: |y32| >= A32 - 2B
        const float thr = (float)((double)A32 - 2.0 * B) * (1.0f - 1e-6f);
        double cmax = 0.0;
        if constexpr (N0 <= 16) {
          if (lmax >= thr) {  // lane-local (divergent) scan of the quads
#pragma unroll
            for (int p = 0; p < P; ++p) {
              uint32_t m = 0;
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (qmx[p][q] >= thr) {
#pragma unroll
                  for (int i = 4 * q; i < 4 * q + 4; ++i) {
                    m |= (fabsf(v[p][i].x) >= thr ? 1u : 0u) << i;
                    m |= (fabsf(v[p][i].y) >= thr ? 1u : 0u) << (16 + i);
                  }
                }
              if (m) {
                float2 vl[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) vl[i] = v[p][i];
                cmax = fmax(cmax, k1_cands_lane<F32, N0>(m, vl, rowp,
                                                     ((int64_t)(2 * p) * W + w) * 32 + lane,
                                                     cstride, nchunks, a.group, a.kind,
                                                     a.rot_cols));
              }
            }
          }
        } else {
#pragma unroll
          for (int p = 0; p < P; ++p) {
            uint32_t m = 0;
            if (lmax >= thr) {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (qmx[p][q] >= thr) {
#pragma unroll
                  for (int i = 4 * q; i < 4 * q + 4; ++i) {
                    m |= (fabsf(v[p][i].x) >= thr ? 1u : 0u) << i;
                    m |= (fabsf(v[p][i].y) >= thr ? 1u : 0u) << (16 + i);
                  }
                }
            }
            if (__any_sync(0xffffffffu, m != 0))
              cmax = fmax(cmax, k1_cands_warp<F32>(m, rowp, ((int64_t)(2 * p) * W + w) * 32 + lane,
                                                   cstride, nchunks, a.group, a.kind,
                                                   a.rot_cols));
          }
        }
        amax_ref = team_max_d(cmax, &ts, team, w, W);
      }
    } else {
      amax_ref = team_max_d(k1_slow_row_amax<F32>(rowp, C, W, w, nchunks, a.group, a.kind,
                                                  a.rot_cols),
                            &ts, team, w, W);
    }
    if (a.amax_in) amax_ref = a.amax_in[row];  // global row max (row-parallel shard)
    const bool invalid = !isfinite(amax_ref);
    const double s = invalid ? 1.0 : (amax_ref == 0.0 ? 1.0 : amax_ref / (double)QMAX);
    if (invalid && lane == 0 && w == 0) flag_invalid_value(a.err);

    uint8_t* crow = a.codes + row * a.ldc;
    int csum = 0;                       // this lane's code sum (BITS == 5)
    bool resum = (a.K & 15) != 0;       // register sums stale -> re-read the row
    if (!slow_row) {
      // ---- certified quantisation + pack + store ------------------------------
      // t = M + rint(y*inv) with M = 1.5*2^23 (ulp 1): the low byte of its
      // bit pattern is the two's-complement code; e = y*inv - rint(y*inv)
      // certifies the decision against the reference's double rint(y/s).
      // inv = fl32(rk / fl32(s)) is within 2 ulp of rk/s: covered by the
      // (QMAX + 4) ulp slack of the margin.
      // inv = rk/s = rk*QMAX/amax, from an fp32 reciprocal (the double s is
      // off this critical path; it is only stored and used by exact paths):
      // within 3 ulp of rk/s, covered by the (QMAX + 4) * 4 ulp slack.
      const float inv = amax_ref == 0.0 ? (float)rk
                                        : (float)(rk * QMAX) * __frcp_rn((float)amax_ref);
      const float margin = (float)B * (inv * 1.05f) +
                           (float)(QMAX + 4) * 2.384185791015625e-7f + 1e-9f;
      const float thr = 0.5f - margin;
      // 4-bit codes use the biased magic M + 8, so the low nibble of t is
      // code + 8 in [1, 15] with nothing above it: one IMAD packs a byte
      // (odd*16 + even) in offset binary and one XOR 0x88888888 per word
      // turns it into two's-complement nibbles.
      // 4-bit packing wants the +8-biased magic (low nibble = code + 8); int8
      // codes (BITS 5, 8) the plain one: the low byte IS the two's-complement code
      const float mg = __uint_as_float(kMagic23 + (BITS == 4 ? 8u : 0u));
      const float2 iv = make_float2(inv, inv);
      const float2 cc = make_float2(mg, mg);
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int64_t c0 = ((int64_t)(2 * p) * W + w) * 32 + lane;
        uint32_t tb[2][16];
        float em[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 t = __ffma2_rn(v[p][i], iv, cc);                   // M + rint(y*inv)
          const float2 nr = __ffma2_rn(t, make_float2(-1.f, -1.f), cc);   // -rint(y*inv)
          const float2 e = __ffma2_rn(v[p][i], iv, nr);                   // y*inv - rint
          em[i & 3] = max3_abs(e.x, e.y, em[i & 3]);
          tb[0][i] = __float_as_uint(t.x);
          tb[1][i] = __float_as_uint(t.y);
        }
        int ps = 0;  // this pair's code sum (BITS == 5)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t chunk = c0 + h * cstride;
          if (!FULL && chunk >= nchunks) continue;
          if constexpr (BITS == 4) {
            uint32_t by[8];
#pragma unroll
            for (int b2 = 0; b2 < 8; ++b2)  // low byte = 16*(odd+8) + (even+8)
              by[b2] = tb[h][2 * b2 + 1] * 16u + tb[h][2 * b2];
            uint2 out;
            out.x = __byte_perm(__byte_perm(by[0], by[1], 0x0040),
                                __byte_perm(by[2], by[3], 0x0040), 0x5410) ^ 0x88888888u;
            out.y = __byte_perm(__byte_perm(by[4], by[5], 0x0040),
                                __byte_perm(by[6], by[7], 0x0040), 0x5410) ^ 0x88888888u;
            *reinterpret_cast<uint2*>(crow + chunk * 8) = out;
          } else {
            uint32_t wds[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              wds[q] = __byte_perm(__byte_perm(tb[h][4 * q], tb[h][4 * q + 1], 0x0040),
                                   __byte_perm(tb[h][4 * q + 2], tb[h][4 * q + 3], 0x0040),
                                   0x5410);
              if constexpr (BITS == 5) ps = __dp4a((int)wds[q], 0x01010101, ps);
            }
            *reinterpret_cast<uint4*>(crow + chunk * 16) =
                make_uint4(wds[0], wds[1], wds[2], wds[3]);
          }
        }
        // rare: elements within the certified margin of a rounding boundary
        // (exact ties y/s = k + 1/2 are common with discrete bf16 data):
        // decided exactly; the owner re-writes the bytes it just stored.
        uint32_t fm = 0u;
        if (!(max_nan(max_nan(em[0], em[1]), max_nan(em[2], em[3])) <= thr)) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float ex = fmaf(v[p][i].x, inv, mg - __uint_as_float(tb[0][i]));
            const float ey = fmaf(v[p][i].y, inv, mg - __uint_as_float(tb[1][i]));
            fm |= (fabsf(ex) <= thr ? 0u : 1u) << i;
            fm |= (fabsf(ey) <= thr ? 0u : 1u) << (16 + i);
          }
        }
        if constexpr (N0 <= 16) {
          if (fm) {
            float2 vl[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) vl[i] = v[p][i];
            k1_redecide_lane<F32, BITS, N0>(fm, vl, rowp, crow, c0, cstride, nchunks, s, a.group,
                                        a.kind, a.rot_cols);
            if constexpr (BITS == 5) ps = reread_pair_sum<FULL>(crow, c0, cstride, nchunks);
          }
        } else {
          if (__any_sync(0xffffffffu, fm != 0u)) {
            k1_redecide<F32, BITS>(fm, rowp, crow, c0, cstride, nchunks, s, a.group, a.kind,
                                   a.rot_cols);
            if constexpr (BITS == 5) {
              __syncwarp();
              ps = reread_pair_sum<FULL>(crow, c0, cstride, nchunks);
            }
          }
        }
        csum += ps;
      }
    } else {
      resum = true;
      k1_slow_row_codes<F32, BITS>(rowp, crow, C, W, w, nchunks, invalid, s, a.group, a.kind,
                                   a.rot_cols);
    }
    if (w == 0 && lane == 0) {
      if (a.s32) a.s32[row] = (float)s;
      if (a.s64) a.s64[row] = s;
      if (a.amax) a.amax[row] = amax_ref;  // exact max|y_ref| (outlier analysis)
    }
    if constexpr (BULK) {
      // every lane of the team is done with this stage: refill it with the
      // row `stages` ahead.
      if (a.rowsum && W > 1) rowsum_publish(csum, resum, &ts, team, it & 1);
      if (W == 1) __syncwarp();
      else named_bar_sync(1 + team, W * 32);
      if (a.rowsum) {
        const int sum = W == 1 ? team_row_sum(csum, resum, crow, a.K, 1, 0, &ts, team)
                               : rowsum_collect(crow, a.K, W, w, &ts, team, it & 1);
        if (leader) a.rowsum[row] = sum;
      }
      if (leader) {
        const int64_t r = row + (int64_t)S * row_step;
        if (r < a.M) {
          fence_proxy_async();
          mbar_arrive_expect_tx(&full_bar[team][stage], row_bytes);
          bulk_g2s(ring + (size_t)stage * row_bytes,
                   reinterpret_cast<const char*>(a.x) + r * a.ldx * esz, row_bytes,
                   &full_bar[team][stage]);
        }
      }
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
  constexpr int QMAX = BITS == 8 ? 127 : 7;  // BITS 5: 4-bit codes stored as int8
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
    if (a.amax_in) {  // global row max (row-parallel shard)
      m = a.amax_in[row];
      bad = !isfinite(m);
    }
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
      if (a.amax) a.amax[row] = bad ? INFINITY : m;
      if (a.rowsum) {
        int sum = 0;
        for (int64_t j = 0; j < a.K; ++j) sum += scodes[j];
        a.rowsum[row] = sum;
      }
    }
    __syncthreads();
  }
}

template <bool F32, int BITS>
cudaError_t k1_exact_launch(const K1Args& a, cudaStream_t st);

template <int N0, bool F32, int BITS>
cudaError_t launch_rolled(const K1Args& a0, cudaStream_t st, int64_t* launches) {
  const int num_sms = device_sm_count();
  K1Args a = a0;
  const int W = a.team_warps;
  const size_t rb = (size_t)a.K * (F32 ? 4 : 2);
  // Teams per CTA: fill the CTA, but never more teams than rows per SM.
  int teams = kK1Threads / (W * 32);
  teams = teams < 1 ? 1 : (teams > kK1MaxTeams ? kK1MaxTeams : teams);
  const int64_t rows_per_sm = (a.M + num_sms - 1) / num_sms;
  if (teams > rows_per_sm) teams = (int)(rows_per_sm < 1 ? 1 : rows_per_sm);
  // Shared-memory row ring: ~216 KB per SM split over the CTAs that fit by
  // registers (kK1MinBlocks); as many stages as fit, up to kK1MaxStages.
  const size_t budget = (size_t)216 * 1024 / kK1MinBlocks;
  int S = (int)(budget / ((size_t)teams * rb));
  if (S > kK1MaxStages) S = kK1MaxStages;
  const bool bulk = S >= 1 && ((uintptr_t)a.x % 16 == 0) && ((a.ldx * (F32 ? 4 : 2)) % 16 == 0);
  a.stages = bulk ? S : 1;
  const int threads = teams * W * 32;
  const size_t smem = bulk ? (size_t)teams * S * rb : 0;
  // Rows too wide for one shared-memory stage (K > 36864 bf16) go to the
  // exact kernel: the direct-load rolled variants are not built (ptxas 12.9
  // crashes on the module that contains them with the others).
  if (!bulk) {
    ++*launches;
    return k1_exact_launch<F32, BITS>(a0, st);
  }
  const bool full = a.K / 16 == (int64_t)a.chunks * W * 32;
  auto kern = full ? k1_rolled<N0, F32, BITS, true, true> : k1_rolled<N0, F32, BITS, true, false>;
  if (bulk) {
    static SmemAttr attr[2];  // per instantiation, [full]
    const cudaError_t e = ensure_dyn_smem(kern, smem, attr[full], true);
    if (e != cudaSuccess) return e;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (a.M + teams - 1) / teams;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  cudaError_t le = launch_pdl(kern, dim3((unsigned)grid), dim3(threads), smem, st, a);
  ++*launches;
  return le;
}

template <int C, int N0, bool F32, int BITS>
cudaError_t launch_fast(const K1Args& a0, cudaStream_t st, int64_t* launches) {
  const int num_sms = device_sm_count();
  K1Args a = a0;
  const int W = a.team_warps;
  const size_t rb = (size_t)a.K * (F32 ? 4 : 2);
  int teams = kK1FThreads / (W * 32);
  teams = teams < 1 ? 1 : (teams > kK1MaxTeams ? kK1MaxTeams : teams);
  const int64_t rows_per_sm = (a.M + num_sms - 1) / num_sms;
  if (teams > rows_per_sm) teams = (int)(rows_per_sm < 1 ? 1 : rows_per_sm);
  const size_t budget = (size_t)216 * 1024 / k1_fast_min_blocks(C);
  int S = (int)(budget / ((size_t)teams * rb));
  if (S > kK1MaxStages) S = kK1MaxStages;
  const bool bulk = S >= 1 && ((uintptr_t)a.x % 16 == 0) && ((a.ldx * (F32 ? 4 : 2)) % 16 == 0);
  a.stages = bulk ? S : 1;
  const int threads = teams * W * 32;
  const size_t smem = bulk ? (size_t)teams * S * rb : 0;
  if (!bulk) {  // unaligned rows: exact kernel (direct-load variants not built)
    ++*launches;
    return k1_exact_launch<F32, BITS>(a0, st);
  }
  const bool full = a.K / 16 == (int64_t)C * W * 32;  // every lane owns C whole chunks
  auto kern = full ? k1_fast<C, N0, F32, BITS, true, true> : k1_fast<C, N0, F32, BITS, true, false>;
  {
    static SmemAttr attr[2];  // per instantiation, [full]
    const cudaError_t e = ensure_dyn_smem(kern, smem, attr[full], true);
    if (e != cudaSuccess) return e;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (a.M + teams - 1) / teams;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, threads, smem, st>>>(a);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace crt
#include "k1_mma.cuh"
#include "k1_team.cuh"
#include "k1_tc.cuh"
namespace crt {

template <int N0, bool F32, int BITS>
cudaError_t launch_any(const K1Args& a, cudaStream_t st, int64_t* l) {
  // Default: the two-pass rolled kernel (128 registers, 16 warps/SM, no
  // spills) -- measured faster than the register-resident single-pass kernel
  // at every FLUX shape (M=4608: K=3072 24.6 vs 28.7 us, K=12288 69.6 vs
  // 92.1 us; N0 sweep profiles/r01_n0_sweep.jsonl).  The single-pass kernel
  // stays as an opt-in (CRT_K1_FAST=1, C <= 8), the tensor-core one as
  // CRT_K1_MMA=1; tests/test_alt_paths.py keeps both bit-exact.
  if constexpr (!F32 && (N0 == 4 || N0 == 16) && BITS != 5) {
    if (mma_path_ok(a, N0, F32)) {
      const cudaError_t e = launch_mma<N0, BITS>(a, st, l);
      if (e != cudaErrorInvalidValue) return e;
    }
  }
  if constexpr (!F32 && (N0 == 4 || N0 == 16)) {
    if (k1_tc_ok(a, BITS)) return launch_tc<N0, BITS>(a, st, l);
  }
  if (k1_team_ok(a, F32, BITS)) return launch_team<N0, F32, BITS>(a, st, l);
  static const bool fast = [] {
    const char* e = getenv("CRT_K1_FAST");
    return e && e[0] == '1';
  }();
  if (fast && a.team_warps == 1) {
    switch (a.chunks) {
      case 2: return launch_fast<2, N0, F32, BITS>(a, st, l);
      case 4: return launch_fast<4, N0, F32, BITS>(a, st, l);
      case 6: return launch_fast<6, N0, F32, BITS>(a, st, l);
      case 8: return launch_fast<8, N0, F32, BITS>(a, st, l);
    }
  }
  return launch_rolled<N0, F32, BITS>(a, st, l);
}

template <bool F32, int BITS>
cudaError_t k1_dispatch(const K1Args& a, int n0, cudaStream_t st, int64_t* l) {
  switch (n0) {
    case 1: return launch_any<1, F32, BITS>(a, st, l);
    case 4: return launch_any<4, F32, BITS>(a, st, l);
    case 16: return launch_any<16, F32, BITS>(a, st, l);
    case 64: return launch_any<64, F32, BITS>(a, st, l);
    case 256: return launch_any<256, F32, BITS>(a, st, l);
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
