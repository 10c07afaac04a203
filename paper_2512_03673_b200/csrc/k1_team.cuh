// k1_team.cuh -- K1 "team" kernel: one CTA per row team, the whole row in
// registers after ONE rotation, rows software-pipelined two deep per warp.
// The default K1 for K <= 16384.
//
// Same contract as k1_rolled (k1_kernels.cuh): group_rotate
// (pipeline.cpp:111-151), compute_scales (quant.cpp:10-24), quantize
// (quant.cpp:26-52), pack_int4 (quant.cpp:64-81); codes and f64 scales
// bit-identical to the reference.  Different work decomposition:
//
//  * A CTA of W warps owns one row at a time; every lane holds CPL chunks of
//    16 elements (CPL = 2: chunks t and t + 32W as fp32x2 pairs; CPL = 1:
//    one chunk as v[i] = (x[i], x[i+8]), the second radix-4 stage using the
//    free swapped-half operand of FADD2/FFMA2).  W*32*16*CPL >= K.
//  * Two phases per row.  P1: load the lane's chunks from the shared-memory
//    ring, rotate once, |y| max, settle the warp's own row-max candidates
//    exactly (the element holding the row's exact max is a candidate of its
//    own warp: |y32| >= |y_ref| - B >= Aw - 2B), publish (fp32 max, exact
//    max) in per-stage slots and arrive on the stage's mbarrier.  P2: wait
//    for that mbarrier (all W warps published), take the row max and scale,
//    quantise the registers, pack, store.
//    Each warp runs P1(row i+1) BEFORE P2(row i): the exchange of row i is
//    normally complete by the time a warp needs it, so no warp waits for the
//    others (no __syncthreads in the loop), and every warp has two rows of
//    independent work.
//  * The last warp to finish P2 of a row (shared-memory counter) does that
//    row's bookkeeping: row code sum (K3 v3 operand), the f32/f64 scales,
//    and the refill of the row's ring stage with the row S ahead (1-D bulk
//    copy, TMA engine, L2 evict-first).
//  * Certified rounding exactly as k1_rolled; the
//    thresholds are per-kernel constants (see below).
//
// Compile with -DCRT_K1_TRACE for per-row %globaltimer stamps
// (crt_debug_k1_trace, tools/k1_trace.py).

namespace crt {

constexpr int kK1PMaxWarps = 32;
constexpr int kK1PMaxStages = 8;
constexpr int kK1TraceRows = 8;  // trace: 2 + 3 * kK1TraceRows words per CTA

#ifndef CRT_K1P_REGS1
#define CRT_K1P_REGS1 80
#endif
#ifndef CRT_K1P_REGS2
#define CRT_K1P_REGS2 120
#endif
template <int CPL>
struct K1PRegs {
  // No spills at these caps.  CPL 1 (two rows x 16 registers of values):
  // 80, so CTAs of up to 25 warps fit (K <= 12800); CPL 2 (two rows x 32):
  // 120, for the wider rows (up to 17 warps, K <= 17408).
  static constexpr int value = CPL == 2 ? CRT_K1P_REGS2 : CRT_K1P_REGS1;
};

// ---- CPL = 1 helpers (one 16-element chunk per lane) ----------------------
template <bool F32, bool FULL>
__device__ __forceinline__ void load_chunk1(float2 (&v)[8], const void* rowp, int64_t c,
                                            int64_t nchunks) {
  constexpr int CB = F32 ? 64 : 32;
  uint32_t u[CB / 4];
#pragma unroll
  for (int i = 0; i < CB / 4; ++i) u[i] = 0u;
  if (FULL || c < nchunks) {
    const uint32_t sa = smem_u32(rowp) + (uint32_t)c * CB;
#pragma unroll
    for (int j = 0; j < CB / 16; ++j) {
      const uint4 t = ld_shared_v4(sa + j * 16);
      u[4 * j] = t.x;
      u[4 * j + 1] = t.y;
      u[4 * j + 2] = t.z;
      u[4 * j + 3] = t.w;
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if constexpr (F32) {
      v[i] = make_float2(__uint_as_float(u[i]), __uint_as_float(u[i + 8]));
    } else {
      const uint32_t lo = u[i >> 1], hi = u[4 + (i >> 1)];
      v[i] = (i & 1) ? make_float2(__uint_as_float(lo & 0xFFFF0000u),
                                   __uint_as_float(hi & 0xFFFF0000u))
                     : make_float2(__uint_as_float(lo << 16), __uint_as_float(hi << 16));
    }
  }
}

__device__ __forceinline__ float2 swap2(float2 a) { return make_float2(a.y, a.x); }

// Regular-Hadamard butterflies on v[i] = (x[i], x[i+8]): in-chunk digit 0
// (elements 4g..4g+3) is bfly4 over v[0..3] / v[4..7] (.x: groups 0,1;
// .y: groups 2,3); digit 1 (elements j, j+4, j+8, j+12) combines the two
// halves: S = (a+b) + (c+d) via one FADD2 with swapped operand.  Outer
// digits (N0 >= 64) are lane shuffles as in rotate_pair.
template <int N0>
__device__ __forceinline__ void rotate_chunk1(float2 (&v)[8]) {
  if constexpr (N0 >= 4) {
    bfly4(v[0], v[1], v[2], v[3]);
    bfly4(v[4], v[5], v[6], v[7]);
  }
  if constexpr (N0 >= 16) {
    const float2 m2 = make_float2(-2.f, -2.f);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 p = __fadd2_rn(v[j], v[j + 4]);            // (a+b, c+d)
      const float2 ss = __fadd2_rn(p, swap2(p));              // (S, S)
      const float2 nj = __ffma2_rn(m2, swap2(v[j + 4]), ss);  // (S-2d, S-2b)
      const float2 nj4 = __ffma2_rn(m2, swap2(v[j]), ss);     // (S-2c, S-2a)
      v[j] = nj;
      v[j + 4] = nj4;
    }
  }
  if constexpr (N0 >= 64) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i].x = xlane4(v[i].x, 1);
      v[i].y = xlane4(v[i].y, 1);
    }
  }
  if constexpr (N0 >= 256) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[i].x = xlane4(v[i].x, 4);
      v[i].y = xlane4(v[i].y, 4);
    }
  }
}

// Element numbering of a lane's values (the bits of the masks below; the
// CPL 2 numbering is the one k1_cands_warp / k1_redecide use):
//   CPL 2: bit = 16 h + i  <->  v[i].{x,y}[h], chunk c0 + h*cstride, position i
//   CPL 1: bit = p         <->  v[p & 7].{x,y}[p >> 3], chunk c0, position p
template <int CPL>
__device__ __forceinline__ float y32_of(const float2* vl, int bit) {
  if constexpr (CPL == 2) return (bit >> 4) ? vl[bit & 15].y : vl[bit & 15].x;
  else return (bit >> 3) ? vl[bit & 7].y : vl[bit & 7].x;
}
template <int CPL>
__device__ __forceinline__ void bit_pos(int bit, int64_t c0, int64_t cstride, int64_t& chunk,
                                        int& pos) {
  if constexpr (CPL == 2) {
    chunk = c0 + (bit >> 4) * cstride;
    pos = bit & 15;
  } else {
    chunk = c0;
    pos = bit;
  }
}
template <int CPL>
__device__ __forceinline__ uint32_t mask_ge(const float2 (&v)[8 * CPL], float thr) {
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 8 * CPL; ++i) {
    m |= (fabsf(v[i].x) >= thr ? 1u : 0u) << i;
    m |= (fabsf(v[i].y) >= thr ? 1u : 0u) << (8 * CPL + i);
  }
  return m;
}

// Lane-local exact max |y_ref| over the flagged elements (N0 <= 16).
template <bool F32, int N0, int CPL>
__device__ __noinline__ double k1p_cands_lane(uint32_t m, const float2* vl, const void* rowp,
                                              int64_t c0, int64_t cstride, int64_t nchunks,
                                              int kind, int64_t rot_cols) {
  double cmax = 0.0;
  while (m) {
    const int bit = __ffs(m) - 1;
    m &= m - 1;
    int64_t chunk;
    int pos;
    bit_pos<CPL>(bit, c0, cstride, chunk, pos);
    if (chunk >= nchunks) continue;
    cmax = fmax(cmax, fabs(y_exact_chunk<F32, N0>(rowp, chunk, pos, kind, rot_cols,
                                                  y32_of<CPL>(vl, bit))));
  }
  return cmax;
}

// Lane-local exact re-decision of flagged elements (N0 <= 16).
template <bool F32, int BITS, int N0, int CPL>
__device__ __noinline__ void k1p_redecide_lane(uint32_t m, const float2* vl, const void* rowp,
                                               uint8_t* crow, int64_t c0, int64_t cstride,
                                               int64_t nchunks, double s, int kind,
                                               int64_t rot_cols) {
  constexpr int QMAX = BITS == 8 ? 127 : 7;
  while (m) {
    const int bit = __ffs(m) - 1;
    m &= m - 1;
    int64_t chunk;
    int pos;
    bit_pos<CPL>(bit, c0, cstride, chunk, pos);
    if (chunk >= nchunks) continue;
    const int code = exact_code(
        y_exact_chunk<F32, N0>(rowp, chunk, pos, kind, rot_cols, y32_of<CPL>(vl, bit)), s, QMAX);
    if constexpr (BITS == 4) {
      uint8_t* bp = crow + chunk * 8 + (pos >> 1);
      const uint8_t old = *bp;
      *bp = (pos & 1) ? (uint8_t)((old & 0x0F) | ((code & 0x0F) << 4))
                      : (uint8_t)((old & 0xF0) | (code & 0x0F));
    } else {
      crow[chunk * 16 + pos] = (uint8_t)code;
    }
  }
}

// Code sum of the lane's stored int8-code chunks (after a re-decision or
// the exact slow path rewrote some of their bytes).
template <int CPL, bool FULL>
__device__ __forceinline__ int reread_sum(const uint8_t* crow, int64_t c0, int64_t cstride,
                                          int64_t nchunks) {
  int r = 0;
#pragma unroll
  for (int h = 0; h < CPL; ++h) {
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

// Pack the magic-rounded values of one 16-element chunk (tb[p] = bits of
// M + rint(y*inv) for position p) and store it; returns the code sum
// (BITS 5).
template <int BITS>
__device__ __forceinline__ int pack_store_chunk(const uint32_t (&tb)[16], uint8_t* crow,
                                                int64_t chunk) {
  int cs = 0;
  if constexpr (BITS == 4) {
    uint32_t by[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) by[b] = tb[2 * b + 1] * 16u + tb[2 * b];
    uint2 out;
    out.x = __byte_perm(__byte_perm(by[0], by[1], 0x0040), __byte_perm(by[2], by[3], 0x0040),
                        0x5410) ^ 0x88888888u;
    out.y = __byte_perm(__byte_perm(by[4], by[5], 0x0040), __byte_perm(by[6], by[7], 0x0040),
                        0x5410) ^ 0x88888888u;
    *reinterpret_cast<uint2*>(crow + chunk * 8) = out;
  } else {
    uint32_t wd[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      wd[q] = __byte_perm(__byte_perm(tb[4 * q], tb[4 * q + 1], 0x0040),
                          __byte_perm(tb[4 * q + 2], tb[4 * q + 3], 0x0040), 0x5410);
      if constexpr (BITS == 5) cs = __dp4a((int)wd[q], 0x01010101, cs);
    }
    *reinterpret_cast<uint4*>(crow + chunk * 16) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
  }
  return cs;
}

// Relaxed 64-bit shared-memory add (ATOMS, no fence): the row-done counter
// lives in the high word, the biased code sum in the low word.  Nothing
// else is published through it, so no release/acquire (which would make
// every warp wait for its outstanding global code stores) is needed; the
// stage's shared-memory reads it orders against the refill have all been
// consumed (data-dependent) before the atomic issues.
__device__ __forceinline__ uint64_t atom_add_relaxed_u64(uint32_t saddr, uint64_t v) {
  uint64_t old;
  asm volatile("atom.relaxed.cta.shared::cta.add.u64 %0, [%1], %2;"
               : "=l"(old)
               : "r"(saddr), "l"(v)
               : "memory");
  return old;
}
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_u32(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

template <int N0, bool F32, int BITS, int CPL, bool FULL>
__global__ void __maxnreg__(K1PRegs<CPL>::value) k1_team(K1Args a) {
  constexpr int L = Stages<N0>::L;
  constexpr int QMAX = BITS == 8 ? 127 : 7;  // BITS 5: 4-bit codes stored as int8
  constexpr int NV = 8 * CPL;                 // float2 registers per row
  griddep_launch();
  __shared__ __align__(8) uint64_t full_bar[kK1PMaxStages];
  __shared__ __align__(8) uint64_t max_bar[kK1PMaxStages];
  __shared__ uint32_t s_amax[kK1PMaxStages][kK1PMaxWarps];  // per warp: fp32 |y| max bits
  __shared__ double s_cmax[kK1PMaxStages][kK1PMaxWarps];    // per warp: exact candidate max
  // per stage: (warps done with the row) << 32 | sum over them of (code sum + kSumBias)
  __shared__ __align__(8) uint64_t s_done[kK1PMaxStages];
  extern __shared__ __align__(128) uint8_t k1_ring[];

  const int W = blockDim.x >> 5;
  const int w = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nchunks = a.K / 16;
  const int64_t cstride = (int64_t)W * 32;
  const int64_t c0 = (int64_t)w * 32 + lane;  // my chunk(s): c0 (+ cstride)
  const int esz = F32 ? 4 : 2;
  const int S = a.stages;
  const uint32_t row_bytes = (uint32_t)(a.K * esz);
  const int64_t row_step = gridDim.x;
  const int64_t n_rows = a.M > (int64_t)blockIdx.x ? (a.M - 1 - blockIdx.x) / row_step + 1 : 0;
  const uint32_t full_u = smem_u32(full_bar), max_u = smem_u32(max_bar);
  const uint32_t done_u = smem_u32(s_done);

#ifdef CRT_K1_TRACE
  unsigned long long* trace =
      a.trace ? a.trace + (size_t)blockIdx.x * (2 + 3 * kK1TraceRows) : nullptr;
  if (trace && threadIdx.x == 0) trace[0] = globaltimer();
#endif
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&max_bar[s], (uint32_t)W);
      s_done[s] = 0ull;
    }
    mbar_init_fence();
  }
  __syncthreads();
  griddep_wait();  // the prologue above overlaps the predecessor's tail
#ifdef CRT_K1_TRACE
  if (trace && threadIdx.x == 0) trace[1] = globaltimer();
#endif
  if (threadIdx.x == 0) {
    for (int s = 0; s < S && s < n_rows; ++s) {
      const int64_t r = (int64_t)blockIdx.x + (int64_t)s * row_step;
      mbar_arrive_expect_tx(&full_bar[s], row_bytes);
      bulk_g2s(k1_ring + (size_t)s * row_bytes,
               reinterpret_cast<const char*>(a.x) + r * a.ldx * esz, row_bytes, &full_bar[s]);
    }
  }

  const double rk = N0 == 1 ? 1.0 : 1.0 / sqrt((double)N0);
  const double sqrtn = N0 == 1 ? 1.0 : sqrt((double)N0);
  // |y32 - y_ref| <= B = bound_rel * A, A = max |y32| over the group's warp
  const double bound_rel = L == 0 ? 0.0
                                  : (6.0 * L * sqrtn) * 5.9604644775390625e-8 +
                                        (double)N0 * sqrtn * 2.220446049250313e-16;
  // Row-max candidates of a warp: |y32| >= (Aw - 2B)(1 - 1e-6), B = 1.01
  // bound_rel Aw: one fp32 multiply of the warp max Aw (factor rounded
  // down; the product's own rounding is inside the slack).
  const float cand_scale = (float)((1.0 - 2.02 * bound_rel) * (1.0 - 2e-6));
  // Certification margin of the rounding decision, one constant for every
  // row: B * inv <= 1.0605 bound_rel QMAX (inv = rk QMAX / amax_ref and
  // amax_ref >= (A32 - B) rk, the exact max or a caller-given global max that
  // is at least the local one; k1_rolled's per-row B * inv * 1.05), plus
  // (QMAX + 4) * 2^-20 for the fp32 reciprocal (rcp.approx), the products
  // and the fma.
  const float q_thr =
      (float)(0.5 - (1.1 * bound_rel * QMAX + (QMAX + 4) * 9.5367431640625e-7 + 1e-9));
  const bool fast_cert = !F32 && a.kind == kRotRegular && a.rot_cols >= a.K;
  const float mg = __uint_as_float(kMagic23 + (BITS == 4 ? 8u : 0u));

  // ---- P1: rotate, max, warp-local exact settlement, publish --------------
  auto p1 = [&](int64_t i, int st, uint32_t ph, float2 (&v)[NV]) {
    mbar_wait_u32(full_u + 8u * st, ph);
#ifdef CRT_K1_TRACE
    if (trace && threadIdx.x == 0 && i < kK1TraceRows) trace[2 + 3 * i] = globaltimer();
#endif
    const void* rowp = k1_ring + (size_t)st * row_bytes;
    float mh[2];
    if constexpr (CPL == 2) {
      load_pair<F32, true, FULL>(v, rowp, c0, cstride, nchunks);
      rotate_pair<N0>(v);
      pair_absmax2(v, mh[0], mh[1]);
    } else {
      load_chunk1<F32, FULL>(v, rowp, c0, nchunks);
      rotate_chunk1<N0>(v);
      float m4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < 8; ++k) m4[k & 3] = max3_abs(v[k].x, v[k].y, m4[k & 3]);
      mh[0] = max_nan(max_nan(m4[0], m4[1]), max_nan(m4[2], m4[3]));
      mh[1] = 0.f;
    }
    const float lm = max_nan(mh[0], mh[1]);
    const uint32_t wm = __reduce_max_sync(0xffffffffu, __float_as_uint(lm));
    const float Aw = __uint_as_float(wm);
    double cmax = 0.0;
    if (!a.amax_in) {
      if (!(Aw <= 3.0e38f)) {  // non-finite input / fp32 overflow: the exact loop
        cmax = k1_slow_row_amax<F32>(rowp, CPL, W, w, nchunks, a.group, a.kind, a.rot_cols);
      } else if (N0 == 1) {
        cmax = (double)Aw;  // no rotation: y32 == x exactly
      } else if (Aw != 0.f) {
        const float thr = Aw * cand_scale;
        if constexpr (N0 <= 16) {
          const bool ha = mh[0] >= thr, hb = CPL == 2 && mh[1] >= thr;
          if (ha || hb) {
            bool settled = false;
            if constexpr (!F32) {
              // candidates only in chunks that pass the exponent-span
              // certificate: their y32 are exact, the exact max is lmax * rk
              if (fast_cert && (!ha || chunk_certified_bf16<N0, true>(rowp, c0)) &&
                  (!hb || chunk_certified_bf16<N0, true>(rowp, c0 + cstride))) {
                cmax = (double)fmaxf(ha ? mh[0] : 0.f, hb ? mh[1] : 0.f) * rk;
                settled = true;
              }
            }
            if (!settled) {
              const uint32_t m = mask_ge<CPL>(v, thr);
              float2 vl[NV];
#pragma unroll
              for (int k = 0; k < NV; ++k) vl[k] = v[k];
              cmax = k1p_cands_lane<F32, N0, CPL>(m, vl, rowp, c0, cstride, nchunks, a.kind,
                                                  a.rot_cols);
            }
          }
        } else {
          const uint32_t m = lm >= thr ? mask_ge<CPL>(v, thr) : 0u;
          if (__any_sync(0xffffffffu, m != 0u))
            cmax = k1_cands_warp<F32>(m, rowp, c0, cstride, nchunks, a.group, a.kind, a.rot_cols);
        }
      }
    }
    const double wc = warp_max_d(cmax);
    if (lane == 0) {
      s_amax[st][w] = wm;
      s_cmax[st][w] = wc;
      mbar_arrive_u32(max_u + 8u * st);  // release: the slots above
    }
  };

  // ---- P2: row max + scale, quantise, pack, store; last warp: bookkeeping --
  auto p2 = [&](int64_t i, int st, uint32_t ph, const float2 (&v)[NV]) {
    const int64_t row = (int64_t)blockIdx.x + i * row_step;
    mbar_wait_u32(max_u + 8u * st, ph);
    const void* rowp = k1_ring + (size_t)st * row_bytes;
    const float A32 =
        __uint_as_float(__reduce_max_sync(0xffffffffu, lane < W ? s_amax[st][lane] : 0u));
    const double amax_ref =
        a.amax_in ? a.amax_in[row] : warp_max_d(lane < W ? s_cmax[st][lane] : 0.0);
    const bool slow_row = !(A32 <= 3.0e38f);  // uniform over the team
    const bool invalid = !isfinite(amax_ref);
    // s = amax/QMAX in double (quant.cpp:21): only the bookkeeping warp and
    // the rare exact paths need it
    auto scale = [&]() -> double {
      return invalid ? 1.0 : (amax_ref == 0.0 ? 1.0 : amax_ref / (double)QMAX);
    };
    uint8_t* crow = a.codes + row * a.ldc;
    int csum = 0;
    if (!slow_row) {
      const float inv =
          amax_ref == 0.0 ? (float)rk : (float)(rk * QMAX) * rcp_approx((float)amax_ref);
      const float2 iv = make_float2(inv, inv);
      const float2 cc = make_float2(mg, mg);
      uint32_t tb[CPL][16];  // magic-rounded bits per chunk and position
      float em[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const float2 t = __ffma2_rn(v[k], iv, cc);
        const float2 nr = __ffma2_rn(t, make_float2(-1.f, -1.f), cc);
        const float2 e = __ffma2_rn(v[k], iv, nr);
        em[k & 3] = max3_abs(e.x, e.y, em[k & 3]);
        if constexpr (CPL == 2) {
          tb[0][k] = __float_as_uint(t.x);
          tb[1][k] = __float_as_uint(t.y);
        } else {
          tb[0][k] = __float_as_uint(t.x);      // positions 0..7
          tb[0][k + 8] = __float_as_uint(t.y);  // positions 8..15
        }
      }
#pragma unroll
      for (int h = 0; h < CPL; ++h) {
        const int64_t chunk = c0 + h * cstride;
        if (FULL || chunk < nchunks) csum += pack_store_chunk<BITS>(tb[h], crow, chunk);
      }
      // rare: elements within the certified margin of a rounding boundary
      // (exact ties y/s = k + 1/2 are common with discrete bf16 data) are
      // decided exactly; the owner re-writes the bytes it just stored
      const float thr = q_thr;
      uint32_t fm = 0u;
      if (!(max_nan(max_nan(em[0], em[1]), max_nan(em[2], em[3])) <= thr)) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const float ex = fmaf(v[k].x, inv, mg - fmaf(v[k].x, inv, mg));
          const float ey = fmaf(v[k].y, inv, mg - fmaf(v[k].y, inv, mg));
          fm |= (fabsf(ex) <= thr ? 0u : 1u) << k;
          fm |= (fabsf(ey) <= thr ? 0u : 1u) << (NV + k);
        }
      }
      if constexpr (N0 <= 16) {
        if (fm) {
          float2 vl[NV];
#pragma unroll
          for (int k = 0; k < NV; ++k) vl[k] = v[k];
          k1p_redecide_lane<F32, BITS, N0, CPL>(fm, vl, rowp, crow, c0, cstride, nchunks,
                                                scale(), a.kind, a.rot_cols);
          if constexpr (BITS == 5) csum = reread_sum<CPL, FULL>(crow, c0, cstride, nchunks);
        }
      } else {
        if (__any_sync(0xffffffffu, fm != 0u)) {
          k1_redecide<F32, BITS>(fm, rowp, crow, c0, cstride, nchunks, scale(), a.group, a.kind,
                                 a.rot_cols);
          if constexpr (BITS == 5) {
            __syncwarp();  // the warp's re-decisions may have rewritten my bytes
            csum = reread_sum<CPL, FULL>(crow, c0, cstride, nchunks);
          }
        }
      }
    } else {
      k1_slow_row_codes<F32, BITS>(rowp, crow, CPL, W, w, nchunks, invalid, scale(), a.group,
                                   a.kind, a.rot_cols);
      if constexpr (BITS == 5) csum = reread_sum<CPL, FULL>(crow, c0, cstride, nchunks);
    }
    int wsum = 0;
    if constexpr (BITS == 5) wsum = __reduce_add_sync(0xffffffffu, csum);
    // ---- done with the row: the last warp does the bookkeeping --------------
    // |warp code sum| <= 32 lanes * 32 codes * 7 < kSumBias, W <= 32: the
    // biased sums never carry into the count.
    constexpr uint32_t kSumBias = 8192u;
    __syncwarp();  // the whole warp is past its reads of the stage
    uint64_t old = 0;
    if (lane == 0)
      old = atom_add_relaxed_u64(done_u + 8u * st, (1ull << 32) | (uint32_t)(wsum + (int)kSumBias));
    old = __shfl_sync(0xffffffffu, old, 0);
    const bool last = (uint32_t)(old >> 32) == (uint32_t)(W - 1);
    if (last && lane == 0) {
      if (a.rowsum)
        a.rowsum[row] = (int)((uint32_t)old + (uint32_t)(wsum + (int)kSumBias) - (uint32_t)W * kSumBias);
      const double s = scale();
      if (invalid) flag_invalid_value(a.err);
      if (a.s32) a.s32[row] = (float)s;
      if (a.s64) a.s64[row] = s;
      if (a.amax) a.amax[row] = amax_ref;  // exact max|y_ref| (outlier analysis)
      s_done[st] = 0ull;
      const int64_t r = row + (int64_t)S * row_step;  // refill: the row S ahead
      if (r < a.M) {
        mbar_arrive_expect_tx(&full_bar[st], row_bytes);
        bulk_g2s(k1_ring + (size_t)st * row_bytes,
                 reinterpret_cast<const char*>(a.x) + r * a.ldx * esz, row_bytes, &full_bar[st]);
      }
    }
#ifdef CRT_K1_TRACE
    if (trace && threadIdx.x == 0 && i < kK1TraceRows) trace[3 + 3 * i] = globaltimer();
    if (trace && last && lane == 0 && i < kK1TraceRows) trace[4 + 3 * i] = globaltimer();
#endif
  };

  // ---- two-deep software pipeline over this CTA's rows ----------------------
  float2 va[NV], vb[NV];
  int st1 = 0, st2 = 0;
  uint32_t ph1 = 0u, ph2 = 0u;
  auto adv = [&](int& st, uint32_t& ph) {
    if (++st == S) {
      st = 0;
      ph ^= 1u;
    }
  };
  if (n_rows > 0) {
    p1(0, st1, ph1, va);
    adv(st1, ph1);
  }
  for (int64_t i = 0; i < n_rows;) {
    if (i + 1 < n_rows) {
      p1(i + 1, st1, ph1, vb);
      adv(st1, ph1);
    }
    p2(i, st2, ph2, va);
    adv(st2, ph2);
    if (++i >= n_rows) break;
    if (i + 1 < n_rows) {
      p1(i + 1, st1, ph1, va);
      adv(st1, ph1);
    }
    p2(i, st2, ph2, vb);
    adv(st2, ph2);
    ++i;
  }
}

// Use the team kernel?  Rows of up to 17 warps x 64 chunks (K <= 17408),
// 16-byte aligned rows (bulk copies), row sums only for the int8-code layout.
inline bool k1_team_ok(const K1Args& a, bool f32, int bits) {
  static const bool off = [] {
    const char* e = getenv("CRT_K1_TEAM");
    return e && e[0] == '0';
  }();
  if (off) return false;
  const int64_t nchunks = a.K / 16;
  if (a.K % 16 != 0 || nchunks < 1 || (nchunks + 63) / 64 > 17) return false;
  if (a.rowsum && bits != 5) return false;
  const int esz = f32 ? 4 : 2;
  return ((uintptr_t)a.x % 16 == 0) && ((a.ldx * esz) % 16 == 0);
}

template <int N0, bool F32, int BITS, int CPL>
cudaError_t launch_team_cpl(const K1Args& a0, cudaStream_t st, int64_t* launches) {
  const int num_sms = device_sm_count();
  K1Args a = a0;
  const int64_t nchunks = a.K / 16;
  const int W = (int)((nchunks + 32 * CPL - 1) / (32 * CPL));
  const int threads = W * 32;
  const size_t rb = (size_t)a.K * (F32 ? 4 : 2);
  const bool full = nchunks == (int64_t)32 * CPL * W;
  auto kern = full ? k1_team<N0, F32, BITS, CPL, true> : k1_team<N0, F32, BITS, CPL, false>;
  // ring depth: as many stages (<= 8) as fit in ~220 KB per SM next to the
  // CTAs the registers allow; at least 3 (two rows in compute + one loading)
  int per_sm_r = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_r, kern, threads, 0);
  if (per_sm_r < 1) per_sm_r = 1;
  int S = kK1PMaxStages;
  while (S > 3 && (size_t)per_sm_r * ((size_t)S * rb + 2048) > (size_t)220 * 1024) --S;
  a.stages = S;
  const size_t smem = (size_t)S * rb;
  {
    static SmemAttr attr[2];  // per instantiation, [full]
    const cudaError_t e = ensure_dyn_smem(kern, smem, attr[full], true);
    if (e != cudaSuccess) return e;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (grid > a.M) grid = a.M;
  if (grid < 1) grid = 1;
  const cudaError_t le = launch_pdl(kern, dim3((unsigned)grid), dim3(threads), smem, st, a);
  ++*launches;
  return le;
}

// One chunk per lane while the CTA fits the register file (W <= 25 at 80
// registers, K <= 12800), two chunks per lane above (K <= 16384 -> W <= 16).
// CRT_K1_CPL=1|2 forces one where it fits (dev aid).
template <int N0, bool F32, int BITS>
cudaError_t launch_team(const K1Args& a, cudaStream_t st, int64_t* launches) {
  static const int force = [] {
    const char* e = getenv("CRT_K1_CPL");
    return e ? atoi(e) : 0;
  }();
  const int64_t nchunks = a.K / 16;
  const bool fits1 = (nchunks + 31) / 32 <= 65536 / (32 * K1PRegs<1>::value);
  const int cpl = (force == 2 || !fits1) ? 2 : 1;
  if (cpl == 1) return launch_team_cpl<N0, F32, BITS, 1>(a, st, launches);
  return launch_team_cpl<N0, F32, BITS, 2>(a, st, launches);
}

}  // namespace crt
