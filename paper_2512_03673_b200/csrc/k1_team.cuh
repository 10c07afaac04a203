// k1_team.cuh -- K1 single-pass "team" kernel (the default for K <= 16384).
//
// Same contract as k1_rolled (k1_kernels.cuh: group_rotate pipeline.cpp:111-151,
// compute_scales quant.cpp:10-24, quantize quant.cpp:26-52, pack_int4
// quant.cpp:64-81; codes and f64 scales bit-identical to the reference),
// different work decomposition:
//
//  * ONE CTA = one row team of W = ceil(K / 1024) warps.  Every lane owns
//    exactly one chunk pair (chunks t and t + 32W, t = 32w + lane; 32
//    elements), so the whole row lives in registers after ONE rotation: no
//    second butterfly pass, no loop over pairs, and a short per-row chain
//    (the rolled kernel holds 96-384 elements per lane and re-rotates them).
//  * Small CTAs (96 threads at K = 3072, 384 at K = 12288) at ~80 registers
//    give 24+ warps per SM; rows are independent CTAs' work, so one CTA's
//    serial settlement / scale chain overlaps the others' streaming.
//  * Rows stream through an S-stage shared-memory ring filled by 1-D bulk
//    copies (TMA engine, L2 evict-first); S - 1 rows are in flight while one
//    is processed.
//  * Two team barriers per row: (A) the fp32 row max, (B) the exact row max
//    (skipped when the row needs no settlement: kind none, all-zero rows, or
//    a caller-given global max).  Everything that has to wait until the whole
//    team is done with a row (the row code sum for K3 v3, refilling the ring
//    stage) is done by thread 0 right after the NEXT row's barrier A, so no
//    end-of-row barrier exists.  Slots read across a barrier that may be
//    skipped are double-buffered by row parity.
//
// Certified rounding is exactly k1_rolled's.

namespace crt {

constexpr int kK1TMaxWarps = 16;   // K <= 16384 elements per row
constexpr int kK1TMaxStages = 4;
constexpr int kK1TThreads = kK1TMaxWarps * 32;
constexpr int kK1TraceRows = 8;  // trace: 2 + 3 * kK1TraceRows words per CTA
#ifndef CRT_K1T_REGS
#define CRT_K1T_REGS 80
#endif
constexpr int kK1TRegs = CRT_K1T_REGS;      // 24 warps per SM at K = 3072 (8 CTAs) and 12288 (2 CTAs), no spills

// near_tie_mask with t recomputed from v (bit h*16 + i flags element i of
// chunk h of the pair).
__device__ __forceinline__ uint32_t near_tie_mask_v(const float2 (&v)[16], float inv, float mg,
                                                    float thr) {
  uint32_t fm = 0u;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float ex = fmaf(v[i].x, inv, mg - fmaf(v[i].x, inv, mg));
    const float ey = fmaf(v[i].y, inv, mg - fmaf(v[i].y, inv, mg));
    fm |= (fabsf(ex) <= thr ? 0u : 1u) << i;
    fm |= (fabsf(ey) <= thr ? 0u : 1u) << (16 + i);
  }
  return fm;
}

// The reference's element-by-element max / codes over the calling lane's
// chunk pair (c0, c0 + cstride): rows the fp32 path cannot certify
// (non-finite input, fp32 overflow) in the lane-pair layout (XG below).
// Same arithmetic as k1_slow_row_*.
template <bool F32>
__device__ __noinline__ double k1_slow_pair_amax(const void* rowp, int64_t c0, int64_t cstride,
                                                 int64_t nchunks, int64_t group, int kind,
                                                 int64_t rot_cols) {
  double m = 0.0;
  bool bad = false;
  for (int h = 0; h < 2; ++h) {
    const int64_t chunk = c0 + h * cstride;
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
__device__ __noinline__ void k1_slow_pair_codes(const void* rowp, uint8_t* crow, int64_t c0,
                                                int64_t cstride, int64_t nchunks, bool invalid,
                                                double s, int64_t group, int kind,
                                                int64_t rot_cols) {
  constexpr int QMAX = BITS == 8 ? 127 : 7;  // BITS 5: 4-bit codes stored as int8
  for (int h = 0; h < 2; ++h) {
    const int64_t chunk = c0 + h * cstride;
    if (chunk >= nchunks) continue;
    for (int i = 0; i < 16; i += 2) {
      int q0 = 0, q1 = 0;
      if (!invalid) {
        q0 = exact_code(y_ref<F32>(rowp, chunk * 16 + i, group, kind, rot_cols), s, QMAX);
        q1 = exact_code(y_ref<F32>(rowp, chunk * 16 + i + 1, group, kind, rot_cols), s, QMAX);
      }
      if constexpr (BITS == 4) {
        crow[chunk * 8 + i / 2] = (uint8_t)((q0 & 0x0F) | ((q1 & 0x0F) << 4));
      } else {
        crow[chunk * 16 + i] = (uint8_t)q0;
        crow[chunk * 16 + i + 1] = (uint8_t)q1;
      }
    }
  }
}

// rotate_team's input chunks in the lane-pair layout (bf16 rows in shared memory): the
// lane pairs' chunks sit at 128-byte-periodic offsets {0, 32}, so the two
// 16-byte halves are read in an order alternating with lane bit 1 (2-way
// instead of 4-way bank conflicts, like load_pair's consecutive chunks).
template <bool FULL>
__device__ __forceinline__ void load_pair_xg(float2 (&v)[16], const void* rowp, int64_t c0i,
                                             int64_t csi, int64_t nchunks, int lane) {
  const uint32_t sw = (uint32_t)(lane >> 1) & 1u;
  const uint32_t sb = smem_u32(rowp);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t chunk = c0i + h * csi;
    uint4 lo = make_uint4(0u, 0u, 0u, 0u), hi = lo;
    if (FULL || chunk < nchunks) {
      const uint32_t ca = sb + (uint32_t)chunk * 32u;
      const uint4 ta = ld_shared_v4(ca + 16u * sw), tb = ld_shared_v4(ca + 16u * (sw ^ 1u));
      lo = sw ? tb : ta;
      hi = sw ? ta : tb;
    }
    const uint32_t u[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float f = __uint_as_float((i & 1) ? (u[i >> 1] & 0xFFFF0000u) : (u[i >> 1] << 16));
      if (h == 0) v[i].x = f;
      else v[i].y = f;
    }
  }
}

// Sum certificate of the calling lane's group (lane-pair layout: both of its
// chunks lie in one group spanning lane bits 0 .. log2(N0 / 32) - 1), from
// the bf16 inputs v before the rotation.  Every value the butterflies form
// -- any stage's output, xlane4's partial sums, rotate_team's u -- is a +-1
// combination of a subset of the group's inputs, so its magnitude is at
// most S = sum |x|, and all are integer multiples of the smallest nonzero
// input's bf16 ulp 2^(E_min - 134) (E_min its biased exponent).  S <= 2^24
// ulps => every fp32 operation is exact.  S is accumulated in fp32 (relative
// error < 2^-16 for 256 terms), so the test is S <= 2^(E_min - 110) (1 -
// 2^-12).  inf / NaN fail the comparison; subnormal inputs are excluded.
// Gaussian rows: ~95% of 64-groups and ~50% of 256-groups pass (the
// exponent-span test: 82% / 4%).  Warp-uniform call (shuffles).
template <int N0>
__device__ __forceinline__ bool group_sum_certified(const float2 (&v)[16]) {
  float2 sa = make_float2(0.f, 0.f);
  uint32_t m0 = 0xFFFFFFFFu, m1 = 0xFFFFFFFFu;  // min |x| bits - 1 (zeros -> top)
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float2 a = make_float2(fabsf(v[i].x), fabsf(v[i].y));
    sa = __fadd2_rn(sa, a);
    m0 = min(m0, __float_as_uint(a.x) - 1u);
    m1 = min(m1, __float_as_uint(a.y) - 1u);
  }
  float s = sa.x + sa.y;
  uint32_t m = min(m0, m1);
#pragma unroll
  for (int o = 1; o < N0 / 32; o <<= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  const uint32_t b = m + 1u;          // smallest nonzero |x| bits; 0: all zero
  if (b == 0u) return true;           // all-zero group: y = 0
  if (b < 0x00800000u) return false;  // subnormal input
  const uint32_t e = b >> 23;         // E_min (inf / NaN fail the comparison)
  if (e > 237u) return false;         // bound not representable
  return s <= __uint_as_float((e + 17u) << 23) * 0.999755859375f;
}

// Exact re-decision of the flagged elements (bit h*16 + i: element i of
// chunk c0 + h*cstride) of a lane whose group passed the exponent-span
// certificate: y32 * rk is the reference's value, so the decision is
// quant.cpp:26-52's nearbyint(y / s) on it, lane-local.
template <int BITS>
__device__ __noinline__ void k1_redecide_cert(uint32_t m, const float2* vl, uint8_t* crow,
                                              int64_t c0, int64_t cstride, int64_t nchunks,
                                              double s, double rk) {
  constexpr int QMAX = BITS == 8 ? 127 : 7;  // BITS 5: 4-bit codes stored as int8
  while (m) {
    const int bit = __ffs(m) - 1;
    m &= m - 1;
    const int i = bit & 15;
    const int64_t chunk = c0 + (bit >> 4) * cstride;
    if (chunk >= nchunks) continue;
    const float y32 = (bit >> 4) ? vl[i].y : vl[i].x;
    const int code = exact_code((double)y32 * rk, s, QMAX);
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

// The team's rotation.  !XG: rotate_pair (in-chunk butterflies, outer
// digits by xlane4).  XG (the lane-pair layout, N0 >= 64): the third radix-4 digit (element bits 4-5, the chunk's position
// in its 4-chunk block) is split over the lane pair (lane, lane ^ 1): with
// H4 = J - 2 antidiag = diag(1,1,1,-1) (H2 (x) H2) P, P the signed
// permutation x -> (x0, x2, x1, -x3), lane a = lane & 1 loads INPUT chunks
// {a, a + 2} of the block and holds OUTPUT chunks {2a, 2a + 1} (c0i / c0
// in k1_team), so the digit is one in-register H2 plus one shuffled H2: 2 shuffles
// and 4 FFMA per element pair instead of xlane4's 6 shuffles and 6 FADD/FFMA.
// Each output takes two roundings (xlane4: three) with partial sums of the
// same four terms, inside the error bound B.  N0 = 256
// adds the fourth digit across lane bits 1-2 (xlane4, stride 2).
template <int N0, bool XG>
__device__ __forceinline__ void rotate_team(float2 (&v)[16], int lane) {
  if constexpr (!XG) {
    rotate_pair<N0>(v);
  } else {
    rotate_pair<16>(v);
    const float sa = (lane & 1) ? -1.f : 1.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float ux = fmaf(v[i].y, sa, v[i].x);   // a = 0: x + y   a = 1: x - y
      const float uy = fmaf(v[i].y, -sa, v[i].x);  //        x - y          x + y
      const float px = __shfl_xor_sync(0xffffffffu, ux, 1);
      const float py = __shfl_xor_sync(0xffffffffu, uy, 1);
      v[i].x = fmaf(ux, sa, px);  // a = 0: u0 + u1 (y0)   a = 1: u0 - u1 (y2)
      v[i].y = fmaf(py, sa, uy);  //        u0 + u1 (y1)          u1 - u0 (y3)
    }
    if constexpr (N0 >= 256) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        v[i].x = xlane4(v[i].x, 2);
        v[i].y = xlane4(v[i].y, 2);
      }
    }
  }
}

// WC > 0: the team width as a compile-time constant (the FLUX widths of the
// production instantiation), so the per-row team loops and index math fold;
// those instantiations also fix forward's outputs (PROD below).  W = 15 runs
// one CTA per SM whatever its registers, so it gets up to 128 (74.8 vs 78.1
// us at K = 15360: fewer rematerialisations); 3 and 12 keep 80 (8 and 2
// CTAs per SM).
template <int N0, bool F32, int BITS, bool FULL, int WC = 0>
__global__ void __maxnreg__(WC == 15 ? 128 : kK1TRegs) k1_team(K1Args a) {
  constexpr int L = Stages<N0>::L;
  constexpr int QMAX = BITS == 8 ? 127 : 7;  // BITS 5: 4-bit codes stored as int8
  griddep_launch();
  __shared__ uint64_t full_bar[kK1TMaxStages];
  __shared__ uint32_t s_amax[2][kK1TMaxWarps];  // per-warp fp32 |y| max bits, by row parity
  __shared__ double s_cmax[2][kK1TMaxWarps];    // per-warp exact candidate max, by row parity
  __shared__ int s_sum[2][kK1TMaxWarps];        // per-warp int8 code sums, by row parity
  extern __shared__ __align__(128) uint8_t k1_ring[];

  const int W = WC > 0 ? WC : (int)(blockDim.x >> 5);
  const int w = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nchunks = a.K / 16;
  // my (output) chunks c0 and c0 + cstride; inputs c0i and c0i + csi (the
  // lane-pair layout of rotate_team for N0 >= 64)
  constexpr bool XG = N0 >= 64;
  // lane-local settlement of certified groups (N0 >= 64, bf16 rows)
  constexpr bool CERTG = !F32 && N0 >= 64;
  const int64_t gl = (int64_t)w * 32 + lane;
  const int64_t cstride = XG ? 1 : (int64_t)W * 32;
  const int64_t c0 = XG ? 4 * (gl >> 1) + 2 * (lane & 1) : gl;
  const int64_t csi = XG ? 2 : cstride;
  const int64_t c0i = XG ? 4 * (gl >> 1) + (lane & 1) : c0;
  const int esz = F32 ? 4 : 2;
  const int S = a.stages;
  const uint32_t row_bytes = (uint32_t)(a.K * esz);
  const int64_t row_step = gridDim.x;
  const bool t0 = threadIdx.x == 0;
  // The compile-time-width instantiations serve only forward's K1 (launcher):
  // codes, row sums and fp32 scales present, no caller max, no outlier max.
  constexpr bool PROD = WC > 0;
  const double* const amax_in = PROD ? nullptr : a.amax_in;
  double* const amax_out = PROD ? nullptr : a.amax;
  int32_t* const rowsum = a.rowsum;
  const bool has_rowsum = PROD || rowsum != nullptr;
  const bool has_codes = PROD || a.codes != nullptr;

#ifdef CRT_K1_TRACE  // dev aid, compiled out by default (costs ~4%: fc2 53.4 vs 51.4 us)
  unsigned long long* trace = a.trace ? a.trace + (size_t)blockIdx.x * (2 + 3 * kK1TraceRows) : nullptr;
#else
  unsigned long long* const trace = nullptr;
#endif
  if (trace && t0) trace[0] = globaltimer();
  if (t0) {
    for (int s = 0; s < S; ++s) mbar_init(&full_bar[s], 1);
    mbar_init_fence();
  }
  __syncthreads();
  griddep_wait();  // the prologue above overlaps the predecessor's tail
  if (trace && t0) trace[1] = globaltimer();
  // (ring stage s holds the CTA's rows s, s + S, ...; stage == it % S)
  // Only the first two rows are requested up front, so every CTA's first
  // row is not queued behind the whole input in HBM; the later stages are
  // filled one per row (below).
  if (t0) {
    for (int s = 0; s < (S < 2 ? S : 2); ++s) {
      const int64_t r = (int64_t)blockIdx.x + (int64_t)s * row_step;
      if (r >= a.M) break;
      mbar_arrive_expect_tx(&full_bar[s], row_bytes);
      bulk_g2s(k1_ring + (size_t)s * row_bytes,
               reinterpret_cast<const char*>(a.x) + r * a.ldx * esz, row_bytes, &full_bar[s]);
    }
  }

  const double rk = N0 == 1 ? 1.0 : 1.0 / sqrt((double)N0);
  const double sqrtn = N0 == 1 ? 1.0 : sqrt((double)N0);
  // |y32 - y_ref| <= B = bound_rel * A (A = the max |y32| of the warp or row)
  const double bound_rel = L == 0 ? 0.0
                                  : (6.0 * L * sqrtn) * 5.9604644775390625e-8 +
                                        (double)N0 * sqrtn * 2.220446049250313e-16;
  // Row-max candidates of a warp: |y32| >= (Aw - 2 B) (1 - 1e-6) with
  // B = 1.01 bound_rel Aw, as ONE fp32 multiply of the warp max Aw (the
  // factor rounded down; the fp32 product's rounding is inside the 1e-6).
  const float cand_scale = (float)((1.0 - 2.02 * bound_rel) * (1.0 - 2e-6));
  // Certification margin of the rounding decision.  B * inv <= 1.0605
  // bound_rel QMAX for every row: inv = rk QMAX / amax_ref and amax_ref >=
  // (A32 - B) rk (the exact max, or a caller-given global max that is at
  // least the local one), so one constant replaces the per-row expression
  // B * inv * 1.05 of k1_rolled; (QMAX + 4) * 2^-22 covers the fp32
  // reciprocal, the products and the fma.
  const float q_thr = (float)(0.5 - (1.1 * bound_rel * QMAX + (QMAX + 4) * 2.384185791015625e-7 +
                                     1e-9));
  const bool fast_cert = !F32 && a.kind == kRotRegular && a.rot_cols >= a.K;

  int stage = 0, pstage = 0, par = 0, it = 0;
  uint32_t phase = 0;
  int64_t prev = -1;
  for (int64_t row = blockIdx.x; row < a.M; row += row_step) {
    mbar_wait(&full_bar[stage], phase);
    const void* rowp = k1_ring + (size_t)stage * row_bytes;
    unsigned long long* tr = (trace && t0 && it < kK1TraceRows) ? trace + 2 + 3 * it : nullptr;
    if (tr) tr[0] = globaltimer();

    // ---- load + rotate once; per-chunk |y| maxima ---------------------------
    float2 v[16];
    if constexpr (XG && !F32)
      load_pair_xg<FULL>(v, rowp, c0i, csi, nchunks, lane);
    else
      load_pair<F32, true, FULL>(v, rowp, c0i, csi, nchunks);
    // gcert: my group (both chunks of the pair, N0 >= 64) passes the sum
    // certificate (every fp32 partial sum exact), so its y32 * rk are the
    // reference's values: row-max candidates and near-ties settle lane-locally
    bool gcert = false;
    if constexpr (CERTG) gcert = fast_cert && group_sum_certified<N0>(v);
    rotate_team<N0, XG>(v, lane);
    float mx, my;
    pair_absmax2(v, mx, my);

    // ---- this warp's exact max over its candidates (before the barrier) ----
    // The element holding the row's exact max is a candidate of its own warp
    // (|y32| >= |y_ref| - B >= Aw - 2B), so the row's exact max is the max of
    // the warps' exact candidate maxima: no second team reduction.
    const uint32_t wm = __reduce_max_sync(0xffffffffu, __float_as_uint(max_nan(mx, my)));
    const float Aw = __uint_as_float(wm);
    double cmax = 0.0;
    if (!amax_in) {
      if (!(Aw <= 3.0e38f)) {  // non-finite input / fp32 overflow: exact loop
        if constexpr (XG)
          cmax = k1_slow_pair_amax<F32>(rowp, c0, cstride, nchunks, a.group, a.kind, a.rot_cols);
        else
          cmax = k1_slow_row_amax<F32>(rowp, 2, W, w, nchunks, a.group, a.kind, a.rot_cols);
      } else if (N0 == 1) {
        cmax = (double)Aw;  // no rotation: y32 == x exactly
      } else if (Aw != 0.f) {
        const float thr = Aw * cand_scale;
        if constexpr (N0 <= 16) {
          const bool ha = mx >= thr, hb = my >= thr;
          if (ha || hb) {
            bool settled = false;
            if constexpr (!F32) {
              // candidates only in chunks that pass the exponent-span
              // certificate: their y32 are exact, the exact max is lmax * rk
              if (fast_cert && (!ha || chunk_certified_bf16<N0, true>(rowp, c0)) &&
                  (!hb || chunk_certified_bf16<N0, true>(rowp, c0 + cstride))) {
                cmax = (double)fmaxf(ha ? mx : 0.f, hb ? my : 0.f) * rk;
                settled = true;
              }
            }
            if (!settled) {
              uint32_t m = 0;
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                m |= (fabsf(v[i].x) >= thr ? 1u : 0u) << i;
                m |= (fabsf(v[i].y) >= thr ? 1u : 0u) << (16 + i);
              }
              float2 vl[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) vl[i] = v[i];
              cmax = k1_cands_lane<F32, N0>(m, vl, rowp, c0, cstride, nchunks, a.group, a.kind,
                                            a.rot_cols);
            }
          }
        } else {
          uint32_t m = 0;
          if (max_nan(mx, my) >= thr) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              m |= (fabsf(v[i].x) >= thr ? 1u : 0u) << i;
              m |= (fabsf(v[i].y) >= thr ? 1u : 0u) << (16 + i);
            }
          }
          if constexpr (CERTG) {
            // candidates of a certified group are exact as y32 * rk (no
            // warp-cooperative double sums)
            if (gcert && m != 0u) {
              cmax = (double)max_nan(mx, my) * rk;
              m = 0u;
            }
          }
          if (__any_sync(0xffffffffu, m != 0u))
            cmax = fmax(cmax, k1_cands_warp<F32>(m, rowp, c0, cstride, nchunks, a.group, a.kind,
                                                 a.rot_cols));
        }
      }
    }
    const double wc = warp_max_d(cmax);
    if (lane == 0) {
      s_amax[par][w] = wm;
      s_cmax[par][w] = wc;
    }

    // ---- the one team barrier of the row -----------------------------------
    __syncthreads();
    if (tr) tr[1] = globaltimer();
    // Bookkeeping that needs the whole team past a row, spread over warps:
    // the last warp (re)fills the ring, warp 1 publishes the previous row's
    // code sum, warp 0 stores this row's scales.  (No proxy fence before
    // the refill: the stage was only read by the generic proxy, ordered by
    // the barrier.)
    if (w == W - 1 && lane == 0) {
      const int ahead = it + 2;  // initial fill of stages 2 .. S-1
      if (ahead < S) {
        const int64_t r = row + 2 * row_step;
        if (r < a.M) {
          mbar_arrive_expect_tx(&full_bar[ahead], row_bytes);
          bulk_g2s(k1_ring + (size_t)ahead * row_bytes,
                   reinterpret_cast<const char*>(a.x) + r * a.ldx * esz, row_bytes,
                   &full_bar[ahead]);
        }
      }
      if (prev >= 0) {  // the previous row's stage is free: the row S ahead of it
        const int64_t r = prev + (int64_t)S * row_step;
        if (r < a.M) {
          mbar_arrive_expect_tx(&full_bar[pstage], row_bytes);
          bulk_g2s(k1_ring + (size_t)pstage * row_bytes,
                   reinterpret_cast<const char*>(a.x) + r * a.ldx * esz, row_bytes,
                   &full_bar[pstage]);
        }
      }
    }
    if (has_rowsum && prev >= 0 && w == (W > 1 ? 1 : 0)) {
      const int sum = __reduce_add_sync(0xffffffffu, lane < W ? s_sum[par ^ 1][lane] : 0);
      if (lane == 0) rowsum[prev] = sum;
    }
    const float A32 = __uint_as_float(
        __reduce_max_sync(0xffffffffu, lane < W ? s_amax[par][lane] : 0u));
    const double amax_ref =
        amax_in ? amax_in[row] : warp_max_d(lane < W ? s_cmax[par][lane] : 0.0);
    const bool slow_row = !(A32 <= 3.0e38f);  // uniform over the team
    const bool invalid = !isfinite(amax_ref);
    // s = amax/QMAX in double (quant.cpp:21) is needed only by thread 0 (the
    // stored scales) and by the rare exact paths
    auto scale = [&]() -> double {
      return invalid ? 1.0 : (amax_ref == 0.0 ? 1.0 : amax_ref / (double)QMAX);
    };
    if (t0) {
      const double s = scale();
      if (invalid) flag_invalid_value(a.err);
      if (PROD || a.s32) a.s32[row] = (float)s;
      if (a.s64) a.s64[row] = s;
      if (amax_out) amax_out[row] = amax_ref;  // exact max|y_ref| (outlier analysis)
    }

    // ---- certified quantisation + pack + store from registers --------------
    uint8_t* crow = a.codes + row * a.ldc;
    int csum = 0;
    if (!has_codes) {
      // amax only (crt_rotated_row_absmax): no codes
    } else if (!slow_row) {
      // inv = rk*QMAX/amax from an fp32 reciprocal (within 3 ulp of rk/s,
      // covered by the margin's slack); t = M + rint(y*inv) (low bits = code),
      // e = y*inv - rint(y*inv) certifies the decision (see k1_rolled)
      const float inv = amax_ref == 0.0 ? (float)rk
                                        : (float)(rk * QMAX) * __frcp_rn((float)amax_ref);
      const float thr = q_thr;
      const float mg = __uint_as_float(kMagic23 + (BITS == 4 ? 8u : 0u));
      const float2 iv = make_float2(inv, inv);
      const float2 cc = make_float2(mg, mg);
      // codes are packed four elements at a time (few live registers); the
      // rare near-tie path recomputes t from v (the same FFMA2 rounding)
      constexpr int NW = BITS == 4 ? 2 : 4;  // code words per chunk
      uint32_t wd[2][NW];
      float em[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t tq[2][4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int i = 4 * q + k;
          const float2 t = __ffma2_rn(v[i], iv, cc);
          const float2 nr = __ffma2_rn(t, make_float2(-1.f, -1.f), cc);
          const float2 e = __ffma2_rn(v[i], iv, nr);
          em[k] = max3_abs(e.x, e.y, em[k]);
          tq[0][k] = __float_as_uint(t.x);
          tq[1][k] = __float_as_uint(t.y);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if constexpr (BITS == 4) {
            // low byte = 16*(odd+8) + (even+8): offset-binary nibbles
            const uint32_t hw = __byte_perm(tq[h][1] * 16u + tq[h][0], tq[h][3] * 16u + tq[h][2],
                                            0x0040);
            if (q & 1) wd[h][q >> 1] = __byte_perm(wd[h][q >> 1], hw, 0x5410) ^ 0x88888888u;
            else wd[h][q >> 1] = hw;
          } else {
            wd[h][q] = __byte_perm(__byte_perm(tq[h][0], tq[h][1], 0x0040),
                                   __byte_perm(tq[h][2], tq[h][3], 0x0040), 0x5410);
            if constexpr (BITS == 5) csum = __dp4a((int)wd[h][q], 0x01010101, csum);
          }
        }
      }
      if constexpr (XG) {
        // the lane's two chunks are adjacent: one 16-byte (packed) or 32-byte
        // (int8) store when the row allows it
        if (FULL || c0 < nchunks) {
          if constexpr (BITS == 4) {
            uint8_t* p = crow + c0 * 8;
            if (((uintptr_t)p & 15) == 0) {
              *reinterpret_cast<uint4*>(p) = make_uint4(wd[0][0], wd[0][1], wd[1][0], wd[1][1]);
            } else {
              *reinterpret_cast<uint2*>(p) = make_uint2(wd[0][0], wd[0][1]);
              *reinterpret_cast<uint2*>(p + 8) = make_uint2(wd[1][0], wd[1][1]);
            }
          } else {
            uint8_t* p = crow + c0 * 16;
            const uint4 lo = make_uint4(wd[0][0], wd[0][1], wd[0][2], wd[0][3]);
            const uint4 hi = make_uint4(wd[1][0], wd[1][1], wd[1][2], wd[1][3]);
            if (((uintptr_t)p & 31) == 0) {
              st_v8(p, lo, hi);
            } else {
              *reinterpret_cast<uint4*>(p) = lo;
              *reinterpret_cast<uint4*>(p + 16) = hi;
            }
          }
        } else if constexpr (BITS == 5) {  // zero-filled chunks: their codes are not stored
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int q = 0; q < NW; ++q) csum -= __dp4a((int)wd[h][q], 0x01010101, 0);
        }
      } else {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t chunk = c0 + h * cstride;
        if (!FULL && chunk >= nchunks) {
          if constexpr (BITS == 5) {  // zero-filled chunk: its codes are not stored
#pragma unroll
            for (int q = 0; q < NW; ++q) csum -= __dp4a((int)wd[h][q], 0x01010101, 0);
          }
          continue;
        }
        if constexpr (BITS == 4)
          *reinterpret_cast<uint2*>(crow + chunk * 8) = make_uint2(wd[h][0], wd[h][1]);
        else
          *reinterpret_cast<uint4*>(crow + chunk * 16) =
              make_uint4(wd[h][0], wd[h][1], wd[h][2], wd[h][3]);
      }
      }
      uint32_t fm = 0u;
      if (!(max_nan(max_nan(em[0], em[1]), max_nan(em[2], em[3])) <= thr))
        fm = near_tie_mask_v(v, inv, mg, thr);
      if constexpr (N0 <= 16) {
        if (fm) {
          float2 vl[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) vl[i] = v[i];
          k1_redecide_lane<F32, BITS, N0>(fm, vl, rowp, crow, c0, cstride, nchunks, scale(), a.group,
                                          a.kind, a.rot_cols);
          if constexpr (BITS == 5) csum = reread_pair_sum<FULL>(crow, c0, cstride, nchunks);
        }
      } else {
        if constexpr (CERTG) {
          if (gcert && fm != 0u) {
            float2 vl[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) vl[i] = v[i];
            k1_redecide_cert<BITS>(fm, vl, crow, c0, cstride, nchunks, scale(), rk);
            fm = 0u;
            if constexpr (BITS == 5) csum = reread_pair_sum<FULL>(crow, c0, cstride, nchunks);
          }
        }
        if (__any_sync(0xffffffffu, fm != 0u)) {
          k1_redecide<F32, BITS>(fm, rowp, crow, c0, cstride, nchunks, scale(), a.group, a.kind,
                                 a.rot_cols);
          if constexpr (BITS == 5) {
            __syncwarp();
            csum = reread_pair_sum<FULL>(crow, c0, cstride, nchunks);
          }
        }
      }
    } else {
      if constexpr (XG)
        k1_slow_pair_codes<F32, BITS>(rowp, crow, c0, cstride, nchunks, invalid, scale(), a.group,
                                      a.kind, a.rot_cols);
      else  // (the same chunks: c0 = 32 w + lane, cstride = 32 W)
        k1_slow_row_codes<F32, BITS>(rowp, crow, 2, W, w, nchunks, invalid, scale(), a.group,
                                     a.kind, a.rot_cols);
      if constexpr (BITS == 5) csum = reread_pair_sum<FULL>(crow, c0, cstride, nchunks);
    }
    if constexpr (BITS == 5) {
      if (has_rowsum) {
        const int ws = __reduce_add_sync(0xffffffffu, csum);
        if (lane == 0) s_sum[par][w] = ws;
      }
    }
    if (tr) tr[2] = globaltimer();
    ++it;
    prev = row;
    pstage = stage;
    par ^= 1;
    if (++stage == S) {
      stage = 0;
      phase ^= 1u;
    }
  }
  if (has_rowsum && prev >= 0) {
    __syncthreads();
    if (t0) {
      int sum = 0;
      for (int i = 0; i < W; ++i) sum += s_sum[par ^ 1][i];
      rowsum[prev] = sum;
    }
  }
}

// Use the team kernel?  Rows of up to 16 warps x 64 chunks (K <= 16384),
// 16-byte aligned rows (bulk copies), row sums only for the int8-code layout.
inline bool k1_team_ok(const K1Args& a, bool f32, int bits) {
  static const bool off = [] {
    const char* e = getenv("CRT_K1_TEAM");
    return e && e[0] == '0';
  }();
  if (off) return false;
  const int64_t nchunks = a.K / 16;
  if (a.K % 16 != 0 || nchunks < 1 || (nchunks + 63) / 64 > kK1TMaxWarps) return false;
  if (a.rowsum && bits != 5) return false;
  const int esz = f32 ? 4 : 2;
  return ((uintptr_t)a.x % 16 == 0) && ((a.ldx * esz) % 16 == 0);
}

template <int N0, bool F32, int BITS>
cudaError_t launch_team(const K1Args& a0, cudaStream_t st, int64_t* launches) {
  const int num_sms = device_sm_count();
  K1Args a = a0;
  const int64_t nchunks = a.K / 16;
  const int W = (int)((nchunks + 63) / 64);
  const int threads = W * 32;
  const size_t rb = (size_t)a.K * (F32 ? 4 : 2);
  const bool full = nchunks == (int64_t)64 * W;
  auto kern = full ? k1_team<N0, F32, BITS, true> : k1_team<N0, F32, BITS, false>;
  // the production path (bf16, N0 = 16, int8 codes) at the FLUX widths:
  // compile-time team width (CRT_K1_WC=0 keeps the runtime-width kernel)
  static const bool wc_off = [] {
    const char* e = getenv("CRT_K1_WC");
    return e && e[0] == '0';
  }();
  int ki = full ? 1 : 0;  // which kernel (its smem attribute is cached per kernel)
  if constexpr (!F32 && BITS == 5) {
    if (full && !wc_off && a.codes && a.rowsum && a.s32 && !a.amax_in && !a.amax) {
      // K = 3072 (cfg1-3), every N0 (M = 4608, N0 = 64 / 256: 20.3 / 35.6 us
      // vs 20.4 / 38.1 at runtime width)
      if (W == 3) kern = k1_team<N0, F32, BITS, true, 3>, ki = 2;
      if constexpr (N0 == 16) {  // the FLUX MLP / proj_out widths
        if (W == 12) kern = k1_team<N0, F32, BITS, true, 12>, ki = 3;
        else if (W == 15) kern = k1_team<N0, F32, BITS, true, 15>, ki = 4;
      }
    }
  }
  // ring depth: up to 4 stages while every CTA the registers allow still fits
  // in ~220 KB of shared memory per SM; at least 2
  int per_sm_r = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_r, kern, threads, 0);
  if (per_sm_r < 1) per_sm_r = 1;
  int S = kK1TMaxStages;
  while (S > 2 && (size_t)per_sm_r * ((size_t)S * rb + 1024) > (size_t)220 * 1024) --S;
  a.stages = S;
  const size_t smem = (size_t)S * rb;
  {
    static SmemAttr attr[5];  // per kernel: [runtime width, not full / full, W = 3 / 12 / 15]
    const cudaError_t e = ensure_dyn_smem(kern, smem, attr[ki], true);
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

}  // namespace crt
