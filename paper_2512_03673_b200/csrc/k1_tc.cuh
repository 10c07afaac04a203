#include <algorithm>
#include <stdio.h>
// k1_tc.cuh -- K1 with the group rotation on the 5th-generation tensor cores
// (tcgen05.mma kind::f16, bf16 x bf16 -> fp32 in TMEM), the rest of K1 on
// the CUDA cores.  Default K1 for bf16 rows with N0 in {4, 16}, K % 1024 == 0,
// K <= 16384, dense rows (ldx == K).
//
// Replaces group_rotate (pipeline.cpp:111-151), compute_scales
// (quant.cpp:10-24), quantize (quant.cpp:26-52) and pack_int4
// (quant.cpp:64-81) for one activation matrix, bit-identical to the
// reference like every K1 kernel (codes, f64 scales).
//
// The rotation of a 16-element group is a 16x16 product, and the activation
// matrix viewed as [M*K/16 groups] x [16] is exactly an MMA A operand:
//  * a TMA box of 128 groups x 16 bf16 (4 KB, 32-byte swizzle) is the A tile
//    of one tcgen05.mma M=128 N=16 K=16 against B = H16 (N0 = 16) or
//    blockdiag(H4, H4, H4, H4) (N0 = 4), y = x * B lands in TMEM: lane g =
//    group g, columns 0..15 = its 16 rotated values (unnormalised);
//  * a tile is R rows = U such units (K = 3072: 2 rows, 3 units;
//    K = 12288: 1 row, 6 units), double-buffered in TMEM (2 x 16U columns);
//  * warp 4 streams tiles into a shared-memory ring with TMA, warp 5 issues
//    the MMAs (one elected thread), warps 0-3 (one warpgroup: TMEM lanes
//    0..127) read y back with tcgen05.ld three times per tile: |y| max, the
//    exact settlement of the row-max candidates, certified quantise + pack +
//    store.  TMEM is the row's y buffer between the passes, so the CUDA cores
//    never unpack bf16 nor run butterflies.
//
// Certification.  The tensor core's fp32 accumulation is not correctly
// rounded and not exact even when the exact sum is fp32-representable
// (alignment truncation; tools/probes/tc_rot_probe.cu: at most 5.2 * 2^-23 *
// max|x| over 6 x 1M groups, exponent spans up to 60 binades).  The bound
// used is B = 64 * 2^-23 * A (A = the max |y| of the warp; max|x| <= max|y|
// for the regular Hadamard), 12x the worst seen and 2x the bound of a
// truncating 24-bit aligner (16 terms x 1 ulp + the final rounding).  Every
// row-max candidate (|y_tc| >= A - 2B) and every near-tie of the rounding
// decision is settled with the reference's own sequential double loop from
// the bf16 inputs still in shared memory; y_tc is never used where it could
// disagree with the reference.  Rows with non-finite input or fp32 overflow
// go element by element.

namespace crt {

constexpr int kK1TcStages = 8;
constexpr int kK1TcThreads = 320;  // 8 compute warps (two warpgroups) + TMA warp + MMA warp
constexpr int kK1TcUnit = 4096;    // bytes of one 128-group A tile

struct K1TcArgs {
  const void* x;         // M x K bf16, dense rows
  int64_t M, K;
  int32_t U, R;          // units per tile, rows per tile
  int64_t tiles;
  int32_t stages;
  uint32_t tmem_cols;    // allocated columns (2 buffers of 16U)
  uint8_t* codes;        // null: amax only
  int64_t ldc;
  float* s32;
  double* s64;
  double* amax;
  int32_t* rowsum;
  const double* amax_in;
  int* err;
  int32_t dbg;           // dev aid (CRT_K1_TC_DBG, timing only, WRONG results): 1 skip the
                         // candidate pass, 2 skip quantise/store, 4 skip the max pass,
                         // 8 skip the MMA
};

__device__ __forceinline__ uint32_t tc_sw32(uint32_t row, uint32_t k) {
  // byte offset of element k of group `row` in a 32B-swizzled K-major tile
  const uint32_t lin = row * 32u + k * 2u;
  return lin ^ (((lin >> 7) & 1u) << 4);
}
__device__ __forceinline__ uint64_t tc_desc_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(256 >> 4) << 32;  // SBO: 8-row groups 256 B apart
  d |= (uint64_t)1 << 46;           // sm100 descriptor version
  d |= (uint64_t)6 << 61;           // SWIZZLE_32B
  return d;
}
__host__ __device__ constexpr uint32_t tc_idesc_bf16(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void tc_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tc_wait(uint32_t bar, uint32_t parity) {
  // pure polling (mbarrier.test_wait): the pipeline's waits are on its
  // critical path, and try_wait's suspend/wake-up costs more than the poll
  asm volatile(
      "{\n.reg .pred P1;\nTCW_%=:\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra TCW_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void tc_tma_2d(uint32_t dst, const CUtensorMap* map, int x, int y,
                                          uint32_t bar) {
  asm volatile(
      "{\n.reg .b64 pol;\ncreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], pol;\n}\n" ::"r"(dst),
      "l"(map), "r"(x), "r"(y), "r"(bar)
      : "memory");
}

// The reference's value of element j (0..N0-1 within its group) of the
// group starting at element e0 of group tile row `grow`: sequential double
// sum in ascending k, products then adds (pipeline.cpp:134-142).
template <int N0>
__device__ __noinline__ double tc_y_ref(const uint8_t* unit_smem, uint32_t grow, int e0, int j) {
  const double r = N0 == 4 ? 0.5 : 0.25;
  double acc = 0.0;
  for (int k = 0; k < N0; ++k) {
    const uint16_t b =
        *reinterpret_cast<const uint16_t*>(unit_smem + grow * 32u + (uint32_t)(e0 + k) * 2u);
    const double xv = (double)__uint_as_float((uint32_t)b << 16);
    acc = __dadd_rn(acc, __dmul_rn(xv, regular_negative((uint32_t)k, (uint32_t)j) ? -r : r));
  }
  return acc;
}

// Exact max |y_ref| over the positions flagged in m (bits 0..15) of group
// row `grow` of a unit in shared memory.
template <int N0>
__device__ __noinline__ double tc_cands_exact(const uint8_t* us, uint32_t grow, uint32_t m) {
  double c = 0.0;
  while (m) {
    const int j = __ffs(m) - 1;
    m &= m - 1;
    const double yr = tc_y_ref<N0>(us, grow, j & ~(N0 - 1), j & (N0 - 1));
    c = isfinite(yr) ? fmax(c, fabs(yr)) : INFINITY;
  }
  return c;
}
// Exact codes of the flagged positions, written over the chunk's bytes
// (s == 0: invalid row, codes 0).
template <int N0, int BITS>
__device__ __noinline__ void tc_redecide(const uint8_t* us, uint32_t grow, uint32_t m, double s,
                                         uint8_t* crow, int64_t gc) {
  constexpr int QMAX = BITS == 8 ? 127 : 7;
  while (m) {
    const int j = __ffs(m) - 1;
    m &= m - 1;
    const int code =
        s == 0.0 ? 0 : exact_code(tc_y_ref<N0>(us, grow, j & ~(N0 - 1), j & (N0 - 1)), s, QMAX);
    if constexpr (BITS == 4) {
      uint8_t* bp = crow + gc * 8 + (j >> 1);
      *bp = (j & 1) ? (uint8_t)((*bp & 0x0F) | ((code & 0x0F) << 4))
                    : (uint8_t)((*bp & 0xF0) | (code & 0x0F));
    } else {
      crow[gc * 16 + j] = (uint8_t)code;
    }
  }
}

template <int N0, int BITS, int UH>
__global__ void __launch_bounds__(kK1TcThreads, 1)
    k1_tc_kernel(K1TcArgs a) {
  constexpr int QMAX = BITS == 8 ? 127 : 7;
  constexpr int U = 2 * UH;  // units per tile; warpgroup h owns units [h*UH, (h+1)*UH)
  griddep_launch();
  extern __shared__ __align__(1024) uint8_t tc_smem[];
  __shared__ __align__(1024) uint8_t hmat[16 * 32];  // B = H16 / blockdiag(H4), 32B swizzle
  __shared__ __align__(8) uint64_t full_bar[kK1TcStages], empty_bar[kK1TcStages];
  __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_base;
  __shared__ uint32_t s_amax[8][4];
  __shared__ double s_cmax[8][4];
  __shared__ int s_sum[8][4];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = a.R, S = a.stages;
  const int64_t GR = a.K / 16;  // groups per row
  const uint32_t ring = smem_u32(tc_smem);
  const uint32_t fb = smem_u32(full_bar), eb = smem_u32(empty_bar);
  const uint32_t tfb = smem_u32(tfull_bar), teb = smem_u32(tempty_bar);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 8);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 8);
    }
    mbar_init_fence();
  }
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {  // B[n][k] = H[k][n]
    const int n = i >> 4, k = i & 15;
    const bool same = N0 == 16 || (k >> 2) == (n >> 2);
    const bool neg = N0 == 16 ? regular_negative((uint32_t)k, (uint32_t)n)
                              : regular_negative((uint32_t)(k & 3), (uint32_t)(n & 3));
    *reinterpret_cast<__nv_bfloat16*>(hmat + tc_sw32((uint32_t)n, (uint32_t)k)) =
        __float2bfloat16(same ? (neg ? -1.f : 1.f) : 0.f);
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // hmat -> MMA (async proxy)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  griddep_wait();  // the prologue above overlaps the predecessor's tail

  const int64_t my_tiles =
      a.tiles > (int64_t)blockIdx.x ? (a.tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (warp == 8) {  // ---------------- TMA producer ----------------
    if (lane == 0) {
      for (int64_t i = 0; i < my_tiles; ++i) {
        const int s = (int)(i % S);
        if (i >= S) tc_wait(eb + 8u * s, (uint32_t)((i / S - 1) & 1));
        const int64_t tile = blockIdx.x + i * gridDim.x;
        // the tile's R whole rows are contiguous: one 1-D bulk copy (linear
        // layout; the MMA reads it through a 32B-swizzle descriptor, see below)
        const int64_t rows = std::min<int64_t>(R, a.M - tile * R);
        const uint32_t bytes = (uint32_t)(rows * a.K * 2);
        mbar_arrive_expect_tx(&full_bar[s], bytes);
        bulk_g2s(tc_smem + (size_t)(s * U) * kK1TcUnit,
                 reinterpret_cast<const char*>(a.x) + tile * R * a.K * 2, bytes, &full_bar[s]);
      }
    }
  } else if (warp == 9) {  // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint64_t hdesc = tc_desc_sw32(smem_u32(hmat));
      const uint32_t idesc = tc_idesc_bf16(128, 16);
      for (int64_t i = 0; i < my_tiles; ++i) {
        const int s = (int)(i % S), b = (int)(i & 1);
        tc_wait(fb + 8u * s, (uint32_t)((i / S) & 1));
        if (i >= 2) tc_wait(teb + 8u * b, (uint32_t)((i / 2 - 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int u = 0; u < ((a.dbg & 8) ? 0 : U); ++u) {
          const uint64_t adesc = tc_desc_sw32(ring + (uint32_t)(s * U + u) * kK1TcUnit);
          const uint32_t d = tmem + (uint32_t)(b * 16 * U + u * 16);
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
              "l"(adesc), "l"(hdesc), "r"(idesc)
              : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                tfb + 8u * b)
            : "memory");
      }
    }
  } else {  // ---------------- compute: two warpgroups (warps 0-3, 4-7) ----------------
    const int wg = warp >> 2;
    const int t = (warp & 3) * 32 + lane;  // my TMEM lane = my group in every unit
    // The A tiles are linear (32 B per group) but read through a 32B-swizzle
    // descriptor, which swaps the two 16-byte halves of groups 4..7 of every
    // 8: the MMA sees x[k ^ 8] there.  H16 (and blockdiag(H4)) commute with
    // that half swap, so those lanes receive y[j ^ 8] in column j; the codes
    // are put back in place when packed and the exact paths index the true
    // elements.
    const bool hswap = (t & 4) != 0;
    constexpr double rk = N0 == 4 ? 0.5 : 0.25;
    constexpr double bound_rel = 64.0 * 1.1920928955078125e-7;  // B = bound_rel * A (header)
    constexpr float cand_scale = (float)((1.0 - 2.02 * bound_rel) * (1.0 - 2e-6));
    constexpr float q_thr =
        (float)(0.5 - (1.1 * bound_rel * QMAX + (QMAX + 4) * 9.5367431640625e-7 + 1e-9));
    constexpr float inv0 = (float)(rk * QMAX);
    const float mg = __uint_as_float(kMagic23 + (BITS == 4 ? 8u : 0u));
    int urow[UH];  // row (within the tile) of my group in each of my units
#pragma unroll
    for (int uu = 0; uu < UH; ++uu) urow[uu] = (int)(((int64_t)(wg * UH + uu) * 128 + t) / GR);
    for (int64_t i = 0; i < my_tiles; ++i) {
      const int s = (int)(i % S), b = (int)(i & 1);
      const int64_t tile = blockIdx.x + i * gridDim.x;
      const int64_t row0 = tile * R;
      const uint8_t* stage = tc_smem + (size_t)(s * U) * kK1TcUnit;
      const uint32_t tbuf = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(b * 16 * U);
      tc_wait(tfb + 8u * b, (uint32_t)((i >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // ---- the one TMEM read: my UH groups' 16 rotated values each -----------
      float y[UH][16];
#pragma unroll
      for (int uu = 0; uu < UH; ++uu) {
        uint32_t* r = reinterpret_cast<uint32_t*>(y[uu]);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
              "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
              "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(tbuf + (uint32_t)((wg * UH + uu) * 16)));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      // TMEM buffer free for the next MMA as soon as every warp has its values
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) tc_arrive(teb + 8u * b);

      // ---- |y| max per unit and per row ------------------------------------
      float um[UH];
#pragma unroll
      for (int uu = 0; uu < UH; ++uu) {
        float m4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < 8; ++k) m4[k & 3] = max3_abs(y[uu][2 * k], y[uu][2 * k + 1], m4[k & 3]);
        um[uu] = max_nan(max_nan(m4[0], m4[1]), max_nan(m4[2], m4[3]));
      }
      float lm[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int uu = 0; uu < UH; ++uu)
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (urow[uu] == r) lm[r] = max_nan(lm[r], um[uu]);
      uint32_t wm[4];
      float Aw[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        wm[r] = r < R ? __reduce_max_sync(0xffffffffu, __float_as_uint(lm[r])) : 0u;
        Aw[r] = __uint_as_float(wm[r]);
      }
      // ---- this warp's row-max candidates, settled exactly ---------------------
      double cmax[4] = {0.0, 0.0, 0.0, 0.0};
      if (!a.amax_in && !(a.dbg & 1)) {
#pragma unroll
        for (int uu = 0; uu < UH; ++uu) {
          float aw = 0.f;
#pragma unroll
          for (int r = 0; r < 4; ++r)
            if (urow[uu] == r) aw = Aw[r];
          const bool slow = !(aw <= 3.0e38f);
          const float thr = aw * cand_scale;
          if (!(slow || (aw != 0.f && um[uu] >= thr))) continue;
          uint32_t m = 0;
#pragma unroll
          for (int j = 0; j < 16; ++j) m |= (slow || fabsf(y[uu][j]) >= thr ? 1u : 0u) << j;
          if (hswap) m = ((m >> 8) | (m << 8)) & 0xFFFFu;
          const double c = tc_cands_exact<N0>(stage + (size_t)(wg * UH + uu) * kK1TcUnit,
                                              (uint32_t)t, m);
#pragma unroll
          for (int r = 0; r < 4; ++r)
            if (urow[uu] == r) cmax[r] = fmax(cmax[r], c);
        }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (r >= R) break;
        const uint64_t bb = (uint64_t)__double_as_longlong(cmax[r]);
        const uint32_t hi = __reduce_max_sync(0xffffffffu, (uint32_t)(bb >> 32));
        const uint32_t lo =
            __reduce_max_sync(0xffffffffu, (uint32_t)(bb >> 32) == hi ? (uint32_t)bb : 0u);
        if (lane == 0) {
          s_amax[warp][r] = wm[r];
          s_cmax[warp][r] = __longlong_as_double((long long)(((uint64_t)hi << 32) | lo));
        }
      }
      tc_named_sync(1, 256);
      float A32[4], inv[4];
      double amax_ref[4];
      bool invalid[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        uint32_t am = 0;
        double cm = 0.0;
        if (r < R) {
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            am = max(am, s_amax[w][r]);
            cm = fmax(cm, s_cmax[w][r]);
          }
        }
        A32[r] = __uint_as_float(am);
        const int64_t row = row0 + r;
        amax_ref[r] = a.amax_in ? (r < R && row < a.M ? a.amax_in[row] : 0.0) : cm;
        invalid[r] = !isfinite(amax_ref[r]);
        inv[r] = amax_ref[r] == 0.0 ? (float)rk : inv0 * __frcp_rn((float)amax_ref[r]);
      }
      // ---- certified quantisation + pack + store from registers ----------------
      int csum[4] = {0, 0, 0, 0};
      if (a.codes && !(a.dbg & 2)) {
#pragma unroll
        for (int uu = 0; uu < UH; ++uu) {
          const int r = urow[uu];
          float ir = 0.f, a32 = 0.f;
          bool inval = false;
          double aref = 0.0;
#pragma unroll
          for (int rr = 0; rr < 4; ++rr)
            if (r == rr) {
              ir = inv[rr];
              a32 = A32[rr];
              inval = invalid[rr];
              aref = amax_ref[rr];
            }
          const int64_t row = row0 + r;
          if (row >= a.M) continue;
          const int64_t gc = (int64_t)(wg * UH + uu) * 128 + t - (int64_t)r * GR;
          uint8_t* crow = a.codes + row * a.ldc;
          const uint8_t* us = stage + (size_t)(wg * UH + uu) * kK1TcUnit;
          uint32_t tb[16];
          const bool exact_all = !(a32 <= 3.0e38f);  // slow row: every element exactly
          uint32_t fm = exact_all ? 0xFFFFu : 0u;
          {
            const float2 iv = make_float2(ir, ir);
            const float2 cc = make_float2(mg, mg);
            float em = 0.f;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float2 yv = make_float2(y[uu][2 * k], y[uu][2 * k + 1]);
              const float2 tt = __ffma2_rn(yv, iv, cc);
              const float2 nr = __ffma2_rn(tt, make_float2(-1.f, -1.f), cc);
              const float2 e = __ffma2_rn(yv, iv, nr);
              em = max3_abs(e.x, e.y, em);
              tb[2 * k] = __float_as_uint(tt.x);
              tb[2 * k + 1] = __float_as_uint(tt.y);
            }
            if (!exact_all && !(em <= q_thr)) {  // rare: near-ties
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float ex = fmaf(y[uu][j], ir, mg - fmaf(y[uu][j], ir, mg));
                fm |= (fabsf(ex) <= q_thr ? 0u : 1u) << j;
              }
            }
          }
          int cs = 0;
          if constexpr (BITS == 4) {
            uint32_t by[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) by[q] = tb[2 * q + 1] * 16u + tb[2 * q];
            uint2 o;
            o.x = __byte_perm(__byte_perm(by[0], by[1], 0x0040), __byte_perm(by[2], by[3], 0x0040),
                              0x5410) ^ 0x88888888u;
            o.y = __byte_perm(__byte_perm(by[4], by[5], 0x0040), __byte_perm(by[6], by[7], 0x0040),
                              0x5410) ^ 0x88888888u;
            *reinterpret_cast<uint2*>(crow + gc * 8) = hswap ? make_uint2(o.y, o.x) : o;
          } else {
            uint32_t wd[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              wd[q] = __byte_perm(__byte_perm(tb[4 * q], tb[4 * q + 1], 0x0040),
                                  __byte_perm(tb[4 * q + 2], tb[4 * q + 3], 0x0040), 0x5410);
              if constexpr (BITS == 5) cs = __dp4a((int)wd[q], 0x01010101, cs);
            }
            *reinterpret_cast<uint4*>(crow + gc * 16) =
                hswap ? make_uint4(wd[2], wd[3], wd[0], wd[1]) : make_uint4(wd[0], wd[1], wd[2], wd[3]);
          }
          if (hswap) fm = ((fm >> 8) | (fm << 8)) & 0xFFFFu;  // true element positions
          if (fm) {  // the owner rewrites the flagged codes it just stored
            const double sr = inval ? 0.0 : (aref == 0.0 ? 1.0 : aref / (double)QMAX);
            tc_redecide<N0, BITS>(us, (uint32_t)t, fm, sr, crow, gc);
            if constexpr (BITS == 5) {
              const uint4 w4 = *reinterpret_cast<const uint4*>(crow + gc * 16);
              cs = __dp4a((int)w4.x, 0x01010101,
                          __dp4a((int)w4.y, 0x01010101,
                                 __dp4a((int)w4.z, 0x01010101, __dp4a((int)w4.w, 0x01010101, 0))));
            }
          }
#pragma unroll
          for (int rr = 0; rr < 4; ++rr)
            if (r == rr) csum[rr] += cs;
        }
      }
      // ---- row bookkeeping; the stage is free once every warp is past it ----
      if constexpr (BITS == 5) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (r >= R) break;
          const int ws = __reduce_add_sync(0xffffffffu, csum[r]);
          if (lane == 0) s_sum[warp][r] = ws;
        }
      }
      __syncwarp();
      if (lane == 0) tc_arrive(eb + 8u * s);
      tc_named_sync(1, 256);
      if (threadIdx.x < R) {
        const int r = threadIdx.x;
        const int64_t row = row0 + r;
        if (row < a.M) {
          double ar = 0.0;
          bool iv = false;
#pragma unroll
          for (int rr = 0; rr < 4; ++rr)
            if (r == rr) {
              ar = amax_ref[rr];
              iv = invalid[rr];
            }
          const double sc = iv ? 1.0 : (ar == 0.0 ? 1.0 : ar / (double)QMAX);
          if (iv) flag_invalid_value(a.err);
          if (a.s32) a.s32[row] = (float)sc;
          if (a.s64) a.s64[row] = sc;
          if (a.amax) a.amax[row] = ar;
          if (BITS == 5 && a.rowsum && a.codes) {
            int sum = 0;
            for (int w = 0; w < 8; ++w) sum += s_sum[w][r];
            a.rowsum[row] = sum;
          }
        }
      }
    }
  }
  __syncthreads();
  if (warp == 9) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                               "r"(a.tmem_cols));
}

}  // namespace crt

namespace crt {

inline PFN_cuTensorMapEncodeTiled_v12000 k1_tc_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
  }();
  return fn;
}

// Use the tensor-core K1?  bf16, regular N0 4/16 without identity tail,
// K % 1024 == 0 (a tile is one or two whole rows of 128-group units),
// K <= 16384, dense 16-byte aligned rows, code rows aligned for the vector
// stores.  CRT_K1_TC=0 turns it off (A/B against the CUDA-core kernels).
inline bool k1_tc_ok(const K1Args& a, int bits) {
  static const bool on = [] {  // opt-in until it beats the team kernel
    const char* e = getenv("CRT_K1_TC");
    return e && e[0] == '1';
  }();
  if (!on || a.kind != kRotRegular || (a.group != 4 && a.group != 16)) return false;
  if (a.rot_cols != a.K || a.K % 1024 != 0 || a.K > 16384 || a.K <= 0 || a.M <= 0) return false;
  {  // tile geometry: R rows = U units, U even and <= 6, R <= 4
    int R = 1;
    while ((R * a.K) % 4096 != 0) ++R;
    const int64_t U = R * a.K / 2048;
    if (R > 4 || U > 6 || U < 2) return false;
  }
  if (a.ldx != a.K || (uintptr_t)a.x % 16) return false;
  if (a.M * (a.K / 16) >= ((int64_t)1 << 31)) return false;
  if (a.rowsum && bits != 5) return false;
  if (a.codes && ((uintptr_t)a.codes % 16 || a.ldc % 16)) return false;
  return true;
}

template <int N0, int BITS>
cudaError_t launch_tc(const K1Args& a, cudaStream_t st, int64_t* launches) {
  const int num_sms = device_sm_count();
  K1TcArgs t{};
  t.x = a.x;
  t.M = a.M;
  t.K = a.K;
  // a tile is R whole rows = U units of 128 groups, U = 2*UH (two warpgroups)
  t.R = 1;
  while ((t.R * a.K) % 4096 != 0) ++t.R;  // R*K/2048 even
  t.U = (int32_t)(t.R * a.K / 2048);
  t.tiles = (a.M + t.R - 1) / t.R;
  uint32_t cols = 32;
  while (cols < (uint32_t)(32 * t.U)) cols <<= 1;
  t.tmem_cols = cols;
  t.codes = a.codes;
  t.ldc = a.ldc;
  t.s32 = a.s32;
  t.s64 = a.s64;
  t.amax = a.amax;
  t.rowsum = a.rowsum;
  t.amax_in = a.amax_in;
  t.err = a.err;
  {
    const char* e = getenv("CRT_K1_TC_DBG");
    t.dbg = e ? atoi(e) : 0;
  }
  auto kern = t.U == 2 ? k1_tc_kernel<N0, BITS, 1>
              : t.U == 4 ? k1_tc_kernel<N0, BITS, 2> : k1_tc_kernel<N0, BITS, 3>;
  // CTAs per SM: TMEM (512 columns), registers; then the deepest ring that
  // fits next to them (the occupancy API reports 1 for this kernel although
  // several ~50 KB CTAs fit; persistent CTAs over disjoint tile lists, so any
  // residency is correct)
  int per_sm = (int)(512 / cols);
  {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    if (fa.numRegs > 0) per_sm = std::min(per_sm, 65536 / (fa.numRegs * kK1TcThreads));
    if (per_sm < 1) per_sm = 1;
  }
  const size_t stage_bytes = (size_t)t.U * kK1TcUnit;
  int S = kK1TcStages;
  while (S > 2 && (size_t)per_sm * (S * stage_bytes + 4096) > (size_t)220 * 1024) --S;
  while (per_sm > 1 && (size_t)per_sm * (S * stage_bytes + 4096) > (size_t)220 * 1024) --per_sm;
  t.stages = S;
  const size_t smem = (size_t)S * stage_bytes;
  {
    static SmemAttr attr[4];
    const cudaError_t e = ensure_dyn_smem(kern, smem, attr[t.U / 2], true);
    if (e != cudaSuccess) return e;
  }
  static const bool dbg = getenv("CRT_K1_TC_DEBUG") != nullptr;
  if (dbg)
    fprintf(stderr, "[k1_tc] U=%d R=%d tiles=%lld cols=%u S=%d smem=%zu per_sm=%d\n", t.U, t.R,
            (long long)t.tiles, cols, S, smem, per_sm);
  int64_t grid = (int64_t)num_sms * per_sm;
  if (grid > t.tiles) grid = t.tiles;
  const cudaError_t le = launch_pdl(kern, dim3((unsigned)grid), dim3(kK1TcThreads), smem, st, t);
  ++*launches;
  return le;
}

}  // namespace crt
