// k3_gemm_v4.cu -- K3 v4: W4A4 GEMM with the weights expanded in SOFTWARE
// into the shared-memory (SS-form) MMA operand.  The default W4A4 path.
//
// Replaces int_gemm (pipeline.cpp:178-204) and the dequant loop of forward
// (pipeline.cpp:224-230), like v3 (k3_gemm_v3.cu), whose tile, epilogue and
// two-issuer structure it keeps.  The difference is the A operand:
//   * v3 stages the offset-binary weights as padded 4-bit units (TMA
//     16U4_ALIGN16B) and expands them with tcgen05.cp ... b4x16_p64 into
//     TMEM.  Those copies run in the tensor pipe: at fc1 the tc pipe is 85%
//     busy for 65% MMA (ncu), and the same kernel with int8 weights in
//     shared memory (W8A8, SS form, no copies) is 10-22% faster even though
//     it moves twice the weight bytes.
//   * v4 TMA-loads the packed offset-binary bytes as they are (64 B per
//     128-code row block, 64B swizzle), and expander warps turn each row's
//     nibbles n = w + 8 into bytes in registers and write them straight
//     into the TMEM A slot with tcgen05.st (lane = row, 4 codes per
//     column); the MMAs read A from TMEM and B from shared memory.  Per
//     stage this moves 8 KB packed + 12 KB B through shared memory
//     (v3: 16 KB padded + 12 KB written, 16 KB + 12 KB read) and puts
//     nothing but MMAs in the tensor pipe.  (Expanding into a shared-memory
//     SS operand instead measured slower than v3: the extra 24 KB of
//     shared-memory traffic per stage.)
//   * D = sum((w+8)*a) = sum(w*a) + 8*S_a[m], acc = D - 8 S_a (S_a = the
//     per-token code sum K1 stores beside the codes).
// Pair tile 256 channels x 192 tokens; warps: 0 TMA producer (each CTA,
// completing on its own barrier), 1-2 MMA issuers (leader, alternate K
// stages -- see k3_gemm_v3.cu for why two), 4..7 epilogue, 3 and 8..14
// expanders (each CTA; two groups of four, one warp per TMEM lane quarter,
// the groups alternate stages).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "k3_gemm.h"
#include "k3_tc_common.cuh"

namespace crt {
namespace {

constexpr int V4_BM = 128;         // channels per CTA (pair: 256)
#ifndef CRT_K3_V4_PS
#define CRT_K3_V4_PS 10
#endif
constexpr int V4_PS = CRT_K3_V4_PS;  // stages
constexpr int V4_EPI_WARPS = 4;    // epilogue warps 4..7 (one per TMEM lane quarter)
constexpr int V4_EXP_WARPS = 8;    // expander warps per CTA: 3 and 8..14, two groups of 4
constexpr int V4_THREADS = 32 * (4 + V4_EPI_WARPS + V4_EXP_WARPS - 1);
constexpr int V4_EPI_THREADS = 32 * V4_EPI_WARPS;
constexpr int V4_AP = V4_BM * 64;        // 8 KB: packed A, 128 rows x 64 B (128 codes), 64B swizzle
// Token-tile width BT (tokens per pair tile) is a template parameter: 192
// by default, 176 where it saves a wave (k3_v4_pick_bt).  224 measured
// slower (one A slot per expander group: 2108 vs 3032 TOPS at fc1).
template <int BT>
struct V4Cfg {
  static constexpr int BTH = BT / 2;                            // token rows of B per CTA
  static constexpr int B = BTH * 128;                           // int8 activation codes, 128B swizzle
  static constexpr int STAGE = (V4_AP + B + 1023) / 1024 * 1024;  // packed A | B, 1024-aligned
  // TMEM (512 columns): accumulators at 0 and 256 (BT columns each), the
  // rest of each half holds 32-column A slots (one 128-code K block each)
  static constexpr int SLOTS = (256 - BT) / 32 * 2;
  static constexpr int NCH = (BT + 31) / 32;                    // epilogue token chunks
  static constexpr int LASTW = BT - 32 * (NCH - 1);             // width of the last one
  static_assert(SLOTS == 4, "two A slots per accumulator half");
  static_assert(LASTW == 32 || LASTW == 16, "chunks of 32 (+ one of 16)");
  static_assert(BT % 16 == 0 && BT <= 192, "UMMA N");
};

template <int BT>
struct V4Smem {
  uint64_t full[V4_PS];      // each CTA: its own TMA bytes (A packed + B)
  uint64_t empty[V4_PS];     // both: MMA commit multicast
  uint64_t slot_full[4];     // leader: A slot written (4 expander warps x 2 CTAs)
  uint64_t slot_empty[4];    // both: MMA commit multicast
  uint64_t acc_full[2];      // both: one commit per MMA issuer
  uint64_t acc_empty[2];     // leader: 8 epilogue warps x 2 CTAs
  uint32_t tmem_base;
  alignas(16) float sa[BT];
  alignas(16) int sums[BT];
};

__device__ __forceinline__ uint32_t acc_col(int b) { return (uint32_t)b * 256u; }
template <int BT>
__device__ __forceinline__ uint32_t a_col(int s) {
  return (s < 2 ? (uint32_t)BT : 256u + (uint32_t)BT) + (uint32_t)(s & 1) * 32u;
}
// Epilogue output staging (YT): one 32-token x 32-channel bf16 box (2 KB)
// per epilogue warp, written with st.shared and stored by one TMA bulk
// tensor store; the tensor map clips tokens >= M and channels >= N.
constexpr int V4_YSTG = 2048;
__device__ __forceinline__ void st_shared_u16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t saddr, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   map),
               "r"(x), "r"(y), "r"(saddr)
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_zero16(uint32_t taddr) {
  const uint32_t z = 0;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(z)
      : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// 2-D TMA load completing on this CTA's own barrier
__device__ __forceinline__ void tma_load_local(void* dst, const CUtensorMap* map, int x, int y,
                                               uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void sts128(uint32_t saddr, uint32_t a, uint32_t b, uint32_t c,
                                       uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(saddr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
// 8 offset-binary nibbles (pack_int4 order: byte t = n[2t] | n[2t+1] << 4)
// -> the 8 bytes n[0..7]
__device__ __forceinline__ void expand8(uint32_t w, uint32_t& lo4, uint32_t& hi4) {
  const uint32_t ev = w & 0x0F0F0F0Fu;         // n[0], n[2], n[4], n[6]
  const uint32_t od = (w >> 4) & 0x0F0F0F0Fu;  // n[1], n[3], n[5], n[7]
  lo4 = __byte_perm(ev, od, 0x5140);
  hi4 = __byte_perm(ev, od, 0x7362);
}
struct V4Args {
  int64_t M, N, K;
  int32_t ttiles, ctiles;
  const float* a_scales;
  const int32_t* a_sums;
  const float* w_scales;
  const float* bias;
  int32_t out_kind;  // 0 bf16, 1 f32, 2 int32 accumulators
  void* y;
  int64_t ldy;
  int32_t fdq;       // magic-number fp32x2 dequant (bf16 output)
  unsigned long long* trace;  // dev aid (crt_debug_k3_trace), as v3's layout
  int32_t dbg;                // dev aid (builds with -DCRT_K3_DBG; CRT_K3_V4_DBG bitmask, timing only, wrong output):
                              // 1 no A-slot stores, 2 no dequant/stores, 4 no TMEM loads/zeroing
};

// YT: bf16 output through shared-memory boxes and TMA bulk stores (set by
// the launcher when out_kind == bf16 and y is 16-byte aligned).
template <int BT, bool YT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(V4_THREADS, 1)
    k3_v4_kernel(const __grid_constant__ CUtensorMap map_w,
                 const __grid_constant__ CUtensorMap map_x,
                 const __grid_constant__ CUtensorMap map_y, V4Args a) {
  using C = V4Cfg<BT>;
  constexpr int V4_BT = BT, V4_BTH = C::BTH, V4_B = C::B, V4_STAGE = C::STAGE, V4_SLOTS = C::SLOTS;
  using V4Smem = crt::V4Smem<BT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* stg = smem;                          // V4_PS x (packed A 8 KB | B 12 KB)
  V4Smem* ss = reinterpret_cast<V4Smem*>(smem + V4_PS * V4_STAGE);
  uint8_t* ystg = smem + V4_PS * V4_STAGE + ((sizeof(V4Smem) + 127) & ~(size_t)127);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int npairs = gridDim.x >> 1;
  const int pair = blockIdx.x >> 1;
  const int ntiles = a.ttiles * a.ctiles;
  const int KB = (int)((a.K + 127) / 128);
  unsigned long long* const tr = (a.trace && pair == 0 && leader) ? a.trace : nullptr;

  if (threadIdx.x == 0) {
    for (int s = 0; s < V4_PS; ++s) {
      mbar_init(&ss->full[s], 1);
      mbar_init(&ss->empty[s], 1);
    }
    for (int x = 0; x < V4_SLOTS; ++x) {
      mbar_init(&ss->slot_full[x], 8);  // 4 expander warps (one group) x 2 CTAs
      mbar_init(&ss->slot_empty[x], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ss->acc_full[b], 2);  // one commit per MMA issuer
      mbar_init(&ss->acc_empty[b], 2 * V4_EPI_WARPS);
    }
    mbar_init_fence();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&ss->tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = ss->tmem_base;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
    if (YT) asm volatile("prefetch.tensormap [%0];" ::"l"(&map_y) : "memory");
  }
  griddep_launch();
  griddep_wait();

  int my_tiles = 0;
  for (int t = pair; t < ntiles; t += npairs) ++my_tiles;
  const int G = my_tiles * KB;  // this pair's stages

  if (warp == 0) {
    // ===== TMA producer (each CTA; its own full barrier) ====================
    if (lane == 0) {
      int s = 0, g = 0;
      uint32_t ph = 0;
      for (int t = pair; t < ntiles; t += npairs) {
        const int tt = t % a.ttiles, ct = t / a.ttiles;
        const int n0 = ct * 2 * V4_BM + (int)rank * V4_BM;  // this CTA's channels
        const int m0 = tt * V4_BT + (int)rank * V4_BTH;     // this CTA's token rows
        for (int kb = 0; kb < KB; ++kb, ++g) {
          mbar_wait(&ss->empty[s], ph ^ 1);
          k3_stamp(tr, 0, g);
          mbar_arrive_expect_tx(&ss->full[s], V4_AP + V4_B);
          uint8_t* st = stg + s * V4_STAGE;
          tma_load_local(st, &map_w, kb * 64, n0, &ss->full[s]);
          tma_load_local(st + V4_AP, &map_x, kb * 128, m0, &ss->full[s]);
          if (++s == V4_PS) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1 || warp == 2) {
    // ===== MMA issuers (leader): two threads, alternate stages (v3) =========
    const int who = warp - 1;
    if (leader && lane == 0) {
      constexpr uint32_t idesc = idesc_i8(2 * V4_BM, V4_BT);
      int ab = 0, ti = 0;
      uint32_t aph = 0;
      int g = 0;  // global stage index of the tile's first stage
      for (int t = pair; t < ntiles; t += npairs, ++ti, g += KB) {
        mbar_wait(&ss->acc_empty[ab], aph);
        if (who == 0) k3_stamp(tr, 4, ti);
        tc_fence_after();
        const uint32_t dcol = tmem + acc_col(ab);
        for (int kb = ((g & 1) != who) ? 1 : 0; kb < KB; kb += 2) {
          const int gs = g + kb;
          const int s = gs % V4_PS, slot = gs % V4_SLOTS;
          k3_stamp(tr, 7, gs);
          mbar_wait(&ss->slot_full[slot], (uint32_t)(gs / V4_SLOTS) & 1u);  // A in TMEM, both CTAs
          k3_stamp(tr, 3, gs);
          tc_fence_after();
          const uint32_t bbase = smem_u32(stg + s * V4_STAGE + V4_AP);
          const uint32_t acol = tmem + a_col<BT>(slot);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc_mma_pair_ts(dcol, acol + kk * 8, sw128_desc(bbase + kk * 32), idesc, 1u);
          tc_commit_pair(&ss->empty[s]);
          tc_commit_pair(&ss->slot_empty[slot]);
          k3_stamp(tr, 8, gs);
        }
        tc_commit_pair(&ss->acc_full[ab]);
        if (++ab == 2) {
          ab = 0;
          aph ^= 1;
        }
      }
    }
  } else if (warp == 3 || warp >= 4 + V4_EPI_WARPS) {
    // ===== expanders (each CTA): packed offset binary -> TMEM A slot ========
    // Group 0 = warps 8..11, group 1 = warps 12..14 and 3: each group holds
    // one warp per TMEM lane quarter (warp % 4), the groups alternate
    // stages.  Lane = A row 32*(warp%4) + lane: its 64 packed bytes (the
    // 64B-swizzled TMA tile: 16-byte chunk c of row r sits at c ^ (r/2)%4)
    // become 32 columns of 4 codes each, stored with one tcgen05.st.
    const int q = warp & 3;
    const int grp = (warp >= 4 + V4_EPI_WARPS && warp < 8 + V4_EPI_WARPS) ? 0 : 1;
    const uint32_t slot_full0 = mapa(smem_u32(&ss->slot_full[0]), 0);
    const int row = q * 32 + lane;
    const uint32_t rsw = (uint32_t)((row >> 1) & 3);
    // trace rows 1-2 (leader) / 9-10 (peer): stage landed, slot written
    // (%globaltimer ns: comparable across the two SMs, unlike clock64)
    unsigned long long* const xtr =
        (a.trace && pair == 0 && lane == 0 && (warp == 8 || warp == 12)) ? a.trace : nullptr;
    const int xr = leader ? 1 : 9;
    for (int gs = grp; gs < G; gs += 2) {
      const int s = gs % V4_PS, slot = gs % V4_SLOTS;
      mbar_wait(&ss->full[s], (uint32_t)(gs / V4_PS) & 1u);
#ifdef CRT_K3_TRACE
      if (xtr && gs < kK3TraceN) xtr[xr * kK3TraceN + gs] = globaltimer();
#endif
      const uint32_t src = smem_u32(stg + s * V4_STAGE) + (uint32_t)row * 64u;
      uint4 p[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) p[c] = lds128(src + (((uint32_t)c ^ rsw) << 4));
      uint32_t o[32];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        expand8(p[c].x, o[8 * c + 0], o[8 * c + 1]);
        expand8(p[c].y, o[8 * c + 2], o[8 * c + 3]);
        expand8(p[c].z, o[8 * c + 4], o[8 * c + 5]);
        expand8(p[c].w, o[8 * c + 6], o[8 * c + 7]);
      }
      mbar_wait(&ss->slot_empty[slot], ((uint32_t)(gs / V4_SLOTS) & 1u) ^ 1u);
      tc_fence_after();
#ifdef CRT_K3_DBG
      if (!(a.dbg & 1))
#endif
        tmem_st32(tmem + ((uint32_t)(q * 32) << 16) + a_col<BT>(slot), o);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
#ifdef CRT_K3_TRACE
      if (xtr && gs < kK3TraceN) xtr[(xr + 1) * kK3TraceN + gs] = globaltimer();
#endif
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(slot_full0 + (uint32_t)slot * 8u)
                     : "memory");
    }
  } else if (warp >= 4 && warp < 4 + V4_EPI_WARPS) {
    // ===== epilogue (v3's): TMEM -> dequant -> direct stores ===============
    const int q = warp & 3;
    const int et = threadIdx.x - 128;  // 0 .. V4_EPI_THREADS-1
    // two boxes per warp: a chunk's st.shared overlaps the previous box's TMA read
    const uint32_t ybuf0 = smem_u32(ystg) + (uint32_t)(warp - 4) * 2u * V4_YSTG;
    uint32_t ysel = 0;
    const uint32_t empty_acc = mapa(smem_u32(&ss->acc_empty[0]), 0);
    // fdq: acc + (0x4B400000 - 8 S_a) are the float bits of 1.5*2^23 + v,
    // exact while |v| < 2^22 (|v| <= 49 K: K <= 85598)
    const bool fdq = a.out_kind == 0 && a.fdq && a.K <= 85598;
    int ab = 0, ti = 0;
    uint32_t aph = 0;
    unsigned long long* const etr = (warp == 4 && lane == 0) ? tr : nullptr;
    for (int b2 = 0; b2 < 2; ++b2)
      for (int c = 0; c < C::NCH; ++c) {
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + acc_col(b2) + c * 32;
        if (C::LASTW == 32 || c < C::NCH - 1) tmem_zero32(ta);
        else tmem_zero16(ta);
      }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      arrive_cluster(empty_acc);
      arrive_cluster(empty_acc + 8);
    }
    for (int t = pair; t < ntiles; t += npairs, ++ti) {
      const int tt = t % a.ttiles, ct = t / a.ttiles;
      const int64_t mb = (int64_t)tt * V4_BT;
      const int64_t nw = (int64_t)ct * 2 * V4_BM + (int64_t)rank * V4_BM + q * 32;
      const int64_t n = nw + lane;
      const bool nok = n < a.N;
      const float sw = nok ? a.w_scales[n] : 0.f;
      const float bn = (a.bias && nok) ? a.bias[n] : 0.f;
      named_bar_sync(2, V4_EPI_THREADS);
      for (int i = et; i < V4_BT; i += V4_EPI_THREADS) {
        const int64_t m = mb + i;
        ss->sa[i] = m < a.M ? a.a_scales[m] : 0.f;
        const int off = m >= a.M ? 0 : 8 * a.a_sums[m];
        ss->sums[i] = fdq ? (int)(0x4B400000u - (uint32_t)off) : off;
      }
      named_bar_sync(1, V4_EPI_THREADS);
      wait_sleep(&ss->acc_full[ab], aph);
      k3_stamp(etr, 5, ti);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < C::NCH; ++c) {
        uint32_t acc[32];
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + acc_col(ab) + c * 32;
        const int cw = (C::LASTW == 32 || c < C::NCH - 1) ? 32 : 16;  // chunk width
#ifdef CRT_K3_DBG
        if (a.dbg & 4) continue;
#endif
        if (cw == 32) {
          tmem_ld32(ta, acc);
          tmem_zero32(ta);
        } else {
          tmem_ld16(ta, acc);
          tmem_zero16(ta);
        }
        const int64_t m0 = mb + c * 32;
#ifdef CRT_K3_DBG
        if (a.dbg & 2) continue;
#endif
        const int* sm = &ss->sums[c * 32];
        const float* sa = &ss->sa[c * 32];
        if constexpr (YT) {
          if (cw == 32) {
            // the whole 32 x 32 box through shared memory and one TMA store;
            // tokens >= M and channels >= N are clipped by the tensor map
            if (m0 >= a.M || nw >= a.N) continue;
            uint32_t sav[32], smv[32];
            lds_row32(smem_u32(sa), sav);
            lds_row32(smem_u32(sm), smv);
            const uint32_t ybuf = ybuf0 + ysel * V4_YSTG;
            ysel ^= 1u;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();  // the box stored two chunks ago has left this buffer
            if (fdq) {
              const float2 mc = make_float2(-12582912.f, -12582912.f);  // -1.5 * 2^23
              const float2 w2 = make_float2(sw, sw), b2 = make_float2(bn, bn);
#pragma unroll
              for (int j = 0; j < 32; j += 2) {
                const float2 mm = make_float2(__uint_as_float(acc[j] + smv[j]),
                                              __uint_as_float(acc[j + 1] + smv[j + 1]));
                const float2 v = __fadd2_rn(mm, mc);
                const float2 p =
                    __fmul2_rn(v, make_float2(__uint_as_float(sav[j]), __uint_as_float(sav[j + 1])));
                const __nv_bfloat162 o = __float22bfloat162_rn(__ffma2_rn(p, w2, b2));
                st_shared_u16(ybuf + (uint32_t)j * 64u + (uint32_t)lane * 2u, __bfloat16_as_ushort(o.x));
                st_shared_u16(ybuf + (uint32_t)(j + 1) * 64u + (uint32_t)lane * 2u,
                              __bfloat16_as_ushort(o.y));
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const int v = (int)acc[j] - (int)smv[j];
                const __nv_bfloat16 o =
                    __float2bfloat16_rn(fmaf((float)v * __uint_as_float(sav[j]), sw, bn));
                st_shared_u16(ybuf + (uint32_t)j * 64u + (uint32_t)lane * 2u, __bfloat16_as_ushort(o));
              }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&map_y, ybuf, (int)nw, (int)m0);
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            continue;
          }
        }
        if (m0 >= a.M || !nok) continue;
        const int jn = a.M - m0 < cw ? (int)(a.M - m0) : cw;
        if (a.out_kind == 0) {
          __nv_bfloat16* yp = reinterpret_cast<__nv_bfloat16*>(a.y) + m0 * a.ldy + n;
          if (jn == 32) {
            uint32_t sav[32], smv[32];
            lds_row32(smem_u32(sa), sav);
            lds_row32(smem_u32(sm), smv);
            if (fdq) {
              const float2 mc = make_float2(-12582912.f, -12582912.f);  // -1.5 * 2^23
              const float2 w2 = make_float2(sw, sw), b2 = make_float2(bn, bn);
#pragma unroll
              for (int j = 0; j < 32; j += 2) {
                const float2 mm = make_float2(__uint_as_float(acc[j] + smv[j]),
                                              __uint_as_float(acc[j + 1] + smv[j + 1]));
                const float2 v = __fadd2_rn(mm, mc);
                const float2 p =
                    __fmul2_rn(v, make_float2(__uint_as_float(sav[j]), __uint_as_float(sav[j + 1])));
                const __nv_bfloat162 o = __float22bfloat162_rn(__ffma2_rn(p, w2, b2));
                yp[j * a.ldy] = o.x;
                yp[(j + 1) * a.ldy] = o.y;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const int v = (int)acc[j] - (int)smv[j];
                yp[j * a.ldy] = __float2bfloat16_rn(fmaf((float)v * __uint_as_float(sav[j]), sw, bn));
              }
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < jn) {
                const int off = fdq ? (int)(0x4B400000u - (uint32_t)sm[j]) : sm[j];
                const int v = (int)acc[j] - off;
                yp[j * a.ldy] = __float2bfloat16_rn(fmaf((float)v * sa[j], sw, bn));
              }
          }
        } else {
          uint32_t* yp = reinterpret_cast<uint32_t*>(a.y) + m0 * a.ldy + n;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < jn) {
              const int v = (int)acc[j] - sm[j];
              yp[j * a.ldy] = a.out_kind == 2 ? (uint32_t)v
                                              : __float_as_uint(fmaf((float)v * sa[j], sw, bn));
            }
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      k3_stamp(etr, 6, ti);
      if (lane == 0) arrive_cluster(empty_acc + ab * 8);
      if (++ab == 2) {
        ab = 0;
        aph ^= 1;
      }
    }
    if (YT && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // boxes written
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn_v4() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace

bool k3_v4_supported(const K3Args& a) {
  if (a.bits != 4 || a.a_layout != 1 || !a.a_sums || !a.w.codes_ob) return false;
  if (a.M <= 0 || a.N <= 0 || a.K <= 0 || a.K > 1277000) return false;
  if ((uintptr_t)a.a_codes % 16 || a.lda % 16) return false;
  if ((uintptr_t)a.w.codes_ob % 16 || a.w.ld_ob % 64) return false;
  return encode_fn_v4() != nullptr;
}

namespace {
template <int BT>
cudaError_t launch_bt(const K3Args& a, cudaStream_t st, int64_t* launches, int num_sms) {
  static const bool ydirect = [] {  // A/B: per-lane global stores instead of TMA boxes
    const char* e = getenv("CRT_K3_V4_YDIRECT");
    return e && e[0] == '1';
  }();
  using C = V4Cfg<BT>;
  auto fn = encode_fn_v4();
  CUtensorMap mw, mx;
  {  // weights: N rows x ld_ob bytes of packed offset-binary codes, 64 B x 128 row boxes
    cuuint64_t dims[2] = {(cuuint64_t)a.w.ld_ob, (cuuint64_t)a.N};
    cuuint64_t strides[1] = {(cuuint64_t)a.w.ld_ob};
    cuuint32_t box[2] = {64, (cuuint32_t)V4_BM};
    cuuint32_t es[2] = {1, 1};
    if (fn(&mw, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a.w.codes_ob), dims, strides,
           box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {  // activations: M rows x K int8 codes
    cuuint64_t dims[2] = {(cuuint64_t)a.K, (cuuint64_t)a.M};
    cuuint64_t strides[1] = {(cuuint64_t)a.lda};
    cuuint32_t box[2] = {128, (cuuint32_t)C::BTH};
    cuuint32_t es[2] = {1, 1};
    if (fn(&mx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a.a_codes), dims, strides,
           box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  V4Args v{};
  static const bool no_fdq = [] {
    const char* e = getenv("CRT_K3_NO_FDQ");
    return e && e[0] == '1';
  }();
  v.fdq = no_fdq ? 0 : 1;
  v.M = a.M;
  v.N = a.N;
  v.K = a.K;
  v.ttiles = (int32_t)((a.M + BT - 1) / BT);
  v.ctiles = (int32_t)((a.N + 2 * V4_BM - 1) / (2 * V4_BM));
  v.a_scales = a.a_scales;
  v.a_sums = a.a_sums;
  v.w_scales = a.w_scales;
  v.bias = a.bias;
  v.out_kind = a.out_kind;
  v.y = a.y;
  v.ldy = a.ldy;
  v.trace = k3_trace();
  static const int dbg = [] {
    const char* e = getenv("CRT_K3_V4_DBG");
    return e ? atoi(e) : 0;
  }();
  v.dbg = dbg;
  // bf16 output map for the TMA-store epilogue: N channels (inner) x M tokens, 32 x 32 boxes
  CUtensorMap my = mx;
  bool yt = false;
  // (the TMA store clips at N in 16-byte units: with N % 8 != 0 it would
  // write up to 7 columns past N, which a caller's wider row may own)
  if (a.out_kind == 0 && !ydirect && (uintptr_t)a.y % 16 == 0 && (a.ldy * 2) % 16 == 0 &&
      a.N % 8 == 0) {
    cuuint64_t dims[2] = {(cuuint64_t)a.N, (cuuint64_t)a.M};
    cuuint64_t strides[1] = {(cuuint64_t)(a.ldy * 2)};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t es[2] = {1, 1};
    yt = fn(&my, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a.y, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    if (!yt) my = mx;
  }
  auto kern = yt ? k3_v4_kernel<BT, true> : k3_v4_kernel<BT, false>;
  const size_t smem = 1024 + V4_PS * C::STAGE + ((sizeof(V4Smem<BT>) + 127) & ~(size_t)127) +
                      (yt ? 2 * V4_EPI_WARPS * V4_YSTG : 0);
  static SmemAttr attr[2];
  {
    const cudaError_t e = ensure_dyn_smem(kern, smem, attr[yt], false);
    if (e != cudaSuccess) return e;
  }
  const int tiles = v.ttiles * v.ctiles;
  int pairs = num_sms / 2;
  if (pairs > tiles) pairs = tiles;
  const cudaError_t le = launch_pdl(kern, dim3((unsigned)(2 * pairs)), dim3(V4_THREADS), smem, st,
                                    mw, mx, my, v);
  ++*launches;
  return le;
}
}  // namespace

// Token-tile width: the persistent grid runs ceil(tiles / pairs) waves of
// tiles, so the time goes as waves x BT -- but a 176-token tile does ~9%
// less work per stage for the same fixed per-stage costs, so 176 is picked
// only when it saves more than 10% of waves x BT.  At cfg1 (M = 4096,
// N = 3072: 4 waves of 192 vs 4 waves of 176) the two measured equal (39.5
// vs 38.8 us), so no FLUX shape picks it today.  CRT_K3_V4_BT=192|176 forces.
int k3_v4_pick_bt(int64_t M, int64_t N, int num_sms) {
  static const int forced = [] {
    const char* e = getenv("CRT_K3_V4_BT");
    return e ? atoi(e) : 0;
  }();
  if (forced == 192 || forced == 176) return forced;
  const int64_t pairs = num_sms / 2, ct = (N + 255) / 256;
  auto cost = [&](int64_t bt) {
    const int64_t tiles = (M + bt - 1) / bt * ct;
    const int64_t p = tiles < pairs ? tiles : pairs;
    return (tiles + p - 1) / p * bt;
  };
  return cost(176) * 11 < cost(192) * 10 ? 176 : 192;
}

cudaError_t k3_v4_launch(const K3Args& a, cudaStream_t st, int64_t* launches) {
  const int num_sms = device_sm_count();
  if (k3_v4_pick_bt(a.M, a.N, num_sms) == 176) return launch_bt<176>(a, st, launches, num_sms);
  return launch_bt<192>(a, st, launches, num_sms);
}

}  // namespace crt
