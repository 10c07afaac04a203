// k3_gemm_v2.cu -- K3 v2: the W4A4 GEMM with fused dequant on a 2-SM pair.
//
// Replaces int_gemm (pipeline.cpp:178-204) and the dequant loop of forward
// (pipeline.cpp:224-230):  y[m][n] = acc[m][n] * s_a[m] * s_w[n] + b[n],
// acc[m][n] = sum_k a[m][k] * w[n][k] (int32, exact).
//
// Design:
//   * One cluster = a CTA pair on one TPC issuing
//     tcgen05.mma.cta_group::2.kind::i8, pair tile 256 (M) x 192 (N): each
//     CTA owns 128 rows of A and 96 rows (output channels) of B.
//     Persistent: pair p walks tiles p, p + #pairs, ...
//   * TMA (cp.async.bulk.tensor, SWIZZLE_64B) stages the PACKED INT4 tiles:
//     A 128 rows x 64 B and B 96 rows x 64 B per 128-code K block.
//   * A expansion: 4 warps, thread = row (= TMEM lane).  Each thread reads
//     its 64 packed bytes (conflict-free thanks to the swizzle), expands
//     nibbles to int8 with the exact x16 trick -- (v<<4)&0xF0F0F0F0 and
//     v&0xF0F0F0F0 are the even / odd codes times 16 -- and writes the
//     32 words straight into TMEM with tcgen05.st (A-from-TMEM MMA): no
//     shared-memory round trip for A.
//   * B expansion: 4 warps expand the packed B half into a 128B-swizzled
//     K-major int8 tile in shared memory (the B operand descriptor).
//     Both operands use the same de-interleave, so the dot products are
//     unchanged; acc = 256 * sum(a*b) is exact for K <= 171,196.
//   * One elected thread of the leader CTA issues the MMAs (M256 N192 K32)
//     into a double-buffered 192-column int32 TMEM accumulator; stage
//     release / accumulator-ready are tcgen05.commit multicast to both CTAs.
//   * 4 epilogue warps tcgen05.ld the accumulator, dequantise in fp32
//     (acc/256 * s_a * s_w + b) and store bf16 / f32 / raw int32 while the
//     next tile accumulates into the other buffer.
// TMEM (512 columns per CTA): acc0 [0,192), A stages 0,1 [192,256),
// acc1 [256,448), A stages 2,3 [448,512).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <stdlib.h>

#include "common.cuh"
#include "k3_gemm.h"

namespace crt {
namespace {

constexpr int V2_BM = 128;         // A rows per CTA (pair: 256)
constexpr int V2_BN = 192;         // output channels per pair tile
constexpr int V2_BNH = V2_BN / 2;  // B rows per CTA
constexpr int V2_BKB = 64;         // packed bytes per row per K block (128 codes)
constexpr int V2_KS = 4;           // K stages (TMEM A + smem int8 B)
constexpr int V2_PS = 8;           // packed (TMA) stages
constexpr int V2_THREADS = 640;  // 20 warps
constexpr int V2_PK_A = V2_BM * V2_BKB;     // 8 KB
constexpr int V2_PK_B = V2_BNH * V2_BKB;    // 6 KB
constexpr int V2_PK_STAGE = 16384;          // A + B, 1 KB aligned
constexpr int V2_B8_STAGE = V2_BNH * 128;   // 12 KB int8 B tile
// TMEM column of accumulator buffer b / of TMEM A stage ks (see header)
__device__ __forceinline__ uint32_t acc_col(int b) { return (uint32_t)b * 256u; }
__device__ __forceinline__ uint32_t a_col(int ks) {
  return (ks < 2 ? 192u : 448u) + (uint32_t)(ks & 1) * 32u;
}

struct V2Smem {
  uint64_t pk_full[V2_PS];
  uint64_t pk_empty[V2_PS];
  uint64_t st_full[V2_KS];   // leader only: A + B expanders of both CTAs (16 arrivals)
  uint64_t st_empty[V2_KS];  // both: MMA commit multicast
  uint64_t acc_full[2];      // both: MMA commit multicast
  uint64_t acc_empty[2];     // leader only: epilogue warps of both CTAs (8 arrivals)
  uint32_t tmem_base;
  float sw[2][V2_BN];
  float bias[2][V2_BN];
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// Address of the same shared variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// Arrive on a barrier in (possibly) the peer CTA.  Default .release.cta
// semantics, as CUTLASS's ClusterBarrier::arrive: a .release.cluster arrive
// compiles to MEMBAR.ALL.GPU + ERRBAR and stalls the expanders for
// microseconds.  Operand visibility to the pair's MMA is carried by
// tcgen05.fence::before_thread_sync (TMEM A) and fence.proxy.async (smem B).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Wait with back-off for warps whose wait is long and off the critical path
// (epilogue waiting for a whole tile, TMA producer): spinning would steal
// issue slots from the expander warps on the same SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  for (;;) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(64);
  }
}
// Local arrive that cannot issue before `dep` is available: releasing a
// stage read with ld.shared must wait for the loads to RETURN, or the TMA
// refill can overwrite the bytes still in flight (WAR across proxies).
__device__ __forceinline__ void mbar_arrive_after(uint64_t* bar, uint32_t dep) {
  asm volatile(
      "{\n"
      ".reg .b32 d;\n"
      "mov.b32 d, %1;\n"
      "mbarrier.arrive.shared::cta.b64 _, [%0];\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(dep)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// commit all prior MMAs of this thread to `bar` in both CTAs of the pair
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tc_mma_pair_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 128B-swizzled, K-major UMMA shared-memory descriptor (rows of 128 bytes,
// 8-row core groups 1024 bytes apart; version 1 for sm_100).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// Instruction descriptor: D s32, A/B signed int8, both K-major, M x N.
constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
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
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct V2Args {
  int64_t M, N, K;
  int32_t mtiles, ntiles;
  const float* a_scales;
  const float* w_scales;
  const float* bias;
  int32_t out_kind;  // 0 bf16, 1 f32, 2 int32 accumulators
  void* y;
  int64_t ldy;
  int32_t w_ob;      // weights in offset binary (flip bit 3 of each nibble)
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(V2_THREADS, 1)
    k3_v2_kernel(const __grid_constant__ CUtensorMap map_a,
                 const __grid_constant__ CUtensorMap map_b, V2Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* pk = smem;                                // V2_PS x 16 KB packed (A 8 KB | B 6 KB)
  uint8_t* b8 = smem + V2_PS * V2_PK_STAGE;          // V2_KS x 12 KB int8 B tiles
  V2Smem* ss = reinterpret_cast<V2Smem*>(b8 + V2_KS * V2_B8_STAGE);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int npairs = gridDim.x >> 1;
  const int pair = blockIdx.x >> 1;
  const int ntiles = a.mtiles * a.ntiles;
  const int KB = (int)((a.K + 127) / 128);
  constexpr int nacc = 2;  // accumulator buffers

  if (threadIdx.x == 0) {
    for (int s = 0; s < V2_PS; ++s) {
      mbar_init(&ss->pk_full[s], 1);
      mbar_init(&ss->pk_empty[s], 8);  // 4 A- + 4 B-expander warps
    }
    for (int s = 0; s < V2_KS; ++s) {
      mbar_init(&ss->st_full[s], 16);  // (4 A + 4 B warps) x 2 CTAs
      mbar_init(&ss->st_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ss->acc_full[b], 1);
      mbar_init(&ss->acc_empty[b], 8);  // 4 epilogue warps x 2 CTAs
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

  if (warp == 0) {
    // ===== TMA producer (each CTA loads its own A rows and B half) ==========
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
      int ps = 0;
      uint32_t pph = 0;
      for (int t = pair; t < ntiles; t += npairs) {
        const int mt = t % a.mtiles, nt = t / a.mtiles;
        const int m0 = mt * 2 * V2_BM + (int)rank * V2_BM;
        const int n0 = nt * V2_BN + (int)rank * V2_BNH;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&ss->pk_empty[ps], pph ^ 1);
          uint8_t* st = pk + ps * V2_PK_STAGE;
          mbar_arrive_expect_tx(&ss->pk_full[ps], V2_PK_A + V2_PK_B);
          tma_load_2d(st, &map_a, kb * V2_BKB, m0, &ss->pk_full[ps]);
          tma_load_2d(st + V2_PK_A, &map_b, kb * V2_BKB, n0, &ss->pk_full[ps]);
          if (++ps == V2_PS) {
            ps = 0;
            pph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (leader CTA, one thread) =================================
    if (leader && lane == 0) {
      constexpr uint32_t idesc = idesc_i8(2 * V2_BM, V2_BN);
      int ks = 0;
      uint32_t kph = 0;
      int ab = 0;
      uint32_t aph = 0;
      for (int t = pair; t < ntiles; t += npairs) {
        mbar_wait_cluster(&ss->acc_empty[ab], aph ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem + acc_col(ab);
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait_cluster(&ss->st_full[ks], kph);
          tc_fence_after();
          const uint32_t acol = tmem + a_col(ks);
          const uint32_t bbase = smem_u32(b8 + ks * V2_B8_STAGE);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc_mma_pair_ts(dcol, acol + kk * 8, sw128_desc(bbase + kk * 32), idesc,
                           (kb | kk) != 0 ? 1u : 0u);
          tc_commit_pair(&ss->st_empty[ks]);
          if (++ks == V2_KS) {
            ks = 0;
            kph ^= 1;
          }
        }
        tc_commit_pair(&ss->acc_full[ab]);
        if (++ab == nacc) {
          ab = 0;
          aph ^= 1;
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ===== A expansion: packed SW64 smem -> int8 x16 -> TMEM ===================
    const int q = warp & 3;
    const int row = q * 32 + lane;  // TMEM lane = A row within the CTA tile
    const uint32_t full_st = mapa(smem_u32(&ss->st_full[0]), 0);
    int ps = 0, ks = 0;
    uint32_t pph = 0, kph = 0;
    for (int t = pair; t < ntiles; t += npairs) {
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(&ss->pk_full[ps], pph);
        const uint32_t src = smem_u32(pk + ps * V2_PK_STAGE) + row * 64;
        const uint32_t sw = (uint32_t)((row >> 1) & 3);
        uint4 p[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) p[j] = ld_shared_v4(src + ((j ^ sw) << 4));
        uint32_t r[32];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t w4[4] = {p[j].x, p[j].y, p[j].z, p[j].w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            r[8 * j + 2 * i] = (w4[i] << 4) & 0xF0F0F0F0u;
            r[8 * j + 2 * i + 1] = w4[i] & 0xF0F0F0F0u;
          }
        }
        // packed stage consumed (all four loads returned) -> release it
        {
          const uint32_t all = __reduce_or_sync(0xffffffffu, r[1] ^ r[9] ^ r[17] ^ r[25]);
          if (lane == 0) mbar_arrive_after(&ss->pk_empty[ps], all);
        }
        mbar_wait(&ss->st_empty[ks], kph ^ 1);
        tc_fence_after();
        tmem_st32(tmem + ((uint32_t)(q * 32) << 16) + a_col(ks), r);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(full_st + ks * 8);
        if (++ps == V2_PS) {
          ps = 0;
          pph ^= 1;
        }
        if (++ks == V2_KS) {
          ks = 0;
          kph ^= 1;
        }
      }
    }
  } else if (warp >= 8 && warp < 16) {
    // ===== B expansion: packed SW64 smem -> int8 x16 -> SW128 K-major tile =====
    // Two groups of 4 warps take alternate K blocks, so each warp has two
    // MMA K-block periods to cover its load -> expand -> store -> fence chain.
    const int grp = (warp - 8) >> 2;
    const int e = threadIdx.x - 256 - grp * 128;  // 0..127
    const uint32_t wflip = a.w_ob ? 0x80808080u : 0u;
    const uint32_t full_st = mapa(smem_u32(&ss->st_full[0]), 0);
    int c = 0;  // global K-block counter of this CTA
    for (int t = pair; t < ntiles; t += npairs) {
      for (int kb = 0; kb < KB; ++kb, ++c) {
        if ((c & 1) != grp) continue;
        const int ps = c % V2_PS, ks = c % V2_KS;
        const uint32_t pph = (uint32_t)(c / V2_PS) & 1u, kph = (uint32_t)(c / V2_KS) & 1u;
        mbar_wait(&ss->pk_full[ps], pph);
        const uint32_t src = smem_u32(pk + ps * V2_PK_STAGE + V2_PK_A);
        uint4 p[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int u = e + i * 128;  // 96 rows x 4 units
          const int r = u >> 2, j = u & 3;
          p[i] = ld_shared_v4(src + r * 64 + ((j ^ ((r >> 1) & 3)) << 4));
        }
        {  // packed stage consumed (all loads returned) -> release it
          const uint32_t dep = p[0].x ^ p[1].x ^ p[2].x;
          const uint32_t all = __reduce_or_sync(0xffffffffu, dep);
          if (lane == 0) mbar_arrive_after(&ss->pk_empty[ps], all);
        }
        mbar_wait(&ss->st_empty[ks], kph ^ 1);
        uint8_t* tile = b8 + ks * V2_B8_STAGE;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int u = e + i * 128;
          const int r = u >> 2, j = u & 3;
          const uint4 v = p[i];
          uint4 c0, c1;
          // offset-binary weights: flipping bit 7 of each code*16 byte is
          // the nibble's bit 3 (one LOP3 with the mask)
          c0.x = ((v.x << 4) & 0xF0F0F0F0u) ^ wflip;
          c0.y = (v.x & 0xF0F0F0F0u) ^ wflip;
          c0.z = ((v.y << 4) & 0xF0F0F0F0u) ^ wflip;
          c0.w = (v.y & 0xF0F0F0F0u) ^ wflip;
          c1.x = ((v.z << 4) & 0xF0F0F0F0u) ^ wflip;
          c1.y = (v.z & 0xF0F0F0F0u) ^ wflip;
          c1.z = ((v.w << 4) & 0xF0F0F0F0u) ^ wflip;
          c1.w = (v.w & 0xF0F0F0F0u) ^ wflip;
          uint8_t* rowp = tile + r * 128;
          const int s7 = r & 7;
          *reinterpret_cast<uint4*>(rowp + (((2 * j) ^ s7) << 4)) = c0;
          *reinterpret_cast<uint4*>(rowp + (((2 * j + 1) ^ s7) << 4)) = c1;
        }
        fence_proxy_async();  // generic-proxy smem writes -> visible to the MMA
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(full_st + ks * 8);
      }
    }
  } else if (warp >= 16) {
    // ===== epilogue: TMEM -> registers -> dequant -> global =====================
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int et = threadIdx.x - 512;  // 0..127
    const uint32_t empty_acc = mapa(smem_u32(&ss->acc_empty[0]), 0);
    int ab = 0;
    uint32_t aph = 0;
    const float acc_scale = 1.0f / 256.0f;  // x16 * x16, exact
    for (int t = pair; t < ntiles; t += npairs) {
      const int mt = t % a.mtiles, nt = t / a.mtiles;
      const int64_t m = (int64_t)mt * 2 * V2_BM + (int64_t)rank * V2_BM + row;
      const int64_t nbase = (int64_t)nt * V2_BN;
      // per-channel scale / bias of this tile into smem (buffer ab)
      for (int i = et; i < V2_BN; i += 128) {
        const int64_t n = nbase + i;
        ss->sw[ab][i] = n < a.N ? a.w_scales[n] : 0.f;
        ss->bias[ab][i] = (a.bias && n < a.N) ? a.bias[n] : 0.f;
      }
      named_bar_sync(1, 128);
      const float sa = m < a.M ? a.a_scales[m] * acc_scale : 0.f;
      mbar_wait_sleep(&ss->acc_full[ab], aph);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < V2_BN / 32; ++c) {
        uint32_t acc[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc_col(ab) + c * 32, acc);
        const int64_t nb = nbase + c * 32;
        if (m >= a.M || nb >= a.N) continue;
        const bool full = nb + 32 <= a.N;
        const float* swp = &ss->sw[ab][c * 32];
        const float* bp = &ss->bias[ab][c * 32];
        if (a.out_kind == 2) {
          int32_t* yp = reinterpret_cast<int32_t*>(a.y) + m * a.ldy + nb;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (full || nb + i < a.N) yp[i] = (int32_t)acc[i] >> 8;
        } else if (a.out_kind == 1) {
          float* yp = reinterpret_cast<float*>(a.y) + m * a.ldy + nb;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float v = fmaf((float)(int32_t)acc[i] * sa, swp[i], bp[i]);
            if (full || nb + i < a.N) yp[i] = v;
          }
        } else {
          __nv_bfloat16* yp = reinterpret_cast<__nv_bfloat16*>(a.y) + m * a.ldy + nb;
          uint32_t packed[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float v0 = fmaf((float)(int32_t)acc[2 * i] * sa, swp[2 * i], bp[2 * i]);
            const float v1 =
                fmaf((float)(int32_t)acc[2 * i + 1] * sa, swp[2 * i + 1], bp[2 * i + 1]);
            __nv_bfloat162 h = __floats2bfloat162_rn(v0, v1);
            packed[i] = *reinterpret_cast<uint32_t*>(&h);
          }
          if (full && ((reinterpret_cast<uintptr_t>(yp) & 15) == 0)) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              reinterpret_cast<uint4*>(yp)[i] = make_uint4(packed[4 * i], packed[4 * i + 1],
                                                           packed[4 * i + 2], packed[4 * i + 3]);
          } else {
            for (int i = 0; i < 32; ++i)
              if (nb + i < a.N) {
                const uint32_t w2 = packed[i >> 1];
                reinterpret_cast<uint16_t*>(yp)[i] =
                    (i & 1) ? (uint16_t)(w2 >> 16) : (uint16_t)(w2 & 0xFFFF);
              }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(empty_acc + ab * 8);
      if (++ab == nacc) {
        ab = 0;
        aph ^= 1;
      }
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// Packed-code matrix rows x bytes_per_row (pitch ld bytes) as a 2-D uint8
// tensor map with box {64 bytes, box_rows}, 64-byte swizzle.
bool make_codes_map(CUtensorMap* map, const uint8_t* base, int64_t rows, int64_t bytes,
                    int64_t ld, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)bytes, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

bool k3_v2_supported(const K3Args& a) {
  if (a.bits != 4 || a.K <= 0 || a.K > 171196) return false;
  if (a.M <= 0 || a.N <= 0) return false;
  if ((uintptr_t)a.a_codes % 16 || a.lda % 16 || (uintptr_t)a.w.codes % 16 || a.w.ld % 16)
    return false;
  if (a.M > (int64_t)1 << 31 || a.N > (int64_t)1 << 31) return false;
  return encode_fn() != nullptr;
}

cudaError_t k3_v2_launch(const K3Args& a, cudaStream_t st, int64_t* launches) {
  const int num_sms = device_sm_count();
  CUtensorMap ma, mb;
  const int64_t kbytes = (a.K + 1) / 2;
  if (!make_codes_map(&ma, a.a_codes, a.M, kbytes, a.lda, V2_BM) ||
      !make_codes_map(&mb, a.w.codes, a.N, kbytes, a.w.ld, V2_BNH))
    return cudaErrorInvalidValue;
  V2Args v{};
  v.M = a.M;
  v.N = a.N;
  v.K = a.K;
  v.mtiles = (int32_t)((a.M + 2 * V2_BM - 1) / (2 * V2_BM));
  v.ntiles = (int32_t)((a.N + V2_BN - 1) / V2_BN);
  v.a_scales = a.a_scales;
  v.w_scales = a.w_scales;
  v.bias = a.bias;
  v.out_kind = a.out_kind;
  v.y = a.y;
  v.ldy = a.ldy;
  v.w_ob = a.w.ob;
  const size_t smem = 1024 + V2_PS * V2_PK_STAGE + V2_KS * V2_B8_STAGE + sizeof(V2Smem);
  static SmemAttr attr;
  {
    const cudaError_t e = ensure_dyn_smem(k3_v2_kernel, smem, attr, false);
    if (e != cudaSuccess) return e;
  }
  const int tiles = v.mtiles * v.ntiles;
  int pairs = num_sms / 2;
  if (pairs > tiles) pairs = tiles;
  k3_v2_kernel<<<(unsigned)(2 * pairs), V2_THREADS, smem, st>>>(ma, mb, v);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace crt
