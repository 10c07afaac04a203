// k3_gemm_v3.cu -- K3 v3: W4A4 GEMM with HARDWARE int4 -> int8 expansion.
//
// Replaces int_gemm (pipeline.cpp:178-204) and the dequant loop of forward
// (pipeline.cpp:224-230).  Same 2-SM tcgen05 kind::i8 machinery as v2, with
// the operands swapped so that no thread touches an operand byte:
//   * A = the prepared WEIGHTS, stored packed in offset binary (nibble =
//     code + 8).  TMA (CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B, 128B swizzle)
//     stages them as padded 4-bit units; the MMA thread expands them with
//     tcgen05.cp ... .b8x16.b4x16_p64 straight into TMEM (measured on B200,
//     tools/probes/tcgen05_cp_probe.cu: byte = nibble << 2), i.e. the A
//     operand holds 4*(w + 8).
//   * B = the ACTIVATION codes from K1 stored one int8 per code (values
//     -7..7); TMA puts them directly into the 128B-swizzled K-major smem
//     operand layout.
//   * D = W * X^T in TMEM (lane = output channel, column = token):
//     acc' = 4*sum(w*a) + 32*S_a[m], S_a = per-token code sum from K1, so
//     acc = (acc' - 32*S_a[m]) >> 2 exactly (|acc'| < 2^31 for K <= 1,277,000).
// Pair tile: 256 channels (128 per CTA, A from its own TMEM) x 192 tokens
// (96 token rows of B per CTA).  Persistent over tiles; warp roles: 0 TMA
// producer, 1 and 2 MMA issuers (alternate K stages, each expanding its
// stage's A with tcgen05.cp right before its MMAs; two issuers because one
// thread's mbarrier wait after its commits drains its MMA pipeline -- see
// the issuer section), 4..11 epilogue (warp 3 idle).  The accumulators are double
// buffered so the epilogue (TMEM -> dequant -> stores, lane = channel)
// overlaps the next tile's MMAs.
// TMEM per CTA (512 columns): acc0 [0,192), A slots 0,1 [192,256), acc1
// [256,448), A slots 2,3 [448,512); one slot = one 128-code K block.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <atomic>

#include "common.cuh"
#include "k3_gemm.h"
#include "k3_tc_common.cuh"

namespace crt {
namespace {

constexpr int V3_BM = 128;         // channels per CTA (pair: 256)
constexpr int V3_BT = 192;         // tokens per pair tile (measured: 160 and 224 both ~20% slower)
constexpr int V3_BTH = V3_BT / 2;  // token rows of B per CTA
constexpr int V3_PS = 8;           // smem stages (8 x 28 KB: the epilogue stages nothing)
constexpr int V3_THREADS = 384;  // 12 warps: producer, 2 MMA issuers, (idle), 8 epilogue
constexpr int V3_A_STAGE = V3_BM * 128;  // 16 KB: 128 rows x (8 x 16 B padded units)
constexpr int V3_B_STAGE = V3_BTH * 128; // 12 KB int8
// TMEM (512 columns): two V3_BT-column accumulators at 0 and 256, the rest of
// each half holds 32-column A slots (one 128-code K block each)
constexpr int V3_SLOTS = (256 - V3_BT) / 32 * 2;
static_assert(V3_SLOTS >= 2, "no TMEM room for A slots");
constexpr int V3_STAGE = V3_A_STAGE + V3_B_STAGE;
// transaction bytes of one stage: a 16U4_ALIGN16B box completes its PACKED
// data bytes (64 per row), not its padded smem footprint (128 per row) --
// measured, tools/probes/tma_u4_probe.cu
constexpr int V3_STAGE_TX = V3_BM * 64 + V3_B_STAGE;
constexpr int V3_STAGE_TX_W8 = V3_BM * 128 + V3_B_STAGE;  // W8A8: int8 weights, no padding

struct V3Smem {
  uint64_t full[V3_PS];   // leader: 2 arrivals (one per CTA) + tx bytes of both CTAs
  uint64_t empty[V3_PS];  // both: MMA commit multicast
  uint64_t acc_full[2];   // both: MMA commit multicast
  uint64_t acc_empty[2];  // leader: 8 epilogue warps x 2 CTAs
  uint64_t dec_empty[V3_SLOTS];  // leader: MMA commit (A slot consumed by its issuer)
  uint32_t tmem_base;
  alignas(16) float sa[V3_BT];  // per-token activation scale of the tile (ld.shared.v4)
  alignas(16) int sums[V3_BT];  // per-token code-sum offsets of the tile
};

__device__ __forceinline__ uint32_t acc_col(int b) { return (uint32_t)b * 256u; }
__device__ __forceinline__ uint32_t a_col(int s) {
  constexpr int H = V3_SLOTS / 2;
  return (s < H ? (uint32_t)V3_BT : 256u + (uint32_t)V3_BT) + (uint32_t)(s % H) * 32u;
}
struct V3Args {
  int64_t M, N, K;
  int32_t ttiles, ctiles;  // token tiles (192), channel tiles (256)
  const float* a_scales;
  const int32_t* a_sums;
  const float* w_scales;
  const float* bias;
  int32_t out_kind;  // 0 bf16, 1 f32, 2 int32 accumulators
  void* y;
  int64_t ldy;
  int32_t w8_ss;     // W8A8: A straight from shared memory (no TMEM copy)
  int32_t fdq;       // magic-number fp32x2 dequant (bf16 output)
  int32_t dbg_skip_epi;       // dev aid (CRT_K3_DBG_SKIP_EPI=1): TMEM reads only, no dequant/stores
  unsigned long long* trace;  // dev aid (crt_debug_k3_trace): pair 0's leader clock64 stamps
};
// trace layout: 9 rows x kK3TraceN; per stage: row 0 producer issue, row 3
// MMA issue (stage landed, slot free), row 7 the issuer before its waits,
// row 8 after its copies, MMAs and commits; per tile: row 4 first issuer's
// tile start, 5 epilogue sees acc_full, 6 epilogue done; rows 1-2 unused

// W8 = false: W4A4 (offset-binary int4 weights, hardware expansion);
// W8 = true: W8A8 (int8 weights and activations).
template <bool W8>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(V3_THREADS, 1)
    k3_v3_kernel(const __grid_constant__ CUtensorMap map_w,
                 const __grid_constant__ CUtensorMap map_x, V3Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* stg = smem;                                        // V3_PS x (A 16 KB | B 12 KB)
  V3Smem* ss = reinterpret_cast<V3Smem*>(smem + V3_PS * V3_STAGE);

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
    for (int s = 0; s < V3_PS; ++s) {
      mbar_init(&ss->full[s], 2);
      mbar_init(&ss->empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ss->acc_full[b], 2);  // one commit per MMA issuer
      mbar_init(&ss->acc_empty[b], 16);
    }
    for (int b = 0; b < V3_SLOTS; ++b) {
      mbar_init(&ss->dec_empty[b], 1);
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
  // PDL: the prologue above (barriers, TMEM allocation) overlapped the
  // previous kernel's tail; no global memory is touched before this wait.
  if (warp == 0 && lane == 0) {  // kernel parameters, not predecessor output
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
  }
  griddep_launch();
  griddep_wait();

  if (warp == 0) {
    // ===== TMA producer (both CTAs; completions land on the leader) ========
    if (lane == 0) {
      const uint32_t full0 = mapa(smem_u32(&ss->full[0]), 0);
      int s = 0, g = 0;
      uint32_t ph = 0;
      for (int t = pair; t < ntiles; t += npairs) {
        const int tt = t % a.ttiles, ct = t / a.ttiles;
        const int n0 = ct * 2 * V3_BM + (int)rank * V3_BM;   // this CTA's channels
        const int m0 = tt * V3_BT + (int)rank * V3_BTH;      // this CTA's token rows
        for (int kb = 0; kb < KB; ++kb, ++g) {
          mbar_wait(&ss->empty[s], ph ^ 1);
          k3_stamp(tr, 0, g);
          if (leader) mbar_arrive_expect_tx(&ss->full[s], 2 * (W8 ? V3_STAGE_TX_W8 : V3_STAGE_TX));
          else arrive_cluster(full0 + s * 8);
          uint8_t* st = stg + s * V3_STAGE;
          tma_load_2sm(st, &map_w, kb * 128, n0, &ss->full[s]);
          tma_load_2sm(st + V3_A_STAGE, &map_x, kb * 128, m0, &ss->full[s]);
          if (++s == V3_PS) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1 || warp == 2) {
    // ===== MMA issuers (leader): two threads, alternate stages ===============
    // An MMA-issuing thread that touches shared memory (an mbarrier wait)
    // while one of its tcgen05.commit arrivals is pending stalls until its
    // MMA pipeline drains: one issuer with K3's per-stage wait + commits
    // keeps the tensor pipe ~70% busy (tools/probes/i8_peak_probe.cu:
    // 137.5 cycles per M256xN192xK32 MMA instead of 96).  The drain is per
    // issuing thread, so two issuers (warps 1 and 2) taking alternate stages
    // keep it full (96.0) -- they accumulate into the same TMEM accumulator,
    // exact for integers in any order (probe: 0 wrong of 3.6M elements).
    // All MMAs accumulate: the epilogue zeroes each accumulator after
    // reading it (and both once at start), so neither issuer orders against
    // the other's first MMA of a tile.  acc_full takes one commit from each.
    // Each issuer also expands the A operand of its stage (tcgen05.cp from
    // the padded smem stage into a TMEM slot) right before the stage's
    // MMAs: cp -> mma from one thread execute in order.  The copies cost
    // tensor-pipe time (ncu at fc1: tc pipe 85% busy, MMA 65%), but every
    // ordering that issues them earlier measured slower (fc1 TOPS, k3_time):
    // one separate expansion thread (its own waits drain its copies: ~580
    // cycles per stage), two expansion threads (copies queue behind issued
    // MMAs; issuers wait ~900 cycles: 2757 vs 2819), an issuer expanding its
    // own next stage (2111), expanding the other issuer's next stage (2248),
    // and issuing each stage's MMAs one own step after its copies (~1650 at
    // 3072^2 vs 2110).
    // A slot's previous readers (this issuer's MMAs two own stages back) are
    // fenced by dec_empty.
    const int who = warp - 1;
    if (leader && lane == 0) {
      constexpr uint32_t idesc = idesc_i8(2 * V3_BM, V3_BT);
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
          const int s = gs % V3_PS;
          const uint32_t ph = (uint32_t)(gs / V3_PS) & 1u;
          if (W8 && a.w8_ss) {  // W8A8, SS form: both operands from the stage
            mbar_wait(&ss->full[s], ph);
            tc_fence_after();
            const uint32_t abase = smem_u32(stg + s * V3_STAGE);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              tc_mma_pair_ss(dcol, sw128_desc(abase + kk * 32),
                             sw128_desc(abase + V3_A_STAGE + kk * 32), idesc, 1u);
            tc_commit_pair(&ss->empty[s]);
            continue;
          }
          const int slot = gs % V3_SLOTS;
          const uint32_t sph = (uint32_t)(gs / V3_SLOTS) & 1u;
          k3_stamp(tr, 7, gs);
          mbar_wait(&ss->full[s], ph);
          mbar_wait(&ss->dec_empty[slot], sph ^ 1);
          k3_stamp(tr, 3, gs);
          tc_fence_after();
          const uint32_t abase = smem_u32(stg + s * V3_STAGE);
          const uint32_t bbase = abase + V3_A_STAGE;
          const uint32_t acol = tmem + a_col(slot);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            if constexpr (W8) tc_cp_raw(acol + kk * 8, sw128_desc(abase + kk * 32));
            else tc_cp_decompress(acol + kk * 8, sw128_desc(abase + kk * 32));
          }
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) tc_mma_pair_ts(dcol, acol + kk * 8, sw128_desc(bbase + kk * 32), idesc, 1u);
          tc_commit_pair(&ss->empty[s]);
          tc_commit_leader(&ss->dec_empty[slot]);
          k3_stamp(tr, 8, gs);
        }
        tc_commit_pair(&ss->acc_full[ab]);
        if (++ab == 2) {
          ab = 0;
          aph ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue: TMEM -> dequant -> direct stores =======================
    // Lane = output channel, so for each token the warp's 32 lanes write 32
    // consecutive channels (64 B bf16 / 128 B f32): coalesced without a
    // transpose or shared-memory staging (staging boxes for TMA stores
    // would cost the eighth operand stage).  Two warps per TMEM lane
    // quarter split the token chunks.
    const int q = warp & 3;
    const int h = (warp - 4) >> 2;
    const int et = threadIdx.x - 128;  // 0..255
    const uint32_t empty_acc = mapa(smem_u32(&ss->acc_empty[0]), 0);
    // fdq: integer-to-float by the magic constant, two tokens per fp32x2
    // instruction; exact while |4*sum(w*a)| < 2^22 (4*49*K < 2^22: K <= 21384)
    const bool fdq = !W8 && a.out_kind == 0 && a.fdq && a.K <= 21384;
    int ab = 0, ti = 0;
    uint32_t aph = 0;
    unsigned long long* const etr = (warp == 4 && lane == 0) ? tr : nullptr;
    // both accumulators start at zero (the MMAs never overwrite), then
    // release them to the issuers (phase 0 of acc_empty)
    for (int b2 = 0; b2 < 2; ++b2)
      for (int c = h; c < V3_BT / 32; c += 2) tmem_zero32(tmem + ((uint32_t)(q * 32) << 16) + acc_col(b2) + c * 32);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      arrive_cluster(empty_acc);
      arrive_cluster(empty_acc + 8);
    }
    for (int t = pair; t < ntiles; t += npairs, ++ti) {
      const int tt = t % a.ttiles, ct = t / a.ttiles;
      const int64_t mb = (int64_t)tt * V3_BT;                                // tile tokens
      const int64_t nw = (int64_t)ct * 2 * V3_BM + (int64_t)rank * V3_BM + q * 32;  // warp's channels
      const int64_t n = nw + lane;
      const bool nok = n < a.N;
      const float sw = nok ? a.w_scales[n] : 0.f;
      const float bn = (a.bias && nok) ? a.bias[n] : 0.f;
      named_bar_sync(2, 256);  // every epilogue warp is done with the previous tile's token data
      for (int i = et; i < V3_BT; i += 256) {
        const int64_t m = mb + i;
        ss->sa[i] = m < a.M ? a.a_scales[m] : 0.f;
        const int off = (W8 || m >= a.M) ? 0 : 32 * a.a_sums[m];
        // magic-number dequant (fdq): acc' + (0x4B400000 - 32 S_a) are the
        // float bits of 1.5*2^23 + 4*sum(w*a)
        ss->sums[i] = fdq ? (int)(0x4B400000u - (uint32_t)off) : off;
      }
      named_bar_sync(1, 256);
      wait_sleep(&ss->acc_full[ab], aph);
      k3_stamp(etr, 5, ti);
      tc_fence_after();
#pragma unroll 1
      for (int c = h; c < V3_BT / 32; c += 2) {
        uint32_t acc[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc_col(ab) + c * 32, acc);
        tmem_zero32(tmem + ((uint32_t)(q * 32) << 16) + acc_col(ab) + c * 32);
        const int64_t m0 = mb + c * 32;  // tokens m0 .. m0+31 of this chunk
        if (m0 >= a.M || !nok || a.dbg_skip_epi) continue;
        const int jn = a.M - m0 < 32 ? (int)(a.M - m0) : 32;
        const int* sm = &ss->sums[c * 32];
        const float* sa = &ss->sa[c * 32];
        if (a.out_kind == 0) {
          __nv_bfloat16* yp = reinterpret_cast<__nv_bfloat16*>(a.y) + m0 * a.ldy + n;
          if (jn == 32) {
            // the chunk's 32 token scales / offsets as shared broadcasts
            // (explicit ld.shared: the generic pointer compiles to LD.E)
            uint32_t sav[32], smv[32];
            lds_row32(smem_u32(sa), sav);
            if constexpr (!W8) lds_row32(smem_u32(sm), smv);
            if (fdq) {
              // v = (acc' - 32 S_a) / 4 exactly: fma(1.5*2^23 + 4v, 1/4, -1.5*2^21);
              // then the same fp32 expression as below, two tokens at a time
              const float2 q4 = make_float2(0.25f, 0.25f), mc = make_float2(-3145728.f, -3145728.f);
              const float2 w2 = make_float2(sw, sw), b2 = make_float2(bn, bn);
#pragma unroll
              for (int j = 0; j < 32; j += 2) {
                const float2 mm = make_float2(__uint_as_float(acc[j] + smv[j]),
                                              __uint_as_float(acc[j + 1] + smv[j + 1]));
                const float2 v = __ffma2_rn(mm, q4, mc);
                const float2 p =
                    __fmul2_rn(v, make_float2(__uint_as_float(sav[j]), __uint_as_float(sav[j + 1])));
                const __nv_bfloat162 o = __float22bfloat162_rn(__ffma2_rn(p, w2, b2));
                yp[j * a.ldy] = o.x;
                yp[(j + 1) * a.ldy] = o.y;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const int v = W8 ? (int)acc[j] : (((int)acc[j] - (int)smv[j]) >> 2);
                yp[j * a.ldy] = __float2bfloat16_rn(fmaf((float)v * __uint_as_float(sav[j]), sw, bn));
              }
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < jn) {
                // fdq offsets hold 0x4B400000 - 32 S_a: recover 32 S_a
                const int off = fdq ? (int)(0x4B400000u - (uint32_t)sm[j]) : sm[j];
                const int v = W8 ? (int)acc[j] : (((int)acc[j] - off) >> 2);
                yp[j * a.ldy] = __float2bfloat16_rn(fmaf((float)v * sa[j], sw, bn));
              }
          }
        } else {
          uint32_t* yp = reinterpret_cast<uint32_t*>(a.y) + m0 * a.ldy + n;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < jn) {
              const int v = W8 ? (int)acc[j] : (((int)acc[j] - sm[j]) >> 2);
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
PFN_cuTensorMapEncodeTiled_v12000 encode_fn_v3() {
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

std::atomic<unsigned long long*> g_k3_trace{nullptr};
}  // namespace

void set_k3_trace(unsigned long long* buf) { g_k3_trace.store(buf); }
unsigned long long* k3_trace() { return g_k3_trace.load(); }

bool k3_v3_supported(const K3Args& a) {
  if (a.M <= 0 || a.N <= 0 || a.K <= 0 || a.K > 1277000) return false;
  if ((uintptr_t)a.a_codes % 16 || a.lda % 16) return false;
  if (a.bits == 8) {  // W8A8: int8 rows on both sides (the reference layout)
    if (a.a_layout != 0 || !a.w.codes || (uintptr_t)a.w.codes % 16 || a.w.ld % 16) return false;
  } else {
    if (a.bits != 4 || a.a_layout != 1 || !a.a_sums || !a.w.codes_ob) return false;
    if ((uintptr_t)a.w.codes_ob % 16 || a.w.ld_ob % 64) return false;
  }
  return encode_fn_v3() != nullptr;
}

cudaError_t k3_v3_launch(const K3Args& a, cudaStream_t st, int64_t* launches) {
  const int num_sms = device_sm_count();
  auto fn = encode_fn_v3();
  CUtensorMap mw, mx;
  const bool w8 = a.bits == 8;
  if (w8) {  // weights: N rows x K int8 codes
    cuuint64_t dims[2] = {(cuuint64_t)a.K, (cuuint64_t)a.N};
    cuuint64_t strides[1] = {(cuuint64_t)a.w.ld};
    cuuint32_t box[2] = {128, (cuuint32_t)V3_BM};
    cuuint32_t es[2] = {1, 1};
    if (fn(&mw, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a.w.codes), dims, strides,
           box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  } else {  // weights: N rows x K 4-bit codes (offset binary), padded 16-code units
    cuuint64_t dims[2] = {(cuuint64_t)(a.w.ld_ob * 2), (cuuint64_t)a.N};
    cuuint64_t strides[1] = {(cuuint64_t)a.w.ld_ob};
    cuuint32_t box[2] = {128, (cuuint32_t)V3_BM};
    cuuint32_t es[2] = {1, 1};
    if (fn(&mw, CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B, 2, const_cast<uint8_t*>(a.w.codes_ob),
           dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {  // activations: M rows x K int8 codes
    cuuint64_t dims[2] = {(cuuint64_t)a.K, (cuuint64_t)a.M};
    cuuint64_t strides[1] = {(cuuint64_t)a.lda};
    cuuint32_t box[2] = {128, (cuuint32_t)V3_BTH};
    cuuint32_t es[2] = {1, 1};
    if (fn(&mx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a.a_codes), dims, strides,
           box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  V3Args v{};
  static const bool no_fdq = [] {  // A/B switch: per-token I2F dequant
    const char* e = getenv("CRT_K3_NO_FDQ");
    return e && e[0] == '1';
  }();
  v.fdq = no_fdq ? 0 : 1;
  v.M = a.M;
  v.N = a.N;
  v.K = a.K;
  v.ttiles = (int32_t)((a.M + V3_BT - 1) / V3_BT);
  v.ctiles = (int32_t)((a.N + 2 * V3_BM - 1) / (2 * V3_BM));
  v.a_scales = a.a_scales;
  v.a_sums = a.a_sums;
  v.w_scales = a.w_scales;
  v.bias = a.bias;
  v.out_kind = a.out_kind;
  v.y = a.y;
  v.ldy = a.ldy;
  static const bool w8_ts = [] {  // A/B switch: W8A8 through the TMEM copy path
    const char* e = getenv("CRT_K3_W8_TS");
    return e && e[0] == '1';
  }();
  v.w8_ss = w8 && !w8_ts;
  v.trace = k3_trace();
  static const bool skip_epi = [] {
    const char* e = getenv("CRT_K3_DBG_SKIP_EPI");
    return e && e[0] == '1';
  }();
  v.dbg_skip_epi = skip_epi ? 1 : 0;
  const size_t smem =
      1024 + V3_PS * V3_STAGE + ((sizeof(V3Smem) + 127) & ~(size_t)127);
  auto kern = w8 ? k3_v3_kernel<true> : k3_v3_kernel<false>;
  static SmemAttr attr[2];
  {
    const cudaError_t e = ensure_dyn_smem(kern, smem, attr[w8], false);
    if (e != cudaSuccess) return e;
  }
  const int tiles = v.ttiles * v.ctiles;
  int pairs = num_sms / 2;
  if (pairs > tiles) pairs = tiles;
  const cudaError_t le = launch_pdl(kern, dim3((unsigned)(2 * pairs)), dim3(V3_THREADS), smem, st,
                                    mw, mx, v);
  ++*launches;
  return le;
}

}  // namespace crt
