// k3_gemm.cu -- K3: the W4A4 (and W8A8) GEMM with fused dequant epilogue.
//
// Replaces int_gemm (pipeline.cpp:178-204) and the dequant loop of forward
// (pipeline.cpp:224-230):  y[m][n] = acc[m][n] * s_a[m] * s_w[n] + b[n],
// acc[m][n] = sum_k a[m][k] * w[n][k]  (int32, exact).
//
// sm_100a design (this file, v1):
//   * CTA tile 128 (M) x 256 (N), K staged in blocks of 128 codes.
//   * Packed INT4 codes are loaded straight from global (16-byte vectors),
//     expanded to int8 in registers and stored into 128B-swizzled K-major
//     shared-memory operand tiles.  Expansion uses the exact "x16" trick:
//     (w << 4) & 0xF0F0F0F0 and w & 0xF0F0F0F0 are the even/odd codes times
//     16 as int8, so acc = 256 * sum(a*b) and acc >> 8 is exact (int32-safe
//     for K <= 171,196).  Both operands go through the same de-interleave,
//     so their K orders agree and the dot products are unchanged.
//   * One elected thread issues tcgen05.mma.cta_group::1.kind::i8
//     (M=128, N=256, K=32) into a 256-column int32 TMEM accumulator; stage
//     release and accumulator-ready are tcgen05.commit -> mbarrier.
//   * Epilogue warps read TMEM with tcgen05.ld.32x32b, dequantise in fp32
//     and store bf16 / f32 / raw int32.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "k3_gemm.h"

namespace crt {
namespace {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BKC = 128;  // codes per K block (= 128 int8 bytes per operand row)
constexpr int STAGES = 2;
constexpr int A_STAGE_BYTES = BM * 128;  // 16 KB int8
constexpr int B_STAGE_BYTES = BN * 128;  // 32 KB int8
constexpr int NUM_EXP_THREADS = 128;     // warps 2..5
constexpr int K3_THREADS = 192;
constexpr int TMEM_COLS = 256;

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 128B-swizzled, K-major UMMA shared-memory descriptor (rows of 128 bytes,
// 8-row core groups 1024 bytes apart; version 1 for sm_100).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);  // start address
  d |= (uint64_t)1 << 16;                   // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;         // SBO
  d |= (uint64_t)1 << 46;                   // version
  d |= (uint64_t)2 << 61;                   // SWIZZLE_128B
  return d;
}

// Instruction descriptor: D s32, A/B signed int8, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
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

struct K3Smem {
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t accf;
  uint32_t tmem_base;
  float sw[BN];
  float bias[BN];
};

// ---------------------------------------------------------------------------
// Expander: one 16-byte global vector -> int8 16-byte chunk(s) in the
// swizzled operand tile.
// ---------------------------------------------------------------------------
template <int BITS>
__device__ __forceinline__ void store_unit(uint8_t* tile, int r, int j, uint4 v) {
  uint8_t* rowp = tile + r * 128;
  const int sw = r & 7;
  if constexpr (BITS == 4) {
    uint4 c0, c1;
    c0.x = (v.x << 4) & 0xF0F0F0F0u;
    c0.y = v.x & 0xF0F0F0F0u;
    c0.z = (v.y << 4) & 0xF0F0F0F0u;
    c0.w = v.y & 0xF0F0F0F0u;
    c1.x = (v.z << 4) & 0xF0F0F0F0u;
    c1.y = v.z & 0xF0F0F0F0u;
    c1.z = (v.w << 4) & 0xF0F0F0F0u;
    c1.w = v.w & 0xF0F0F0F0u;
    *reinterpret_cast<uint4*>(rowp + (((2 * j) ^ sw) << 4)) = c0;
    *reinterpret_cast<uint4*>(rowp + (((2 * j + 1) ^ sw) << 4)) = c1;
  } else {
    *reinterpret_cast<uint4*>(rowp + ((j ^ sw) << 4)) = v;
  }
}

template <int BITS>
__global__ void __launch_bounds__(K3_THREADS, 1) k3_ss_kernel(K3Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;                                   // STAGES x 16 KB
  uint8_t* sB = smem + STAGES * A_STAGE_BYTES;          // STAGES x 32 KB
  K3Smem* ss = reinterpret_cast<K3Smem*>(sB + STAGES * B_STAGE_BYTES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t mt = (a.M + BM - 1) / BM;
  const int64_t m0 = (int64_t)(blockIdx.x % mt) * BM;
  const int64_t n0 = (int64_t)(blockIdx.x / mt) * BN;
  const int KB = (int)((a.K + BKC - 1) / BKC);
  const uint8_t* wcodes = a.w.codes;
  const int64_t ldw = a.w.ld;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&ss->full[s], NUM_EXP_THREADS);
      mbar_init(&ss->empty[s], 1);
    }
    mbar_init(&ss->accf, 1);
    mbar_init_fence();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&ss->tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = threadIdx.x; i < BN; i += blockDim.x) {
    const int64_t n = n0 + i;
    ss->sw[i] = n < a.N ? a.w_scales[n] : 0.f;
    ss->bias[i] = (a.bias && n < a.N) ? a.bias[n] : 0.f;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_acc = ss->tmem_base;

  if (warp == 0) {
    // ===== MMA issuer (one elected lane) =====================================
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_i8(BM, BN);
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&ss->full[s], (uint32_t)((kb / STAGES) & 1));
        tc_fence_after();
        const uint32_t abase = smem_u32(sA + s * A_STAGE_BYTES);
        const uint32_t bbase = smem_u32(sB + s * B_STAGE_BYTES);
#pragma unroll
        for (int kk = 0; kk < BKC / 32; ++kk) {
          tc_mma_i8(tmem_acc, sw128_desc(abase + kk * 32), sw128_desc(bbase + kk * 32), idesc,
                    (kb | kk) != 0 ? 1u : 0u);
        }
        tc_commit(&ss->empty[s]);
      }
      tc_commit(&ss->accf);
    }
    __syncwarp();
  } else if (warp >= 2) {
    // ===== expanders (warps 2..5) ============================================
    const int e = threadIdx.x - 64;
    constexpr int UPR = BITS == 4 ? 4 : 8;  // 16-byte units per row per K block
    constexpr int UNITS = (BM + BN) * UPR;
    constexpr int PER = UNITS / NUM_EXP_THREADS;  // 12 or 24
    constexpr int BATCH = 12;
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES;
      uint8_t* tA = sA + s * A_STAGE_BYTES;
      uint8_t* tB = sB + s * B_STAGE_BYTES;
      const int64_t kbyte0 = (int64_t)kb * (BITS == 4 ? 64 : 128);
      const int64_t kbytes = BITS == 4 ? (a.K + 1) / 2 : a.K;
#pragma unroll 1
      for (int b0 = 0; b0 < PER; b0 += BATCH) {
        uint4 v[BATCH];
#pragma unroll
        for (int q = 0; q < BATCH; ++q) {
          const int u = e + (b0 + q) * NUM_EXP_THREADS;
          const bool isA = u < BM * UPR;
          const int uu = isA ? u : u - BM * UPR;
          const int r = uu / UPR, j = uu % UPR;
          const int64_t kbyte = kbyte0 + j * 16;
          v[q] = make_uint4(0, 0, 0, 0);
          if (isA) {
            const int64_t m = m0 + r;
            if (m < a.M && kbyte < kbytes)
              v[q] = __ldg(reinterpret_cast<const uint4*>(a.a_codes + m * a.lda + kbyte));
          } else {
            const int64_t n = n0 + r;
            if (n < a.N && kbyte < kbytes)
              v[q] = __ldg(reinterpret_cast<const uint4*>(wcodes + n * ldw + kbyte));
            if (BITS == 4 && a.w.ob) {  // offset-binary weights -> two's complement
              v[q].x ^= 0x88888888u;
              v[q].y ^= 0x88888888u;
              v[q].z ^= 0x88888888u;
              v[q].w ^= 0x88888888u;
            }
          }
        }
        if (b0 == 0) mbar_wait(&ss->empty[s], (uint32_t)(((kb / STAGES) & 1) ^ 1));
#pragma unroll
        for (int q = 0; q < BATCH; ++q) {
          const int u = e + (b0 + q) * NUM_EXP_THREADS;
          const bool isA = u < BM * UPR;
          const int uu = isA ? u : u - BM * UPR;
          store_unit<BITS>(isA ? tA : tB, uu / UPR, uu % UPR, v[q]);
        }
      }
      fence_proxy_async();
      mbar_arrive(&ss->full[s]);
    }

    // ===== epilogue: TMEM -> registers -> dequant -> global ====================
    mbar_wait(&ss->accf, 0);
    tc_fence_after();
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int r = q * 32 + lane;
    const int64_t m = m0 + r;
    const float sa = m < a.M ? a.a_scales[m] : 0.f;
    const float acc_scale = BITS == 4 ? (1.0f / 256.0f) : 1.0f;  // exact power of two
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t acc[32];
      tmem_ld32(tmem_acc + ((uint32_t)(q * 32) << 16) + (uint32_t)(c * 32), acc);
      if (m >= a.M) continue;
      const int64_t nb = n0 + c * 32;
      if (nb >= a.N) continue;
      const bool full = nb + 32 <= a.N;
      if (a.out_kind == 2) {
        int32_t* yp = reinterpret_cast<int32_t*>(a.y) + m * a.ldy + nb;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int32_t v = BITS == 4 ? ((int32_t)acc[i] >> 8) : (int32_t)acc[i];
          if (full || nb + i < a.N) yp[i] = v;
        }
      } else if (a.out_kind == 1) {
        float* yp = reinterpret_cast<float*>(a.y) + m * a.ldy + nb;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float av = (float)(int32_t)acc[i] * acc_scale;
          const float v = fmaf(av * sa, ss->sw[c * 32 + i], ss->bias[c * 32 + i]);
          if (full || nb + i < a.N) yp[i] = v;
        }
      } else {
        __nv_bfloat16* yp = reinterpret_cast<__nv_bfloat16*>(a.y) + m * a.ldy + nb;
        uint32_t packed[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float v0 = fmaf((float)(int32_t)acc[2 * i] * acc_scale * sa, ss->sw[c * 32 + 2 * i],
                                ss->bias[c * 32 + 2 * i]);
          const float v1 = fmaf((float)(int32_t)acc[2 * i + 1] * acc_scale * sa,
                                ss->sw[c * 32 + 2 * i + 1], ss->bias[c * 32 + 2 * i + 1]);
          __nv_bfloat162 h = __floats2bfloat162_rn(v0, v1);
          packed[i] = *reinterpret_cast<uint32_t*>(&h);
        }
        if (full && ((reinterpret_cast<uintptr_t>(yp) & 15) == 0)) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            reinterpret_cast<uint4*>(yp)[i] =
                make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
        } else {
          for (int i = 0; i < 32; ++i)
            if (nb + i < a.N) {
              uint32_t w2 = packed[i >> 1];
              uint16_t hb = (i & 1) ? (uint16_t)(w2 >> 16) : (uint16_t)(w2 & 0xFFFF);
              reinterpret_cast<uint16_t*>(yp)[i] = hb;
            }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_acc),
                 "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// Generic CUDA-core kernel for shapes the tensor-core path does not take
// (K not a multiple of 32, unaligned rows).  Exact int32 like int_gemm.
// ---------------------------------------------------------------------------
template <int BITS>
__device__ __forceinline__ int code_at(const uint8_t* row, int64_t k) {
  if constexpr (BITS == 4) {
    uint8_t b = row[k >> 1];
    int nib = (k & 1) ? (b >> 4) : (b & 0x0F);
    return nib >= 8 ? nib - 16 : nib;
  } else {
    return (int)(int8_t)row[k];
  }
}

template <int BITS>
__global__ void k3_generic_kernel(K3Args a) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= a.M * a.N) return;
  const int64_t m = idx / a.N, n = idx % a.N;
  const uint8_t* ar = a.a_codes + m * a.lda;
  const uint8_t* wr = a.w.codes + n * a.w.ld;
  int32_t acc = 0;
  const int wflip = BITS == 4 && a.w.ob ? 8 : 0;  // offset-binary weight nibbles
  for (int64_t k = 0; k < a.K; ++k) {
    int wc = code_at<BITS>(wr, k);
    if (wflip) wc = ((wc & 15) ^ 8) - 8;  // nibble n -> (n ^ 8) as two's complement
    acc += code_at<BITS>(ar, k) * wc;
  }
  if (a.out_kind == 2) {
    reinterpret_cast<int32_t*>(a.y)[m * a.ldy + n] = acc;
  } else {
    float v = fmaf((float)acc * a.a_scales[m], a.w_scales[n], a.bias ? a.bias[n] : 0.f);
    if (a.out_kind == 1) reinterpret_cast<float*>(a.y)[m * a.ldy + n] = v;
    else reinterpret_cast<__nv_bfloat16*>(a.y)[m * a.ldy + n] = __float2bfloat16_rn(v);
  }
}

}  // namespace

__global__ void k3_offset_binary_kernel(const uint8_t* src, int64_t lds, int64_t row_bytes,
                                        uint8_t* dst, int64_t ldd, int64_t n, uint8_t flip) {
  // two's-complement nibble -> offset binary: flip bit 3 (flip = 0x88; 0 if
  // the source is offset binary already); pad = code 0 (0x8)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ldd, c = i - r * ldd;
    dst[i] = c < row_bytes ? src[r * lds + c] ^ flip : 0x88;
  }
}

__global__ void k3_xor_copy_kernel(const uint8_t* src, int64_t lds, uint8_t* dst, int64_t ldd,
                                   int64_t row_bytes, int64_t n) {
  // dst row r = src row r with every nibble's bit 3 flipped (offset binary <->
  // two's complement), row_bytes per row
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / row_bytes, c = i - r * row_bytes;
    dst[r * ldd + c] = src[r * lds + c] ^ 0x88;
  }
}

cudaError_t k3_prepare_weights(const uint8_t* codes, int64_t ldc, int64_t N, int64_t K, int bits,
                               K3Weights* out, cudaStream_t st, int64_t* launches, bool src_ob) {
  out->codes = codes;
  out->codes_ob = nullptr;
  out->ld_ob = 0;
  out->ld = ldc;
  out->N = N;
  out->K = K;
  out->bits = bits;
  out->ob = 0;
  if (bits != 4) return cudaSuccess;
  // the single 4-bit copy: offset binary (TMA 16U4 + tcgen05.cp decompress
  // -> 4*(w+8) for v3; v1 / v2 flip it back as they expand)
  uint8_t* ob = nullptr;
  const int64_t ldo = (K + 127) / 128 * 64;
  cudaError_t e = cudaMalloc(&ob, (size_t)ldo * (N ? N : 1));
  if (e != cudaSuccess) return e;
  const int64_t n = ldo * N;
  if (n > 0) {
    k3_offset_binary_kernel<<<(unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256, 0,
                              st>>>(codes, ldc, (K + 1) / 2, ob, ldo, n, src_ob ? 0x00 : 0x88);
    ++*launches;
  }
  out->codes = ob;
  out->codes_ob = ob;
  out->ld_ob = ldo;
  out->ld = ldo;
  out->ob = 1;
  return cudaGetLastError();
}

cudaError_t k3_export_w4(const K3Weights& w, uint8_t* dst, int64_t ldd, int64_t col_byte0,
                         int64_t row_bytes, cudaStream_t st, int64_t* launches) {
  const int64_t n = row_bytes * w.N;
  if (n <= 0) return cudaSuccess;
  k3_xor_copy_kernel<<<(unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256, 0, st>>>(
      w.codes_ob + col_byte0, w.ld_ob, dst, ldd, row_bytes, n);
  ++*launches;
  return cudaGetLastError();
}

void k3_free_weights(K3Weights* w) {
  cudaFree(const_cast<uint8_t*>(w->codes_ob));
  w->codes_ob = nullptr;
  w->codes = nullptr;
}

cudaError_t k3_launch(const K3Args& a, cudaStream_t st, int64_t* launches) {
  static const bool force_v1 = [] {
    const char* e = getenv("CRT_K3_V1");
    return e && e[0] == '1';
  }();
  static const bool force_v3 = [] {
    const char* e = getenv("CRT_K3_V3");
    return e && e[0] == '1';
  }();
  if (a.a_layout == 1) {  // int8-stored 4-bit activation codes: v4 (default) or v3
    if (!force_v3 && k3_gemv_supported(a)) return k3_gemv_launch(a, st, launches);
    if (!force_v3 && k3_v4_supported(a)) return k3_v4_launch(a, st, launches);
    if (k3_v3_supported(a)) return k3_v3_launch(a, st, launches);
    return cudaErrorInvalidValue;
  }
  if (!force_v1 && a.bits == 8 && k3_v3_supported(a)) return k3_v3_launch(a, st, launches);
  if (!force_v1 && k3_v2_supported(a)) return k3_v2_launch(a, st, launches);
  const bool b4 = a.bits == 4;
  const bool aligned = ((uintptr_t)a.a_codes % 16 == 0) && (a.lda % 16 == 0) &&
                       ((uintptr_t)a.w.codes % 16 == 0) && (a.w.ld % 16 == 0);
  const bool kok = b4 ? (a.K % 32 == 0) : (a.K % 16 == 0);
  const bool cap = !b4 || a.K <= 171196;
  if (aligned && kok && cap && a.K > 0) {
    const size_t smem = 1024 + STAGES * (A_STAGE_BYTES + B_STAGE_BYTES) + sizeof(K3Smem);
    auto kern = b4 ? k3_ss_kernel<4> : k3_ss_kernel<8>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t tiles = ((a.M + BM - 1) / BM) * ((a.N + BN - 1) / BN);
    kern<<<(unsigned)tiles, K3_THREADS, smem, st>>>(a);
    ++*launches;
    return cudaGetLastError();
  }
  const int64_t total = a.M * a.N;
  const unsigned grid = (unsigned)((total + 255) / 256);
  if (b4) k3_generic_kernel<4><<<grid, 256, 0, st>>>(a);
  else k3_generic_kernel<8><<<grid, 256, 0, st>>>(a);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace crt
