// i8_peak_probe.cu -- the dense INT8 tensor-core ceiling of this B200,
// measured directly: every SM runs one CTA that issues back-to-back
// tcgen05.mma kind::i8 (SS form: A and B resident in shared memory, 128B
// swizzle, K-major, M = 128, K = 32, N = 192 or 256) into a TMEM
// accumulator, for `iters` instructions, then commits once.  No loads, no
// epilogue: the MMA pipe alone.  Also kind::f16 (bf16) for comparison with
// the cuBLAS figure in MEASURED_PEAKS.json.  TOPS = 2*M*N*K*iters*SMs / t.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8_peak_probe i8_peak_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(bool i8, int m, int n) {
  // i8: D s32 (2), A/B signed int8; f16 kind: D f32 (1), A/B bf16 (1)
  return (i8 ? (2u << 4) | (1u << 7) | (1u << 10) : (1u << 4) | (1u << 7) | (1u << 10)) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <bool I8, int N>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];  // A 128 x 128 B, B N x 128 B
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < (128 + N) * 128 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (t == 0) {
    const uint64_t a = sw128_desc(smem_u32(sm)), b = sw128_desc(smem_u32(sm + 128 * 128));
    const uint32_t id = idesc(I8, 128, N);
    const uint32_t d = tmem_base;
    const unsigned long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
      // K = 32 bytes per instruction; 4 per 128 B swizzle row (desc + 32 B)
      const uint64_t off = (uint64_t)((i & 3) * 2);  // 32 B >> 4
      if (I8)
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
            "l"(a + off), "l"(b + off), "r"(id), "r"(i));
      else
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
            "l"(a + off), "l"(b + off), "r"(id), "r"(i));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&bar))
                 : "memory");
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar))
        : "memory");
    cycles[blockIdx.x] = clock64() - c0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem_base));
}


// K3's operand path: A from TMEM (ts form) and a tcgen05.cp (int4 -> int8
// decompress, or raw) into the next A slot per MMA, from the same issuing
// thread.  mode 0: ss; 1: ts; 2: ts + decompress cp per MMA; 3: ts + raw cp
// per MMA; 4: ss + decompress cp per MMA (cp result unused).
template <int MODE, int N>
__global__ void __launch_bounds__(128, 1) mma_cp_loop(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];  // A 128 x 128 B, B N x 128 B
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < (128 + N) * 128 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (t == 0) {
    const uint64_t a = sw128_desc(smem_u32(sm)), b = sw128_desc(smem_u32(sm + 128 * 128));
    const uint32_t id = idesc(true, 128, N);
    const uint32_t d = tmem_base;
    const uint32_t aslot = tmem_base + 192;  // 4 slots x 8 columns
    const unsigned long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t off = (uint64_t)((i & 3) * 2);
      const uint32_t ta = aslot + (uint32_t)(i & 3) * 8, tn = aslot + (uint32_t)((i + 2) & 3) * 8;
      if (MODE == 2 || MODE == 4)
        asm volatile("tcgen05.cp.cta_group::1.128x256b.b8x16.b4x16_p64 [%0], %1;" ::"r"(tn), "l"(a + off)
                     : "memory");
      if (MODE == 3)
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tn), "l"(a + off) : "memory");
      if (MODE == 0 || MODE == 4)
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
            "l"(a + off), "l"(b + off), "r"(id), "r"(i));
      else
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
            "r"(ta), "l"(b + off), "r"(id), "r"(i));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&bar))
                 : "memory");
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar))
        : "memory");
    cycles[blockIdx.x] = clock64() - c0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem_base));
}

template <int MODE, int N>
void run_cp(int sms) {
  const int iters = 20000;
  const size_t smem = (size_t)(128 + N) * 128;
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  cudaFuncSetAttribute(mma_cp_loop<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mma_cp_loop<MODE, N><<<sms, 128, smem>>>(100, cyc);
  cudaDeviceSynchronize();
  mma_cp_loop<MODE, N><<<sms, 128, smem>>>(iters, cyc);
  cudaDeviceSynchronize();
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  static const char* names[] = {"ss", "ts", "ts + decompress cp", "ts + raw cp", "ss + decompress cp"};
  printf("kind::i8 M=128 N=%d %-20s: %.1f cycles per MMA (ideal %d) err=%s\n", N, names[MODE],
         (double)c / iters, N / 2, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}


// K3's exact MMA shape: a CTA pair (cta_group::2), M = 256 (128 rows of A
// per CTA), N = 192 (96 rows of B per CTA), K = 32, issued by the leader.
// mode 0: ss; 1: ts; 2: ts + decompress cp per MMA (same thread);
// 3: ts + decompress cp per MMA issued by a second thread (warp 1), as K3.
template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_pair_loop(int iters, unsigned long long* cycles, const uint8_t* gbuf, int ld_bytes) {
  extern __shared__ __align__(1024) uint8_t sm[];  // A 128 x 128 B, B 96 x 128 B, [4 x load stage]
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t lbar[8];
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = t; i < (128 + 96) * 128 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    for (int s = 0; s < 8; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&lbar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint64_t a = sw128_desc(smem_u32(sm)), b = sw128_desc(smem_u32(sm + 128 * 128));
  const uint32_t aslot = tmem_base + 192;
  if (rank == 0 && t == 0) {
    const uint32_t id = idesc(true, 256, 192);
    const uint32_t d = tmem_base;
    const unsigned long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t off = (uint64_t)((i & 3) * 2);
      const uint32_t ta = aslot + (uint32_t)(i & 3) * 8, tn = aslot + (uint32_t)((i + 2) & 3) * 8;
      if (MODE == 2)
        asm volatile("tcgen05.cp.cta_group::2.128x256b.b8x16.b4x16_p64 [%0], %1;" ::"r"(tn), "l"(a + off)
                     : "memory");
      if (MODE == 0 || MODE == 4)
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
            "l"(a + off), "l"(b + off), "r"(id), "r"(i));
      else
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
            "r"(ta), "l"(b + off), "r"(id), "r"(i));
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)), "h"((uint16_t)1)
        : "memory");
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar))
        : "memory");
    cycles[blockIdx.x] = clock64() - c0;
  }
  if (MODE >= 4 && (t == 64 || t == 96)) {
    // K3's smem fill traffic beside the MMAs: two loader threads (both
    // CTAs), each a 4-deep ring of 12 KB bulk copies from an L2-resident
    // buffer, iters * ld_bytes / 2 bytes each; cycles[grid + cta] = their time
    const int w = (t >> 5) - 2;
    uint8_t* ring = sm + (128 + 96) * 128 + w * 4 * 12288;
    uint64_t* lb = &lbar[w * 4];
    uint32_t ph = 0;
    const int n = (int)((long long)iters * ld_bytes / 2 / 12288);
    const unsigned long long c0 = clock64();
    for (int i = 0; i < n; ++i) {
      const int s = i & 3;
      if (i >= 4) {
        asm volatile(
            "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
            "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&lb[s])),
            "r"((ph >> s) & 1u)
            : "memory");
        ph ^= 1u << s;
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&lb[s])),
                   "r"(12288)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(ring + s * 12288)),
          "l"(gbuf + ((size_t)(blockIdx.x * 131 + w * 977 + i) & 2047) * 12288), "r"(12288),
          "r"(smem_u32(&lb[s]))
          : "memory");
    }
    for (int i = n; i < n + 4; ++i) {
      const int s = i & 3;
      if (i >= 4) {
        asm volatile(
            "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
            "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&lb[s])),
            "r"((ph >> s) & 1u)
            : "memory");
        ph ^= 1u << s;
      }
    }
    if (w == 0) cycles[gridDim.x + blockIdx.x] = clock64() - c0;
  }
  if ((MODE == 3 || MODE == 5) && rank == 0 && t == 32) {
    for (int i = 0; i < iters; ++i) {
      const uint64_t off = (uint64_t)((i & 3) * 2);
      asm volatile("tcgen05.cp.cta_group::2.128x256b.b8x16.b4x16_p64 [%0], %1;" ::"r"(
                       aslot + (uint32_t)((i + 2) & 3) * 8),
                   "l"(a + off)
                   : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem_base));
  }
}

template <int MODE>
void run_pair(int sms, int ld_bytes = 0) {
  const int iters = 20000;
  const size_t smem = (size_t)(128 + 96) * 128 + 8 * 12288;
  static uint8_t* gbuf = nullptr;
  if (!gbuf) {
    cudaMalloc(&gbuf, 2048 * 12288);
    cudaMemset(gbuf, 0, 2048 * 12288);
  }
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * 16);
  cudaMemset(cyc, 0, sms * 16);
  cudaFuncSetAttribute(mma_pair_loop<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mma_pair_loop<MODE><<<sms, 128, smem>>>(100, cyc, gbuf, ld_bytes);
  cudaDeviceSynchronize();
  mma_pair_loop<MODE><<<sms, 128, smem>>>(iters, cyc, gbuf, ld_bytes);
  cudaDeviceSynchronize();
  unsigned long long c = 0, cl = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&cl, cyc + sms, 8, cudaMemcpyDeviceToHost);
  if (ld_bytes)
    printf("   loaders: %.1f cycles per MMA-equivalent, %.1f B/cycle/SM loaded\n", (double)cl / iters,
           (double)iters * ld_bytes / cl);
  static const char* names[] = {"ss", "ts", "ts + decompress cp", "ts + cp from 2nd thread",
                                "ss + bulk loads", "ts + 2nd-thread cp + bulk loads"};
  printf("kind::i8 pair M=256 N=192 %-32s (%4d B/MMA loaded): %.1f cycles per MMA (ideal 96) err=%s\n",
         names[MODE], ld_bytes, (double)c / iters, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}


// How deep is the MMA issue queue?  Pair ts MMAs (K3's shape), with, every
// 4 MMAs, one of: (1) a `gap`-cycle clock64 spin, (2) a try_wait on an
// already-complete mbarrier, (3) two tcgen05.commit (K3's per-stage
// commits), (4) the commits + the wait (K3's MMA-thread stage overhead).
template <int EXTRA>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_gap_loop(int iters, int gap, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar, done_bar, cbar[2];
  __shared__ uint32_t flag;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = t; i < (128 + 96) * 128 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done_bar)));
    flag = 1;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(smem_u32(&cbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(smem_u32(&cbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    // complete phase 0 of done_bar once: later waits on parity 0 succeed at once
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&done_bar)) : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint64_t b = sw128_desc(smem_u32(sm + 128 * 128));
  const uint32_t aslot = tmem_base + 192;
  if (rank == 0 && t == 0) {
    const uint32_t id = idesc(true, 256, 192);
    const uint32_t d = tmem_base;
    const unsigned long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t off = (uint64_t)((i & 3) * 2);
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
          "r"(aslot + (uint32_t)(i & 3) * 8), "l"(b + off), "r"(id), "r"(i));
      if ((EXTRA == 15 && (i & 7) == 7) || (EXTRA == 16 && (i & 15) == 15)) {
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&cbar[0])), "h"((uint16_t)3)
            : "memory");
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&cbar[1])), "h"((uint16_t)1)
            : "memory");
        asm volatile(
            "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
            "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&done_bar))
            : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      if ((i & 3) == 3 && EXTRA < 14) {
        if (EXTRA == 1) {
          const unsigned long long s0 = clock64();
          while (clock64() - s0 < (unsigned long long)gap) {
          }
        }
        if (EXTRA == 12) {
          asm volatile(
              "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
              "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&done_bar))
              : "memory");
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        if (EXTRA == 13) {  // relaxed (volatile) flag poll
          uint32_t v;
          do {
            asm volatile("ld.volatile.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(&flag)) : "memory");
          } while (v == 0);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        if (EXTRA >= 3 && EXTRA != 11) {
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&cbar[0])), "h"((uint16_t)3)
              : "memory");
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&cbar[1])), "h"((uint16_t)1)
              : "memory");
        }
        if (EXTRA == 11)
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&cbar[0])), "h"((uint16_t)3)
              : "memory");
        if (EXTRA == 2 || EXTRA == 4 || EXTRA == 11 || (EXTRA == 7 && (i & 7) == 7)) {
          asm volatile(
              "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
              "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&done_bar))
              : "memory");
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        if (EXTRA == 8)
          asm volatile(
              "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
              "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&done_bar))
              : "memory");
        if (EXTRA == 9) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (EXTRA == 10) {  // plain shared-memory flag poll (acquire), already set
          uint32_t v;
          do {
            asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(&flag)) : "memory");
          } while (v == 0);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        if (EXTRA == 5) {
          asm volatile(
              "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.relaxed.cta.shared::cta.b64 P1, [%0], 0;\n"
              "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&done_bar))
              : "memory");
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        if (EXTRA == 6) {
          asm volatile(
              "{\n.reg .pred P1;\nW_%=:\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
              "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&done_bar))
              : "memory");
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
      }
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)), "h"((uint16_t)1)
        : "memory");
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar))
        : "memory");
    cycles[blockIdx.x] = clock64() - c0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem_base));
  }
}

template <int EXTRA>
void run_gap(int sms, int gap) {
  const int iters = 20000;
  const size_t smem = (size_t)(128 + 96) * 128;
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  cudaFuncSetAttribute(mma_gap_loop<EXTRA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mma_gap_loop<EXTRA><<<sms, 128, smem>>>(100, gap, cyc);
  cudaDeviceSynchronize();
  mma_gap_loop<EXTRA><<<sms, 128, smem>>>(iters, gap, cyc);
  cudaDeviceSynchronize();
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  static const char* names[] = {"none", "spin", "try_wait (complete)", "2 commits", "2 commits + try_wait",
                                "2 commits + relaxed try_wait", "2 commits + test_wait",
                                "2 commits, wait every 8", "2 commits + try_wait, no fence",
                                "2 commits + fence only", "2 commits + flag poll", "1 commit + try_wait",
                                "try_wait, then 2 commits", "volatile poll + 2 commits", "-",
                                "8 MMAs: 2 commits + try_wait", "16 MMAs: 2 commits + try_wait"};
  printf("pair ts MMA, every 4 MMAs: %-30s gap %4d: %.1f cycles per 4 MMAs (ideal 384) err=%s\n",
         names[EXTRA], EXTRA == 1 ? gap : 0, 4.0 * c / iters, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}


// The drain comes from a shared-memory access by the thread with pending
// commits.  Here lane 0 issues the MMAs and the commits, and LANE 1 does the
// mbarrier wait (then __syncwarp, then lane 0's tcgen05 fence): every 4 MMAs
// (K3's stage) or, with `every` = 8, every 8.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_lane_wait_loop(int iters, int every, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar, done_bar, cbar[2];
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = t; i < (128 + 96) * 128 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done_bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(smem_u32(&cbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(smem_u32(&cbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&done_bar)) : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint64_t b = sw128_desc(smem_u32(sm + 128 * 128));
  const uint32_t aslot = tmem_base + 192;
  if (every < 0) {  // named-barrier relay: warp 1 waits on the mbarrier, warp 0 bar.syncs
    // handshake per group j: ready[j&1] (ids 1,2: warp 1 arrives, warp 0
    // syncs), done[j&1] (ids 3,4: warp 0 arrives, warp 1 syncs before its
    // arrival for group j+2, so a barrier generation is never aliased)
    const int ev = -every;
    const int groups = iters / ev;
    if (rank == 0 && warp == 1) {
      for (int j = 0; j < groups; ++j) {
        if (lane == 0)
          asm volatile(
              "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
              "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&done_bar))
              : "memory");
        __syncwarp();
        if (j >= 2) asm volatile("barrier.cta.sync.aligned %0, 64;" ::"r"(3 + (j & 1)) : "memory");
        asm volatile("barrier.cta.arrive.aligned %0, 64;" ::"r"(1 + (j & 1)) : "memory");
      }
      for (int j = groups; j < groups + 2; ++j)
        if (j >= 2) asm volatile("barrier.cta.sync.aligned %0, 64;" ::"r"(3 + (j & 1)) : "memory");
    }
    if (rank == 0 && warp == 0) {
      const uint32_t id = idesc(true, 256, 192);
      const uint32_t d = tmem_base;
      const unsigned long long c0 = clock64();
      for (int j = 0; j < groups; ++j) {
        asm volatile("barrier.cta.sync.aligned %0, 64;" ::"r"(1 + (j & 1)) : "memory");
        asm volatile("barrier.cta.arrive.aligned %0, 64;" ::"r"(3 + (j & 1)) : "memory");
        if (lane == 0) {
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          for (int k = 0; k < ev; ++k) {
            const int i = j * ev + k;
            const uint64_t off = (uint64_t)((i & 3) * 2);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                "r"(aslot + (uint32_t)(i & 3) * 8), "l"(b + off), "r"(id), "r"(i));
          }
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&cbar[0])), "h"((uint16_t)3)
              : "memory");
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&cbar[1])), "h"((uint16_t)1)
              : "memory");
        }
        __syncwarp();
      }
      if (lane == 0) {
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)), "h"((uint16_t)1)
            : "memory");
        asm volatile(
            "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
            "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar))
            : "memory");
        cycles[blockIdx.x] = clock64() - c0;
      }
    }
  } else if (rank == 0 && warp == 0) {
    const uint32_t id = idesc(true, 256, 192);
    const uint32_t d = tmem_base;
    const unsigned long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t off = (uint64_t)((i & 3) * 2);
      if (lane == 0)
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
            "r"(aslot + (uint32_t)(i & 3) * 8), "l"(b + off), "r"(id), "r"(i));
      if ((i & (every - 1)) == every - 1) {
        if (lane == 0) {
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&cbar[0])), "h"((uint16_t)3)
              : "memory");
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&cbar[1])), "h"((uint16_t)1)
              : "memory");
        }
        if (lane == 1)
          asm volatile(
              "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
              "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&done_bar))
              : "memory");
        __syncwarp();
        if (lane == 0) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
    }
    if (lane == 0) {
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&bar)), "h"((uint16_t)1)
          : "memory");
      asm volatile(
          "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
          "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar))
          : "memory");
      cycles[blockIdx.x] = clock64() - c0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem_base));
  }
}

void run_lane_wait(int sms, int every) {
  const int iters = 20000;
  const size_t smem = (size_t)(128 + 96) * 128;
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  cudaFuncSetAttribute(mma_lane_wait_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mma_lane_wait_loop<<<sms, 128, smem>>>(100, every, cyc);
  cudaDeviceSynchronize();
  mma_lane_wait_loop<<<sms, 128, smem>>>(iters, every, cyc);
  cudaDeviceSynchronize();
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("pair ts MMA, lane 0 MMAs + 2 commits, %s every %d: %.1f cycles per 4 MMAs (ideal 384) err=%s\n",
         every < 0 ? "warp 1 try_wait -> named barrier" : "LANE 1 try_wait + __syncwarp", every < 0 ? -every : every,
         4.0 * c / iters, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}


// Two MMA-issuing threads (warps 0 and 2 of the leader CTA), each with K3's
// per-stage pattern (4 MMAs, 2 commits, a wait) into its own accumulator:
// is the post-commit drain per issuing thread (hidden by the other
// thread's MMAs) or per SM?
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_two_issuers(int iters, int nissuers, unsigned long long* cycles, int k3like = 0) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[2], done_bar, cbar[4];
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = t; i < (128 + 96) * 128 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (t == 0) {
    for (int k = 0; k < 2; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[k])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done_bar)));
    for (int k = 0; k < 4; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(smem_u32(&cbar[k])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&done_bar)) : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint64_t b = sw128_desc(smem_u32(sm + 128 * 128));
  const int who = warp == 0 ? 0 : (warp == 2 ? 1 : -1);
  if (rank == 0 && lane == 0 && who >= 0 && who < nissuers) {
    const uint32_t id = idesc(true, 256, 192);
    const uint32_t d = tmem_base + (uint32_t)who * 256;
    const uint32_t aslot = d + 192;
    const unsigned long long c0 = clock64();
    const uint64_t adesc = sw128_desc(smem_u32(sm));
    for (int i = 0; i < iters; ++i) {
      const uint64_t off = (uint64_t)((i & 3) * 2);
      if (k3like && (i & 3) == 0) {  // K3's stage head: a second wait, fence, 4 decompress cps
        asm volatile(
            "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
            "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&done_bar))
            : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int k = 0; k < 4; ++k)
          asm volatile("tcgen05.cp.cta_group::2.128x256b.b8x16.b4x16_p64 [%0], %1;" ::"r"(aslot + k * 8),
                       "l"(adesc + (uint64_t)(k * 2))
                       : "memory");
      }
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
          "r"(aslot + (uint32_t)(i & 3) * 8), "l"(b + off), "r"(id), "r"(i));
      if ((i & 3) == 3) {
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&cbar[2 * who])), "h"((uint16_t)3)
            : "memory");
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&cbar[2 * who + 1])), "h"((uint16_t)1)
            : "memory");
        asm volatile(
            "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
            "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&done_bar))
            : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar[who])), "h"((uint16_t)1)
        : "memory");
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar[who]))
        : "memory");
    cycles[2 * blockIdx.x + who] = clock64() - c0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

void run_two(int sms, int n, int k3like = 0) {
  const int iters = 20000;
  const size_t smem = (size_t)(128 + 96) * 128;
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * 16);
  cudaFuncSetAttribute(mma_two_issuers, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mma_two_issuers<<<sms, 128, smem>>>(100, n, cyc, k3like);
  cudaDeviceSynchronize();
  mma_two_issuers<<<sms, 128, smem>>>(iters, n, cyc, k3like);
  cudaDeviceSynchronize();
  unsigned long long c[2] = {0, 0};
  cudaMemcpy(c, cyc, 16, cudaMemcpyDeviceToHost);
  const unsigned long long cm = c[0] > c[1] ? c[0] : c[1];
  printf("%d issuing thread(s), each 4 MMAs + 2 commits + wait%s: %.1f cycles per MMA over all (ideal 96) err=%s\n", n,
         k3like ? " + K3 stage head (wait, 4 cps)" : "",
         (double)cm / (iters * n), cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}


// Correctness of K3's planned split: two issuing threads (warps 1 and 2,
// leader CTA) alternate 4-MMA groups into the SAME accumulator (issuer 1
// starts after issuer 0's first, zeroing, group completed).  A (TMEM, via
// tcgen05.cp) and B are all ones, so every D element must end at
// 32 * iters.  mism[0] counts wrong elements over both CTAs.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_same_d(int iters, unsigned int* mism, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar, start_bar, done_bar, cbar[4];
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = t; i < (128 + 96) * 128 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&start_bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done_bar)));
    for (int k = 0; k < 4; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(smem_u32(&cbar[k])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&done_bar)) : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint64_t a = sw128_desc(smem_u32(sm)), b = sw128_desc(smem_u32(sm + 128 * 128));
  const uint32_t d = tmem_base, aslot = tmem_base + 192;
  if (rank == 0 && t == 0) {  // A slots: 4 x 8 columns of int8 ones (raw copy, both CTAs)
    for (int k = 0; k < 4; ++k)
      asm volatile("tcgen05.cp.cta_group::2.128x256b [%0], %1;" ::"r"(aslot + k * 8), "l"(a + (uint64_t)(k * 2))
                   : "memory");
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&start_bar)), "h"((uint16_t)1)
        : "memory");
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&start_bar))
        : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int who = warp == 1 ? 0 : (warp == 2 ? 1 : -1);
  if (rank == 0 && lane == 0 && who >= 0) {
    const uint32_t id = idesc(true, 256, 192);
    const unsigned long long c0 = clock64();
    if (who == 1) {  // after issuer 0's first (zeroing) group completed: start_bar phase 1
      asm volatile(
          "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 1;\n"
          "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&start_bar))
          : "memory");
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    for (int g = who; g < iters / 4; g += 2) {
      for (int k = 0; k < 4; ++k) {
        const int i = g * 4 + k;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
            "r"(aslot + (uint32_t)k * 8), "l"(b + (uint64_t)(k * 2)), "r"(id), "r"(i));
      }
      if (g == 0)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&start_bar)), "h"((uint16_t)1)
            : "memory");
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&cbar[2 * who])), "h"((uint16_t)3)
          : "memory");
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&cbar[2 * who + 1])), "h"((uint16_t)1)
          : "memory");
      asm volatile(
          "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
          "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&done_bar))
          : "memory");
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)), "h"((uint16_t)3)
        : "memory");
    if (who == 0) {
      asm volatile(
          "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
          "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar))
          : "memory");
      cycles[blockIdx.x] = clock64() - c0;
    }
  }
  // every CTA: wait for both issuers' completion (both commits multicast here)
  if (lane == 0)
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar))
        : "memory");
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  unsigned int bad = 0;
  const uint32_t want = 32u * (uint32_t)iters;
  for (int c = 0; c < 192; c += 32) {
    uint32_t r[32];
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
        : "r"(d + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 32; ++j) bad += r[j] != want;
  }
  if (bad) atomicAdd(mism, bad);
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem_base));
  }
}

void run_same_d(int sms) {
  unsigned long long* cyc;
  unsigned int* mism;
  cudaMalloc(&cyc, sms * 8);
  cudaMalloc(&mism, 4);
  const size_t smem = (size_t)(128 + 96) * 128;
  cudaFuncSetAttribute(mma_same_d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int iters : {8, 64, 20000}) {
    cudaMemset(mism, 0, 4);
    mma_same_d<<<sms, 128, smem>>>(iters, mism, cyc);
    cudaDeviceSynchronize();
    unsigned int m = 0;
    unsigned long long c = 0;
    cudaMemcpy(&m, mism, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("two issuers, same accumulator, %5d MMAs: %u wrong of %d elements; %.1f cycles per MMA err=%s\n", iters, m,
           sms * 128 * 192, (double)c / iters, cudaGetErrorString(cudaGetLastError()));
  }
}


// K3's inline pattern with 1..4 issuing threads (warps 0..3 of the leader),
// all into ONE accumulator (as K3): per 4-MMA stage each issuer waits,
// expands its stage's A (4 decompress copies into its own 32-column slot),
// issues the 4 dependent MMAs and 2 commits.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_n_issuers(int iters, int nissuers, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[4], done_bar, cbar[8];
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = t; i < (128 + 96) * 128 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (t == 0) {
    for (int k = 0; k < 4; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[k])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done_bar)));
    for (int k = 0; k < 8; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(smem_u32(&cbar[k])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&done_bar)) : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint64_t b = sw128_desc(smem_u32(sm + 128 * 128));
  const uint64_t adesc = sw128_desc(smem_u32(sm));
  const int who = warp;
  if (rank == 0 && lane == 0 && who < nissuers) {
    const uint32_t id = idesc(true, 256, 192);
    const uint32_t d = tmem_base;
    const uint32_t aslot = tmem_base + 192 + (uint32_t)who * 32;
    const unsigned long long c0 = clock64();
    for (int st = who; st < iters / 4; st += nissuers) {
      asm volatile(
          "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
          "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&done_bar))
          : "memory");
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int k = 0; k < 4; ++k)
        asm volatile("tcgen05.cp.cta_group::2.128x256b.b8x16.b4x16_p64 [%0], %1;" ::"r"(aslot + k * 8),
                     "l"(adesc + (uint64_t)(k * 2))
                     : "memory");
      for (int k = 0; k < 4; ++k)
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
            "r"(aslot + (uint32_t)k * 8), "l"(b + (uint64_t)(k * 2)), "r"(id), "r"(1));
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&cbar[2 * who])), "h"((uint16_t)3)
          : "memory");
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&cbar[2 * who + 1])), "h"((uint16_t)1)
          : "memory");
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar[who])), "h"((uint16_t)1)
        : "memory");
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar[who]))
        : "memory");
    cycles[4 * blockIdx.x + who] = clock64() - c0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

void run_n(int sms, int n) {
  const int iters = 20000;
  const size_t smem = (size_t)(128 + 96) * 128;
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * 32);
  cudaMemset(cyc, 0, sms * 32);
  cudaFuncSetAttribute(mma_n_issuers, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mma_n_issuers<<<sms, 128, smem>>>(100, n, cyc);
  cudaDeviceSynchronize();
  mma_n_issuers<<<sms, 128, smem>>>(iters, n, cyc);
  cudaDeviceSynchronize();
  unsigned long long c[4];
  cudaMemcpy(c, cyc, 32, cudaMemcpyDeviceToHost);
  unsigned long long cm = 0;
  for (int k = 0; k < n; ++k) cm = c[k] > cm ? c[k] : cm;
  printf("%d issuers, K3 inline stage (wait, 4 cps, 4 dependent MMAs, 2 commits), one accumulator: %.1f cycles per MMA (ideal 96) err=%s\n",
         n, (double)cm / iters, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}


// Pair ts MMAs (K3's shape) from one thread while warps 1..4 store into TMEM
// A-slot columns with tcgen05.st at K3 v4's rate (4 KB per warp per 4 MMAs),
// in shape SHAPE: 0 = 32x32b.x32, 1 = 32x32b.x8 (four per 4 KB), 2 =
// 16x256b.x8 (16 lanes x 8 cols x 8 reps... = 4 KB per instruction pair).
template <int SHAPE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(160, 1)
    mma_tmem_st_loop(int iters, int store, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = t; i < (128 + 96) * 128 / 4; i += 160) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint64_t b = sw128_desc(smem_u32(sm + 128 * 128));
  const uint32_t d = tmem_base, aslot = tmem_base + 192;
  if (rank == 0 && t == 0) {
    const uint32_t id = idesc(true, 256, 192);
    const unsigned long long c0 = clock64();
    for (int i = 0; i < iters; ++i)
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
          "r"(aslot + (uint32_t)(i & 3) * 8), "l"(b + (uint64_t)((i & 3) * 2)), "r"(id), "r"(i));
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)), "h"((uint16_t)1)
        : "memory");
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar))
        : "memory");
    cycles[blockIdx.x] = clock64() - c0;
  }
  if (store && warp >= 1) {  // warps 1..4: lane quarter (warp % 4); store into columns 448.. (unused)
    const uint32_t q = (uint32_t)(warp & 3);
    const uint32_t ta = tmem_base + 448 + (q * 32 << 16);
    uint32_t r[32];
    for (int k = 0; k < 32; ++k) r[k] = (uint32_t)(k * 0x01010101);
    // K3 v4: 4 KB per warp per stage of 4 MMAs (~384 cycles); pace with the clock
    const unsigned long long c0 = clock64();
    for (int j = 0; j < iters / 4; ++j) {
      while (clock64() - c0 < (unsigned long long)j * 384) {
      }
      if (SHAPE == 0) {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
            "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
            "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
            "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
            "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
            "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
            "r"(r[29]), "r"(r[30]), "r"(r[31])
            : "memory");
      } else {
        for (int h = 0; h < 4; ++h)
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta + h * 8),
              "r"(r[8 * h]), "r"(r[8 * h + 1]), "r"(r[8 * h + 2]), "r"(r[8 * h + 3]), "r"(r[8 * h + 4]),
              "r"(r[8 * h + 5]), "r"(r[8 * h + 6]), "r"(r[8 * h + 7])
              : "memory");
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

template <int SHAPE>
void run_st(int sms, int store) {
  const int iters = 20000;
  const size_t smem = (size_t)(128 + 96) * 128;
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  cudaFuncSetAttribute(mma_tmem_st_loop<SHAPE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mma_tmem_st_loop<SHAPE><<<sms, 160, smem>>>(100, store, cyc);
  cudaDeviceSynchronize();
  mma_tmem_st_loop<SHAPE><<<sms, 160, smem>>>(iters, store, cyc);
  cudaDeviceSynchronize();
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("pair ts MMA + TMEM stores (%s, %s): %.1f cycles per MMA (ideal 96) err=%s\n",
         store ? "on" : "off", SHAPE == 0 ? "32x32b.x32" : "4 x 32x32b.x8", (double)c / iters,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

template <bool I8, int N>
void run(int sms) {
  const int iters = 20000;
  const size_t smem = (size_t)(128 + N) * 128;
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  cudaFuncSetAttribute(mma_loop<I8, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mma_loop<I8, N><<<sms, 128, smem>>>(100, cyc);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma_loop<I8, N><<<sms, 128, smem>>>(iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const int KE = I8 ? 32 : 16;  // K elements per instruction (32 bytes either way)
  const double ops = 2.0 * 128 * N * KE * (double)iters * sms;
  printf("kind::%s M=128 N=%d K=32B SS, %d SMs x %d MMAs: %.1f us -> %.0f TOPS (%.1f cycles/MMA/SM, "
         "%.0f MACs/cycle/SM) err=%s\n",
         I8 ? "i8 " : "f16", N, sms, iters, ms * 1e3, ops / (ms * 1e-3) / 1e12, (double)c / iters,
         128.0 * N * KE * iters / (double)c, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<true, 192>(sms);
  run<true, 256>(sms);
  run<false, 192>(sms);
  run<false, 256>(sms);
  run_gap<0>(sms, 0);
  for (int g : {50, 100, 200, 300, 400}) run_gap<1>(sms, g);
  run_gap<2>(sms, 0);
  run_gap<3>(sms, 0);
  run_gap<4>(sms, 0);
  run_gap<5>(sms, 0);
  run_gap<6>(sms, 0);
  run_gap<7>(sms, 0);
  run_gap<8>(sms, 0);
  run_gap<9>(sms, 0);
  run_gap<10>(sms, 0);
  run_gap<11>(sms, 0);
  run_gap<12>(sms, 0);
  run_gap<13>(sms, 0);
  run_st<0>(sms, 0);
  run_st<0>(sms, 1);
  run_st<1>(sms, 1);
  for (int n = 1; n <= 4; ++n) run_n(sms, n);
  run_same_d(sms);
  run_two(sms, 1);
  run_two(sms, 2);
  run_two(sms, 1, 1);
  run_two(sms, 2, 1);
  run_lane_wait(sms, 4);
  run_lane_wait(sms, 8);
  run_lane_wait(sms, -4);
  run_lane_wait(sms, -8);
  run_gap<15>(sms, 0);
  run_gap<16>(sms, 0);
  run_pair<0>(sms);
  run_pair<1>(sms);
  run_pair<2>(sms);
  run_pair<3>(sms);
  for (int lb : {2048, 4096, 5120, 7168, 8192}) run_pair<5>(sms, lb);
  for (int lb : {4096, 7168}) run_pair<4>(sms, lb);
  run_cp<0, 192>(sms);
  run_cp<1, 192>(sms);
  run_cp<2, 192>(sms);
  run_cp<3, 192>(sms);
  run_cp<4, 192>(sms);
  run_cp<1, 256>(sms);
  run_cp<2, 256>(sms);
  run_cp<2, 96>(sms);
  run_cp<1, 96>(sms);
  return 0;
}
