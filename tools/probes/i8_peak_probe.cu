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
  return 0;
}
