// l2_bw_probe.cu -- L2 -> shared-memory bandwidth of this B200 with every SM
// pulling L2-resident data through cp.async.bulk (the path K3's TMA loads
// take), to decide whether K3's operand streams are L2-bound.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_bw_probe l2_bw_probe.cu
// One CTA per SM, one thread issues `chunk`-byte bulk copies into an 8-deep
// smem ring (mbarrier complete_tx), walking a `span`-byte window of a buffer
// that stays in L2.  mode 0: CTAs read disjoint offsets; mode 1: groups of
// 4 CTAs read the same offsets at the same time (K3's shared operand tiles).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(32, 1) pull(const uint8_t* buf, size_t span, int chunk, int iters,
                                               int mode, unsigned long long* cyc, int depth = 8, int poll = 0) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[32];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < depth; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const size_t nchunks = span / chunk;
  const size_t start = mode == 0 ? (size_t)blockIdx.x * 977 : (size_t)(blockIdx.x / 4) * 977;
  size_t ci = start % nchunks;  // chunk index, wrapped incrementally (no division in the loop)
  int s = 0;
  const unsigned long long c0 = clock64();
  uint32_t phase = 0;
  for (int i = 0; i < iters + depth; ++i) {
    if (i >= depth) {
      if (poll)
        asm volatile(
            "{\n.reg .pred P1;\nW_%=:\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
            "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar[s])),
            "r"((phase >> s) & 1u)
            : "memory");
      else
      asm volatile(
          "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
          "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar[s])),
          "r"((phase >> s) & 1u)
          : "memory");
      phase ^= 1u << s;
    }
    if (i < iters) {
      const uint8_t* src = buf + ci * chunk;
      if (++ci == nchunks) ci = 0;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])),
                   "r"(chunk)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(sm + s * chunk)),
          "l"(src), "r"(chunk), "r"(smem_u32(&bar[s]))
          : "memory");
    }
    if (++s == depth) s = 0;
  }
  cyc[blockIdx.x] = clock64() - c0;
}


// W issuing warps per CTA (lane 0 of each runs its own ring of `depth`
// copies of `chunk` bytes): is the ~240-cycle per-copy cost per issuing
// thread (overlappable) or per SM (the TMA unit's request rate)?
__global__ void __launch_bounds__(256, 1) pull_multi(const uint8_t* buf, size_t span, int chunk, int iters,
                                                     int depth, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[8][16];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0) return;
  for (int s = 0; s < depth; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[w][s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const size_t nchunks = span / chunk;
  size_t ci = ((size_t)blockIdx.x * 977 + w * 131) % nchunks;
  uint8_t* ring = sm + (size_t)w * depth * chunk;
  const unsigned long long c0 = clock64();
  uint32_t phase = 0;
  int s = 0;
  for (int i = 0; i < iters + depth; ++i) {
    if (i >= depth) {
      asm volatile(
          "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
          "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar[w][s])),
          "r"((phase >> s) & 1u)
          : "memory");
      phase ^= 1u << s;
    }
    if (i < iters) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[w][s])),
                   "r"(chunk)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(ring + s * chunk)),
          "l"(buf + ci * chunk), "r"(chunk), "r"(smem_u32(&bar[w][s]))
          : "memory");
      if (++ci == nchunks) ci = 0;
    }
    if (++s == depth) s = 0;
  }
  if (w == 0) cyc[blockIdx.x] = clock64() - c0;
}


// Where the per-copy cost of one issuing thread goes: clock64 around each
// instruction of the ring step (expect_tx, the copy, the wait on a barrier
// whose copy landed long ago).
__global__ void __launch_bounds__(32, 1) step_cost(const uint8_t* buf, int chunk, int tensor_like,
                                                    unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[32];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < 32; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  unsigned long long te = 0, tc = 0, tw = 0;
  for (int i = 0; i < 32 * 8; ++i) {
    const int s = i & 31;
    unsigned long long c0 = clock64();
    if (i >= 32) {
      asm volatile(
          "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
          "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar[s])),
          "r"(((i >> 5) - 1) & 1)
          : "memory");
    }
    unsigned long long c1 = clock64();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])),
                 "r"(chunk * (tensor_like ? 2 : 1))
                 : "memory");
    unsigned long long c2 = clock64();
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(sm + (s & 3) * 2 * chunk)),
        "l"(buf + (size_t)(i & 255) * chunk * 2), "r"(chunk), "r"(smem_u32(&bar[s]))
        : "memory");
    if (tensor_like)
      asm volatile(
          "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(sm + (s & 3) * 2 * chunk + chunk)),
          "l"(buf + (size_t)(i & 255) * chunk * 2 + chunk), "r"(chunk), "r"(smem_u32(&bar[s]))
          : "memory");
    unsigned long long c3 = clock64();
    if (i >= 64) {
      tw += c1 - c0;
      te += c2 - c1;
      tc += c3 - c2;
    }
  }
  out[0] = tw;
  out[1] = te;
  out[2] = tc;
}


// Unloaded latency of one bulk copy (depth 1, one SM), same source each
// time (L2-resident after the first), by size.
__global__ void __launch_bounds__(32, 1) lat1(const uint8_t* buf, int chunk, int iters, int stride,
                                               unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x != 0) return;
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  asm volatile("fence.mbarrier_init.release.cluster;");
  unsigned long long tot = 0;
  for (int i = 0; i < iters; ++i) {
    const unsigned long long c0 = clock64();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(chunk)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(sm)),
        "l"(buf + (size_t)(i % 16) * stride), "r"(chunk), "r"(smem_u32(&bar))
        : "memory");
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar)),
        "r"(i & 1)
        : "memory");
    if (i >= 16) tot += clock64() - c0;
  }
  out[0] = tot / (iters - 16);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t span = 32ull << 20;  // 32 MB: L2-resident
  uint8_t* buf;
  cudaMalloc(&buf, span);
  cudaMemset(buf, 1, span);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  for (int chunk : {128, 1024, 4096, 16384}) {
    cudaFuncSetAttribute(lat1, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    lat1<<<1, 32, 16384>>>(buf, chunk, 200, 16384, cyc);
    cudaDeviceSynchronize();
    unsigned long long h = 0;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("one bulk copy of %5d B, nothing else running: %llu cycles round trip %s\n", chunk, h,
           cudaGetErrorString(cudaGetLastError()));
  }
  for (int tl = 0; tl < 2; ++tl)
    for (int chunk : {1024, 8192}) {
      cudaFuncSetAttribute(step_cost, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * chunk);
      step_cost<<<1, 32, 8 * chunk>>>(buf, chunk, tl, cyc);
      cudaDeviceSynchronize();
      unsigned long long h[3];
      cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
      const double n = 32 * 6;
      printf("one thread, %d copy(ies) of %d B per step: wait(landed) %.0f, expect_tx %.0f, copies %.0f cycles %s\n",
             tl + 1, chunk, h[0] / n, h[1] / n, h[2] / n, cudaGetErrorString(cudaGetLastError()));
    }
  struct Cfg { int grid, chunk, depth, poll; };
  for (Cfg k : {Cfg{1, 16384, 8, 0}, Cfg{148, 16384, 8, 0}, Cfg{1, 16384, 8, 1}, Cfg{1, 4096, 8, 0},
                Cfg{1, 4096, 16, 0}, Cfg{1, 4096, 32, 0}, Cfg{1, 1024, 32, 0}, Cfg{1, 8192, 24, 0},
                Cfg{148, 8192, 24, 0}, Cfg{148, 8192, 24, 1}}) {
    const int grid = k.grid, chunk = k.chunk, mode = 0;
    const int iters = 4000;
    cudaFuncSetAttribute(pull, cudaFuncAttributeMaxDynamicSharedMemorySize, k.depth * chunk);
    pull<<<grid, 32, k.depth * chunk>>>(buf, span, chunk, iters, mode, cyc, k.depth, k.poll);
    cudaDeviceSynchronize();
    unsigned long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("grid %3d chunk %5d x %2d in flight%s: %.1f B/cycle/SM -> %.0f cycles per copy round trip, %.0f cycles/iter\n",
           grid, chunk, k.depth, k.poll ? " (test_wait poll)" : "", (double)chunk * iters / c,
           (double)k.depth * chunk / ((double)chunk * iters / c), (double)c / iters);
  }
  for (int W : {1, 2, 4, 8})
    for (int chunk : {2048, 8192}) {
      const int depth = 8, iters = 2000;
      const int smem = W * depth * chunk;
      if (smem > 200 * 1024) continue;
      cudaFuncSetAttribute(pull_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      pull_multi<<<148, 32 * W, smem>>>(buf, span, chunk, iters, depth, cyc);
      cudaDeviceSynchronize();
      unsigned long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("148 CTAs x %d issuing warps, chunk %5d x %d: %.1f B/cycle/SM, %.0f cycles per copy per SM %s\n", W,
             chunk, depth, (double)W * chunk * iters / c, (double)c / (W * iters),
             cudaGetErrorString(cudaGetLastError()));
    }
  for (int mode = 0; mode < 2; ++mode)
    for (int chunk : {16384, 20480, 24576, 27648}) {
      const int iters = (int)((2ull << 30) / ((size_t)chunk * sms));  // ~2 GB total
      const size_t smem = (size_t)8 * chunk;
      cudaFuncSetAttribute(pull, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      pull<<<sms, 32, smem>>>(buf, span, chunk, 64, mode, cyc);
      cudaDeviceSynchronize();
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      pull<<<sms, 32, smem>>>(buf, span, chunk, iters, mode, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)chunk * iters * sms;
      printf("mode %d (%s) chunk %5d: %.2f TB/s, %.0f B/cycle chip (%.1f B/cycle/SM at CTA0's clock) %s\n",
             mode, mode ? "4 CTAs share offsets" : "disjoint", chunk, bytes / (ms * 1e-3) / 1e12,
             bytes / c, bytes / c / sms, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
