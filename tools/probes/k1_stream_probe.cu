// Memory-structure ceiling for K1: rows of K bf16 streamed through a
// per-CTA TMA (cp.async.bulk) ring into shared memory, each lane turning its
// 16-element chunks into 16 int8 bytes (low byte of the bf16 high half) and
// storing them -- K1's HBM traffic (2 B in + 1 B out per element) with no
// arithmetic.  Variants: CTA = W warps (one row at a time), S stages; and a
// direct-load variant (ld.global.nc.v8 into registers, no shared memory).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o k1_stream_probe k1_stream_probe.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(b) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("{\n.reg .b64 pol;\ncreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
               "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n}\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__global__ void ring_kernel(const uint16_t* x, uint8_t* out, int M, int K, int S) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ uint64_t bar[8];
  const int W = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x & 31;
  const uint32_t rb = K * 2;
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < S; ++s) { int r = blockIdx.x + s * gridDim.x; if (r >= M) break; mbar_expect(&bar[s], rb); bulk(ring + s * rb, x + (size_t)r * K, rb, &bar[s]); }
  int st = 0; uint32_t ph = 0;
  const int nch = K / 16;
  for (int r = blockIdx.x; r < M; r += gridDim.x) {
    mbar_wait(&bar[st], ph);
    const uint8_t* rowp = ring + st * rb;
    for (int c = threadIdx.x; c < nch; c += blockDim.x) {
      const uint4 a = *reinterpret_cast<const uint4*>(rowp + c * 32);
      const uint4 b = *reinterpret_cast<const uint4*>(rowp + c * 32 + 16);
      uint4 o;
      o.x = __byte_perm(a.x, a.y, 0x7531); o.y = __byte_perm(a.z, a.w, 0x7531);
      o.z = __byte_perm(b.x, b.y, 0x7531); o.w = __byte_perm(b.z, b.w, 0x7531);
      *reinterpret_cast<uint4*>(out + (size_t)r * K + c * 16) = o;
    }
    __syncthreads();
    if (threadIdx.x == 0) { int rn = r + S * gridDim.x; if (rn < M) { mbar_expect(&bar[st], rb); bulk(ring + st * rb, x + (size_t)rn * K, rb, &bar[st]); } }
    if (++st == S) { st = 0; ph ^= 1; }
  }
}

__global__ void direct_kernel(const uint16_t* x, uint8_t* out, int M, int K) {
  // grid-stride over 16-element chunks of the whole matrix, 256-bit loads
  const size_t nch = (size_t)M * K / 16;
  for (size_t c = blockIdx.x * (size_t)blockDim.x + threadIdx.x; c < nch; c += (size_t)gridDim.x * blockDim.x) {
    uint32_t v[8];
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "l"(x + c * 16));
    uint4 o;
    o.x = __byte_perm(v[0], v[1], 0x7531); o.y = __byte_perm(v[2], v[3], 0x7531);
    o.z = __byte_perm(v[4], v[5], 0x7531); o.w = __byte_perm(v[6], v[7], 0x7531);
    *reinterpret_cast<uint4*>(out + c * 16) = o;
  }
}

int main() {
  const int L2 = 126 << 20;
  int shapes[][2] = {{4608, 3072}, {4608, 12288}};
  for (auto& sh : shapes) {
    const int M = sh[0], K = sh[1];
    const size_t in_b = (size_t)M * K * 2, out_b = (size_t)M * K;
    const int nbuf = (int)((3 * (size_t)L2) / in_b) + 2;
    std::vector<uint16_t*> xs(nbuf); std::vector<uint8_t*> os(nbuf);
    for (int i = 0; i < nbuf; ++i) { cudaMalloc(&xs[i], in_b); cudaMalloc(&os[i], out_b); cudaMemset(xs[i], 0x3f, in_b); }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
      for (int i = 0; i < nbuf; ++i) launch(i);
      cudaDeviceSynchronize();
      const int reps = 5;
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) for (int i = 0; i < nbuf; ++i) launch(i);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1e3 / (reps * nbuf);
      printf("M=%d K=%d %-34s %7.2f us  %6.0f GB/s (3 B/elem)  err=%s\n", M, K, name, us, (in_b + out_b) / us / 1e3, cudaGetErrorString(cudaGetLastError()));
    };
    for (int W : {3, 6, 12, 24}) for (int S : {2, 4, 8}) for (int cps : {4, 8}) {
      const size_t smem = (size_t)S * K * 2;
      if (W * 32 > 1024 || smem > 200 * 1024) continue;
      cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ring_kernel, W * 32, smem);
      if (occ < 1) continue;
      if (occ > cps) occ = cps;
      const int grid = 148 * occ;
      char nm[64]; snprintf(nm, 64, "ring W=%d S=%d ctas/sm=%d", W, S, occ);
      run(nm, [&](int i) { ring_kernel<<<grid, W * 32, smem>>>(xs[i], os[i], M, K, S); });
    }
    for (int g : {148 * 4, 148 * 8, 148 * 16}) {
      char nm[64]; snprintf(nm, 64, "direct grid=%d x256", g);
      run(nm, [&](int i) { direct_kernel<<<g, 256>>>(xs[i], os[i], M, K); });
    }
    for (int i = 0; i < nbuf; ++i) { cudaFree(xs[i]); cudaFree(os[i]); }
  }
  return 0;
}
