// Probe: semantics of tcgen05.cp.cta_group::1.128x128b.b8x16.b4x16_p64
// (smem 16 x 4-bit + 64-bit pad per row -> TMEM 16 x 8-bit per lane).
// Prints, for rows 0..3, the 16 source nibbles and the 16 destination bytes.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(uint32_t* out) {
  __shared__ __align__(1024) uint8_t src[128 * 16];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // source layout: K-major, no swizzle, core matrices of 8 rows x 16 B
  // (row r at (r/8)*128 + (r%8)*16); bytes 0..7 = 16 nibbles, 8..15 = pad 0xA5
  for (int r = tid; r < 128; r += blockDim.x) {
    uint8_t* row = src + (r / 8) * 128 + (r % 8) * 16;
    for (int b = 0; b < 8; ++b) {
      const int e0 = 2 * b, e1 = 2 * b + 1;
      const int n0 = (r + e0) & 0xF, n1 = (r + 3 * e1) & 0xF;
      row[b] = (uint8_t)(n0 | (n1 << 4));
    }
    for (int b = 8; b < 16; ++b) row[b] = 0xA5;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" :: "r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = tbase;
  if (tid == 0) {
    const uint32_t sa = smem_u32(src);
    uint64_t d = 0;
    d |= (uint64_t)((sa & 0x3FFFF) >> 4);      // start
    d |= (uint64_t)(128 >> 4) << 16;            // LBO (next K core matrix; unused)
    d |= (uint64_t)(128 >> 4) << 32;            // SBO: next 8-row group
    d |= (uint64_t)1 << 46;                     // version
    asm volatile("tcgen05.cp.cta_group::1.128x128b.b8x16.b4x16_p64 [%0], %1;" :: "r"(t), "l"(d));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)) : "memory");
  }
  // wait for the copy
  asm volatile("{\n.reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}" :: "r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(t + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  const int row = warp * 32 + lane;
  for (int i = 0; i < 4; ++i) out[row * 4 + i] = v[i];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" :: "r"(t));
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 128 * 16);
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  uint32_t h[128 * 4];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int r = 0; r < 4; ++r) {
    printf("row %d src nibbles:", r);
    for (int i = 0; i < 16; ++i) printf(" %x", i % 2 == 0 ? ((r + i) & 0xF) : ((r + 3 * i) & 0xF));
    printf("\n      dst bytes:  ");
    const uint8_t* b = reinterpret_cast<const uint8_t*>(h + r * 4);
    for (int i = 0; i < 16; ++i) printf(" %02x", b[i]);
    printf("\n");
  }
  return 0;
}
