// Probe: what a CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B TMA box writes to smem
// (bytes per row, padding placement) and how many transaction bytes it
// completes.  Box {128 elements, 8 rows}, no swizzle.  Uses a bounded wait.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap map, uint8_t* out, int* status, uint32_t expect) {
  __shared__ __align__(1024) uint8_t buf[4096];
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = 0xEE;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar)), "r"(expect) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 :: "r"(smem_u32(buf)), "l"(&map), "r"(0), "r"(0), "r"(smem_u32(&bar)) : "memory");
    long long t0 = clock64();
    uint32_t done = 0;
    while (!done && clock64() - t0 < 200000000LL) {
      asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\nselp.u32 %0, 1, 0, P1;\n}" : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
    }
    *status = done;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int rows = 8, K = 256;  // 256 nibbles per row = 128 bytes packed
  uint8_t h[rows * K / 2];
  for (int r = 0; r < rows; ++r)
    for (int b = 0; b < K / 2; ++b) h[r * K / 2 + b] = (uint8_t)(((2 * b) & 0xF) | (((2 * b + 1) & 0xF) << 4)) ^ (r << 4);
  uint8_t *dg, *dout; int* dst;
  cudaMalloc(&dg, sizeof(h)); cudaMalloc(&dout, 4096); cudaMalloc(&dst, 4);
  cudaMemcpy(dg, h, sizeof(h), cudaMemcpyHostToDevice);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(K / 2)};
  cuuint32_t box[2] = {128, (cuuint32_t)rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_16U4_ALIGN16B, 2, dg, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  for (uint32_t expect : {512u, 1024u, 2048u}) {
    int st = -1;
    cudaMemset(dst, 0xFF, 4);
    probe<<<1, 128>>>(map, dout, dst, expect);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&st, dst, 4, cudaMemcpyDeviceToHost);
    printf("expect_tx=%u -> completed=%d (%s)\n", expect, st, cudaGetErrorString(e));
    if (st == 1) {
      uint8_t o[4096];
      cudaMemcpy(o, dout, 4096, cudaMemcpyDeviceToHost);
      for (int row = 0; row < 2; ++row) {
        printf("smem row %d (first 48 B at offset %d):", row, row * 128);
        for (int i = 0; i < 48; ++i) printf(" %02x", o[row * 128 + i]);
        printf("\n");
      }
      int last = 0; for (int i = 0; i < 4096; ++i) if (o[i] != 0xEE) last = i;
      printf("last written byte offset: %d\n", last);
    }
  }
  return 0;
}
