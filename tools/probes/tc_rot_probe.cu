// tc_rot_probe.cu -- accumulation error of tcgen05.mma kind::f16 (bf16 x bf16
// -> fp32 in TMEM) on the group rotation y = x * H16 (the regular Hadamard
// of order 16, entries +-1), against the exact sums (double, exact for these
// inputs).  Also validates the K1-TC operand layouts: A = 128 groups x 16
// bf16, K-major, 32-byte swizzle (what a TMA SWIZZLE_32B box writes); B = H16
// in the same layout; D = TMEM lanes 0..127 x 16 fp32 columns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_rot_probe tc_rot_probe.cu
// Prints, per input family, max |y_tc - y_exact| / max|x| in units of 2^-23
// and how many groups were exact.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <random>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// byte offset of element (row, k) (bf16, 16 per row) in a 32B-swizzled
// K-major tile: rows 32 B apart; within each 8-row (256 B) atom the two
// 16-byte halves of rows 4..7 are swapped (Swizzle<1,4,3>: addr bit 4 ^= bit 7)
__device__ __forceinline__ uint32_t sw32_off(int row, int k) {
  const uint32_t lin = (uint32_t)row * 32u + (uint32_t)k * 2u;
  return lin ^ (((lin >> 7) & 1u) << 4);
}
__device__ __forceinline__ uint64_t sw32_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);  // start address
  d |= (uint64_t)1 << 16;                    // LBO (unused for swizzled K-major)
  d |= (uint64_t)(256 >> 4) << 32;           // SBO: 8-row groups 256 B apart
  d |= (uint64_t)1 << 46;                    // version (sm100)
  d |= (uint64_t)6 << 61;                    // SWIZZLE_32B
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ bool regular_negative(uint32_t k, uint32_t j) {
  uint32_t d = k ^ j;
  return (__popc(d & (d >> 1) & 0x55555555u) & 1u) != 0;
}

__global__ void __launch_bounds__(128, 1) probe(const __nv_bfloat16* x, float* y, int groups) {
  __shared__ __align__(1024) uint8_t sa[128 * 32];
  __shared__ __align__(1024) uint8_t sb[16 * 32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // B = H16 (n = output j, k = input element): B[n][k] = H[k][n]
  for (int i = t; i < 256; i += 128) {
    const int n = i >> 4, k = i & 15;
    const __nv_bfloat16 v = __float2bfloat16(regular_negative(k, n) ? -1.f : 1.f);
    *reinterpret_cast<__nv_bfloat16*>(sb + sw32_off(n, k)) = v;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  uint32_t phase = 0;
  for (int g0 = 0; g0 < groups; g0 += 128) {
    // A: group t of the block
    const int g = g0 + t;
    for (int k = 0; k < 16; ++k)
      *reinterpret_cast<__nv_bfloat16*>(sa + sw32_off(t, k)) =
          g < groups ? x[(size_t)g * 16 + k] : __float2bfloat16(0.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\n"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
          "l"(sw32_desc(smem_u32(sa))), "l"(sw32_desc(smem_u32(sb))),
          "r"(idesc_bf16(128, 16)));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bar))
                   : "memory");
    }
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar)),
        "r"(phase)
        : "memory");
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (g < groups)
      for (int j = 0; j < 16; ++j) y[(size_t)g * 16 + j] = __uint_as_float(r[j]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
  }
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

static uint16_t bf16_bits(float f) {  // round to nearest even
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFF + ((u >> 16) & 1);
  return (uint16_t)(u >> 16);
}
static float bf16_val(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static bool neg(uint32_t k, uint32_t j) {
  uint32_t d = k ^ j;
  return (__builtin_popcount(d & (d >> 1) & 0x55555555u) & 1u) != 0;
}

int main() {
  const int G = 1 << 20;  // groups per family
  std::mt19937_64 rng(12345);
  std::normal_distribution<double> nd;
  std::uniform_real_distribution<double> ud(-1, 1);
  const char* fam[] = {"gaussian", "span 8 binades", "span 20 binades", "span 60 binades",
                       "cancellation (x, -x + tiny)", "equal magnitudes"};
  std::vector<uint16_t> hx((size_t)G * 16);
  std::vector<float> hy((size_t)G * 16);
  __nv_bfloat16* dx;
  float* dy;
  cudaMalloc(&dx, hx.size() * 2);
  cudaMalloc(&dy, hy.size() * 4);
  for (int f = 0; f < 6; ++f) {
    for (size_t i = 0; i < hx.size(); ++i) {
      double v;
      switch (f) {
        case 0: v = nd(rng); break;
        case 1: v = ud(rng) * ldexp(1.0, (int)(rng() % 8)); break;
        case 2: v = ud(rng) * ldexp(1.0, (int)(rng() % 20) - 10); break;
        case 3: v = ud(rng) * ldexp(1.0, (int)(rng() % 60) - 30); break;
        case 4: v = (i % 2) ? -bf16_val(hx[i - 1]) + ldexp(ud(rng), -20) : nd(rng) * 64; break;
        default: v = (rng() & 1 ? 1.0 : -1.0) * (1.0 + (double)(rng() % 128) / 128.0); break;
      }
      hx[i] = bf16_bits((float)v);
    }
    cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
    probe<<<1, 128>>>(dx, dy, G);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("CUDA error %s\n", cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(hy.data(), dy, hy.size() * 4, cudaMemcpyDeviceToHost);
    double worst = 0;
    long exact_groups = 0, fp32_exact_mismatch = 0;
    for (int g = 0; g < G; ++g) {
      double mx = 0;
      for (int k = 0; k < 16; ++k) mx = fmax(mx, fabs((double)bf16_val(hx[(size_t)g * 16 + k])));
      bool ex = true;
      for (int j = 0; j < 16; ++j) {
        double s = 0;
        for (int k = 0; k < 16; ++k) {
          const double v = bf16_val(hx[(size_t)g * 16 + k]);
          s += neg(k, j) ? -v : v;
        }
        const double err = fabs((double)hy[(size_t)g * 16 + j] - s);
        if (err != 0) ex = false;
        if (mx > 0) worst = fmax(worst, err / mx * 8388608.0);
        if ((double)(float)s == s && (double)hy[(size_t)g * 16 + j] != s) ++fp32_exact_mismatch;
      }
      exact_groups += ex;
    }
    printf("%-30s max |y_tc - y| / max|x| = %8.3f * 2^-23   exact groups %ld / %d   "
           "fp32-representable sums missed %ld\n",
           fam[f], worst, exact_groups, G, fp32_exact_mismatch);
  }
  return 0;
}
