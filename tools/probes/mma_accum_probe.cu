// Probe: error of mma.sync.m16n8k16 bf16 x bf16 -> f32 (C = 0) against the
// exact sum, for 16-term dot products x . h with h = +-1 (regular Hadamard
// columns), on inputs with wide exponent spans.  Reports the max error in
// units of 2^-23 * max|x| (the bound the K1 certification would use) and
// the fraction of results that are not exactly the correctly rounded sum.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>
#include <random>

__global__ void probe(const __nv_bfloat16* X, const __nv_bfloat16* H, float* Y, int tiles) {
  // tile: 16 rows (dot products) x 16 K; B = H (16 x 8) twice (cols 0-7, 8-15)
  const int lane = threadIdx.x & 31;
  for (int t = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; t < tiles;
       t += gridDim.x * (blockDim.x / 32)) {
    const __nv_bfloat16* A = X + (size_t)t * 256;
    uint32_t a[4];
    const int r = lane / 4, c = 2 * (lane % 4);
    auto pk = [](const __nv_bfloat16* p) {
      return (uint32_t)__bfloat16_as_ushort(p[0]) | ((uint32_t)__bfloat16_as_ushort(p[1]) << 16);
    };
    a[0] = pk(A + r * 16 + c);
    a[1] = pk(A + (r + 8) * 16 + c);
    a[2] = pk(A + r * 16 + c + 8);
    a[3] = pk(A + (r + 8) * 16 + c + 8);
    for (int nb = 0; nb < 2; ++nb) {
      // B col-major 16 x 8: b0 = (k = c, c+1; n = r), b1 = (k = c+8, c+9; n = r)
      const int n = nb * 8 + r;
      uint32_t b0 = (uint32_t)__bfloat16_as_ushort(H[c * 16 + n]) |
                    ((uint32_t)__bfloat16_as_ushort(H[(c + 1) * 16 + n]) << 16);
      uint32_t b1 = (uint32_t)__bfloat16_as_ushort(H[(c + 8) * 16 + n]) |
                    ((uint32_t)__bfloat16_as_ushort(H[(c + 9) * 16 + n]) << 16);
      float d[4] = {0.f, 0.f, 0.f, 0.f};
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
      float* Yt = Y + (size_t)t * 256;
      Yt[r * 16 + nb * 8 + c] = d[0];
      Yt[r * 16 + nb * 8 + c + 1] = d[1];
      Yt[(r + 8) * 16 + nb * 8 + c] = d[2];
      Yt[(r + 8) * 16 + nb * 8 + c + 1] = d[3];
    }
  }
}

int main() {
  const int tiles = 1 << 16;
  const size_t n = (size_t)tiles * 256;
  std::vector<__nv_bfloat16> hx(n), hh(256);
  // regular Hadamard 16: sign(k, j) = (-1)^{popc(d & d>>1 & 0x55)} with d = k ^ j
  for (int k = 0; k < 16; ++k)
    for (int j = 0; j < 16; ++j) {
      unsigned d = k ^ j;
      hh[k * 16 + j] = __float2bfloat16(__builtin_popcount(d & (d >> 1) & 0x55u) & 1 ? -1.f : 1.f);
    }
  std::mt19937_64 rng(7);
  std::normal_distribution<double> g(0, 1);
  std::uniform_int_distribution<int> ex(-40, 40);
  for (size_t i = 0; i < n; ++i) {
    double v = g(rng);
    const int mode = (i / 256) % 4;  // tile families: gaussian, wide span, huge span, cancellation
    if (mode == 1) v = std::ldexp(v, ex(rng) / 4);
    if (mode == 2) v = std::ldexp(v, ex(rng));
    if (mode == 3 && (i % 2)) v = -std::ldexp(std::round(std::ldexp(v, 8)), -8);
    hx[i] = __float2bfloat16((float)v);
  }
  __nv_bfloat16 *dx, *dh;
  float* dy;
  cudaMalloc(&dx, n * 2);
  cudaMalloc(&dh, 512);
  cudaMalloc(&dy, n * 4);
  cudaMemcpy(dx, hx.data(), n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dh, hh.data(), 512, cudaMemcpyHostToDevice);
  probe<<<1024, 256>>>(dx, dh, dy, tiles);
  std::vector<float> hy(n);
  cudaMemcpy(hy.data(), dy, n * 4, cudaMemcpyDeviceToHost);
  double worst[4] = {0, 0, 0, 0};
  size_t inexact[4] = {0, 0, 0, 0}, cnt[4] = {0, 0, 0, 0}, notrn[4] = {0, 0, 0, 0};
  for (int t = 0; t < tiles; ++t) {
    const int mode = t % 4;
    for (int r = 0; r < 16; ++r) {
      double mx = 0;
      for (int k = 0; k < 16; ++k) mx = std::fmax(mx, std::fabs((double)__bfloat162float(hx[(size_t)t * 256 + r * 16 + k])));
      for (int j = 0; j < 16; ++j) {
        long double s = 0;  // exact (all terms are bf16)
        for (int k = 0; k < 16; ++k)
          s += (long double)__bfloat162float(hx[(size_t)t * 256 + r * 16 + k]) * __bfloat162float(hh[k * 16 + j]);
        const double got = hy[(size_t)t * 256 + r * 16 + j];
        const double err = std::fabs((double)(got - s));
        ++cnt[mode];
        if (got != (double)s) ++inexact[mode];
        if (got != (double)(float)s) ++notrn[mode];
        if (mx > 0) worst[mode] = std::fmax(worst[mode], err / (std::ldexp(mx, -23)));
      }
    }
  }
  const char* names[4] = {"gaussian", "span2^20", "span2^80", "cancel"};
  for (int m = 0; m < 4; ++m)
    printf("%-10s n=%zu inexact=%zu not_fp32_RN=%zu worst_err=%.3f x 2^-23*max|x|\n", names[m], cnt[m],
           inexact[m], notrn[m], worst[m]);
  return 0;
}
