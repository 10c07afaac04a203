// k3_gemv.cu -- K3 for a handful of tokens (M <= 8: the FLUX AdaLN
// modulation linears run at M = 1): int_gemm (pipeline.cpp:178-204) + the
// dequant of forward (pipeline.cpp:224-230) as a weight-streaming GEMV on
// the CUDA cores.  The 2-SM tensor-core kernel (k3_gemm_v4.cu) pays its
// whole per-tile pipeline for one token (13.5 us for a 3072 x 18432 layer
// whose 28 MB of packed weights HBM streams in ~4.5 us); here every weight
// byte is read once, expanded in registers and dotted with the (L1-resident)
// int8 activation codes by DP4A.
//
// One warp per output channel and token group: lane l reads 16-byte chunks
// l, l + 32, ... of the channel's offset-binary packed row (nibble n = w + 8,
// pack_int4 order), expands each to 32 bytes n (as v4's expanders do) and
// accumulates sum(n * a) over the matching 32 activation codes of every
// token; a warp reduction gives D = sum(w * a) + 8 S_a, and the dequant is
// v4's epilogue expression, so outputs are bit-identical to the tensor-core
// path.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "k3_gemm.h"

namespace crt {
namespace {

constexpr int GV_MAXM = 8;
constexpr int GV_WARPS = 8;  // channels per CTA

__device__ __forceinline__ void gv_expand8(uint32_t w, uint32_t& lo4, uint32_t& hi4) {
  const uint32_t ev = w & 0x0F0F0F0Fu;         // n[0], n[2], n[4], n[6]
  const uint32_t od = (w >> 4) & 0x0F0F0F0Fu;  // n[1], n[3], n[5], n[7]
  lo4 = __byte_perm(ev, od, 0x5140);
  hi4 = __byte_perm(ev, od, 0x7362);
}

// dot products of one channel's packed row with the M token rows: this
// lane's share (chunks lane, lane + 32, ...), given its loaded chunks
template <int MT>
__device__ __forceinline__ void gv_dot(const K3Args& a, int64_t c, uint4 p, int (&acc)[MT]) {
  uint32_t o[8];
  gv_expand8(p.x, o[0], o[1]);
  gv_expand8(p.y, o[2], o[3]);
  gv_expand8(p.z, o[4], o[5]);
  gv_expand8(p.w, o[6], o[7]);
  const bool full = (c + 1) * 32 <= a.K;
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    if (m >= a.M) break;
    const uint8_t* ar = a.a_codes + m * a.lda + c * 32;
    uint32_t av[8];
    if (full) {
      const uint4 t0 = __ldg(reinterpret_cast<const uint4*>(ar));
      const uint4 t1 = __ldg(reinterpret_cast<const uint4*>(ar) + 1);
      av[0] = t0.x, av[1] = t0.y, av[2] = t0.z, av[3] = t0.w;
      av[4] = t1.x, av[5] = t1.y, av[6] = t1.z, av[7] = t1.w;
    } else {  // the row's last, partial chunk: codes beyond K count as 0
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int64_t k = c * 32 + q * 4 + b;
          if (k < a.K) v |= (uint32_t)ar[q * 4 + b] << (8 * b);
        }
        av[q] = v;
      }
    }
    int s = acc[m];
#pragma unroll
    for (int q = 0; q < 8; ++q) s = __dp4a((int)o[q], (int)av[q], s);
    acc[m] = s;
  }
}

template <int MT>
__device__ __forceinline__ void gv_finish(const K3Args& a, int64_t n, int lane, int (&acc)[MT]) {
  const float sw = a.w_scales[n];
  const float bn = a.bias ? a.bias[n] : 0.f;
#pragma unroll
  for (int m = 0; m < MT; ++m) {
    if (m >= a.M) break;
    int s = acc[m];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
    if (lane != 0) continue;
    const int v = s - 8 * a.a_sums[m];  // D = sum(w a) + 8 S_a
    if (a.out_kind == 2) {
      reinterpret_cast<int32_t*>(a.y)[m * a.ldy + n] = v;
    } else {
      // v4's epilogue expression (v exact in fp32: |v| <= 49 K < 2^24)
      const float o = fmaf((float)v * a.a_scales[m], sw, bn);
      if (a.out_kind == 0)
        reinterpret_cast<__nv_bfloat16*>(a.y)[m * a.ldy + n] = __float2bfloat16_rn(o);
      else
        reinterpret_cast<float*>(a.y)[m * a.ldy + n] = o;
    }
  }
}

// One warp per output channel (a short-lived warp per channel measured as
// fast as persistent warps taking two channels per pass: 7.8 vs 8.3 us at
// 3072 x 18432).
template <int MT>
__global__ void __launch_bounds__(GV_WARPS * 32) k3_gemv_kernel(K3Args a) {
  const int lane = threadIdx.x & 31;
  const int64_t n = (int64_t)blockIdx.x * GV_WARPS + (threadIdx.x >> 5);
  griddep_launch();
  griddep_wait();
  if (n >= a.N) return;
  const uint4* wrow = reinterpret_cast<const uint4*>(a.w.codes_ob + n * a.w.ld_ob);
  const int64_t nch = (a.K + 31) / 32;  // 32-code chunks (the packed row is padded to 128 codes)
  int acc[MT];
#pragma unroll
  for (int m = 0; m < MT; ++m) acc[m] = 0;
  for (int64_t c = lane; c < nch; c += 32) gv_dot<MT>(a, c, __ldg(wrow + c), acc);
  gv_finish<MT>(a, n, lane, acc);
}

}  // namespace

bool k3_gemv_supported(const K3Args& a) {
  static const bool off = [] {  // A/B: CRT_K3_GEMV=0 keeps the tensor-core kernel
    const char* e = getenv("CRT_K3_GEMV");
    return e && e[0] == '0';
  }();
  if (off || a.bits != 4 || a.a_layout != 1 || !a.a_sums || !a.w.codes_ob) return false;
  if (a.M < 1 || a.M > GV_MAXM || a.N < 1 || a.K < 1 || a.K > 342392) return false;  // 49 K < 2^24
  return (uintptr_t)a.a_codes % 16 == 0 && a.lda % 16 == 0 && (uintptr_t)a.w.codes_ob % 16 == 0 &&
         a.w.ld_ob % 64 == 0;
}

cudaError_t k3_gemv_launch(const K3Args& a, cudaStream_t st, int64_t* launches) {
  const dim3 grid((unsigned)((a.N + GV_WARPS - 1) / GV_WARPS));
  const dim3 block(GV_WARPS * 32);
  cudaError_t e;
  if (a.M == 1) e = launch_pdl(k3_gemv_kernel<1>, grid, block, 0, st, a);
  else if (a.M <= 2) e = launch_pdl(k3_gemv_kernel<2>, grid, block, 0, st, a);
  else if (a.M <= 4) e = launch_pdl(k3_gemv_kernel<4>, grid, block, 0, st, a);
  else e = launch_pdl(k3_gemv_kernel<8>, grid, block, 0, st, a);
  ++*launches;
  return e;
}

}  // namespace crt
