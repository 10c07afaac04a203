// k1_rotate_quant.cu -- K1 host side: plan (fast vs exact kernel) + launch.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "k1_rotate_quant.h"

namespace crt {

template <bool F32, int BITS>
cudaError_t k1_dispatch(const K1Args& a, int c, int n0, cudaStream_t st, int64_t* l);
template <bool F32, int BITS>
cudaError_t k1_exact_launch(const K1Args& a, cudaStream_t st);

// ---------------------------------------------------------------------------
// Host launcher
// ---------------------------------------------------------------------------
K1Plan plan_k1(int64_t K, int64_t n0, int kind, bool identity_tail, bool f32, int bits,
               const void* x, int64_t ldx, const void* codes, int64_t ldc) {
  K1Plan p{};
  p.fast = false;
  const int esz = f32 ? 4 : 2;
  bool ok = K > 0 && K % 16 == 0 && (kind == kRotNone || kind == kRotRegular);
  int fast_n0 = kind == kRotNone ? 1 : (int)n0;
  ok = ok && (fast_n0 == 1 || fast_n0 == 4 || fast_n0 == 16 || fast_n0 == 64 || fast_n0 == 256);
  ok = ok && (kind == kRotNone || K % n0 == 0);
  ok = ok && ((uintptr_t)x % 32 == 0) && ((ldx * esz) % 32 == 0);
  const int cbytes = bits == 4 ? 8 : 16;
  ok = ok && ((uintptr_t)codes % cbytes == 0) && (ldc % cbytes == 0);
  (void)identity_tail;
  if (!ok) return p;
  const int64_t nchunks = K / 16;
  // pick C (chunks per lane) and W (warps per team): exact fit preferred,
  // W must divide 8 or be >= 8.
  int bestC = 0, bestW = 0;
  int64_t best_waste = INT64_MAX;
  for (int c : {4, 2, 6, 8}) {
    int64_t w = (nchunks + 32 * c - 1) / (32 * c);
    if (w > 8) continue;
    if (w < 8 && 8 % w != 0) {
      // round W up to a divisor of 8
      int64_t ww = w;
      while (8 % ww != 0) ++ww;
      w = ww;
    }
    int64_t waste = w * 32 * c - nchunks;
    if (waste < best_waste) {
      best_waste = waste;
      bestC = c;
      bestW = (int)w;
    }
  }
  if (bestC == 0) return p;
  p.fast = true;
  p.C = bestC;
  p.W = bestW;
  return p;
}

cudaError_t launch_k1(const K1Args& a, const K1Plan& p, bool f32, int bits, cudaStream_t st,
                      int64_t* launches) {
  if (p.fast) {
    K1Args b = a;
    b.team_warps = p.W;
    const int n0 = a.kind == kRotNone ? 1 : (int)a.group;
    if (f32) {
      return bits == 4 ? k1_dispatch<true, 4>(b, p.C, n0, st, launches)
                       : k1_dispatch<true, 8>(b, p.C, n0, st, launches);
    }
    return bits == 4 ? k1_dispatch<false, 4>(b, p.C, n0, st, launches)
                     : k1_dispatch<false, 8>(b, p.C, n0, st, launches);
  }
  cudaError_t e = f32 ? (bits == 4 ? k1_exact_launch<true, 4>(a, st) : k1_exact_launch<true, 8>(a, st))
                      : (bits == 4 ? k1_exact_launch<false, 4>(a, st) : k1_exact_launch<false, 8>(a, st));
  ++*launches;
  return e;
}

}  // namespace crt
