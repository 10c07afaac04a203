// k1_rotate_quant.cu -- K1 host side: plan (fast vs exact kernel) + launch.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "k1_rotate_quant.h"
#include <stdio.h>
#include <atomic>

namespace crt {

template <bool F32, int BITS>
cudaError_t k1_dispatch(const K1Args& a, int n0, cudaStream_t st, int64_t* l);
template <bool F32, int BITS>
cudaError_t k1_exact_launch(const K1Args& a, cudaStream_t st);

namespace {
std::atomic<unsigned long long*> g_trace{nullptr};
}
void set_k1_trace(unsigned long long* buf) { g_trace.store(buf); }
unsigned long long* k1_trace() { return g_trace.load(); }

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
  // Team of W warps per row with C (even) chunks per lane: about 6 chunks
  // (96 elements) per lane amortises the per-row work (reductions, scale,
  // certification).  Single-pass kernels hold C <= 8 chunks in registers
  // with W <= 6 (one 192-thread CTA); wider rows use the rolled two-pass
  // kernel (W <= 8).
  int64_t W = (nchunks + 191) / 192;
  if (W < 1) W = 1;
  int64_t C = (nchunks + 32 * W - 1) / (32 * W);
  C += C & 1;
  if (C < 2) C = 2;
  if (W > 6) {
    W = (nchunks + 255) / 256;
    C = 8;
    if (W > 6) {  // rolled kernel
      W = 8;
      C = (nchunks + 255) / 256;
      C += C & 1;
      if (C <= 8) C = 10;
    }
  }
  int bestC = (int)C, bestW = (int)W;
  // dev aid: CRT_K1_PLAN="W,C" forces the team shape (single-pass when W <= 6,
  // C <= 8 and C even) -- used by tools/k1_sweep.sh
  static const char* force = getenv("CRT_K1_PLAN");
  if (force) {
    int fw = 0, fc = 0;
    if (sscanf(force, "%d,%d", &fw, &fc) == 2 && fw >= 1 && fw <= 8 && fc >= 2 && fc % 2 == 0 &&
        (int64_t)fw * 32 * fc >= nchunks) {
      bestW = fw;
      bestC = fc;
    }
  }
  p.fast = true;
  p.C = bestC;
  p.W = bestW;
  return p;
}

cudaError_t launch_k1(const K1Args& a, const K1Plan& p, bool f32, int bits, cudaStream_t st,
                      int64_t* launches) {
  if (p.fast) {
    K1Args b = a;
    b.trace = k1_trace();
    b.team_warps = p.W;
    b.chunks = p.C;
    const int n0 = a.kind == kRotNone ? 1 : (int)a.group;
    if (f32) {
      return bits == 4   ? k1_dispatch<true, 4>(b, n0, st, launches)
             : bits == 5 ? k1_dispatch<true, 5>(b, n0, st, launches)
                         : k1_dispatch<true, 8>(b, n0, st, launches);
    }
    return bits == 4   ? k1_dispatch<false, 4>(b, n0, st, launches)
           : bits == 5 ? k1_dispatch<false, 5>(b, n0, st, launches)
                       : k1_dispatch<false, 8>(b, n0, st, launches);
  }
  cudaError_t e =
      f32 ? (bits == 4 ? k1_exact_launch<true, 4>(a, st)
             : bits == 5 ? k1_exact_launch<true, 5>(a, st) : k1_exact_launch<true, 8>(a, st))
          : (bits == 4 ? k1_exact_launch<false, 4>(a, st)
             : bits == 5 ? k1_exact_launch<false, 5>(a, st) : k1_exact_launch<false, 8>(a, st));
  ++*launches;
  return e;
}

}  // namespace crt
