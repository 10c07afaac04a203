// k3_gemm.h -- host interface of K3 (W4A4 / W8A8 GEMM + dequant epilogue).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace crt {

// Prepared weight operand.  Codes are row-major per output channel (n), in
// the reference pack_int4 nibble order (bits 4) or int8 (bits 8), with a
// 16-byte aligned row pitch `ld` so every 32-code K-chunk is one aligned
// 16-byte vector (the unit K3 stages).
struct K3Weights {
  const uint8_t* codes;
  int64_t ld;
  int64_t N;
  int64_t K;
  int32_t bits;
};

struct K3Args {
  const uint8_t* a_codes;  // M x lda bytes
  int64_t lda;
  const float* a_scales;   // M
  K3Weights w;             // by value (device pointers inside)
  const float* w_scales;   // N
  const float* bias;       // N or null
  int64_t M, N, K;
  int32_t bits;
  int32_t out_kind;        // 0 bf16, 1 f32, 2 int32 accumulators
  void* y;
  int64_t ldy;
};

cudaError_t k3_prepare_weights(const uint8_t* codes, int64_t ldc, int64_t N, int64_t K, int bits,
                               K3Weights* out, cudaStream_t st, int64_t* launches);
void k3_free_weights(K3Weights* w);
cudaError_t k3_launch(const K3Args& a, cudaStream_t st, int64_t* launches);

// v2: persistent 2-SM (cta_group::2) kernel, TMA-staged packed tiles, A
// expanded into TMEM (k3_gemm_v2.cu).  W4A4 only.
bool k3_v2_supported(const K3Args& a);
cudaError_t k3_v2_launch(const K3Args& a, cudaStream_t st, int64_t* launches);

}  // namespace crt
