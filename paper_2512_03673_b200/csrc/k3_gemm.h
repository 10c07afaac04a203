// k3_gemm.h -- host interface of K3 (W4A4 / W8A8 GEMM + dequant epilogue).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace crt {

// Prepared weight operand.  Codes are row-major per output channel (n) with
// a 16-byte aligned row pitch `ld`, so every 32-code K-chunk is one aligned
// 16-byte vector (the unit K3 stages).
//  * bits 8: int8 codes (the layer's own buffer).
//  * bits 4: ONE copy, owned here, in offset binary (nibble = code + 8, the
//    pack_int4 nibble order, K padded to 128 codes with code 0 = 0x8):
//    codes == codes_ob, ob = 1.  v3 feeds it to TMA 16U4 + tcgen05.cp
//    decompression as is; v1 / v2 / the generic kernel flip bit 3 of every
//    nibble (XOR 0x88) as they expand, and export converts on the way out.
struct K3Weights {
  const uint8_t* codes;
  const uint8_t* codes_ob;  // bits 4: the offset-binary codes (== codes); else null
  int64_t ld_ob;            // its row pitch: K rounded up to 128 codes (64 B; TMA 16U4 needs it)
  int64_t ld;
  int64_t N;
  int64_t K;
  int32_t bits;
  int32_t ob;               // codes are offset binary (bits 4)
};

struct K3Args {
  const uint8_t* a_codes;  // M x lda bytes
  int64_t lda;
  int32_t a_layout;        // 0: packed like pack_int4 (bits 4) / int8 (bits 8); 1: int8 per 4-bit code
  const int32_t* a_sums;   // layout 1: per-row sum of the codes (K1 rowsum)
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

// bits 4: builds the owned offset-binary copy from `codes` (reference
// pack_int4 layout, row pitch ldc; or already offset binary when src_ob);
// the caller may free `codes` afterwards (stream-ordered).  bits 8: refers
// to `codes`, which must outlive the weights.
cudaError_t k3_prepare_weights(const uint8_t* codes, int64_t ldc, int64_t N, int64_t K, int bits,
                               K3Weights* out, cudaStream_t st, int64_t* launches,
                               bool src_ob = false);
// Reference-layout copy of prepared 4-bit weights (XOR 0x88 back to two's
// complement): row r of dst gets (K + 1) / 2 bytes.
cudaError_t k3_export_w4(const K3Weights& w, uint8_t* dst, int64_t ldd, int64_t col_byte0,
                         int64_t row_bytes, cudaStream_t st, int64_t* launches);
void k3_free_weights(K3Weights* w);
cudaError_t k3_launch(const K3Args& a, cudaStream_t st, int64_t* launches);

// v2: persistent 2-SM (cta_group::2) kernel, TMA-staged packed tiles, A
// expanded into TMEM (k3_gemm_v2.cu).  W4A4 only.
bool k3_v2_supported(const K3Args& a);
// v3: hardware int4 expansion (tcgen05.cp decompress) of offset-binary
// weights into TMEM, int8 activation codes as the smem operand (k3_gemm_v3.cu).
bool k3_v3_supported(const K3Args& a);
cudaError_t k3_v3_launch(const K3Args& a, cudaStream_t st, int64_t* launches);
// v4: v3's kernel with the offset-binary weights TMA'd packed and expanded
// by expander warps into the shared-memory MMA operand (no tcgen05.cp);
// the default W4A4 path (k3_gemm_v4.cu).  CRT_K3_V3=1 selects v3.
bool k3_v4_supported(const K3Args& a);
cudaError_t k3_v4_launch(const K3Args& a, cudaStream_t st, int64_t* launches);
int k3_v4_pick_bt(int64_t M, int64_t N, int num_sms);  // token-tile width v4 uses
// M <= 8 (FLUX AdaLN): a weight-streaming CUDA-core GEMV on the same operands
// (k3_gemv.cu); CRT_K3_GEMV=0 keeps the tensor-core kernel.
bool k3_gemv_supported(const K3Args& a);
cudaError_t k3_gemv_launch(const K3Args& a, cudaStream_t st, int64_t* launches);
// Dev aid (crt_debug_k3_trace): when set, k3_v3 records clock64 stamps of
// pair 0's leader CTA (9 rows x 4096, see k3_gemm_v3.cu); null = off.
void set_k3_trace(unsigned long long* buf);
unsigned long long* k3_trace();
cudaError_t k3_v2_launch(const K3Args& a, cudaStream_t st, int64_t* launches);

}  // namespace crt
