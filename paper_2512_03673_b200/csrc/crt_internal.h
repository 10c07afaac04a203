// crt_internal.h -- library-internal state shared by the C-ABI translation
// units (crt_api.cu: single-GPU entry points; crt_tp.cu: tensor-parallel
// entry points over NCCL).  Not installed; the public surface is
// include/crt/convlinear4bit.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/crt/convlinear4bit.h"
#include "k3_gemm.h"

// A prepared layer (reference PreparedLayer, pipeline.hpp:55-65): immutable
// after prepare, shareable across threads and streams.
struct crt_layer {
  crt_layer_desc desc;
  int64_t n_total;      // N of the full layer (== desc.out_features unless sharded)
  int64_t row_offset;   // first output channel of this shard
  uint8_t* codes;       // bits 8: N x ldc int8 codes (K3's operand); bits 4: null --
                        // the only copy is tiles' offset-binary one
  int64_t ldc;          // reference-layout row pitch (scratch / export layout)
  float* s32;           // N
  double* s64;          // N
  float* bias;          // N or null
  crt::K3Weights tiles; // K3 operand layout
  int32_t tp_mode;      // 0, CRT_TP_COLUMN or CRT_TP_ROW (crt_tp_layer_prepare)
  int32_t tp_rank, tp_nranks;
  int64_t k_total;      // CRT_TP_ROW: in_features of the full layer
};

// Forward scratch owned by the caller (no hidden allocation on the forward
// path) plus its own device error word: a forward on one workspace never
// reports, or clears, another caller's non-finite input.
struct crt_workspace {
  int64_t max_m, max_k;
  uint8_t* codes;
  float* s32;
  int32_t* rowsum;
  int* err;
  void* tp_buf;      // crt_tp_forward scratch (gathered shards / row maxima +
  size_t tp_bytes;   // int32 partials), grown on first use, owned here
};

// NVTX ranges around the C-ABI entry points (nvtx3 is header-only; the
// ranges cost one branch unless CRT_NVTX=1 and a tool such as nsys or ncu
// --nvtx is attached).  SURVEY.md 5 tracing.
#include <nvtx3/nvToolsExt.h>
namespace crt_detail {
bool nvtx_on();
struct NvtxRange {
  bool on;
  explicit NvtxRange(const char* name) : on(nvtx_on()) {
    if (on) nvtxRangePushA(name);
  }
  ~NvtxRange() {
    if (on) nvtxRangePop();
  }
};
}  // namespace crt_detail

namespace crt_detail {
// ws->tp_buf with at least `bytes` (grows once: synchronises `st`, frees,
// reallocates); null on failure.
void* workspace_tp_scratch(crt_workspace* ws, size_t bytes, cudaStream_t st);
}  // namespace crt_detail

namespace crt_detail {

extern thread_local std::string g_err;
extern std::atomic<int64_t> g_launches;

crt_status fail(crt_status st, const std::string& msg);
crt_status cuda_fail(cudaError_t e, const char* where);
int* device_error_word();
crt_status resolve_rotation(const crt_rotation_spec* rot, int64_t cols, int64_t* group,
                            int64_t* rot_cols);
// K1 launch (bits 4 packed, 5 int8 codes + row sums, 8 int8).  codes may be
// null when only amax is wanted (amax-only: no code stores).  err: the
// device error word to flag non-finite input in (null: the device's).
crt_status run_k1(const void* x, int32_t x_dtype, int64_t M, int64_t K, int64_t ldx,
                  const crt_rotation_spec* rot, int32_t bits, uint8_t* codes, int64_t ldc,
                  float* s32, double* s64, cudaStream_t st, double* amax = nullptr,
                  int32_t* rowsum = nullptr, const double* amax_in = nullptr, int* err = nullptr);
crt_status prepare_impl(const crt_layer_desc* d, const void* w, int64_t ldw, const float* bias,
                        int32_t rank, int32_t nranks, cudaStream_t st, crt_layer** out);
crt_status quant_gemm_impl(const uint8_t* a_codes, int64_t lda, const float* a_scales,
                           const int32_t* a_sums, int32_t layout, int32_t bits_a,
                           const crt_layer* L, int64_t M, int32_t out_kind, void* y, int64_t ldy,
                           void* stream);

}  // namespace crt_detail
