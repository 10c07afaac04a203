// convrot_b200.hpp -- C++ host mirror of the reference's ConvLinear4bit API
// (/root/reference/proj/core/include/convrot/{pipeline,quant,hadamard}.hpp)
// over the C-ABI in convlinear4bit.h.  Header-only; link
// paper_2512_03673_b200/libconvrot_b200.so.
//
// Same names, argument meaning and error classes as the reference
// (errors.hpp:9-67), but buffers live on the GPU: pointers are device
// pointers, work is ordered on a CUDA stream (passed as void*, nullptr =
// legacy stream) and nothing here synchronises except DeviceStatus().
#ifndef CRT_CONVROT_B200_HPP_
#define CRT_CONVROT_B200_HPP_

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "convlinear4bit.h"

namespace convrot_b200 {

// ---- error taxonomy (errors.hpp:9-67) --------------------------------------
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class InvalidOrderError : public Error { public: using Error::Error; };
class InvalidValueError : public Error { public: using Error::Error; };
class ShapeError : public Error { public: using Error::Error; };
class CapacityError : public Error { public: using Error::Error; };
class FormatError : public Error { public: using Error::Error; };
class CudaError : public Error { public: using Error::Error; };
class UnsupportedError : public Error { public: using Error::Error; };

inline void check(crt_status s) {
  if (s == CRT_OK) return;
  const std::string m = crt_last_error();
  switch (s) {
    case CRT_ERR_INVALID_ORDER: throw InvalidOrderError(m);
    case CRT_ERR_INVALID_VALUE: throw InvalidValueError(m);
    case CRT_ERR_SHAPE: throw ShapeError(m);
    case CRT_ERR_CAPACITY: throw CapacityError(m);
    case CRT_ERR_FORMAT: throw FormatError(m);
    case CRT_ERR_CUDA: throw CudaError(m);
    case CRT_ERR_UNSUPPORTED: throw UnsupportedError(m);
    default: throw Error(m);
  }
}

// ---- value types (pipeline.hpp:14-30, quant.hpp:15-20) -------------------
enum class RotationKind { none = CRT_ROT_NONE, sylvester = CRT_ROT_SYLVESTER, regular = CRT_ROT_REGULAR };

struct RotationSpec {
  RotationKind kind = RotationKind::none;
  int group_size = 0;  // 0 = global (one block over K)
  uint64_t seed = 0;
  bool identity_tail = false;
  crt_rotation_spec c() const {
    return crt_rotation_spec{static_cast<int32_t>(kind), group_size, seed, identity_tail ? 1 : 0};
  }
};

struct QuantSpec {
  int bits = 4;
  int qmax() const { return (1 << (bits - 1)) - 1; }
};

enum class DType { bf16 = CRT_DTYPE_BF16, f32 = CRT_DTYPE_F32 };
enum class Out { bf16 = CRT_OUT_BF16, f32 = CRT_OUT_F32, i32_acc = CRT_OUT_I32_ACC };

// ---- a1: regular(n) (hadamard.cpp:91-106) -> host n x n signs -------------
inline std::vector<int8_t> regular(int n) {
  std::vector<int8_t> h(n > 0 && n <= 4096 ? (size_t)n * n : 1);
  check(crt_regular_hadamard(n, h.data()));
  return h;
}

// ---- K1: group_rotate + compute_scales + quantize + pack_int4 ------------
// (pipeline.cpp:111-151, quant.cpp:10-81).  Device buffers.
inline void rotate_quantize(const void* x, DType dt, int64_t m, int64_t k, int64_t ldx,
                            const RotationSpec& rot, QuantSpec q, uint8_t* codes,
                            int64_t ld_codes, float* scales_f32, double* scales_f64 = nullptr,
                            void* stream = nullptr) {
  const crt_rotation_spec r = rot.c();
  check(crt_rotate_quant(x, static_cast<int32_t>(dt), m, k, ldx, &r, q.bits, codes, ld_codes,
                         scales_f32, scales_f64, stream));
}

// ---- a7: PreparedLayer / prepare_layer (pipeline.hpp:55-65, .cpp:158-176)
class PreparedLayer {
 public:
  PreparedLayer() = default;
  explicit PreparedLayer(crt_layer* h) : h_(h) {}
  PreparedLayer(PreparedLayer&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  PreparedLayer& operator=(PreparedLayer&& o) noexcept {
    reset();
    h_ = std::exchange(o.h_, nullptr);
    return *this;
  }
  PreparedLayer(const PreparedLayer&) = delete;
  PreparedLayer& operator=(const PreparedLayer&) = delete;
  ~PreparedLayer() { reset(); }

  const crt_layer* handle() const { return h_; }
  crt_layer_desc desc() const {
    crt_layer_desc d{};
    check(crt_layer_info(h_, &d));
    return d;
  }
  int64_t out_features() const { return desc().out_features; }
  int64_t in_features() const { return desc().in_features; }

 private:
  void reset() {
    if (h_) crt_layer_destroy(h_);
    h_ = nullptr;
  }
  crt_layer* h_ = nullptr;
};

// w: device N x K (row stride ldw elements), bias: device fp32 N or nullptr.
inline PreparedLayer prepare_layer(const void* w, DType dt, int64_t n, int64_t k, int64_t ldw,
                                   const float* bias, const RotationSpec& rot,
                                   QuantSpec wq = {}, void* stream = nullptr) {
  crt_layer_desc d{n, k, rot.c(), wq.bits, static_cast<int32_t>(dt)};
  crt_layer* h = nullptr;
  check(crt_layer_prepare(&d, w, ldw, bias, stream, &h));
  return PreparedLayer(h);
}

// Column-parallel shard: output channels [r*N/P, (r+1)*N/P).
inline PreparedLayer prepare_layer_shard(const void* w, DType dt, int64_t n, int64_t k,
                                         int64_t ldw, const float* bias, const RotationSpec& rot,
                                         QuantSpec wq, int rank, int nranks,
                                         void* stream = nullptr) {
  crt_layer_desc d{n, k, rot.c(), wq.bits, static_cast<int32_t>(dt)};
  crt_layer* h = nullptr;
  check(crt_layer_prepare_shard(&d, w, ldw, bias, rank, nranks, stream, &h));
  return PreparedLayer(h);
}

// Row-parallel shard (SURVEY.md 8e "K", 8f row f3): input columns
// [r*K/P, (r+1)*K/P) of the full layer's codes, full-K channel scales.
inline PreparedLayer prepare_layer_kshard(const void* w, DType dt, int64_t n, int64_t k,
                                          int64_t ldw, const float* bias,
                                          const RotationSpec& rot, QuantSpec wq, int rank,
                                          int nranks, void* stream = nullptr) {
  crt_layer_desc d{n, k, rot.c(), wq.bits, static_cast<int32_t>(dt)};
  crt_layer* h = nullptr;
  check(crt_layer_prepare_kshard(&d, w, ldw, bias, rank, nranks, stream, &h));
  return PreparedLayer(h);
}

// ---- forward workspace (no hidden allocation on the forward path) --------
class Workspace {
 public:
  Workspace(int64_t max_m, int64_t max_k) { check(crt_workspace_create(max_m, max_k, &h_)); }
  Workspace(const Workspace&) = delete;
  Workspace& operator=(const Workspace&) = delete;
  ~Workspace() {
    if (h_) crt_workspace_destroy(h_);
  }
  crt_workspace* handle() const { return h_; }
  // Raises InvalidValueError if a forward run with this workspace saw a
  // non-finite input (compute_scales, quant.cpp:16-18); its own error word.
  // Synchronises the stream.
  void status(void* stream = nullptr, bool reset = true) {
    check(crt_workspace_status(h_, stream, reset ? 1 : 0));
  }

 private:
  crt_workspace* h_ = nullptr;
};

// ---- a8 + a9: int_gemm + dequant (pipeline.cpp:178-233) ------------------
inline void quant_gemm(const uint8_t* a_codes, int64_t lda, const float* a_scales, QuantSpec aq,
                       const PreparedLayer& layer, int64_t m, Out out, void* y, int64_t ldy,
                       void* stream = nullptr) {
  check(crt_quant_gemm(a_codes, lda, a_scales, aq.bits, layer.handle(), m,
                       static_cast<int32_t>(out), y, ldy, stream));
}

// W4A4 fast path pieces: K1 with int8-stored codes + per-row code sums, and
// the hardware-expansion GEMM (K3 v3) that consumes them.
inline void rotate_quantize_i8(const void* x, DType dt, int64_t m, int64_t k, int64_t ldx,
                               const RotationSpec& rot, uint8_t* codes, int64_t ld_codes,
                               float* scales_f32, int32_t* code_sums, void* stream = nullptr) {
  const crt_rotation_spec r = rot.c();
  check(crt_rotate_quant_i8(x, static_cast<int32_t>(dt), m, k, ldx, &r, codes, ld_codes,
                            scales_f32, code_sums, stream));
}
inline void quant_gemm_i8(const uint8_t* a_codes, int64_t lda, const float* a_scales,
                          const int32_t* code_sums, const PreparedLayer& layer, int64_t m,
                          Out out, void* y, int64_t ldy, void* stream = nullptr) {
  check(crt_quant_gemm_i8(a_codes, lda, a_scales, code_sums, layer.handle(), m,
                          static_cast<int32_t>(out), y, ldy, stream));
}

// Row-parallel pieces: K1 with the global per-row max (after a MAX
// all-reduce of every rank's crt_rotated_row_absmax), and the dequant of the
// SUM-all-reduced int32 accumulators.
inline void rotated_row_absmax(const void* x, DType dt, int64_t m, int64_t k, int64_t ldx,
                               const RotationSpec& rot, double* amax_rows,
                               void* stream = nullptr) {
  const crt_rotation_spec r = rot.c();
  check(crt_rotated_row_absmax(x, static_cast<int32_t>(dt), m, k, ldx, &r, amax_rows, stream));
}
inline void rotate_quantize_amax(const void* x, DType dt, int64_t m, int64_t k, int64_t ldx,
                                 const RotationSpec& rot, const double* amax_rows, QuantSpec aq,
                                 uint8_t* codes, int64_t ld_codes, float* scales_f32,
                                 double* scales_f64, int32_t* code_sums,
                                 void* stream = nullptr) {
  const crt_rotation_spec r = rot.c();
  check(crt_rotate_quant_amax(x, static_cast<int32_t>(dt), m, k, ldx, &r, amax_rows, aq.bits,
                              codes, ld_codes, scales_f32, scales_f64, code_sums, stream));
}
inline void dequant(const int32_t* acc, int64_t ld_acc, int64_t m, const float* a_scales,
                    const PreparedLayer& layer, Out out, void* y, int64_t ldy,
                    void* stream = nullptr) {
  check(crt_dequant(acc, ld_acc, m, a_scales, layer.handle(), static_cast<int32_t>(out), y, ldy,
                    stream));
}

// forward(x, layer, aq) on device buffers: K1 then K3.
inline void forward(const void* x, DType dt, int64_t m, int64_t ldx, const PreparedLayer& layer,
                    QuantSpec aq, Out out, void* y, int64_t ldy, Workspace& ws,
                    void* stream = nullptr) {
  check(crt_forward(layer.handle(), x, static_cast<int32_t>(dt), m, ldx, aq.bits,
                    static_cast<int32_t>(out), y, ldy, ws.handle(), stream));
}

// Raises InvalidValueError if a free-standing K1 call (rotate_quantize*,
// rotated_row_absmax) saw a non-finite input (compute_scales,
// quant.cpp:16-18).  Forwards report through Workspace::status;
// prepare_layer throws by itself.  Synchronises the stream.
inline void device_status(void* stream = nullptr, bool reset = true) {
  check(crt_device_status(stream, reset ? 1 : 0));
}

}  // namespace convrot_b200

#endif  // CRT_CONVROT_B200_HPP_
