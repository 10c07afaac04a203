// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the UNMODIFIED reference library
// (/root/reference/proj/core/src/*.cpp, compiled in place by
// oracle/Makefile into oracle/_ref/libconvrot_ref.so).  Used to validate the
// plain-C restatement (oracle/convrot_oracle.c), to generate the committed
// golden vectors (tests/golden/make_golden.py) and as the CPU arm of
// bench.py (--impl reference / cpu_baseline).  Never linked by the product.
//
// Exceptions map onto the same status numbering as the C-ABI
// (include/crt/convlinear4bit.h), following errors.hpp:9-67.
#include <cstdint>
#include <cstring>
#include <optional>
#include <string>
#include <vector>

#include "convrot/analysis.hpp"
#include "convrot/errors.hpp"
#include "convrot/hadamard.hpp"
#include "convrot/parallel.hpp"
#include "convrot/pipeline.hpp"
#include "convrot/quant.hpp"
#include "convrot/rng.hpp"
#include "convrot/tensorio.hpp"

using namespace convrot;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const InvalidOrderError& e) {
    g_err = e.what();
    return 1;
  } catch (const InvalidValueError& e) {
    g_err = e.what();
    return 2;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return 3;
  } catch (const CapacityError& e) {
    g_err = e.what();
    return 4;
  } catch (const FormatError& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

MatrixD to_matrix(const double* p, int64_t rows, int64_t cols) {
  return MatrixD(rows, cols, std::vector<double>(p, p + rows * cols));
}

RotationSpec spec_of(int kind, int group, int identity_tail) {
  RotationSpec s;
  s.kind = kind == 0 ? RotationKind::none
           : kind == 1 ? RotationKind::sylvester
                       : RotationKind::regular;
  s.group_size = group;
  s.identity_tail = identity_tail != 0;
  return s;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

unsigned ref_thread_count() { return thread_count(); }

int ref_regular(int n, int8_t* out) {
  return guarded([&] {
    HadamardMatrix h = regular(n);
    for (size_t i = 0; i < h.entries.size(); ++i)
      out[i] = static_cast<int8_t>(h.entries.data()[i]);
  });
}

int ref_sign_text_len(int n) { return n * (n + 1); }

int ref_group_rotate(const double* x, int64_t rows, int64_t cols, int kind,
                     int group, int identity_tail, double* out) {
  return guarded([&] {
    MatrixD r = group_rotate(to_matrix(x, rows, cols),
                             spec_of(kind, group, identity_tail));
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  });
}

int ref_compute_scales(const double* x, int64_t rows, int64_t cols, int bits,
                       double* scales) {
  return guarded([&] {
    auto s = compute_scales(to_matrix(x, rows, cols), QuantSpec{bits});
    std::memcpy(scales, s.data(), sizeof(double) * s.size());
  });
}

int ref_quantize(const double* x, int64_t rows, int64_t cols,
                 const double* scales, int bits, int8_t* codes) {
  return guarded([&] {
    QuantizedTensor q = quantize(to_matrix(x, rows, cols),
                                 std::vector<double>(scales, scales + rows),
                                 QuantSpec{bits});
    std::memcpy(codes, q.codes.data(), q.codes.size());
  });
}

// Row-wise CRT1 packed_i4 payload (tensorio.cpp:162-171).
int ref_pack_rows(const int8_t* codes, int64_t rows, int64_t cols,
                  uint8_t* out) {
  return guarded([&] {
    MatrixI8 m(rows, cols, std::vector<int8_t>(codes, codes + rows * cols));
    Tensor t = tensor_from_packed_i4(m);
    std::memcpy(out, t.payload.data(), t.payload.size());
  });
}

int ref_int_gemm(const int8_t* a, const int8_t* b, int64_t m, int64_t n,
                 int64_t k, int bits_a, int bits_b, int32_t* out) {
  return guarded([&] {
    MatrixI8 am(m, k, std::vector<int8_t>(a, a + m * k));
    MatrixI8 bm(n, k, std::vector<int8_t>(b, b + n * k));
    MatrixI32 r = int_gemm(am, bm, bits_a, bits_b);
    std::memcpy(out, r.data(), sizeof(int32_t) * r.size());
  });
}

// prepare_layer (pipeline.cpp:158-176); bias may be null.
int ref_prepare_layer(const double* w, int64_t n, int64_t k, const double* bias,
                      int kind, int group, int identity_tail, int bits,
                      int8_t* codes, double* scales) {
  return guarded([&] {
    std::optional<std::vector<double>> b;
    if (bias) b = std::vector<double>(bias, bias + n);
    PreparedLayer l = prepare_layer(to_matrix(w, n, k), b,
                                    spec_of(kind, group, identity_tail),
                                    QuantSpec{bits}, "ref");
    std::memcpy(codes, l.prepared_weights.codes.data(),
                l.prepared_weights.codes.size());
    std::memcpy(scales, l.prepared_weights.scales.data(), sizeof(double) * n);
  });
}

// prepare_layer + forward (pipeline.cpp:206-233).  Optional outputs:
// act_codes (M*K int8), act_scales (M), acc (M*N int32) recomputed with the
// same library calls forward() makes, in the same order.
int ref_forward(const double* x, int64_t m, int64_t k, const double* w,
                int64_t n, const double* bias, int kind, int group,
                int identity_tail, int bits_a, int bits_w, double* out,
                int8_t* act_codes, double* act_scales, int32_t* acc) {
  return guarded([&] {
    std::optional<std::vector<double>> b;
    if (bias) b = std::vector<double>(bias, bias + n);
    RotationSpec rot = spec_of(kind, group, identity_tail);
    PreparedLayer l = prepare_layer(to_matrix(w, n, k), b, rot,
                                    QuantSpec{bits_w}, "ref");
    MatrixD xm = to_matrix(x, m, k);
    LayerOutput o = forward(xm, l, QuantSpec{bits_a});
    std::memcpy(out, o.values.data(), sizeof(double) * o.values.size());
    if (act_codes || act_scales || acc) {
      MatrixD rotated = group_rotate(xm, rot);
      auto sa = compute_scales(rotated, QuantSpec{bits_a});
      QuantizedTensor q = quantize(rotated, sa, QuantSpec{bits_a});
      if (act_codes) std::memcpy(act_codes, q.codes.data(), q.codes.size());
      if (act_scales) std::memcpy(act_scales, sa.data(), sizeof(double) * m);
      if (acc) {
        MatrixI32 a = int_gemm(q.codes, l.prepared_weights.codes, bits_a, bits_w);
        std::memcpy(acc, a.data(), sizeof(int32_t) * a.size());
      }
    }
  });
}

// forward() against an already prepared layer given as codes/scales/bias.
int ref_forward_prepared(const double* x, int64_t m, int64_t k,
                         const int8_t* w_codes, const double* w_scales,
                         const double* bias, int64_t n, int kind, int group,
                         int identity_tail, int bits_a, int bits_w,
                         double* out) {
  return guarded([&] {
    PreparedLayer l;
    l.out_features = n;
    l.in_features = k;
    l.rotation = spec_of(kind, group, identity_tail);
    l.weight_quant = QuantSpec{bits_w};
    l.prepared_weights.rows = n;
    l.prepared_weights.cols = k;
    l.prepared_weights.bits = bits_w;
    l.prepared_weights.codes =
        MatrixI8(n, k, std::vector<int8_t>(w_codes, w_codes + n * k));
    l.prepared_weights.scales = std::vector<double>(w_scales, w_scales + n);
    if (bias) l.bias = std::vector<double>(bias, bias + n);
    LayerOutput o = forward(to_matrix(x, m, k), l, QuantSpec{bits_a});
    std::memcpy(out, o.values.data(), sizeof(double) * o.values.size());
  });
}

int ref_reference_forward(const double* x, const double* w, const double* bias,
                          int64_t m, int64_t n, int64_t k, double* out) {
  return guarded([&] {
    std::optional<std::vector<double>> b;
    if (bias) b = std::vector<double>(bias, bias + n);
    LayerOutput o = reference_forward(to_matrix(x, m, k), to_matrix(w, n, k), b);
    std::memcpy(out, o.values.data(), sizeof(double) * o.values.size());
  });
}

int ref_synth_outliers(int64_t rows, int64_t cols, int mode, double magnitude,
                       double fraction, uint64_t seed, double* out) {
  return guarded([&] {
    OutlierMode om = mode == 0 ? OutlierMode::rowwise
                     : mode == 1 ? OutlierMode::colwise
                                 : OutlierMode::gaussian;
    MatrixD x = synth_outliers(rows, cols, om, magnitude, fraction, seed);
    std::memcpy(out, x.data(), sizeof(double) * x.size());
  });
}

void ref_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed,
                         double* out) {
  Rng rng(seed);
  for (int64_t i = 0; i < rows * cols; ++i) out[i] = rng.next_gaussian();
}

void ref_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
  Rng rng(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = rng.next_u64();
}

// Prepared-layer persistence (pipeline.cpp:257-314), for the f2 row.
int ref_save_prepared_layer(const char* dir, const double* w, int64_t n,
                            int64_t k, const double* bias, int kind, int group,
                            int identity_tail, int bits) {
  return guarded([&] {
    std::optional<std::vector<double>> b;
    if (bias) b = std::vector<double>(bias, bias + n);
    PreparedLayer l = prepare_layer(to_matrix(w, n, k), b,
                                    spec_of(kind, group, identity_tail),
                                    QuantSpec{bits}, "ref");
    save_prepared_layer(dir, l);
  });
}

}  // extern "C"
