// C++ host mirror (include/crt/convrot_b200.hpp) smoke tests, modelled on the
// reference's doctest cases.  `cpu` mode needs no GPU (host-only entry
// points and synchronous error reporting); `gpu` mode runs tiny forwards.
//   test_host_api cpu | gpu
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "crt/convrot_b200.hpp"

namespace cb = convrot_b200;
static int failures = 0;
#define EXPECT(c)                                                   \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                                   \
    }                                                               \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static void cpu_tests() {
  // H4 literal and sign text (test_hadamard.cpp:75-84, :233-236)
  std::vector<int8_t> h = cb::regular(4);
  std::string text;
  for (int r = 0; r < 4; ++r) {
    for (int c = 0; c < 4; ++c) text += h[r * 4 + c] > 0 ? '+' : '-';
    text += '\n';
  }
  EXPECT(text == "+++-\n++-+\n+-++\n-+++\n");
  // regular(16) column sums = 4 (test_hadamard.cpp:86-90)
  h = cb::regular(16);
  for (int c = 0; c < 16; ++c) {
    int s = 0;
    for (int r = 0; r < 16; ++r) s += h[r * 16 + c];
    EXPECT(s == 4);
  }
  // order rejection (test_hadamard.cpp:106-111)
  EXPECT(throws<cb::InvalidOrderError>([] { cb::regular(8); }));
  EXPECT(throws<cb::InvalidOrderError>([] { cb::regular(16384); }));
  // group_rotate divisibility / order errors are host-side (pipeline.cpp:27-50, :124-130)
  cb::RotationSpec bad{cb::RotationKind::regular, 8};
  EXPECT(throws<cb::InvalidOrderError>(
      [&] { cb::prepare_layer(nullptr, cb::DType::bf16, 4, 64, 64, nullptr, bad); }));
  cb::RotationSpec nodiv{cb::RotationKind::regular, 16};
  EXPECT(throws<cb::ShapeError>(
      [&] { cb::prepare_layer(nullptr, cb::DType::bf16, 4, 40, 40, nullptr, nodiv); }));
  cb::QuantSpec q3{3};
  EXPECT(throws<cb::InvalidValueError>(
      [&] { cb::prepare_layer(nullptr, cb::DType::bf16, 4, 64, 64, nullptr, nodiv, q3); }));
}

static void gpu_tests() {
  // 1x1 exact forward -> 49 (test_pipeline.cpp:154-162): x = 7, w = 7, no rotation
  float hx = 7.f, hw = 7.f, hb = 0.f;
  float *dx, *dw, *db, *dy;
  cudaMalloc(&dx, 4);
  cudaMalloc(&dw, 4);
  cudaMalloc(&db, 4);
  cudaMalloc(&dy, 4);
  cudaMemcpy(dx, &hx, 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, &hw, 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, &hb, 4, cudaMemcpyHostToDevice);
  cb::RotationSpec none{};
  cb::PreparedLayer L = cb::prepare_layer(dw, cb::DType::f32, 1, 1, 1, db, none);
  EXPECT(L.out_features() == 1 && L.in_features() == 1);
  cb::Workspace ws(1, 1);
  cb::forward(dx, cb::DType::f32, 1, 1, L, cb::QuantSpec{4}, cb::Out::f32, dy, 1, ws);
  float y1 = 0.f;
  cudaMemcpy(&y1, dy, 4, cudaMemcpyDeviceToHost);
  EXPECT(y1 == 49.f);
  // zero activations give the bias (test_pipeline.cpp:164-180)
  const int M = 8, K = 64, N = 16;
  std::vector<float> x(M * K, 0.f), w(N * K), b(N);
  for (int i = 0; i < N * K; ++i) w[i] = (float)((i * 37) % 11) - 5.f;
  for (int n = 0; n < N; ++n) b[n] = 0.25f * n - 1.f;
  float *x2, *w2, *b2, *y2;
  cudaMalloc(&x2, x.size() * 4);
  cudaMalloc(&w2, w.size() * 4);
  cudaMalloc(&b2, b.size() * 4);
  cudaMalloc(&y2, M * N * 4);
  cudaMemcpy(x2, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(w2, w.data(), w.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(b2, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
  cb::RotationSpec reg{cb::RotationKind::regular, 16};
  cb::PreparedLayer L2 = cb::prepare_layer(w2, cb::DType::f32, N, K, K, b2, reg);
  cb::Workspace ws2(M, K);
  cb::forward(x2, cb::DType::f32, M, K, L2, cb::QuantSpec{4}, cb::Out::f32, y2, N, ws2);
  ws2.status();
  std::vector<float> y(M * N);
  cudaMemcpy(y.data(), y2, y.size() * 4, cudaMemcpyDeviceToHost);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) EXPECT(y[m * N + n] == b[n]);
  // non-finite input -> InvalidValueError at the next status check (quant.cpp:16-18)
  x[3] = NAN;
  cudaMemcpy(x2, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  cb::forward(x2, cb::DType::f32, M, K, L2, cb::QuantSpec{4}, cb::Out::f32, y2, N, ws2);
  EXPECT(throws<cb::InvalidValueError>([&] { ws2.status(); }));
  ws2.status();  // cleared by the previous check
  // non-finite weights: prepare_layer throws itself (compute_scales)
  {
    std::vector<float> wn(w);
    wn[7] = INFINITY;
    float* wn2;
    cudaMalloc(&wn2, wn.size() * 4);
    cudaMemcpy(wn2, wn.data(), wn.size() * 4, cudaMemcpyHostToDevice);
    EXPECT(throws<cb::InvalidValueError>([&] {
      cb::prepare_layer(wn2, cb::DType::f32, N, K, K, b2, reg);
    }));
    cudaFree(wn2);
  }
  // int_gemm capacity precheck (pipeline.cpp:184-192) is host-side
  EXPECT(throws<cb::InvalidValueError>([&] {
    cb::forward(x2, cb::DType::f32, M, K, L2, cb::QuantSpec{5}, cb::Out::f32, y2, N, ws2);
  }));
  // row-parallel (K-sharded) forward, P = 2 shards run one after the other:
  // global row max, per-shard K1 + int32 partial GEMM, summed, dequant ==
  // the unsharded forward bit for bit
  for (int i = 0; i < M * K; ++i) x[i] = (float)((i * 29) % 17) - 8.f;
  cudaMemcpy(x2, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
  float* yref;
  cudaMalloc(&yref, M * N * 4);
  cb::forward(x2, cb::DType::f32, M, K, L2, cb::QuantSpec{4}, cb::Out::f32, yref, N, ws2);
  const int P = 2, Ks = K / P;
  double *am, *am_s;
  float *sa;
  int32_t *acc, *part, *sums;
  uint8_t* codes;
  cudaMalloc(&am, M * 8);
  cudaMalloc(&am_s, M * 8);
  cudaMalloc(&sa, M * 4);
  cudaMalloc(&acc, M * N * 4);
  cudaMalloc(&part, M * N * 4);
  cudaMalloc(&sums, M * 4);
  cudaMalloc(&codes, M * 64);
  std::vector<double> amax(M, 0.0), part_amax(M);
  for (int r = 0; r < P; ++r) {  // exact local maxima, MAX-reduced on the host here
    cb::rotated_row_absmax(x2 + r * Ks, cb::DType::f32, M, Ks, K, reg, am_s);
    cudaMemcpy(part_amax.data(), am_s, M * 8, cudaMemcpyDeviceToHost);
    for (int m = 0; m < M; ++m) amax[m] = std::max(amax[m], part_amax[m]);
  }
  cudaMemcpy(am, amax.data(), M * 8, cudaMemcpyHostToDevice);
  std::vector<int32_t> total(M * N, 0), p(M * N);
  cb::PreparedLayer shard0 = cb::prepare_layer_kshard(w2, cb::DType::f32, N, K, K, b2, reg,
                                                      cb::QuantSpec{4}, 0, P);
  for (int r = 0; r < P; ++r) {
    cb::PreparedLayer sh = cb::prepare_layer_kshard(w2, cb::DType::f32, N, K, K, b2, reg,
                                                    cb::QuantSpec{4}, r, P);
    cb::rotate_quantize_amax(x2 + r * Ks, cb::DType::f32, M, Ks, K, reg, am, cb::QuantSpec{4},
                             codes, 64, sa, nullptr, sums);
    cb::quant_gemm_i8(codes, 64, sa, sums, sh, M, cb::Out::i32_acc, part, N);
    cudaMemcpy(p.data(), part, M * N * 4, cudaMemcpyDeviceToHost);
    for (int i = 0; i < M * N; ++i) total[i] += p[i];
  }
  cudaMemcpy(acc, total.data(), M * N * 4, cudaMemcpyHostToDevice);
  cb::dequant(acc, N, M, sa, shard0, cb::Out::f32, y2, N);
  cudaDeviceSynchronize();
  std::vector<float> yr(M * N), yt(M * N);
  cudaMemcpy(yr.data(), yref, M * N * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(yt.data(), y2, M * N * 4, cudaMemcpyDeviceToHost);
  EXPECT(std::memcmp(yr.data(), yt.data(), M * N * 4) == 0);
  EXPECT(throws<cb::ShapeError>([&] {  // 64 / 3 shards do not divide K
    cb::prepare_layer_kshard(w2, cb::DType::f32, N, K, K, b2, reg, cb::QuantSpec{4}, 0, 3);
  }));
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  try {
    cpu_tests();
    if (gpu) gpu_tests();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "unexpected exception: %s\n", e.what());
    return 2;
  }
  std::printf("%s: %d failure(s)\n", gpu ? "cpu+gpu" : "cpu", failures);
  return failures ? 1 : 0;
}
