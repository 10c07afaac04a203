// crt_api.cu -- the C-ABI (include/crt/convlinear4bit.h): host-side
// validation with the reference's error behaviour, resource ownership, and
// the launches of K1 (rotate+quant), K2 (weight prep) and K3 (GEMM).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/crt/convlinear4bit.h"
#include "common.cuh"
#include "crt_internal.h"
#include "k1_rotate_quant.h"
#include "k3_gemm.h"

namespace crt_detail {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

// One device error word per device for the free-standing K1 entry points
// (crt_rotate_quant*, crt_device_status), lazily allocated under a mutex,
// never freed.  Forward calls use their workspace's own word and layer
// preparation a per-call word (crt_workspace_status, prepare_impl).
int* device_error_word() {
  static int* words[64] = {nullptr};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!words[dev]) {
    int* p = nullptr;
    if (cudaMalloc(&p, sizeof(int)) != cudaSuccess) return nullptr;
    const int zero = 0;
    if (cudaMemcpy(p, &zero, sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    words[dev] = p;
  }
  return words[dev];
}

bool nvtx_on() {
  static const bool on = [] {
    const char* e = getenv("CRT_NVTX");
    return e && e[0] == '1';
  }();
  return on;
}

crt_status fail(crt_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

crt_status cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return CRT_ERR_CUDA;
}

bool is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }
bool is_pow4(int64_t n) { return is_pow2(n) && (n & 0x5555555555555555LL) != 0; }

// Resolve and validate a rotation spec against a width the way group_rotate
// does (pipeline.cpp:111-130, check_group_order :27-50).  On success
// *group is the block width (1 for kind none) and *rot_cols the columns
// covered by whole blocks.
crt_status resolve_rotation(const crt_rotation_spec* rot, int64_t cols, int64_t* group,
                            int64_t* rot_cols) {
  crt_rotation_spec none{CRT_ROT_NONE, 0, 0, 0};
  if (rot == nullptr) rot = &none;
  if (rot->kind == CRT_ROT_NONE) {  // :114 returns x unchanged, no checks
    *group = 1;
    *rot_cols = cols;
    return CRT_OK;
  }
  if (rot->kind != CRT_ROT_REGULAR && rot->kind != CRT_ROT_SYLVESTER)
    return fail(CRT_ERR_UNSUPPORTED, "rotation kind not supported (random_orthogonal is out of scope)");
  if (cols == 0) return fail(CRT_ERR_SHAPE, "group_rotate: empty input");
  if (rot->group_size < 0) return fail(CRT_ERR_INVALID_VALUE, "group_rotate: negative group size");
  int64_t g = rot->group_size == 0 ? cols : rot->group_size;
  if (rot->kind == CRT_ROT_SYLVESTER && !is_pow2(g))
    return fail(CRT_ERR_INVALID_ORDER,
                "sylvester rotation needs a power-of-two group size, got " + std::to_string(g));
  if (rot->kind == CRT_ROT_REGULAR && (!is_pow4(g) || g < 4))
    return fail(CRT_ERR_INVALID_ORDER,
                "regular rotation needs a power-of-four group size, got " + std::to_string(g));
  if (g > 4096)  // hadamard.hpp:12 kMaxHadamardOrder
    return fail(CRT_ERR_INVALID_ORDER, "order " + std::to_string(g) + " exceeds maximum 4096");
  int64_t blocks = cols / g;
  if (blocks * g != cols && !rot->identity_tail)
    return fail(CRT_ERR_SHAPE, "group_rotate: " + std::to_string(cols) +
                                   " columns not divisible by group size " + std::to_string(g));
  *group = g;
  *rot_cols = blocks * g;
  return CRT_OK;
}

crt_status run_k1(const void* x, int32_t x_dtype, int64_t M, int64_t K, int64_t ldx,
                  const crt_rotation_spec* rot, int32_t bits, uint8_t* codes, int64_t ldc,
                  float* s32, double* s64, cudaStream_t st, double* amax,
                  int32_t* rowsum, const double* amax_in, int* err) {
  // bits 5 (internal): 4-bit codes stored one int8 per code, + row code sums
  if (x_dtype != CRT_DTYPE_BF16 && x_dtype != CRT_DTYPE_F32)
    return fail(CRT_ERR_INVALID_VALUE, "unsupported input dtype");
  if (bits != 4 && bits != 8 && bits != 5) return fail(CRT_ERR_INVALID_VALUE, "bits must be 4 or 8");
  if (M < 0 || K < 0) return fail(CRT_ERR_SHAPE, "negative shape");
  int64_t group = 1, rot_cols = K;
  crt_status rs = resolve_rotation(rot, K, &group, &rot_cols);
  if (rs != CRT_OK) return rs;
  if (M == 0) return CRT_OK;
  if (K == 0) {  // reference: zero-width rows -> scale 1.0, no codes
    std::vector<float> ones32(M, 1.f);
    std::vector<double> ones64(M, 1.0);
    if (s32) cudaMemcpyAsync(s32, ones32.data(), M * 4, cudaMemcpyHostToDevice, st);
    if (s64) cudaMemcpyAsync(s64, ones64.data(), M * 8, cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
    return CRT_OK;
  }
  if (ldx < K) return fail(CRT_ERR_SHAPE, "ldx < K");
  const int64_t row_bytes = bits == 4 ? (K + 1) / 2 : K;  // bits 5, 8: one byte per code
  if (x == nullptr) return fail(CRT_ERR_INVALID_VALUE, "null buffer");
  const bool f32 = x_dtype == CRT_DTYPE_F32;
  // amax only (codes == null): the team kernel skips the code stores; other
  // kernels quantise into a stream-ordered scratch buffer
  uint8_t* scratch = nullptr;
  const bool amax_only = codes == nullptr;
  if (amax_only) {
    if (!amax || rowsum) return fail(CRT_ERR_INVALID_VALUE, "null buffer");
    ldc = 16;
  } else if (ldc < row_bytes) {
    return fail(CRT_ERR_SHAPE, "ld_codes too small for one packed row");
  }
  const int kind = rot ? rot->kind : CRT_ROT_NONE;
  crt::K1Args a{};
  a.x = x;
  a.ldx = ldx;
  a.M = M;
  a.K = K;
  a.group = group;
  a.rot_cols = rot_cols;
  a.kind = kind;
  a.codes = codes;
  a.ldc = ldc;
  a.s32 = s32;
  a.s64 = s64;
  a.amax = amax;
  a.rowsum = rowsum;
  a.amax_in = amax_in;
  a.err = err ? err : device_error_word();
  if (!a.err) return fail(CRT_ERR_CUDA, "device error word allocation failed");
  crt::K1Plan plan = crt::plan_k1(K, group, kind, rot && rot->identity_tail, f32, bits, x, ldx,
                                  codes, ldc);
  if (amax_only && !(plan.fast && crt::k1_team_eligible(a, f32, bits))) {
    a.ldc = (row_bytes + 15) / 16 * 16;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&scratch), (size_t)a.ldc * M, st);
    if (e != cudaSuccess) return cuda_fail(e, "scratch alloc");
    a.codes = scratch;
    plan = crt::plan_k1(K, group, kind, rot && rot->identity_tail, f32, bits, x, ldx, scratch,
                        a.ldc);
  }
  int64_t launches = 0;
  cudaError_t e = crt::launch_k1(a, plan, f32, bits, st, &launches);
  g_launches += launches;
  if (scratch) cudaFreeAsync(scratch, st);
  if (e != cudaSuccess) return cuda_fail(e, "rotate_quant launch");
  return CRT_OK;
}

}  // namespace crt_detail

using namespace crt_detail;

extern "C" {

int32_t crt_abi_version(void) { return CRT_ABI_VERSION; }
const char* crt_last_error(void) { return g_err.c_str(); }
int64_t crt_launch_count(void) { return g_launches.load(); }
void crt_debug_k1_trace(void* buf) { crt::set_k1_trace(static_cast<unsigned long long*>(buf)); }
void crt_debug_k3_trace(void* buf) { crt::set_k3_trace(static_cast<unsigned long long*>(buf)); }

// hadamard.cpp:91-106 / :108-126.  H_{4^L}[r][c] = prod_s H4[r_s][c_s]; the
// Kronecker rule puts the right factor on the least significant base-4
// digit, and H4[a][b] = -1 iff a + b == 3.
crt_status crt_regular_hadamard(int32_t n, int8_t* signs) {
  if (!is_pow4(n) || n < 4)
    return fail(CRT_ERR_INVALID_ORDER,
                "regular: order must be a power of four >= 4, got " + std::to_string(n));
  if (n > 4096) return fail(CRT_ERR_INVALID_ORDER, "regular: order exceeds maximum 4096");
  if (!signs) return fail(CRT_ERR_INVALID_VALUE, "null output");
  for (int32_t r = 0; r < n; ++r)
    for (int32_t c = 0; c < n; ++c) {
      uint32_t d = (uint32_t)(r ^ c);
      int neg = __builtin_popcount(d & (d >> 1) & 0x55555555u) & 1;
      signs[(int64_t)r * n + c] = neg ? -1 : 1;
    }
  return CRT_OK;
}

// hadamard.cpp:70-89: H[r][c] = (-1)^popcount(r & c).
crt_status crt_sylvester_hadamard(int32_t n, int8_t* signs) {
  if (!is_pow2(n)) return fail(CRT_ERR_INVALID_ORDER, "sylvester: order must be a power of two");
  if (n > 4096) return fail(CRT_ERR_INVALID_ORDER, "sylvester: order exceeds maximum 4096");
  if (!signs) return fail(CRT_ERR_INVALID_VALUE, "null output");
  for (int32_t r = 0; r < n; ++r)
    for (int32_t c = 0; c < n; ++c)
      signs[(int64_t)r * n + c] = (__builtin_popcount((uint32_t)(r & c)) & 1) ? -1 : 1;
  return CRT_OK;
}

crt_status crt_rotate_quant(const void* x, int32_t x_dtype, int64_t M, int64_t K, int64_t ldx,
                            const crt_rotation_spec* rot, int32_t bits, uint8_t* codes,
                            int64_t ld_codes, float* scales_f32, double* scales_f64,
                            void* stream) {
  NvtxRange nvtx_("crt_rotate_quant (K1)");
  if (bits != 4 && bits != 8) return fail(CRT_ERR_INVALID_VALUE, "bits must be 4 or 8");
  return run_k1(x, x_dtype, M, K, ldx, rot, bits, codes, ld_codes, scales_f32, scales_f64,
                (cudaStream_t)stream);
}

// Row-parallel K1: quantise a column shard of X with the GLOBAL exact row
// maxima `amax_rows` (the MAX all-reduce of every shard's
// crt_rotated_row_absmax), so scales and codes equal the unsharded
// compute_scales / quantize (quant.cpp:10-52) on those columns.
// row_sums != null (bits 4 only) stores the codes one int8 per code with the
// per-row code sums (crt_quant_gemm_i8 operand); else packed / int8 by bits.
crt_status crt_rotate_quant_amax(const void* x, int32_t x_dtype, int64_t M, int64_t K,
                                 int64_t ldx, const crt_rotation_spec* rot,
                                 const double* amax_rows, int32_t bits, uint8_t* codes,
                                 int64_t ld_codes, float* scales_f32, double* scales_f64,
                                 int32_t* row_sums, void* stream) {
  if (bits != 4 && bits != 8) return fail(CRT_ERR_INVALID_VALUE, "bits must be 4 or 8");
  if (!amax_rows && M > 0) return fail(CRT_ERR_INVALID_VALUE, "null amax_rows");
  if (row_sums && bits != 4) return fail(CRT_ERR_INVALID_VALUE, "row sums are for 4-bit codes");
  return run_k1(x, x_dtype, M, K, ldx, rot, row_sums ? 5 : bits, codes, ld_codes, scales_f32,
                scales_f64, (cudaStream_t)stream, nullptr, row_sums, amax_rows);
}

// f4: outlier_amplitude(group_rotate(x)) per row (analysis.cpp:12-17,
// pipeline.cpp:111-151) -- the exact max |y_ref| K1 already settles.  The
// codes go to a stream-ordered scratch buffer.
crt_status crt_rotated_row_absmax(const void* x, int32_t x_dtype, int64_t M, int64_t K,
                                  int64_t ldx, const crt_rotation_spec* rot, double* amax_rows,
                                  void* stream) {
  if (!amax_rows) return fail(CRT_ERR_INVALID_VALUE, "null output");
  if (M <= 0 || K <= 0) return fail(CRT_ERR_SHAPE, "outlier_amplitude: empty matrix");
  // amax-only K1 (no code stores where the team kernel applies)
  return run_k1(x, x_dtype, M, K, ldx, rot, 4, nullptr, 0, nullptr, nullptr, (cudaStream_t)stream,
                amax_rows);
}

crt_status crt_device_status(void* stream, int32_t reset) {
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "device_status sync");
  int v = 0;
  int* word = device_error_word();
  if (!word) return fail(CRT_ERR_CUDA, "device error word allocation failed");
  e = cudaMemcpy(&v, word, sizeof(int), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "device_status read");
  if (reset && v) cudaMemset(word, 0, sizeof(int));
  if (v) return fail(CRT_ERR_INVALID_VALUE, "compute_scales: non-finite input");
  return CRT_OK;
}

// ---------------------------------------------------------------------------
// K2: prepare_layer (pipeline.cpp:158-176)
// ---------------------------------------------------------------------------
}  // extern "C"

crt_status crt_detail::prepare_impl(const crt_layer_desc* d, const void* w, int64_t ldw,
                               const float* bias, int32_t rank, int32_t nranks,
                               cudaStream_t st, crt_layer** out) {
  NvtxRange nvtx_("crt_layer_prepare (K2)");
  if (!d || !out) return fail(CRT_ERR_INVALID_VALUE, "null argument");
  *out = nullptr;
  if (d->bits_w != 4 && d->bits_w != 8) return fail(CRT_ERR_INVALID_VALUE, "bits_w must be 4 or 8");
  if (d->out_features < 0 || d->in_features < 0) return fail(CRT_ERR_SHAPE, "negative shape");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(CRT_ERR_INVALID_VALUE, "bad rank / nranks");
  const int64_t N = d->out_features, K = d->in_features;
  if (N % nranks != 0) return fail(CRT_ERR_SHAPE, "out_features not divisible by nranks");
  const int64_t Ns = N / nranks, off = (int64_t)rank * Ns;
  int64_t group = 1, rot_cols = K;
  crt_status rs = resolve_rotation(&d->rotation, K, &group, &rot_cols);
  if (rs != CRT_OK) return rs;
  const int esz = d->w_dtype == CRT_DTYPE_F32 ? 4 : 2;
  crt_layer* L = new crt_layer();
  L->desc = *d;
  L->desc.out_features = Ns;
  L->n_total = N;
  L->row_offset = off;
  L->ldc = d->bits_w == 4 ? ((K + 1) / 2 + 15) / 16 * 16 : (K + 15) / 16 * 16;
  cudaError_t e = cudaSuccess;
  size_t nalloc = (size_t)(Ns ? Ns : 1);
  // bits 4: K1 writes the reference layout into a stream-ordered scratch
  // buffer; the layer keeps only K3's offset-binary copy (one copy of the
  // weights, like the reference PreparedLayer, pipeline.hpp:55-65)
  uint8_t* wcodes = nullptr;
  if (d->bits_w == 4) e = cudaMallocAsync(reinterpret_cast<void**>(&wcodes), (size_t)L->ldc * nalloc, st);
  else e = cudaMalloc(&L->codes, (size_t)L->ldc * nalloc), wcodes = L->codes;
  if (e == cudaSuccess) e = cudaMalloc(&L->s32, 4 * nalloc);
  if (e == cudaSuccess) e = cudaMalloc(&L->s64, 8 * nalloc);
  if (e == cudaSuccess && bias) {
    e = cudaMalloc(&L->bias, 4 * nalloc);
    if (e == cudaSuccess && Ns)
      e = cudaMemcpyAsync(L->bias, bias + off, 4 * Ns, cudaMemcpyDeviceToDevice, st);
  }
  auto drop_scratch = [&]() {
    if (d->bits_w == 4 && wcodes) cudaFreeAsync(wcodes, st);
    wcodes = nullptr;
  };
  if (e != cudaSuccess) {
    drop_scratch();
    crt_layer_destroy(L);
    return cuda_fail(e, "layer alloc");
  }
  // K1 on the weight rows: rotation along K, per-output-channel scales.
  // Non-finite weights are reported synchronously, as compute_scales throws
  // (quant.cpp:16-18), through a word of this call's own.
  int* err = nullptr;
  e = cudaMallocAsync(reinterpret_cast<void**>(&err), sizeof(int), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(err, 0, sizeof(int), st);
  if (e != cudaSuccess) {
    drop_scratch();
    crt_layer_destroy(L);
    return cuda_fail(e, "error word");
  }
  const char* wbase = reinterpret_cast<const char*>(w) + off * ldw * esz;
  crt_status s = run_k1(wbase, d->w_dtype, Ns, K, ldw, &d->rotation, d->bits_w, wcodes, L->ldc,
                        L->s32, L->s64, st, nullptr, nullptr, nullptr, err);
  int bad = 0;
  if (s == CRT_OK) {
    e = cudaMemcpyAsync(&bad, err, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) s = cuda_fail(e, "prepare_layer status");
    else if (bad) s = fail(CRT_ERR_INVALID_VALUE, "compute_scales: non-finite weight");
  }
  cudaFreeAsync(err, st);
  if (s != CRT_OK) {
    drop_scratch();
    crt_layer_destroy(L);
    return s;
  }
  int64_t launches = 0;
  e = crt::k3_prepare_weights(wcodes, L->ldc, Ns, K, d->bits_w, &L->tiles, st, &launches);
  g_launches += launches;
  drop_scratch();
  if (e != cudaSuccess) {
    crt_layer_destroy(L);
    return cuda_fail(e, "weight tiling");
  }
  *out = L;
  return CRT_OK;
}

extern "C" {

// f2: a layer prepared elsewhere (reference save_prepared_layer,
// pipeline.cpp:257-314): codes already rotated + quantised, given on the host
// in the reference layout (pack_int4 rows of ceil(K/2) bytes, or int8 rows),
// per-channel fp32 scales (weights.scales.crt is f32) and an optional f64
// bias.  No rotation or quantisation is applied.
crt_status crt_layer_from_codes(const crt_layer_desc* d, const uint8_t* codes_host,
                                int64_t ld_codes, const float* scales_host,
                                const double* bias_host, void* stream, crt_layer** out) {
  if (!d || !out || !codes_host || !scales_host) return fail(CRT_ERR_INVALID_VALUE, "null argument");
  *out = nullptr;
  if (d->bits_w != 4 && d->bits_w != 8) return fail(CRT_ERR_INVALID_VALUE, "bits_w must be 4 or 8");
  const int64_t N = d->out_features, K = d->in_features;
  if (N < 0 || K < 0) return fail(CRT_ERR_SHAPE, "negative shape");
  const int64_t row = d->bits_w == 4 ? (K + 1) / 2 : K;
  if (ld_codes < row) return fail(CRT_ERR_SHAPE, "ld_codes smaller than one packed row");
  int64_t group = 1, rot_cols = K;
  crt_status rs = resolve_rotation(&d->rotation, K, &group, &rot_cols);
  if (rs != CRT_OK) return rs;
  cudaStream_t st = (cudaStream_t)stream;
  crt_layer* L = new crt_layer();
  L->desc = *d;
  L->n_total = N;
  L->row_offset = 0;
  L->ldc = d->bits_w == 4 ? ((K + 1) / 2 + 15) / 16 * 16 : (K + 15) / 16 * 16;
  const size_t nalloc = (size_t)(N ? N : 1);
  std::vector<double> s64(nalloc);
  std::vector<float> b32(nalloc, 0.f);
  for (int64_t n = 0; n < N; ++n) {
    if (!(scales_host[n] > 0.f) || !std::isfinite(scales_host[n]))  // quant.cpp:31-35
      return delete L, fail(CRT_ERR_INVALID_VALUE, "weight scale not positive and finite");
    s64[n] = (double)scales_host[n];
    if (bias_host) b32[n] = (float)bias_host[n];
  }
  // bits 4: the host codes are staged in a scratch buffer and kept only as
  // K3's offset-binary copy
  uint8_t* wcodes = nullptr;
  cudaError_t e = cudaMalloc(&wcodes, (size_t)L->ldc * nalloc);
  if (d->bits_w == 8) L->codes = wcodes;
  if (e == cudaSuccess) e = cudaMalloc(&L->s32, 4 * nalloc);
  if (e == cudaSuccess) e = cudaMalloc(&L->s64, 8 * nalloc);
  if (e == cudaSuccess && bias_host) e = cudaMalloc(&L->bias, 4 * nalloc);
  if (e == cudaSuccess) e = cudaMemsetAsync(wcodes, 0, (size_t)L->ldc * nalloc, st);
  if (e == cudaSuccess && N && row)
    e = cudaMemcpy2DAsync(wcodes, L->ldc, codes_host, ld_codes, row, N, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && N) e = cudaMemcpyAsync(L->s32, scales_host, 4 * N, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && N) e = cudaMemcpyAsync(L->s64, s64.data(), 8 * N, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && bias_host && N)
    e = cudaMemcpyAsync(L->bias, b32.data(), 4 * N, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // host staging vectors go out of scope
  if (e != cudaSuccess) {
    if (d->bits_w == 4) cudaFree(wcodes);
    crt_layer_destroy(L);
    return cuda_fail(e, "layer_from_codes");
  }
  int64_t launches = 0;
  e = crt::k3_prepare_weights(wcodes, L->ldc, N, K, d->bits_w, &L->tiles, st, &launches);
  g_launches += launches;
  if (d->bits_w == 4) {
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(wcodes);
  }
  if (e != cudaSuccess) {
    crt_layer_destroy(L);
    return cuda_fail(e, "weight tiling");
  }
  *out = L;
  return CRT_OK;
}

crt_status crt_layer_prepare(const crt_layer_desc* desc, const void* w, int64_t ldw,
                             const float* bias, void* stream, crt_layer** out) {
  return prepare_impl(desc, w, ldw, bias, 0, 1, (cudaStream_t)stream, out);
}

crt_status crt_layer_prepare_shard(const crt_layer_desc* desc, const void* w, int64_t ldw,
                                   const float* bias, int32_t rank, int32_t nranks,
                                   void* stream, crt_layer** out) {
  return prepare_impl(desc, w, ldw, bias, rank, nranks, (cudaStream_t)stream, out);
}

// Row-parallel (K-sharded) layer: rank r keeps
// input columns [r*K/P, (r+1)*K/P) of the full layer's codes.  The
// per-channel scales are the full layer's (prepare_layer quantises each
// output channel over all of K, pipeline.cpp:158-176), so the shards' int32
// partial accumulators sum to int_gemm's exactly.  Rotation groups must not
// straddle shards.
crt_status crt_layer_prepare_kshard(const crt_layer_desc* d, const void* w, int64_t ldw,
                                    const float* bias, int32_t rank, int32_t nranks,
                                    void* stream, crt_layer** out) {
  if (!d || !out) return fail(CRT_ERR_INVALID_VALUE, "null argument");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(CRT_ERR_INVALID_VALUE, "bad rank / nranks");
  const int64_t N = d->out_features, K = d->in_features;
  if (K < 0 || N < 0) return fail(CRT_ERR_SHAPE, "negative shape");
  if (K % nranks != 0) return fail(CRT_ERR_SHAPE, "in_features not divisible by nranks");
  const int64_t Ks = K / nranks;
  int64_t group = 1, rot_cols = K;
  crt_status rs = resolve_rotation(&d->rotation, K, &group, &rot_cols);
  if (rs != CRT_OK) return rs;
  if (rot_cols != K || (group > 1 && Ks % group != 0) ||
      (d->rotation.kind != CRT_ROT_NONE && d->rotation.group_size == 0 && nranks > 1))
    return fail(CRT_ERR_SHAPE, "rotation groups would straddle the K shards");
  if (d->bits_w == 4 && Ks % 2 != 0) return fail(CRT_ERR_SHAPE, "odd K shard splits a packed byte");
  cudaStream_t st = (cudaStream_t)stream;
  crt_layer* full = nullptr;
  crt_status s = prepare_impl(d, w, ldw, bias, 0, 1, st, &full);
  if (s != CRT_OK) return s;
  crt_layer* L = new crt_layer();
  L->desc = *d;
  L->desc.in_features = Ks;
  L->n_total = N;
  L->row_offset = 0;
  const int64_t row = d->bits_w == 4 ? Ks / 2 : Ks;
  L->ldc = (row + 15) / 16 * 16;
  const size_t nalloc = (size_t)(N ? N : 1);
  cudaError_t e = cudaSuccess;
  if (d->bits_w == 8) {
    e = cudaMalloc(&L->codes, (size_t)L->ldc * nalloc);
    if (e == cudaSuccess) e = cudaMemsetAsync(L->codes, 0, (size_t)L->ldc * nalloc, st);
    if (e == cudaSuccess && N && row)
      e = cudaMemcpy2DAsync(L->codes, L->ldc, full->codes + (int64_t)rank * row, full->ldc, row, N,
                            cudaMemcpyDeviceToDevice, st);
  }
  if (e == cudaSuccess) e = cudaMalloc(&L->s32, 4 * nalloc);
  if (e == cudaSuccess) e = cudaMalloc(&L->s64, 8 * nalloc);
  if (e == cudaSuccess && bias) e = cudaMalloc(&L->bias, 4 * nalloc);
  if (e == cudaSuccess && N) e = cudaMemcpyAsync(L->s32, full->s32, 4 * N, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess && N) e = cudaMemcpyAsync(L->s64, full->s64, 8 * N, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess && bias && N)
    e = cudaMemcpyAsync(L->bias, full->bias, 4 * N, cudaMemcpyDeviceToDevice, st);
  int64_t launches = 0;
  if (e == cudaSuccess) {
    // bits 4: the shard's columns straight from the full layer's
    // offset-binary copy (byte offset rank * Ks/2 of every row)
    e = d->bits_w == 4
            ? crt::k3_prepare_weights(full->tiles.codes_ob + (int64_t)rank * row, full->tiles.ld_ob,
                                      N, Ks, 4, &L->tiles, st, &launches, /*src_ob=*/true)
            : crt::k3_prepare_weights(L->codes, L->ldc, N, Ks, 8, &L->tiles, st, &launches);
  }
  g_launches += launches;
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  crt_layer_destroy(full);
  if (e != cudaSuccess) {
    crt_layer_destroy(L);
    return cuda_fail(e, "weight tiling");
  }
  *out = L;
  return CRT_OK;
}

crt_status crt_layer_destroy(crt_layer* L) {
  if (!L) return CRT_OK;
  cudaFree(L->codes);
  cudaFree(L->s32);
  cudaFree(L->s64);
  cudaFree(L->bias);
  crt::k3_free_weights(&L->tiles);
  delete L;
  return CRT_OK;
}

crt_status crt_layer_info(const crt_layer* L, crt_layer_desc* out) {
  if (!L || !out) return fail(CRT_ERR_INVALID_VALUE, "null argument");
  *out = L->desc;
  return CRT_OK;
}

crt_status crt_layer_export(const crt_layer* L, uint8_t* codes, int64_t ld_codes, float* s32,
                            double* s64, void* stream) {
  if (!L) return fail(CRT_ERR_INVALID_VALUE, "null layer");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t N = L->desc.out_features, K = L->desc.in_features;
  const int64_t row = L->desc.bits_w == 4 ? (K + 1) / 2 : K;
  cudaError_t e = cudaSuccess;
  if (codes && N && row) {
    if (ld_codes < row) return fail(CRT_ERR_SHAPE, "ld_codes too small");
    if (L->desc.bits_w == 4) {  // back from the offset-binary copy
      int64_t launches = 0;
      e = crt::k3_export_w4(L->tiles, codes, ld_codes, 0, row, st, &launches);
      g_launches += launches;
    } else {
      e = cudaMemcpy2DAsync(codes, ld_codes, L->codes, L->ldc, row, N, cudaMemcpyDeviceToDevice, st);
    }
  }
  if (e == cudaSuccess && s32 && N) e = cudaMemcpyAsync(s32, L->s32, 4 * N, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess && s64 && N) e = cudaMemcpyAsync(s64, L->s64, 8 * N, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "layer export");
  return CRT_OK;
}

// ---------------------------------------------------------------------------
// K3 + forward
// ---------------------------------------------------------------------------
}  // extern "C"

void* crt_detail::workspace_tp_scratch(crt_workspace* ws, size_t bytes, cudaStream_t st) {
  if (ws->tp_bytes >= bytes) return ws->tp_buf;
  if (cudaStreamSynchronize(st) != cudaSuccess) return nullptr;
  cudaFree(ws->tp_buf);
  ws->tp_buf = nullptr;
  ws->tp_bytes = 0;
  if (cudaMalloc(&ws->tp_buf, bytes) != cudaSuccess) return nullptr;
  ws->tp_bytes = bytes;
  return ws->tp_buf;
}

crt_status crt_detail::quant_gemm_impl(const uint8_t* a_codes, int64_t lda, const float* a_scales,
                                  const int32_t* a_sums, int32_t layout, int32_t bits_a,
                                  const crt_layer* L, int64_t M, int32_t out_kind, void* y,
                                  int64_t ldy, void* stream) {
  if (!L) return fail(CRT_ERR_INVALID_VALUE, "null layer");
  if (bits_a != 4 && bits_a != 8) return fail(CRT_ERR_INVALID_VALUE, "activation bits must be 4 or 8");
  if (out_kind < CRT_OUT_BF16 || out_kind > CRT_OUT_I32_ACC)
    return fail(CRT_ERR_INVALID_VALUE, "bad out_kind");
  const int64_t N = L->desc.out_features, K = L->desc.in_features;
  // int_gemm capacity precheck (pipeline.cpp:184-192)
  const int64_t qa = (1 << (bits_a - 1)) - 1, qw = (1 << (L->desc.bits_w - 1)) - 1;
  if (qa * qw * K > 2147483647LL)
    return fail(CRT_ERR_CAPACITY, "int_gemm: " + std::to_string(K) +
                                      "-deep accumulation can overflow int32");
  if (bits_a != L->desc.bits_w)
    return fail(CRT_ERR_UNSUPPORTED, "mixed activation/weight bit widths are not built");
  if (M < 0) return fail(CRT_ERR_SHAPE, "negative M");
  if (M == 0 || N == 0) return CRT_OK;
  if (ldy < N) return fail(CRT_ERR_SHAPE, "ldy < N");
  int64_t launches = 0;
  crt::K3Args a{};
  a.a_codes = a_codes;
  a.lda = lda;
  a.a_layout = layout;
  a.a_sums = a_sums;
  a.a_scales = a_scales;
  a.w = L->tiles;
  a.w_scales = L->s32;
  a.bias = L->bias;
  a.M = M;
  a.N = N;
  a.K = K;
  a.bits = bits_a;
  a.out_kind = out_kind;
  a.y = y;
  a.ldy = ldy;
  if (layout == 1 && !crt::k3_v3_supported(a))
    return fail(CRT_ERR_UNSUPPORTED, "int8-stored activation codes need the v3 GEMM shapes");
  cudaError_t e = crt::k3_launch(a, (cudaStream_t)stream, &launches);
  g_launches += launches;
  if (e != cudaSuccess) return cuda_fail(e, "quant_gemm launch");
  return CRT_OK;
}

extern "C" {

crt_status crt_quant_gemm(const uint8_t* a_codes, int64_t lda, const float* a_scales,
                          int32_t bits_a, const crt_layer* L, int64_t M, int32_t out_kind,
                          void* y, int64_t ldy, void* stream) {
  NvtxRange nvtx_("crt_quant_gemm (K3)");
  return quant_gemm_impl(a_codes, lda, a_scales, nullptr, 0, bits_a, L, M, out_kind, y, ldy,
                         stream);
}

crt_status crt_rotate_quant_i8(const void* x, int32_t x_dtype, int64_t M, int64_t K, int64_t ldx,
                               const crt_rotation_spec* rot, uint8_t* codes, int64_t ld_codes,
                               float* scales_f32, int32_t* code_sums, void* stream) {
  NvtxRange nvtx_("crt_rotate_quant_i8 (K1)");
  if (!code_sums) return fail(CRT_ERR_INVALID_VALUE, "null code_sums");
  return run_k1(x, x_dtype, M, K, ldx, rot, 5, codes, ld_codes, scales_f32, nullptr,
                (cudaStream_t)stream, nullptr, code_sums);
}

crt_status crt_quant_gemm_i8(const uint8_t* a_codes, int64_t lda, const float* a_scales,
                             const int32_t* code_sums, const crt_layer* L, int64_t M,
                             int32_t out_kind, void* y, int64_t ldy, void* stream) {
  NvtxRange nvtx_("crt_quant_gemm_i8 (K3 v3)");
  if (!code_sums) return fail(CRT_ERR_INVALID_VALUE, "null code_sums");
  return quant_gemm_impl(a_codes, lda, a_scales, code_sums, 1, 4, L, M, out_kind, y, ldy, stream);
}

// The dequant loop of forward (pipeline.cpp:224-230) on int32 accumulators
// that were summed outside K3 (row-parallel: the SUM all-reduce of the
// shards' partial int_gemm results).  Same fp32 expression as the K3
// epilogues, so the output equals the unsharded forward bit for bit.
__global__ void crt_dequant_kernel(const int32_t* __restrict__ acc, int64_t lda, int64_t M,
                                   int64_t N, const float* __restrict__ sa,
                                   const float* __restrict__ sw, const float* __restrict__ bias,
                                   int32_t out_kind, void* y, int64_t ldy) {
  // one row per blockIdx.y, 8 consecutive columns per thread
  const int64_t m = blockIdx.y;
  const float s = sa[m];
  const int32_t* ar = acc + m * lda;
  for (int64_t n0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; n0 < N;
       n0 += (int64_t)gridDim.x * blockDim.x * 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t n = n0 + j;
      if (n >= N) break;
      const int32_t v = ar[n];
      if (out_kind == CRT_OUT_I32_ACC) {
        reinterpret_cast<int32_t*>(y)[m * ldy + n] = v;
        continue;
      }
      const float r = fmaf((float)v * s, sw[n], bias ? bias[n] : 0.f);
      if (out_kind == CRT_OUT_BF16) reinterpret_cast<__nv_bfloat16*>(y)[m * ldy + n] = __float2bfloat16_rn(r);
      else reinterpret_cast<float*>(y)[m * ldy + n] = r;
    }
  }
}

crt_status crt_dequant(const int32_t* acc, int64_t ld_acc, int64_t M, const float* a_scales,
                       const crt_layer* L, int32_t out_kind, void* y, int64_t ldy, void* stream) {
  NvtxRange nvtx_("crt_dequant");
  if (!L) return fail(CRT_ERR_INVALID_VALUE, "null layer");
  if (out_kind < CRT_OUT_BF16 || out_kind > CRT_OUT_I32_ACC)
    return fail(CRT_ERR_INVALID_VALUE, "bad out_kind");
  const int64_t N = L->desc.out_features;
  if (M < 0) return fail(CRT_ERR_SHAPE, "negative M");
  if (M == 0 || N == 0) return CRT_OK;
  if (ld_acc < N || ldy < N) return fail(CRT_ERR_SHAPE, "ld < N");
  if (!acc || !y || !a_scales) return fail(CRT_ERR_INVALID_VALUE, "null buffer");
  const int64_t bx = std::min<int64_t>((N + 2047) / 2048, 64);
  for (int64_t m0 = 0; m0 < M; m0 += 65535) {  // gridDim.y limit
    const int64_t mr = std::min<int64_t>(M - m0, 65535);
    crt_dequant_kernel<<<dim3((unsigned)bx, (unsigned)mr), 256, 0, (cudaStream_t)stream>>>(
        acc + m0 * ld_acc, ld_acc, mr, N, a_scales + m0, L->s32, L->bias, out_kind,
        static_cast<char*>(y) + m0 * ldy * (out_kind == CRT_OUT_BF16 ? 2 : 4), ldy);
  }
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "dequant launch");
  return CRT_OK;
}

crt_status crt_workspace_create(int64_t max_m, int64_t max_k, crt_workspace** out) {
  if (!out) return fail(CRT_ERR_INVALID_VALUE, "null argument");
  if (max_m < 0 || max_k < 0) return fail(CRT_ERR_SHAPE, "negative workspace size");
  crt_workspace* w = new crt_workspace();
  w->max_m = max_m;
  w->max_k = max_k;
  const int64_t ld = (max_k + 15) / 16 * 16;  // room for int8 codes too
  cudaError_t e = cudaMalloc(&w->codes, (size_t)ld * (max_m ? max_m : 1));
  if (e == cudaSuccess) e = cudaMalloc(&w->s32, 4 * (size_t)(max_m ? max_m : 1));
  if (e == cudaSuccess) e = cudaMalloc(&w->rowsum, 4 * (size_t)(max_m ? max_m : 1));
  if (e == cudaSuccess) e = cudaMalloc(&w->err, sizeof(int));
  const int zero = 0;
  if (e == cudaSuccess) e = cudaMemcpy(w->err, &zero, sizeof(int), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(w->codes);
    cudaFree(w->s32);
    cudaFree(w->rowsum);
    cudaFree(w->err);
    delete w;
    return cuda_fail(e, "workspace alloc");
  }
  *out = w;
  return CRT_OK;
}

crt_status crt_workspace_destroy(crt_workspace* w) {
  if (!w) return CRT_OK;
  cudaFree(w->tp_buf);
  cudaFree(w->codes);
  cudaFree(w->s32);
  cudaFree(w->rowsum);
  cudaFree(w->err);
  delete w;
  return CRT_OK;
}

crt_status crt_workspace_status(crt_workspace* w, void* stream, int32_t reset) {
  if (!w) return fail(CRT_ERR_INVALID_VALUE, "null workspace");
  cudaStream_t st = (cudaStream_t)stream;
  int v = 0;
  cudaError_t e = cudaMemcpyAsync(&v, w->err, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "workspace_status");
  if (reset && v) {
    e = cudaMemsetAsync(w->err, 0, sizeof(int), st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "workspace_status reset");
  }
  if (v) return fail(CRT_ERR_INVALID_VALUE, "compute_scales: non-finite input");
  return CRT_OK;
}

crt_status crt_forward(const crt_layer* L, const void* x, int32_t x_dtype, int64_t M, int64_t ldx,
                       int32_t bits_a, int32_t out_kind, void* y, int64_t ldy, crt_workspace* ws,
                       void* stream) {
  NvtxRange nvtx_("crt_forward (K1 + K3)");
  if (!L || !ws) return fail(CRT_ERR_INVALID_VALUE, "null layer / workspace");
  const int64_t K = L->desc.in_features;
  if (bits_a != 4 && bits_a != 8)  // pipeline.cpp:213-215
    return fail(CRT_ERR_INVALID_VALUE, "forward: activation bits must be 4 or 8");
  if (M > ws->max_m || K > ws->max_k) return fail(CRT_ERR_SHAPE, "workspace too small");
  bool v3 = bits_a == 4 && L->desc.bits_w == 4 && L->tiles.codes_ob && M > 0;
  if (v3) {  // the v3 GEMM's limits (K, TMA encode entry point); else the packed path
    crt::K3Args probe{};
    probe.a_codes = ws->codes;
    probe.lda = (K + 15) / 16 * 16;
    probe.a_layout = 1;
    probe.a_sums = ws->rowsum;
    probe.w = L->tiles;
    probe.M = M;
    probe.N = L->desc.out_features;
    probe.K = K;
    probe.bits = 4;
    v3 = probe.N == 0 || crt::k3_v3_supported(probe);
  }
  if (v3) {
    // v3: int8-stored codes + code sums -> hardware-expanded weights GEMM
    const int64_t ldc = (K + 15) / 16 * 16;
    crt_status s = run_k1(x, x_dtype, M, K, ldx, &L->desc.rotation, 5, ws->codes, ldc, ws->s32,
                          nullptr, (cudaStream_t)stream, nullptr, ws->rowsum, nullptr, ws->err);
    if (s != CRT_OK) return s;
    return quant_gemm_impl(ws->codes, ldc, ws->s32, ws->rowsum, 1, 4, L, M, out_kind, y, ldy,
                           stream);
  }
  const int64_t ldc = bits_a == 4 ? ((K + 1) / 2 + 15) / 16 * 16 : (K + 15) / 16 * 16;
  crt_status s = run_k1(x, x_dtype, M, K, ldx, &L->desc.rotation, bits_a, ws->codes, ldc, ws->s32,
                        nullptr, (cudaStream_t)stream, nullptr, nullptr, nullptr, ws->err);
  if (s != CRT_OK) return s;
  return crt_quant_gemm(ws->codes, ldc, ws->s32, bits_a, L, M, out_kind, y, ldy, stream);
}

crt_status crt_forward_host(const crt_layer* L, const void* x_host, int32_t x_dtype, int64_t M,
                            int32_t bits_a, int32_t out_kind, void* y_host, void* x_dev,
                            void* y_dev, crt_workspace* ws, void* stream) {
  if (!L) return fail(CRT_ERR_INVALID_VALUE, "null layer");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t K = L->desc.in_features, N = L->desc.out_features;
  const size_t xbytes = (size_t)M * K * (x_dtype == CRT_DTYPE_F32 ? 4 : 2);
  const size_t ybytes = (size_t)M * N * (out_kind == CRT_OUT_BF16 ? 2 : 4);
  cudaError_t e = cudaMemcpyAsync(x_dev, x_host, xbytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "h2d");
  crt_status s = crt_forward(L, x_dev, x_dtype, M, K, bits_a, out_kind, y_dev, N, ws, stream);
  if (s != CRT_OK) return s;
  e = cudaMemcpyAsync(y_host, y_dev, ybytes, cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return cuda_fail(e, "d2h");
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "sync");
  return CRT_OK;
}

}  // extern "C"
