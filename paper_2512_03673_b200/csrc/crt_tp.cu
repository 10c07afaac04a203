// crt_tp.cu -- tensor-parallel entry points of the C-ABI over NCCL
// (include/crt/convlinear4bit.h "Tensor parallelism").
//
// NCCL is resolved at first use with dlopen("libnccl.so.2"): inside a
// process that already loaded one (PyTorch's), that same library is used,
// so a communicator created by the caller's NCCL can be passed in; a plain
// C++ host gets the system NCCL.  No link-time dependency.
//
// Column parallel (wide layers, FLUX fc1 N = 12288): the rank's output
// channels are a crt_layer_prepare_shard layer; K1 + K3 on the full input,
// then ncclAllGather of the [M, N/P] shards (rank-major) and one interleave
// kernel into [M, N].  Row parallel (FLUX fc2 K = 12288, fed by a gather-free
// column-parallel fc1): amax-only K1 on the shard, MAX all-reduce of M
// doubles, K1 with the global max, K3 int32 partials, SUM all-reduce, the
// dequant kernel.  Reference operator: forward, pipeline.cpp:206-233.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only; the functions come from dlsym
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "crt_internal.h"

using namespace crt_detail;

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommCount)(const ncclComm_t, int*);
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
  bool ok;
};

const NcclApi& nccl() {
  static NcclApi api{};
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's own, if any
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    auto sym = [h](const char* n) { return dlsym(h, n); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.CommCount = reinterpret_cast<decltype(api.CommCount)>(sym("ncclCommCount"));
    api.CommUserRank = reinterpret_cast<decltype(api.CommUserRank)>(sym("ncclCommUserRank"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.CommCount &&
             api.CommUserRank && api.AllGather && api.AllReduce && api.GetErrorString;
  });
  return api;
}

crt_status nccl_fail(ncclResult_t r, const char* where) {
  const NcclApi& n = nccl();
  return fail(CRT_ERR_NCCL, std::string(where) + ": " +
                                (n.GetErrorString ? n.GetErrorString(r) : "nccl error"));
}

crt_status need_nccl() {
  if (!nccl().ok) return fail(CRT_ERR_NCCL, "libnccl.so.2 not found (or missing symbols)");
  return CRT_OK;
}

crt_status comm_info(void* comm, int* rank, int* nranks) {
  if (!comm) return fail(CRT_ERR_INVALID_VALUE, "null communicator");
  crt_status s = need_nccl();
  if (s != CRT_OK) return s;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  ncclResult_t r = nccl().CommUserRank(c, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommUserRank");
  r = nccl().CommCount(c, nranks);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommCount");
  return CRT_OK;
}

// [P][M][ns] rank-major all-gather buffer -> y[M][P*ns] (row pitch ldy), 16-
// or 32-bit elements, one thread per element.
template <typename T>
__global__ void interleave_kernel(const T* __restrict__ g, int64_t M, int64_t ns, int P, T* y,
                                  int64_t ldy) {
  const int64_t total = (int64_t)P * M * ns;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % ns, mr = i / ns, m = mr % M, r = mr / M;
    y[m * ldy + r * ns + c] = g[i];
  }
}

}  // namespace

extern "C" {

crt_status crt_nccl_unique_id(uint8_t* id128) {
  if (!id128) return fail(CRT_ERR_INVALID_VALUE, "null id");
  crt_status s = need_nccl();
  if (s != CRT_OK) return s;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  ncclResult_t r = nccl().GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id128, &id, 128);
  return CRT_OK;
}

crt_status crt_nccl_comm_create(int32_t nranks, int32_t rank, const uint8_t* id128, void** comm) {
  if (!id128 || !comm) return fail(CRT_ERR_INVALID_VALUE, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(CRT_ERR_INVALID_VALUE, "bad rank / nranks");
  crt_status s = need_nccl();
  if (s != CRT_OK) return s;
  ncclUniqueId id;
  memcpy(&id, id128, 128);
  ncclComm_t c = nullptr;
  ncclResult_t r = nccl().CommInitRank(&c, nranks, id, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  *comm = c;
  return CRT_OK;
}

crt_status crt_nccl_comm_destroy(void* comm) {
  if (!comm) return CRT_OK;
  crt_status s = need_nccl();
  if (s != CRT_OK) return s;
  ncclResult_t r = nccl().CommDestroy(static_cast<ncclComm_t>(comm));
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return CRT_OK;
}

crt_status crt_nccl_comm_info(void* comm, int32_t* rank, int32_t* nranks) {
  if (!rank || !nranks) return fail(CRT_ERR_INVALID_VALUE, "null argument");
  int r = 0, n = 0;
  crt_status s = comm_info(comm, &r, &n);
  if (s != CRT_OK) return s;
  *rank = r;
  *nranks = n;
  return CRT_OK;
}

crt_status crt_tp_layer_prepare(const crt_layer_desc* desc, const void* w, int64_t ldw,
                                const float* bias, int32_t mode, void* comm, void* stream,
                                crt_layer** out) {
  if (!desc || !out) return fail(CRT_ERR_INVALID_VALUE, "null argument");
  if (mode != CRT_TP_COLUMN && mode != CRT_TP_ROW) return fail(CRT_ERR_INVALID_VALUE, "bad tp mode");
  int rank = 0, P = 1;
  crt_status s = comm_info(comm, &rank, &P);
  if (s != CRT_OK) return s;
  s = mode == CRT_TP_COLUMN
          ? prepare_impl(desc, w, ldw, bias, rank, P, (cudaStream_t)stream, out)
          : crt_layer_prepare_kshard(desc, w, ldw, bias, rank, P, stream, out);
  if (s != CRT_OK) return s;
  (*out)->tp_mode = mode;
  (*out)->tp_rank = rank;
  (*out)->tp_nranks = P;
  (*out)->k_total = desc->in_features;
  return CRT_OK;
}

crt_status crt_tp_forward(const crt_layer* L, const void* x, int32_t x_dtype, int64_t M,
                          int64_t ldx, int32_t out_kind, void* y, int64_t ldy, int32_t gather,
                          crt_workspace* ws, void* comm, void* stream) {
  NvtxRange nvtx_("crt_tp_forward");
  if (!L || !ws || !y) return fail(CRT_ERR_INVALID_VALUE, "null layer / workspace / output");
  if (L->tp_mode != CRT_TP_COLUMN && L->tp_mode != CRT_TP_ROW)
    return fail(CRT_ERR_INVALID_VALUE, "layer was not prepared with crt_tp_layer_prepare");
  if (out_kind < CRT_OUT_BF16 || out_kind > CRT_OUT_I32_ACC)
    return fail(CRT_ERR_INVALID_VALUE, "bad out_kind");
  int rank = 0, P = 1;
  crt_status s = comm_info(comm, &rank, &P);
  if (s != CRT_OK) return s;
  if (rank != L->tp_rank || P != L->tp_nranks)
    return fail(CRT_ERR_INVALID_VALUE, "communicator does not match the layer's rank / size");
  if (M < 0) return fail(CRT_ERR_SHAPE, "negative M");
  cudaStream_t st = (cudaStream_t)stream;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  const int32_t bits = L->desc.bits_w;
  const int64_t Ns = L->desc.out_features, K = L->desc.in_features;
  const size_t esz = out_kind == CRT_OUT_BF16 ? 2 : 4;

  if (L->tp_mode == CRT_TP_COLUMN) {
    const int64_t N = Ns * P;
    if (ldy < (gather ? N : Ns)) return fail(CRT_ERR_SHAPE, "ldy too small");
    if (M == 0) return CRT_OK;
    if (!gather || P == 1) return crt_forward(L, x, x_dtype, M, ldx, bits, out_kind, y, ldy, ws, stream);
    const size_t lbytes = ((size_t)M * Ns * esz + 255) / 256 * 256;
    char* buf = static_cast<char*>(workspace_tp_scratch(ws, lbytes + (size_t)P * M * Ns * esz, st));
    if (!buf) return fail(CRT_ERR_CUDA, "tp scratch allocation failed");
    void* local = buf;
    void* gbuf = buf + lbytes;
    cudaError_t e = cudaSuccess;
    s = crt_forward(L, x, x_dtype, M, ldx, bits, out_kind, local, Ns, ws, stream);
    if (s == CRT_OK) {
      const ncclDataType_t dt = out_kind == CRT_OUT_BF16 ? ncclBfloat16
                                : out_kind == CRT_OUT_F32 ? ncclFloat32 : ncclInt32;
      ncclResult_t r = nccl().AllGather(local, gbuf, (size_t)M * Ns, dt, c, st);
      if (r != ncclSuccess) s = nccl_fail(r, "ncclAllGather");
    }
    if (s == CRT_OK) {
      const int64_t total = (int64_t)P * M * Ns;
      const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
      if (esz == 2)
        interleave_kernel<uint16_t><<<blocks, 256, 0, st>>>(static_cast<const uint16_t*>(gbuf), M,
                                                            Ns, P, static_cast<uint16_t*>(y), ldy);
      else
        interleave_kernel<uint32_t><<<blocks, 256, 0, st>>>(static_cast<const uint32_t*>(gbuf), M,
                                                            Ns, P, static_cast<uint32_t*>(y), ldy);
      ++g_launches;
      e = cudaGetLastError();
      if (e != cudaSuccess) s = cuda_fail(e, "interleave launch");
    }
    return s;
  }

  // ---- row parallel: x is this rank's [M, K/P] input shard ------------------
  const int64_t N = Ns;
  if (ldy < N) return fail(CRT_ERR_SHAPE, "ldy too small");
  const int64_t qa = (1 << (bits - 1)) - 1;
  if (qa * qa * L->k_total > 2147483647LL)  // int_gemm capacity of the FULL K (pipeline.cpp:184-192)
    return fail(CRT_ERR_CAPACITY, "int_gemm: " + std::to_string(L->k_total) +
                                      "-deep accumulation can overflow int32");
  if (M == 0) return CRT_OK;
  if (M > ws->max_m || K > ws->max_k) return fail(CRT_ERR_SHAPE, "workspace too small");
  const size_t abytes = ((size_t)M * 8 + 255) / 256 * 256;
  char* buf = static_cast<char*>(workspace_tp_scratch(ws, abytes + (size_t)M * N * 4, st));
  if (!buf) return fail(CRT_ERR_CUDA, "tp scratch allocation failed");
  double* amax = reinterpret_cast<double*>(buf);
  int32_t* acc = reinterpret_cast<int32_t*>(buf + abytes);
  // 1. exact per-row max of the shard (amax-only K1), 2. global max
  s = run_k1(x, x_dtype, M, K, ldx, &L->desc.rotation, bits, nullptr, 0, nullptr, nullptr, st,
             amax, nullptr, nullptr, ws->err);
  if (s == CRT_OK) {
    ncclResult_t r = nccl().AllReduce(amax, amax, (size_t)M, ncclFloat64, ncclMax, c, st);
    if (r != ncclSuccess) s = nccl_fail(r, "ncclAllReduce(max)");
  }
  // 3. K1 with the global max (the unsharded codes), K3 partial accumulators
  const bool i8 = bits == 4 && L->tiles.codes_ob;
  const int64_t ldc = i8 || bits == 8 ? (K + 15) / 16 * 16 : ((K + 1) / 2 + 15) / 16 * 16;
  if (s == CRT_OK)
    s = run_k1(x, x_dtype, M, K, ldx, &L->desc.rotation, i8 ? 5 : bits, ws->codes, ldc, ws->s32,
               nullptr, st, nullptr, i8 ? ws->rowsum : nullptr, amax, ws->err);
  if (s == CRT_OK)
    s = quant_gemm_impl(ws->codes, ldc, ws->s32, i8 ? ws->rowsum : nullptr, i8 ? 1 : 0, bits, L, M,
                        CRT_OUT_I32_ACC, acc, N, stream);
  // 4. exact int32 sum of the partials, 5. dequant
  if (s == CRT_OK) {
    ncclResult_t r = nccl().AllReduce(acc, acc, (size_t)M * N, ncclInt32, ncclSum, c, st);
    if (r != ncclSuccess) s = nccl_fail(r, "ncclAllReduce(sum)");
  }
  if (s == CRT_OK) s = crt_dequant(acc, N, M, ws->s32, L, out_kind, y, ldy, stream);
  return s;
}

}  // extern "C"
