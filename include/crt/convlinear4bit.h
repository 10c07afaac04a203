/*
 * convlinear4bit.h -- the drop-in C-ABI of the B200-native ConvLinear4bit
 * forward path (one shared library: paper_2512_03673_b200/libconvrot_b200.so).
 *
 * The reference (/root/reference/proj) is a C++20 library with no C or FFI
 * surface; each entry point below replaces one reference function on the
 * ConvLinear4bit hot path and keeps its argument meaning
 * and error behaviour.  Reference paths are relative to /root/reference/proj.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Pointers documented "device" must be
 *     CUDA device (or managed) memory; "host" pointers are CPU memory
 *     (pinned memory makes the *_host entry points asynchronous-capable).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *     All device work is stream-ordered; no entry point synchronises unless
 *     documented.
 *   - Shape / order / divisibility / capacity errors are detected on the
 *     host before any launch and returned synchronously.  Data-dependent
 *     errors (non-finite input, reference: compute_scales throws
 *     InvalidValueError, quant.cpp:16-18) set a device error word that
 *     crt_device_status() reports.
 *   - crt_last_error() returns a thread-local message for the last failure.
 */
#ifndef CRT_CONVLINEAR4BIT_H_
#define CRT_CONVLINEAR4BIT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CRT_ABI_VERSION 1

/* Status codes, 1:1 with the reference exception taxonomy (errors.hpp:9-67). */
typedef enum crt_status {
  CRT_OK = 0,
  CRT_ERR_INVALID_ORDER = 1, /* InvalidOrderError (errors.hpp:18-22) */
  CRT_ERR_INVALID_VALUE = 2, /* InvalidValueError (errors.hpp:24-29) */
  CRT_ERR_SHAPE = 3,         /* ShapeError        (errors.hpp:31-35) */
  CRT_ERR_CAPACITY = 4,      /* CapacityError     (errors.hpp:37-41) */
  CRT_ERR_FORMAT = 5,        /* FormatError       (errors.hpp:43-54) */
  CRT_ERR_CUDA = 6,          /* CUDA runtime/driver failure */
  CRT_ERR_UNSUPPORTED = 7,   /* valid for the reference, not built here */
  CRT_ERR_NCCL = 8           /* NCCL unavailable or a collective failed (crt_tp_*) */
} crt_status;

/* RotationKind (pipeline.hpp:14); random_orthogonal is out of scope. */
typedef enum crt_rotation_kind {
  CRT_ROT_NONE = 0,
  CRT_ROT_SYLVESTER = 1,
  CRT_ROT_REGULAR = 2
} crt_rotation_kind;

/* Element types of the activations / weights handed to the library. */
typedef enum crt_dtype {
  CRT_DTYPE_BF16 = 0,
  CRT_DTYPE_F32 = 1
} crt_dtype;

/* Output flavours of the GEMM epilogue. */
typedef enum crt_out_kind {
  CRT_OUT_BF16 = 0,    /* y = acc*s_a*s_w + b, rounded to bf16 (production) */
  CRT_OUT_F32 = 1,     /* same in fp32 (dequant parity, pipeline.cpp:224-230) */
  CRT_OUT_I32_ACC = 2  /* raw int32 accumulators (int_gemm parity, :178-204) */
} crt_out_kind;

/* RotationSpec (pipeline.hpp:23-30).  group_size 0 = global (one block
 * spanning K, pipeline.cpp:120-122).  seed is accepted for layout parity
 * (random_orthogonal only in the reference) and ignored. */
typedef struct crt_rotation_spec {
  int32_t kind;
  int32_t group_size;
  uint64_t seed;
  int32_t identity_tail;
} crt_rotation_spec;

/* -------------------------------------------------------------------------
 * a1: regular(n) -- replaces convrot::regular (hadamard.cpp:91-106) and the
 * Kronecker rule of convrot::kronecker (hadamard.cpp:108-126).  Writes the
 * n x n sign matrix (+1/-1, row-major) to HOST memory.  INVALID_ORDER unless
 * n is a power of four in [4, 4096] (hadamard.cpp:92-96). */
crt_status crt_regular_hadamard(int32_t n, int8_t* signs_host);

/* Sylvester sign matrix (hadamard.cpp:70-89), power of two <= 4096. */
crt_status crt_sylvester_hadamard(int32_t n, int8_t* signs_host);

/* -------------------------------------------------------------------------
 * K1: group_rotate + compute_scales + quantize + pack_int4 --
 * replaces pipeline.cpp:111-151 (group_rotate), quant.cpp:10-24
 * (compute_scales), quant.cpp:26-52 (quantize) and quant.cpp:64-81
 * (pack_int4), i.e. the activation half of forward (pipeline.cpp:216-218).
 *
 *   x        device, M rows x K, row stride ldx ELEMENTS, dtype x_dtype
 *   rot      rotation spec (kind none/regular; sylvester accepted)
 *   bits     4 (codes nibble-packed exactly as pack_int4: element 2t in the
 *            low nibble of byte t, rows padded to a whole byte) or 8 (int8)
 *   codes    device, M rows x ld_codes BYTES (>= ceil(K/2) for bits 4,
 *            >= K for bits 8)
 *   scales_f32 device, M floats, (float)s           (nullable)
 *   scales_f64 device, M doubles, s exactly as compute_scales (nullable)
 *
 * Codes and the f64 scales are bit-identical to the reference's
 * quantize(group_rotate(x)) / compute_scales on the same inputs widened to
 * double. */
crt_status crt_rotate_quant(const void* x, int32_t x_dtype, int64_t M, int64_t K,
                            int64_t ldx, const crt_rotation_spec* rot, int32_t bits,
                            uint8_t* codes, int64_t ld_codes, float* scales_f32,
                            double* scales_f64, void* stream);

/* f4: per-row exact max |group_rotate(x)| (device, M
 * doubles; +inf for a row with a non-finite value).  The reference's
 * outlier_amplitude(group_rotate(x)) (analysis.cpp:12-17) is the max over
 * rows; rotation_sweep (analysis.cpp:89-117) runs it per (kind, group). */
crt_status crt_rotated_row_absmax(const void* x, int32_t x_dtype, int64_t M, int64_t K,
                                  int64_t ldx, const crt_rotation_spec* rot, double* amax_rows,
                                  void* stream);

/* -------------------------------------------------------------------------
 * K2: prepare_layer -- replaces pipeline.cpp:158-176.  Rotates W (N x K,
 * device, row stride ldw elements) along K, quantizes per output channel and
 * stores the codes in the K3 tile layout inside an opaque, immutable layer
 * handle that owns all its device memory.  bias is device fp32 (N) or NULL.
 * The reference's bias-length check (pipeline.cpp:162-164) is implicit: the
 * bias is read as N values. */
typedef struct crt_layer crt_layer;

typedef struct crt_layer_desc {
  int64_t out_features; /* N */
  int64_t in_features;  /* K */
  crt_rotation_spec rotation;
  int32_t bits_w;       /* 4 or 8 (QuantSpec, quant.hpp:15-20) */
  int32_t w_dtype;      /* crt_dtype of W */
} crt_layer_desc;

crt_status crt_layer_prepare(const crt_layer_desc* desc, const void* w, int64_t ldw,
                             const float* bias, void* stream, crt_layer** out);

/* Column-parallel shard of a layer: output channels
 * [rank*N/nranks, (rank+1)*N/nranks) of the full W.
 * Codes and scales equal the corresponding rows of the full layer. */
crt_status crt_layer_prepare_shard(const crt_layer_desc* desc, const void* w,
                                   int64_t ldw, const float* bias, int32_t rank,
                                   int32_t nranks, void* stream, crt_layer** out);

/* f2: a layer prepared and saved by the reference
 * (save_prepared_layer, pipeline.cpp:257-314; loaded there by
 * load_prepared_layer, :288-314).  HOST buffers: codes in the reference
 * layout (bits 4: pack_int4 rows of ceil(K/2) bytes, tensorio.cpp:162-171;
 * bits 8: int8 rows), ld_codes bytes per row; fp32 per-channel scales
 * (weights.scales.crt is f32); optional f64 bias (bias.crt).  Codes are used
 * as given (no rotation / quantisation); INVALID_VALUE if a scale is not
 * positive and finite (quant.cpp:31-35).  Synchronises `stream`. */
crt_status crt_layer_from_codes(const crt_layer_desc* desc, const uint8_t* codes_host,
                                int64_t ld_codes, const float* scales_host,
                                const double* bias_host, void* stream, crt_layer** out);

crt_status crt_layer_destroy(crt_layer* layer);

/* Geometry of a prepared layer (host query). */
crt_status crt_layer_info(const crt_layer* layer, crt_layer_desc* desc_out);

/* Export the prepared weights in the reference layout for parity checks:
 * codes row-major packed like pack_int4 (bits 4) or int8 (bits 8), ld_codes
 * bytes per row; per-channel scales as f32 and/or f64 (nullable). Device. */
crt_status crt_layer_export(const crt_layer* layer, uint8_t* codes, int64_t ld_codes,
                            float* scales_f32, double* scales_f64, void* stream);

/* -------------------------------------------------------------------------
 * K3: int_gemm + dequant -- replaces pipeline.cpp:178-204 (int_gemm, with
 * its CapacityError precheck :184-192) and the dequant loop of forward
 * (pipeline.cpp:224-230).
 *
 *   a_codes   device, K1 output (M rows, lda BYTES per row, bits_a layout)
 *   a_scales  device, M fp32 activation scales
 *   y         device, M x N (ldy ELEMENTS) of bf16 / f32 / int32 per out_kind
 */
crt_status crt_quant_gemm(const uint8_t* a_codes, int64_t lda, const float* a_scales,
                          int32_t bits_a, const crt_layer* layer, int64_t M,
                          int32_t out_kind, void* y, int64_t ldy, void* stream);

/* W4A4 fast path (K3 v3, hardware int4 expansion): K1 with the 4-bit codes
 * stored ONE INT8 PER CODE (values -7..7, same codes as crt_rotate_quant)
 * plus the per-row code sums, and the GEMM that consumes them.  Device
 * buffers; codes M x ld_codes (>= K) bytes, code_sums M int32.
 * crt_quant_gemm_i8 needs 16-byte aligned rows and a layer with 4-bit
 * weights, else UNSUPPORTED (use crt_rotate_quant + crt_quant_gemm). */
crt_status crt_rotate_quant_i8(const void* x, int32_t x_dtype, int64_t M, int64_t K, int64_t ldx,
                               const crt_rotation_spec* rot, uint8_t* codes, int64_t ld_codes,
                               float* scales_f32, int32_t* code_sums, void* stream);
crt_status crt_quant_gemm_i8(const uint8_t* a_codes, int64_t lda, const float* a_scales,
                             const int32_t* code_sums, const crt_layer* layer, int64_t M,
                             int32_t out_kind, void* y, int64_t ldy, void* stream);

/* -------------------------------------------------------------------------
 * Row-parallel (K-sharded) layers -- SURVEY.md 8(e) "K (row-parallel)" and
 * 8(f) row f3 (fc1 column-parallel -> fc2 row-parallel, int32 all-reduce).
 * Rank r of P holds input columns [r*K/P, (r+1)*K/P):
 *   1. crt_rotated_row_absmax on its column shard of X; MAX all-reduce
 *      (exact) -> the global per-row max |y_ref|;
 *   2. crt_rotate_quant_amax with that max: scales and codes equal the
 *      unsharded compute_scales / quantize (quant.cpp:10-52) on its columns;
 *   3. crt_quant_gemm(_i8) with out_kind I32_ACC on a crt_layer_prepare_kshard
 *      layer: partial int_gemm accumulators; SUM all-reduce (int32, exact,
 *      order-free; the caller checks int_gemm's capacity for the full K);
 *   4. crt_dequant: the dequant loop of forward (pipeline.cpp:224-230).
 * The result equals the unsharded forward bit for bit. */

/* K-shard of a layer: the full layer is prepared (per-channel scales over all
 * of K, pipeline.cpp:158-176) and input columns [rank*K/nranks,
 * (rank+1)*K/nranks) of its codes are kept.  SHAPE if K % nranks != 0, if a
 * rotation group would straddle shards (global rotation, K/nranks % n0 != 0)
 * or if an odd 4-bit shard would split a packed byte. */
crt_status crt_layer_prepare_kshard(const crt_layer_desc* desc, const void* w, int64_t ldw,
                                    const float* bias, int32_t rank, int32_t nranks,
                                    void* stream, crt_layer** out);

/* K1 with given exact per-row maxima amax_rows (device, M doubles; +inf ->
 * InvalidValueError at the next crt_device_status, like compute_scales).
 * row_sums != NULL (bits 4 only): codes one int8 per code + per-row code
 * sums (crt_quant_gemm_i8 operand); else the crt_rotate_quant layout. */
crt_status crt_rotate_quant_amax(const void* x, int32_t x_dtype, int64_t M, int64_t K,
                                 int64_t ldx, const crt_rotation_spec* rot,
                                 const double* amax_rows, int32_t bits, uint8_t* codes,
                                 int64_t ld_codes, float* scales_f32, double* scales_f64,
                                 int32_t* row_sums, void* stream);

/* Dequant of int32 accumulators (M x N, ld_acc elements) summed outside K3:
 * y = acc * s_a[m] * s_w[n] + b[n] with the K3 epilogue's fp32 expression
 * (forward, pipeline.cpp:224-230), bf16 / f32 / int32 copy per out_kind. */
crt_status crt_dequant(const int32_t* acc, int64_t ld_acc, int64_t M, const float* a_scales,
                       const crt_layer* layer, int32_t out_kind, void* y, int64_t ldy,
                       void* stream);

/* -------------------------------------------------------------------------
 * a9: forward -- replaces pipeline.cpp:206-233: K1 on x, then K3 against the
 * layer.  bits_a in {4, 8} else INVALID_VALUE (:213-215); x must have
 * in_features columns else SHAPE (:208-212).  The workspace holds the
 * activation codes/scales (no hidden allocation on the forward path). */
typedef struct crt_workspace crt_workspace;

crt_status crt_workspace_create(int64_t max_m, int64_t max_k, crt_workspace** out);
crt_status crt_workspace_destroy(crt_workspace* ws);
/* Non-finite input seen by forwards run with this workspace (its own error
 * word: other callers' inputs never show up here).  Synchronises `stream`;
 * INVALID_VALUE (compute_scales, quant.cpp:16-18) if set, then clears it
 * when reset != 0. */
crt_status crt_workspace_status(crt_workspace* ws, void* stream, int32_t reset);

crt_status crt_forward(const crt_layer* layer, const void* x, int32_t x_dtype,
                       int64_t M, int64_t ldx, int32_t bits_a, int32_t out_kind,
                       void* y, int64_t ldy, crt_workspace* ws, void* stream);

/* forward with HOST buffers: copies x host->device, runs crt_forward and
 * copies y device->host, all on `stream`; synchronises the stream before
 * returning.  x_dev/y_dev are caller-owned device staging buffers. */
crt_status crt_forward_host(const crt_layer* layer, const void* x_host, int32_t x_dtype,
                            int64_t M, int32_t bits_a, int32_t out_kind, void* y_host,
                            void* x_dev, void* y_dev, crt_workspace* ws, void* stream);


/* -------------------------------------------------------------------------
 * Tensor parallelism over NCCL (SURVEY.md 8(b) "Multi-GPU", 8(e)): one
 * process per GPU.  The collectives are NCCL's, resolved at first use from
 * the libnccl.so.2 already loaded in the process (e.g. PyTorch's) or the
 * system one -- so a communicator made by the caller's NCCL may be passed.
 * `comm` is an ncclComm_t passed as void*.  NCCL missing or a failing
 * collective -> CRT_ERR_NCCL.
 *
 *   CRT_TP_COLUMN  rank r of P owns output channels [r*N/P, (r+1)*N/P) (the
 *                  full layer's rows: codes, scales, bias); x is the full
 *                  [M, K] input on every rank.  crt_tp_forward runs K1 + K3
 *                  on the shard and, with gather != 0, all-gathers the shards
 *                  into y [M, N] (rank-major NCCL buffer interleaved by a
 *                  kernel); gather == 0 leaves the rank's [M, N/P] columns in
 *                  y -- the input shard of a following CRT_TP_ROW layer.
 *   CRT_TP_ROW     rank r owns input features [r*K/P, (r+1)*K/P) (per-channel
 *                  scales over all of K); x is the rank's [M, K/P] shard.
 *                  crt_tp_forward: exact per-row max |group_rotate| of the
 *                  shard, MAX all-reduce (M doubles), K1 with the global max
 *                  (codes = the unsharded ones), K3 partial int32
 *                  accumulators, SUM all-reduce (exact, order-free), dequant
 *                  -> y [M, N] on every rank.
 * Both equal the single-GPU forward bit for bit. */
typedef enum crt_tp_mode { CRT_TP_COLUMN = 1, CRT_TP_ROW = 2 } crt_tp_mode;

/* NCCL bootstrap for hosts without their own: a 128-byte ncclUniqueId made
 * on one rank and shared with the others by any transport, then one
 * communicator per rank on the CURRENT device. */
crt_status crt_nccl_unique_id(uint8_t* id128);
crt_status crt_nccl_comm_create(int32_t nranks, int32_t rank, const uint8_t* id128, void** comm);
crt_status crt_nccl_comm_destroy(void* comm);
/* rank / size of a communicator (ncclCommUserRank / ncclCommCount). */
crt_status crt_nccl_comm_info(void* comm, int32_t* rank, int32_t* nranks);

/* The rank's shard of a layer (rank and P from `comm`); SHAPE if N (column)
 * or K (row) is not divisible by P, or a rotation group would straddle
 * K shards. */
crt_status crt_tp_layer_prepare(const crt_layer_desc* desc, const void* w, int64_t ldw,
                                const float* bias, int32_t mode, void* comm, void* stream,
                                crt_layer** out);
/* Forward of a crt_tp_layer_prepare layer (see above); W4A4 / W8A8 as the
 * layer's bits.  Collective: every rank of `comm` must call it.  Scratch for
 * the gathered / reduced buffers is the workspace's (grown on first use). */
crt_status crt_tp_forward(const crt_layer* layer, const void* x, int32_t x_dtype, int64_t M,
                          int64_t ldx, int32_t out_kind, void* y, int64_t ldy, int32_t gather,
                          crt_workspace* ws, void* comm, void* stream);

/* -------------------------------------------------------------------------
 * Diagnostics. */
const char* crt_last_error(void);
/* Synchronises `stream`, returns CRT_ERR_INVALID_VALUE if a kernel saw a
 * non-finite input since the last reset (reference: compute_scales throws
 * InvalidValueError, quant.cpp:16-18), then clears the word if reset != 0. */
crt_status crt_device_status(void* stream, int32_t reset);
/* Number of CUDA kernels this library has launched (process lifetime). */
int64_t crt_launch_count(void);

/* Dev aid (not part of the reference surface): when buf is non-null, the
 * K1 team kernel records %globaltimer stamps into it, 26 uint64 words per
 * CTA (kernel start, after the PDL wait, then per row: data ready, team
 * barrier passed, row done, for the first 8 rows).  NULL turns it off. */
void crt_debug_k1_trace(void* buf);  /* effective in builds with -DCRT_K1_TRACE */
/* Dev aid: K3 (v3) clock64 stamps of the first CTA pair's leader CTA into
 * buf (11 x 4096 uint64: per stage and per tile, see k3_gemm_v3.cu).  NULL
 * turns it off. */
void crt_debug_k3_trace(void* buf);  /* effective in builds with -DCRT_K3_TRACE */
int32_t crt_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* CRT_CONVLINEAR4BIT_H_ */
