// common.cuh -- shared device helpers for the sm_100a ConvLinear4bit kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <atomic>
#include <mutex>

namespace crt {

enum : int { kRotNone = 0, kRotSylvester = 1, kRotRegular = 2 };

// Device error word (passed by pointer): set by a kernel that sees a
// non-finite input -- the reference throws InvalidValueError from
// compute_scales (quant.cpp:16-18).
__device__ __forceinline__ void flag_invalid_value(int* err) { atomicOr(err, 1); }

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---- packed fp32x2 arithmetic (FADD2 / FFMA2 on sm_100) -------------------
__device__ __forceinline__ uint64_t f2_bits(float2 a) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
  return r;
}
__device__ __forceinline__ float2 f2_from(uint64_t r) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
__device__ __forceinline__ float2 f2_add(float2 a, float2 b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
  return f2_from(r);
}
// a * b + c, one rounding per lane
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
  return f2_from(r);
}

// NaN-propagating max of |a|, |b| and c (FMNMX3.NAN with abs modifiers).
__device__ __forceinline__ float max3_abs(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(fabsf(a)), "f"(fabsf(b)), "f"(c));
  return r;
}
__device__ __forceinline__ float max_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// 256-bit streaming load (LDG.E.NA.ENL2.256): 8 words, no L1 allocation.
__device__ __forceinline__ void ld_nc_v8(const void* p, uint32_t (&v)[8]) {
  asm("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
        "=r"(v[6]), "=r"(v[7])
      : "l"(p));
}

// 256-bit store (STG.E.ENL2.256): 8 words at a 32-byte aligned address.
__device__ __forceinline__ void st_v8(void* p, uint4 lo, uint4 hi) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(lo.x), "r"(lo.y),
               "r"(lo.z), "r"(lo.w), "r"(hi.x), "r"(hi.y), "r"(hi.z), "r"(hi.w)
               : "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- shared memory, mbarriers, bulk async copies ---------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 1-D bulk copy global -> shared (TMA engine, UBLKCP), completion counted in
// bytes on `bar`.  dst/src 16-byte aligned, bytes a multiple of 16.  The
// source is streamed (read once): evict-first in L2.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .b64 pol;\n"
      "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], pol;\n"
      "}\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Sign of entry (k, j) of the order-4^L regular Hadamard matrix:
// H = H4^{(x)L} with H4[a][b] = -1 iff a + b == 3 (hadamard.cpp:97-102,119);
// per base-4 digit, a + b == 3  <=>  (a ^ b) == 3.
__device__ __forceinline__ bool regular_negative(uint32_t k, uint32_t j) {
  uint32_t d = k ^ j;
  return (__popc(d & (d >> 1) & 0x55555555u) & 1u) != 0;
}
// Sylvester (hadamard.cpp:70-89): H[k][j] = (-1)^popcount(k & j).
__device__ __forceinline__ bool sylvester_negative(uint32_t k, uint32_t j) {
  return (__popc(k & j) & 1u) != 0;
}

// ---------------------------------------------------------------------------
// Host-side launch helpers, safe for concurrent callers and several devices
// in one process (layer handles may be used from many threads, convlinear4bit.h).
// ---------------------------------------------------------------------------
constexpr int kMaxDevices = 64;

inline int device_sm_count() {
  static std::atomic<int> cache[kMaxDevices];
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& slot = cache[dev % kMaxDevices];
  int v = slot.load(std::memory_order_relaxed);
  if (v == 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    slot.store(v, std::memory_order_relaxed);
  }
  return v;
}

// Per (kernel, device): the largest dynamic shared-memory size requested so
// far.  The attribute only ever grows (under the mutex), so a concurrent
// caller can never lower a limit another launch relies on.
struct SmemAttr {
  std::atomic<size_t> granted[kMaxDevices];
  std::mutex mu;
};
template <typename Kernel>
inline cudaError_t ensure_dyn_smem(Kernel kern, size_t bytes, SmemAttr& c, bool max_carveout) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<size_t>& g = c.granted[dev % kMaxDevices];
  if (g.load(std::memory_order_acquire) >= bytes) return cudaSuccess;
  std::lock_guard<std::mutex> lock(c.mu);
  if (g.load(std::memory_order_relaxed) >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess && max_carveout)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e == cudaSuccess) g.store(bytes, std::memory_order_release);
  return e;
}

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL).  A kernel launched with
// launch_pdl may start (prologue: barriers, TMEM, descriptor prefetch) while
// its stream predecessor drains; every thread calls griddep_wait() before
// its first global-memory access (read OR write: forward reuses the
// workspace, so the next K1 must not overwrite codes the previous K3 still
// reads).  griddep_launch() lets this kernel's own successor be scheduled.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("CRT_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

}  // namespace crt
