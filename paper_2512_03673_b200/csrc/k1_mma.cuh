#pragma once
// k1_mma.cuh -- K1 with the group rotation on the tensor cores (bf16 input,
// N0 in {4, 16}).  Included by k1_kernels.cuh.
//
// The rotation of a 16-element group is a 16x16 matrix product.  A warp takes
// a row 256 elements (16 groups) at a time: ldmatrix loads the tile from the
// shared-memory row copy as the A operand (16 groups x 16 elements, bf16) and
// two mma.sync.m16n8k16 (bf16 x bf16 -> fp32) multiply it by H (N0 = 16:
// regular H16; N0 = 4: blockdiag of four H4) whose columns are permuted so
// that lane j of each quad receives elements 4j..4j+3 of its two groups --
// two packed code bytes per group, stored as one 16-bit word.  This replaces
// the bf16 unpack and the butterflies (2.75 of ~11 CUDA-core instructions
// per element) with 3 instructions per 256 elements per warp.
//
// Certification: the tensor core's fp32 accumulation is not correctly
// rounded (tools/probes/mma_accum_probe.cu measured at most 4.8 * 2^-23 *
// max|x| over 16.7M dot products, exponent spans up to 2^80); the bound used
// is 64 * 2^-23 * max|x| <= 64 * 2^-23 * A (max|x_k| <= max_j |y_j| for the
// unnormalised regular Hadamard, x = H^T y / N0).  Row-max candidates and
// near-ties are settled with the exact double sum (y_exact_dbl), never with
// the tensor-core value.

namespace crt {
namespace {

// Exact reference value of element e of the group inside 16-element chunk
// `chunk` (bf16 input, N0 <= 16): the group's terms summed in double are
// exact (any order) when 1 + log2(N0) + span + 8 <= 53; otherwise the
// reference's sequential loop.
template <int N0>
__device__ __noinline__ double y_exact_dbl(const void* row, int64_t chunk, int e) {
  const int g0 = e & ~(N0 - 1);
  const uint32_t jj = (uint32_t)(e - g0);
  const uint16_t* p =
      reinterpret_cast<const uint16_t*>(reinterpret_cast<const char*>(row) + chunk * 32) + g0;
  uint32_t w[N0 / 2];
  if constexpr (N0 == 16) {
    const uint4 a0 = reinterpret_cast<const uint4*>(p)[0];
    const uint4 a1 = reinterpret_cast<const uint4*>(p)[1];
    w[0] = a0.x; w[1] = a0.y; w[2] = a0.z; w[3] = a0.w;
    w[4] = a1.x; w[5] = a1.y; w[6] = a1.z; w[7] = a1.w;
  } else {
    const uint2 a0 = reinterpret_cast<const uint2*>(p)[0];
    w[0] = a0.x; w[1] = a0.y;
  }
  int emin = 1 << 20, emax = -1, bad = 0;
  double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
  for (int i = 0; i < N0; ++i) {
    const uint32_t bits = (i & 1) ? (w[i >> 1] & 0xFFFF0000u) : (w[i >> 1] << 16);
    const float x = __uint_as_float(bits);
    const int ex = (int)((bits >> 23) & 0xFFu);
    const bool nz = (bits & 0x7FFFFFFFu) != 0;
    bad |= (nz && (ex == 0 || ex == 255)) ? 1 : 0;
    emin = nz ? min(emin, ex) : emin;
    emax = nz ? max(emax, ex) : emax;
    const double t = regular_negative((uint32_t)i, jj) ? -(double)x : (double)x;
    if (i & 1) acc1 += t;
    else acc0 += t;
  }
  constexpr int L2 = N0 == 4 ? 2 : 4;
  if (!bad && (emax < 0 || 1 + L2 + (emax - emin) + 8 <= 53))
    return (acc0 + acc1) * (N0 == 4 ? 0.5 : 0.25);
  return y_ref<false>(row, chunk * 16 + e, N0, kRotRegular, INT64_MAX);
}

// B fragments of H for the two m16n8k16 MMAs (columns permuted, see above):
// MMA h (0, 1) column n computes output element 4*(n/2) + 2*h + (n%2).
// [N0 == 16][lane][h*2 + r], filled once by the launcher (mma_h_table)
__device__ uint4 g_k1_hfrag[2][32];

template <int N0>
__device__ __forceinline__ void mma_h_fragments_compute(uint32_t (&b)[2][2]) {
  const int lane = threadIdx.x & 31;
  const int n = lane >> 2, k0 = 2 * (lane & 3);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j = 4 * (n >> 1) + 2 * h + (n & 1);  // output element of this column
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      uint32_t v = 0;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int k = k0 + 8 * r + u;
        uint16_t bits = 0;  // bf16 0
        if (N0 == 16 || (k >> 2) == (j >> 2))
          bits = regular_negative((uint32_t)(N0 == 16 ? k : (k & 3)),
                                  (uint32_t)(N0 == 16 ? j : (j & 3)))
                     ? 0xBF80
                     : 0x3F80;
        v |= (uint32_t)bits << (16 * u);
      }
      b[h][r] = v;
    }
  }
}

// One 256-element tile: D[h] = 16 groups x 8 permuted outputs.  Lane (g, j)
// = (lane/4, lane%4) receives: d[h][0..1] = group g, elements 4j+2h, +1;
// d[h][2..3] = group g+8, same elements.
template <int N0>
__global__ void k1_mma_table_init() {
  uint32_t b[2][2];
  mma_h_fragments_compute<N0>(b);
  g_k1_hfrag[N0 == 16][threadIdx.x & 31] = make_uint4(b[0][0], b[0][1], b[1][0], b[1][1]);
}

__device__ __forceinline__ void mma_tile(uint32_t tile_saddr, const uint32_t (&b)[2][2],
                                         float (&d)[2][4]) {
  const int lane = threadIdx.x & 31;
  const int m = lane >> 3;  // ldmatrix: lane supplies row (lane&7) of matrix m
  const uint32_t addr = tile_saddr + (uint32_t)((((m & 1) << 3) | (lane & 7)) * 32 + (m >> 1) * 16);
  uint32_t a0, a1, a2, a3;
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
               : "r"(addr));
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    d[h][0] = d[h][1] = d[h][2] = d[h][3] = 0.f;
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[h][0]), "+f"(d[h][1]), "+f"(d[h][2]), "+f"(d[h][3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b[h][0]), "r"(b[h][1]));
  }
}

__device__ __forceinline__ float tile_absmax(const float (&d)[2][4]) {
  const float m0 = max3_abs(d[0][0], d[0][1], max3_abs(d[0][2], d[0][3], 0.f));
  return max3_abs(d[1][0], d[1][1], max3_abs(d[1][2], d[1][3], m0));
}

// value / element index of slot (h, q) of a tile for lane (g, j)
__device__ __forceinline__ int slot_elem(int h, int q) {  // element within the 256-tile
  const int lane = threadIdx.x & 31;
  const int g = (lane >> 2) + ((q >> 1) << 3);
  return g * 16 + 4 * (lane & 3) + 2 * h + (q & 1);
}

}  // namespace

constexpr int kK1MThreads = 256;
constexpr int kK1MMinBlocks = 3;

template <int N0, int BITS>
__global__ void __launch_bounds__(kK1MThreads, kK1MMinBlocks) k1_mma(K1Args a) {
  constexpr int QMAX = BITS == 8 ? 127 : 7;
  __shared__ TeamScratch ts;
  __shared__ uint64_t full_bar[kK1MaxTeams][kK1MaxStages];
  extern __shared__ __align__(128) uint8_t k1_ring[];

  const int W = a.team_warps;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int team = warp / W;
  const int w = warp - team * W;
  const int teams = blockDim.x / (32 * W);
  const int ntiles = (int)(a.K / 256);
  const int S = a.stages;
  const uint32_t row_bytes = (uint32_t)(a.K * 2);
  const bool leader = (w == 0 && lane == 0);
  const int64_t row0 = (int64_t)blockIdx.x * teams + team;
  const int64_t row_step = (int64_t)gridDim.x * teams;
  uint8_t* ring = k1_ring + (size_t)team * S * row_bytes;

  if (threadIdx.x == 0) {
    for (int t = 0; t < teams; ++t)
      for (int s = 0; s < S; ++s) mbar_init(&full_bar[t][s], 1);
    mbar_init_fence();
  }
  __syncthreads();
  if (leader) {
    for (int s = 0; s < S; ++s) {
      const int64_t r = row0 + (int64_t)s * row_step;
      if (r >= a.M) break;
      mbar_arrive_expect_tx(&full_bar[team][s], row_bytes);
      bulk_g2s(ring + (size_t)s * row_bytes, reinterpret_cast<const char*>(a.x) + r * a.ldx * 2,
               row_bytes, &full_bar[team][s]);
    }
  }
  uint32_t bfr[2][2];
  {
    const uint4 f = g_k1_hfrag[N0 == 16][lane];
    bfr[0][0] = f.x;
    bfr[0][1] = f.y;
    bfr[1][0] = f.z;
    bfr[1][1] = f.w;
  }
  const float rk = N0 == 4 ? 0.5f : 0.25f;
  constexpr float kBound = 64.0f * 1.1920928955078125e-7f * 1.01f;  // B = kBound * A

  int it = 0;
  for (int64_t row = row0; row < a.M; row += row_step, ++it) {
    const int stage = it % S;
    mbar_wait(&full_bar[team][stage], (uint32_t)((it / S) & 1));
    const uint8_t* rowb = ring + (size_t)stage * row_bytes;
    const uint32_t rows = smem_u32(rowb);

    // ---- pass 1: rotate (tensor cores) + absmax, best / 2nd tile ------------
    float lmax = 0.f, lmax_nan = 0.f, m2 = 0.f;
    int bt = w;
    int t = w;
#pragma unroll 1
    for (; t + W < ntiles; t += 2 * W) {  // two tiles per iteration (ILP)
      float d0[2][4], d1[2][4];
      mma_tile(rows + (uint32_t)t * 512u, bfr, d0);
      mma_tile(rows + (uint32_t)(t + W) * 512u, bfr, d1);
      const float ma = tile_absmax(d0), mb = tile_absmax(d1);
      lmax_nan = max_nan(lmax_nan, max_nan(ma, mb));
      const float m = fmaxf(ma, mb);
      const int tm = ma >= mb ? t : t + W;
      const float mlo = fminf(ma, mb);
      if (m > lmax) {
        m2 = fmaxf(lmax, mlo);
        lmax = m;
        bt = tm;
      } else {
        m2 = fmaxf(m2, m);
      }
    }
    if (t < ntiles) {
      float d[2][4];
      mma_tile(rows + (uint32_t)t * 512u, bfr, d);
      const float m = tile_absmax(d);
      lmax_nan = max_nan(lmax_nan, m);
      if (m > lmax) {
        m2 = lmax;
        lmax = m;
        bt = t;
      } else {
        m2 = fmaxf(m2, m);
      }
    }
    const float A32 = team_max_nan(lmax_nan, &ts, team, w, W);
    const bool slow_row = !(A32 <= 3.0e38f);
    const float B = kBound * A32;
    double amax_ref = 0.0;
    if (!slow_row) {
      if (A32 == 0.f) {
        amax_ref = 0.0;
      } else {
        const float thr = (A32 - 2.f * B) * (1.0f - 1e-6f);
        double cmax = 0.0;
        // candidates |y| >= thr: a lane's lie in its best tile unless its
        // second-best tile also reaches thr.  ldmatrix / mma.sync are
        // warp-collective, so the tile loop is warp-uniform and each lane
        // settles only its own candidates (exact double sums, lane-local).
        const bool has = lmax >= thr;
        const bool all = m2 >= thr;
        if (__any_sync(0xffffffffu, has)) {
#pragma unroll 1
          for (int t = w; t < ntiles; t += W) {
            const bool need = has && (all || t == bt);
            if (!__any_sync(0xffffffffu, need)) continue;
            float d[2][4];
            mma_tile(rows + (uint32_t)t * 512u, bfr, d);
            if (need) {
#pragma unroll
              for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  if (fabsf(d[h][q]) >= thr) {
                    const int e = t * 256 + slot_elem(h, q);
                    cmax = fmax(cmax, fabs(y_exact_dbl<N0>(rowb, e >> 4, e & 15)));
                  }
            }
          }
        }
        amax_ref = team_max_d(cmax, &ts, team, w, W);
      }
    } else {
      amax_ref = team_max_d(k1_slow_row_amax<false>(rowb, (ntiles * 16 + W * 32 - 1) / (W * 32),
                                                     W, w, a.K / 16, N0, kRotRegular, a.K),
                            &ts, team, w, W);
    }
    const bool invalid = !isfinite(amax_ref);
    const double s = invalid ? 1.0 : (amax_ref == 0.0 ? 1.0 : amax_ref / (double)QMAX);
    if (invalid && lane == 0 && w == 0) flag_invalid_value(a.err);

    uint8_t* crow = a.codes + row * a.ldc;
    if (!slow_row) {
      // ---- pass 2: rotate again, certified quantisation, pack, store --------
      const float inv = amax_ref == 0.0 ? rk : (rk * (float)QMAX) * __frcp_rn((float)amax_ref);
      const float margin = B * (inv * 1.05f) + (float)(QMAX + 4) * 2.384185791015625e-7f + 1e-9f;
      const float thr = 0.5f - margin;
      const float mg = __uint_as_float(kMagic23 + (BITS == 4 ? 8u : 0u));
      const float2 iv = make_float2(inv, inv);
      const float2 cc = make_float2(mg, mg);
      const int g = lane >> 2, j = lane & 3;
#pragma unroll 1
      for (int t = w; t < ntiles; t += W) {
        float d[2][4];
        mma_tile(rows + (uint32_t)t * 512u, bfr, d);
        uint32_t tb[2][4];
        float em = 0.f;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int q = 0; q < 4; q += 2) {
            const float2 v = make_float2(d[h][q], d[h][q + 1]);
            const float2 tt = __ffma2_rn(v, iv, cc);
            const float2 nr = __ffma2_rn(tt, make_float2(-1.f, -1.f), cc);
            const float2 e = __ffma2_rn(v, iv, nr);
            em = max3_abs(e.x, e.y, em);
            tb[h][q] = __float_as_uint(tt.x);
            tb[h][q + 1] = __float_as_uint(tt.y);
          }
        uint8_t* tcodes = crow + (int64_t)t * (BITS == 4 ? 128 : 256);
#pragma unroll
        for (int gg = 0; gg < 2; ++gg) {  // group g (q 0,1) and g + 8 (q 2,3)
          const int q = 2 * gg;
          if constexpr (BITS == 4) {
            // bytes: (4j, 4j+1) from h = 0, (4j+2, 4j+3) from h = 1
            const uint32_t b0 = tb[0][q + 1] * 16u + tb[0][q];
            const uint32_t b1 = tb[1][q + 1] * 16u + tb[1][q];
            const uint16_t v16 = (uint16_t)((__byte_perm(b0, b1, 0x0040) ^ 0x8888u) & 0xFFFFu);
            *reinterpret_cast<uint16_t*>(tcodes + (g + 8 * gg) * 8 + 2 * j) = v16;
          } else {
            const uint32_t v32 = __byte_perm(__byte_perm(tb[0][q], tb[0][q + 1], 0x0040),
                                             __byte_perm(tb[1][q], tb[1][q + 1], 0x0040), 0x5410);
            *reinterpret_cast<uint32_t*>(tcodes + (g + 8 * gg) * 16 + 4 * j) = v32;
          }
        }
        if (!(em <= thr)) {  // rare: near-ties -> exact decisions, owner rewrites
#pragma unroll 1
          for (int h = 0; h < 2; ++h)
#pragma unroll 1
            for (int q = 0; q < 4; ++q) {
              const float v = d[h][q];
              const float ex = fmaf(v, inv, mg - __uint_as_float(tb[h][q]));
              if (fabsf(ex) <= thr) continue;
              const int e = t * 256 + slot_elem(h, q);
              const int code = exact_code(y_exact_dbl<N0>(rowb, e >> 4, e & 15), s, QMAX);
              if constexpr (BITS == 4) {
                uint8_t* bp = crow + (e >> 1);
                const uint8_t old = *bp;
                *bp = (e & 1) ? (uint8_t)((old & 0x0F) | ((code & 0x0F) << 4))
                              : (uint8_t)((old & 0xF0) | (code & 0x0F));
              } else {
                crow[e] = (uint8_t)code;
              }
            }
        }
      }
    } else {
      k1_slow_row_codes<false, BITS>(rowb, crow, (ntiles * 16 + W * 32 - 1) / (W * 32), W, w,
                                     a.K / 16, invalid, s, N0, kRotRegular, a.K);
    }
    if (w == 0 && lane == 0) {
      if (a.s32) a.s32[row] = (float)s;
      if (a.s64) a.s64[row] = s;
      if (a.amax) a.amax[row] = amax_ref;
    }
    if (W == 1) __syncwarp();
    else named_bar_sync(1 + team, W * 32);
    if (leader) {
      const int64_t r = row + (int64_t)S * row_step;
      if (r < a.M) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&full_bar[team][stage], row_bytes);
        bulk_g2s(ring + (size_t)stage * row_bytes,
                 reinterpret_cast<const char*>(a.x) + r * a.ldx * 2, row_bytes,
                 &full_bar[team][stage]);
      }
    }
  }
}

}  // namespace crt

namespace crt {

template <int N0, int BITS>
cudaError_t launch_mma(const K1Args& a0, cudaStream_t st, int64_t* launches) {
  const int num_sms = device_sm_count();
  K1Args a = a0;
  const int ntiles = (int)(a.K / 256);
  int W = (ntiles + 11) / 12;  // ~12 tiles (3072 elements) per warp per row
  if (W > 8) W = 8;
  a.team_warps = W;
  const size_t rb = (size_t)a.K * 2;
  int teams = kK1MThreads / (W * 32);
  teams = teams < 1 ? 1 : (teams > kK1MaxTeams ? kK1MaxTeams : teams);
  const int64_t rows_per_sm = (a.M + num_sms - 1) / num_sms;
  if (teams > rows_per_sm) teams = (int)(rows_per_sm < 1 ? 1 : rows_per_sm);
  const size_t budget = (size_t)216 * 1024 / kK1MMinBlocks;
  int S = (int)(budget / ((size_t)teams * rb));
  if (S > kK1MaxStages) S = kK1MaxStages;
  if (S < 1) return cudaErrorInvalidValue;  // caller falls back
  a.stages = S;
  const int threads = teams * W * 32;
  const size_t smem = (size_t)teams * S * rb;
  auto kern = k1_mma<N0, BITS>;
  {  // the device-side fragment table, once per device (complete before use)
    static std::atomic<bool> table[kMaxDevices];
    static std::mutex mu;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!table[dev % kMaxDevices].load(std::memory_order_acquire)) {
      std::lock_guard<std::mutex> lock(mu);
      if (!table[dev % kMaxDevices].load(std::memory_order_relaxed)) {
        k1_mma_table_init<N0><<<1, 32, 0, st>>>();
        ++*launches;
        const cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return e;
        table[dev % kMaxDevices].store(true, std::memory_order_release);
      }
    }
  }
  static SmemAttr attr;
  {
    const cudaError_t e = ensure_dyn_smem(kern, smem, attr, true);
    if (e != cudaSuccess) return e;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (a.M + teams - 1) / teams;
  int64_t grid = (int64_t)num_sms * per_sm;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, threads, smem, st>>>(a);
  ++*launches;
  return cudaGetLastError();
}

// The tensor-core path applies: bf16 input, regular rotation with N0 4 / 16,
// whole 256-element tiles, 16-byte aligned rows and codes.
inline bool mma_path_ok(const K1Args& a, int n0, bool f32) {
  // Opt-in (CRT_K1_MMA=1): parity-exact, but measured slower than the
  // CUDA-core kernels on B200 (K=3072: 37.9 vs 24.6 us; K=12288: 101 vs
  // 65 us): legacy mma.sync is latency-bound here.
  static const bool on = [] {
    const char* e = getenv("CRT_K1_MMA");
    return e && e[0] == '1';
  }();
  if (!on || f32 || a.amax_in || a.kind != kRotRegular || (n0 != 4 && n0 != 16)) return false;
  if (a.K % 256 != 0 || a.rot_cols != a.K) return false;
  if ((uintptr_t)a.x % 16 || (a.ldx * 2) % 16 || (uintptr_t)a.codes % 16 || a.ldc % 16) return false;
  return (size_t)a.K * 2 <= (size_t)216 * 1024 / kK1MMinBlocks;
}

}  // namespace crt
