// k1_rotate_quant.h -- host interface of K1 (rotate + quantize + pack).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace crt {

struct K1Args {
  const void* x;      // M x K (row stride ldx elements), bf16 or f32
  int64_t ldx;
  int64_t M;
  int64_t K;
  int64_t group;      // resolved group size (K for global); 1 for kind none
  int64_t rot_cols;   // columns covered by whole groups (identity tail beyond)
  int32_t kind;       // kRotNone / kRotSylvester / kRotRegular
  int32_t team_warps; // filled by the plan
  int32_t stages;     // shared-memory row ring depth (launcher)
  int32_t chunks;     // 16-element chunks per lane (even; filled by the plan)
  uint8_t* codes;     // M rows x ldc bytes
  int64_t ldc;
  float* s32;         // nullable
  double* s64;        // nullable
  double* amax;       // nullable: exact per-row max |y_ref| (outlier_amplitude)
  int32_t* rowsum;    // nullable: per-row sum of the int8 codes (bits 5 layout)
  const double* amax_in;  // nullable: use this exact per-row max |y_ref| for the scale
                          // (row-parallel: the MAX all-reduce of the shards' maxima)
  int* err;           // device error word
  unsigned long long* trace;  // nullable dev aid: per-CTA globaltimer stamps (k1_team)
};

// Dev aid (crt_debug_k1_trace): when set, k1_team records globaltimer
// stamps per CTA into this device buffer (kK1TraceWords words per CTA).
void set_k1_trace(unsigned long long* buf);
unsigned long long* k1_trace();

struct K1Plan {
  bool fast;
  int C;  // 16-element chunks per lane (even)
  int W;  // warps per row team
};

K1Plan plan_k1(int64_t K, int64_t n0, int kind, bool identity_tail, bool f32, int bits,
               const void* x, int64_t ldx, const void* codes, int64_t ldc);

cudaError_t launch_k1(const K1Args& a, const K1Plan& p, bool f32, int bits, cudaStream_t st,
                      int64_t* launches);

// Would a fast-plan K1 with these arguments run the team kernel (which
// skips the code stores when a.codes is null: amax-only launches)?
bool k1_team_eligible(const K1Args& a, bool f32, int bits);

}  // namespace crt
