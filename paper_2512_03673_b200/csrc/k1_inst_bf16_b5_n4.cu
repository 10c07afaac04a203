// Explicit instantiation of the K1 fast kernels for one (input dtype, bits,
// N0) triple.  Generated layout: one translation unit per triple keeps each
// ptxas module small (a single module with all ~100 variants crashes ptxas
// 12.9) and lets the variants compile in parallel.
#include "k1_kernels.cuh"

namespace crt {
template cudaError_t launch_any<4, false, 5>(const K1Args&, cudaStream_t, int64_t*);
}  // namespace crt
