// K1 dispatch (N0 -> fast-kernel instantiation in k1_inst_*.cu) and the
// exact kernel instantiations.
#include "k1_kernels.cuh"

namespace crt {
extern template cudaError_t launch_any<1, false, 4>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<4, false, 4>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<16, false, 4>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<64, false, 4>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<256, false, 4>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<1, false, 8>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<4, false, 8>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<16, false, 8>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<64, false, 8>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<256, false, 8>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<1, true, 4>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<4, true, 4>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<16, true, 4>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<64, true, 4>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<256, true, 4>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<1, true, 8>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<4, true, 8>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<16, true, 8>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<64, true, 8>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<256, true, 8>(const K1Args&, cudaStream_t, int64_t*);
bool k1_team_eligible(const K1Args& a, bool f32, int bits) { return k1_team_ok(a, f32, bits); }

template cudaError_t k1_dispatch<false, 4>(const K1Args&, int, cudaStream_t, int64_t*);
template cudaError_t k1_exact_launch<false, 4>(const K1Args&, cudaStream_t);
template cudaError_t k1_dispatch<false, 8>(const K1Args&, int, cudaStream_t, int64_t*);
template cudaError_t k1_exact_launch<false, 8>(const K1Args&, cudaStream_t);
template cudaError_t k1_dispatch<true, 4>(const K1Args&, int, cudaStream_t, int64_t*);
template cudaError_t k1_exact_launch<true, 4>(const K1Args&, cudaStream_t);
template cudaError_t k1_dispatch<true, 8>(const K1Args&, int, cudaStream_t, int64_t*);
template cudaError_t k1_exact_launch<true, 8>(const K1Args&, cudaStream_t);
extern template cudaError_t launch_any<1, false, 5>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<4, false, 5>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<16, false, 5>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<64, false, 5>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<256, false, 5>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<1, true, 5>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<4, true, 5>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<16, true, 5>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<64, true, 5>(const K1Args&, cudaStream_t, int64_t*);
extern template cudaError_t launch_any<256, true, 5>(const K1Args&, cudaStream_t, int64_t*);
template cudaError_t k1_dispatch<false, 5>(const K1Args&, int, cudaStream_t, int64_t*);
template cudaError_t k1_exact_launch<false, 5>(const K1Args&, cudaStream_t);
template cudaError_t k1_dispatch<true, 5>(const K1Args&, int, cudaStream_t, int64_t*);
template cudaError_t k1_exact_launch<true, 5>(const K1Args&, cudaStream_t);
}  // namespace crt
