// Explicit instantiation of the K1 kernels for one (input dtype, bits)
// pair; split so the kernel variants compile in parallel.
#include "k1_kernels.cuh"

namespace crt {
template cudaError_t k1_dispatch<true, 4>(const K1Args&, int, cudaStream_t, int64_t*);
template cudaError_t k1_exact_launch<true, 4>(const K1Args&, cudaStream_t);
}  // namespace crt
