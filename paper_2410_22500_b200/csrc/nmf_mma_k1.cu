// Instantiation of the tensor-core NMF kernel for K = 1 (see nmf_mma.cuh).
#include "nmf_mma.cuh"

namespace hsnct {
template cudaError_t mma_launch_k<1>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, double*,
                                      unsigned*, unsigned*, cudaStream_t);
}  // namespace hsnct
