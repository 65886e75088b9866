// Instantiations of the fused / persistent NMF kernels for K = 16 (see nmf_fused.cuh).
#include "nmf_fused.cuh"

namespace hsnct {
template cudaError_t fused_launch_k<16>(const Geometry&, const NmfPlan&, const NmfWs&, float*, const float*, int,
                                        unsigned*, cudaStream_t);
template cudaError_t persist_launch_k<16>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int,
                                          double*, unsigned*, unsigned*, cudaStream_t);
}  // namespace hsnct
