// Explicit instantiation of the mma.sync row pass for K = 9..16 (parallel nvcc units).
#include "nmf_mma.cuh"

namespace hsnct {
template cudaError_t mma_launch_k<9, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                             double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<9, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                            double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<10, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                             double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<10, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                            double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<11, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                             double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<11, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                            double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<12, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                             double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<12, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                            double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<13, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                             double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<13, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                            double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<14, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                             double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<14, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                            double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<15, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                             double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<15, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                            double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<16, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                             double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<16, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                            double*, unsigned*, unsigned*, cudaStream_t);
}  // namespace hsnct
