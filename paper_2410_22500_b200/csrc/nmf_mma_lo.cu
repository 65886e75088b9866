// Explicit instantiation of the mma.sync row pass for K = 1..8 (parallel nvcc units).
#include "nmf_mma.cuh"

namespace hsnct {
template cudaError_t mma_launch_k<1, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                             double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<1, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                            double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<2, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                             double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<2, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                            double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<3, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                             double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<3, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                            double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<4, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                             double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<4, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                            double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<5, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                             double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<5, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                            double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<6, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                             double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<6, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                            double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<7, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                             double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<7, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                            double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<8, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                             double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k<8, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                            double*, unsigned*, unsigned*, cudaStream_t);
}  // namespace hsnct
