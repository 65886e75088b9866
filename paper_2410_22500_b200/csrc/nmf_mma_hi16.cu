// Explicit instantiation of the 16-warp mma.sync row pass for K = 9..16 (parallel nvcc units).
#include "nmf_mma.cuh"

namespace hsnct {
template cudaError_t mma_launch_k16<9, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                               double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k16<9, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                               double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k16<10, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                               double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k16<10, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                               double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k16<11, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                               double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k16<11, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                               double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k16<12, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                               double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k16<12, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                               double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k16<13, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                               double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k16<13, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                               double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k16<14, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                               double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k16<14, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                               double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k16<15, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                               double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k16<15, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                               double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k16<16, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                               double*, unsigned*, unsigned*, cudaStream_t);
template cudaError_t mma_launch_k16<16, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, int, int,
                                               double*, unsigned*, unsigned*, cudaStream_t);
}  // namespace hsnct
