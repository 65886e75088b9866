// Device helpers shared by the NMF kernels (nmf_fused.cuh, nmf_mma.cuh): mbarriers, bulk
// copies, proxy fences, named barriers, fixed-order reductions, the grid barrier.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hsnct {
namespace {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// mbar_wait on a shared-window address computed once (keeps the address in a register
// instead of re-deriving it from the generic pointer in the hot loop)
__device__ __forceinline__ void mbar_wait_s(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// Warm L2 with `bytes` (multiple of 16) at global address src, no shared-memory destination.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// Orders this thread's (and, after a barrier, the CTA's) generic-proxy shared-memory
// accesses before its subsequent bulk copies into the same buffers.
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Generic -> async proxy ordering for global memory (V rows written by one
// iteration are read by the next iteration's bulk copies).
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Fixed-order block reduction of one double per thread (result valid in thread 0).
__device__ __forceinline__ double block_sum_d(double v, double* sh) {
    v = warp_sum_d(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
    __syncthreads();
    return s;
}

// Grid barrier for a cooperative launch (all CTAs co-resident): a monotone arrival
// counter (zeroed by the host before the launch); barrier number e completes when the
// counter reaches e * nCTA.  One release-add per CTA, acquire polling, no second atomic.
__device__ __forceinline__ void grid_sync(unsigned* count, unsigned& epoch) {
    __syncthreads();
    ++epoch;
    if (threadIdx.x == 0) {
        // release: the CTA's writes (ordered before this thread by __syncthreads) become
        // visible to every CTA whose acquire-load observes the count
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
        const unsigned target = epoch * gridDim.x;
        unsigned cur;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(count) : "memory");
        } while ((int)(cur - target) < 0);
    }
    __syncthreads();
}

// s = sum over cc = q, q + NQ, ... < nC of ld(cc), in that order, with the loads issued
// in predicated batches of 24 so that they are all in flight together.
template <class F>
__device__ __forceinline__ double batched_sum(int q, int NQ, int nC, F&& ld) {
    constexpr int MB = 24;
    double s = 0.0;
    for (int base = q; base < nC; base += NQ * MB) {
        double v[MB];
#pragma unroll
        for (int u = 0; u < MB; ++u) {
            const int cc = base + u * NQ;
            v[u] = cc < nC ? ld(cc) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < MB; ++u) s += v[u];
    }
    return s;
}

// Fixed-order block reduction of one double per thread, result in every thread.
__device__ __forceinline__ double block_sum_all(double v, double* sh) {
    v = warp_sum_d(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
    __syncthreads();
    return s;
}

}  // namespace
}  // namespace hsnct
