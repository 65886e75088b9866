// tcgen05.mma issue/throughput for the small-N shapes of the NMF pass:
// operands resident in shared memory (no HBM), one CTA per SM, one issuing thread; per variant
// `reps` groups of 8 MMAs (kind::f16, K = 16), committed and waited at the end.  Reports ns per
// MMA.  Variants: M (64 / 128), N (16 / 32 / 64), A K-major or MN-major, and the number of
// distinct accumulators the 8 MMAs of a group rotate over (1 = a dependent chain).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tc05_rate tc05_rate.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                               \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess) {                                                            \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                        \
        }                                                                                   \
    } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

// nwarps issuing warps (each its own accumulators); mode 0: lane 0 of each issuing warp runs
// the loop (divergent), mode 1: the whole warp runs it and elect.sync picks the issuing lane
// inside the asm (converged)
__global__ void __launch_bounds__(128, 1) k_rate(int M, int N, int amn, int nacc, int reps, unsigned long long* out,
                                                 int nwarps, int mode) {
    extern __shared__ __align__(1024) uint8_t sm[];  // 64 KB of operands (contents irrelevant)
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(nwarps));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tbase;
    const int lane = threadIdx.x & 31;
    if (mode == 2 && warp < nwarps) {
        // converged warp, every descriptor from warp-uniform values (kernel params, loop
        // counters, a shared-memory base read through __shfl_sync), elect.sync inside the asm
        const uint32_t idesc = (1u << 4) | ((uint32_t)amn << 15) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint32_t a0 = __shfl_sync(0xffffffffu, su32(sm), 0), b0 = a0 + 32768u;
        const uint32_t t0w = __shfl_sync(0xffffffffu, tmem + (uint32_t)(warp * 128), 0);
        const uint64_t ad0 = amn ? sdesc(a0, 1024, 128) : sdesc(a0, 128, 1024);
        const uint64_t bd0 = sdesc(b0, 256, 128);
        unsigned long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint64_t ad = ad0 + (uint64_t)((j & 3) * (amn ? 128 : 16));
                const uint64_t bd = bd0 + (uint64_t)((j & 3) * 32);
                const uint32_t d = t0w + (uint32_t)((j % nacc) * N);
                asm volatile(
                    "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "elect.sync r|e, 0xffffffff;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
            }
        }
        if (lane == 0)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                         : "memory");
        asm volatile(
            "{\n\t.reg .pred p;\nW2:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
            "@!p bra W2;\n}" ::"r"(su32(&bar))
            : "memory");
        unsigned long long t1 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
    } else if (warp < nwarps && (mode == 1 || lane == 0)) {
        const uint32_t idesc = (1u << 4) | ((uint32_t)amn << 15) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        const uint32_t a0 = su32(sm), b0 = su32(sm + 32768);
        unsigned long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint64_t ad = amn ? sdesc(a0 + (j & 3) * 2048, 1024, 128) : sdesc(a0 + (j & 3) * 256, 128, 1024);
                const uint64_t bd = sdesc(b0 + (j & 3) * 512, 256, 128);
                const uint32_t d = tmem + (uint32_t)((j % nacc) * N + warp * 128);
                if (mode == 0)
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                        "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
                else
                    asm volatile(
                        "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "elect.sync r|e, 0xffffffff;\n\t"
                        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                        "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
            }
        }
        if (lane == 0)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                         : "memory");
        asm volatile(
            "{\n\t.reg .pred p;\nW:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
            "@!p bra W;\n}" ::"r"(su32(&bar))
            : "memory");
        unsigned long long t1 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    unsigned long long* dout;
    CK(cudaMalloc(&dout, 8));
    const int reps = 2000;
    struct V { int M, N, amn, nacc, nw, mode; } vs[] = {
        {64, 16, 0, 1, 1, 0}, {64, 16, 0, 1, 1, 2}, {64, 16, 0, 4, 1, 2}, {64, 16, 0, 4, 2, 2},
        {128, 16, 1, 4, 1, 2}, {128, 16, 1, 4, 2, 2}, {64, 16, 0, 4, 4, 2}, {128, 16, 1, 1, 4, 2},
    };
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (auto v : vs) {
        k_rate<<<sms, 128, 65536>>>(v.M, v.N, v.amn, v.nacc, 10, dout, v.nw, v.mode);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        k_rate<<<sms, 128, 65536>>>(v.M, v.N, v.amn, v.nacc, reps, dout, v.nw, v.mode);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long cyc;
        CK(cudaMemcpy(&cyc, dout, 8, cudaMemcpyDeviceToHost));
        const double n = 8.0 * reps * v.nw;
        printf("M=%3d N=%3d A=%s acc=%d warps=%d %s: %.1f ns/MMA (event, all warps), %.1f cycles/MMA\n", v.M, v.N,
               v.amn ? "MN-major" : "K-major", v.nacc, v.nw, v.mode == 2 ? "uniform+elect" : v.mode ? "converged+elect" : "lane-0 loop",
               ms * 1e6 / n, cyc / n);
    }
    return 0;
}
