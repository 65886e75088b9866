// Probe for a TMEM-resident phase 2: (1) where tcgen05.cp.128x256b puts a
// K-major no-swizzle shared-memory matrix of 128 rows x 16 fp16 in TMEM; (2) whether
// tcgen05.mma kind::f16 with the A operand in TMEM (M = 128, K = 16) computes A B^T from that
// copy, against a host reference; (3) its issue cost per MMA (converged warp) vs A in smem.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tc05_tmemA tc05_tmemA.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

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
// K-major core-matrix layout of R rows x 16 fp16: core (rg, kg) at (rg * 2 + kg) * 128 B
__host__ __device__ inline size_t kmaj(int r, int k) { return ((size_t)((r >> 3) * 2 + (k >> 3)) * 8 + (r & 7)) * 8 + (k & 7); }

// out_cp[lane][col] = TMEM words after the copy (128 lanes x 8 columns)
// out_d[lane][n]   = D = A B^T with A from TMEM (128 x 16 fp32)
__global__ void __launch_bounds__(128, 1) k_probe(const __half* __restrict__ Ain, const __half* __restrict__ Bin,
                                                  uint32_t* __restrict__ out_cp, float* __restrict__ out_d,
                                                  int reps, unsigned long long* cyc_tmem,
                                                  unsigned long long* cyc_smem) {
    __shared__ __align__(1024) __half As[128 * 16];
    __shared__ __align__(1024) __half Bs[16 * 16];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 128 * 16; i += 128) As[i] = Ain[i];
    for (int i = tid; i < 16 * 16; i += 128) Bs[i] = Bin[i];
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tbase;
    const uint32_t ta = tmem;         // A copy: columns [0, 8)
    const uint32_t td = tmem + 64;    // D: columns [64, 80)
    if (warp == 0) {
        // (1) smem -> TMEM copy of the 128 x 16 fp16 matrix (K-major: LBO = 128 B, SBO = 256 B)
        const uint64_t ad = sdesc(su32(As), 128, 256);
        asm volatile(
            "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
            "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(ta),
            "l"(ad)
            : "memory");
        // (2) D = A B^T with A in TMEM, B (N = 16 x K = 16, K-major) in smem
        const uint32_t idesc = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t bd = sdesc(su32(Bs), 128, 256);
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\tsetp.ne.b32 p, 0, 0;\n\telect.sync r|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(td),
            "r"(ta), "l"(bd), "r"(idesc)
            : "memory");
        asm volatile(
            "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bar))
            : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred p;\nW1:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra W1;\n}" ::"r"(su32(&bar))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(ta + ((uint32_t)(32 * warp) << 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 8; ++j) out_cp[tid * 8 + j] = v[j];
        uint32_t d[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
              "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
            : "r"(td + ((uint32_t)(32 * warp) << 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 16; ++j) out_d[tid * 16 + j] = __uint_as_float(d[j]);
    }
    // (3) issue cost: reps x 8 MMAs, A from TMEM vs A from smem (converged warp 0)
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) {
        const uint32_t idesc = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t bd = sdesc(__shfl_sync(0xffffffffu, su32(Bs), 0), 128, 256);
        const uint64_t ad = sdesc(__shfl_sync(0xffffffffu, su32(As), 0), 128, 256);
        const uint32_t tt = __shfl_sync(0xffffffffu, tmem, 0);
        for (int mode = 0; mode < 2; ++mode) {
            unsigned long long t0 = clock64();
            for (int r = 0; r < reps; ++r) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t d = tt + 64 + (uint32_t)((j & 3) * 16);
                    if (mode == 0)
                        asm volatile(
                            "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\tsetp.ne.b32 p, 1, 0;\n\telect.sync r|e, 0xffffffff;\n\t"
                            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                            "r"(tt), "l"(bd), "r"(idesc)
                            : "memory");
                    else
                        asm volatile(
                            "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\tsetp.ne.b32 p, 1, 0;\n\telect.sync r|e, 0xffffffff;\n\t"
                            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                            "l"(ad), "l"(bd), "r"(idesc)
                            : "memory");
                }
            }
            asm volatile(
                "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
                "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bar))
                : "memory");
            asm volatile(
                "{\n\t.reg .pred p;\nW2:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                "@!p bra W2;\n}" ::"r"(su32(&bar)),
                "r"((unsigned)((mode + 1) & 1))
                : "memory");
            unsigned long long t1 = clock64();
            if (lane == 0 && blockIdx.x == 0) (mode == 0 ? *cyc_tmem : *cyc_smem) = t1 - t0;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
    std::vector<__half> A(128 * 16), B(16 * 16);
    std::vector<float> Af(128 * 16), Bf(16 * 16);
    srand(5);
    for (int r = 0; r < 128; ++r)
        for (int k = 0; k < 16; ++k) {
            // identifiable values for the layout check: r + k / 32 (exact in fp16 for r < 64; random later)
            const float v = (float)(rand() % 256) / 64.f;
            Af[r * 16 + k] = v;
            A[kmaj(r, k)] = __float2half(v);
        }
    for (int n = 0; n < 16; ++n)
        for (int k = 0; k < 16; ++k) {
            const float v = (float)(rand() % 64) / 32.f;
            Bf[n * 16 + k] = v;
            B[kmaj(n, k)] = __float2half(v);
        }
    __half *dA, *dB;
    uint32_t* dcp;
    float* dd;
    unsigned long long* dcyc;
    CK(cudaMalloc(&dA, A.size() * 2));
    CK(cudaMalloc(&dB, B.size() * 2));
    CK(cudaMalloc(&dcp, 128 * 8 * 4));
    CK(cudaMalloc(&dd, 128 * 16 * 4));
    CK(cudaMalloc(&dcyc, 16));
    CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
    const int reps = 2000;
    k_probe<<<148, 128>>>(dA, dB, dcp, dd, reps, dcyc, dcyc + 1);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<uint32_t> cp(128 * 8);
    std::vector<float> D(128 * 16);
    unsigned long long cyc[2];
    CK(cudaMemcpy(cp.data(), dcp, cp.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(D.data(), dd, D.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(cyc, dcyc, 16, cudaMemcpyDeviceToHost));
    // (1) layout: is TMEM lane r, column c = {A[r][2c], A[r][2c+1]} (low half first)?
    int ok = 0, tot = 0;
    for (int r = 0; r < 128; ++r)
        for (int c = 0; c < 8; ++c) {
            const uint32_t w = cp[r * 8 + c];
            __half lo, hi;
            uint16_t l16 = (uint16_t)(w & 0xffff), h16 = (uint16_t)(w >> 16);
            memcpy(&lo, &l16, 2);
            memcpy(&hi, &h16, 2);
            ok += (__half2float(lo) == Af[r * 16 + 2 * c]) && (__half2float(hi) == Af[r * 16 + 2 * c + 1]);
            ++tot;
        }
    printf("tcgen05.cp.128x256b: lane r, column c = (A[r][2c], A[r][2c+1]): %d of %d words match\n", ok, tot);
    if (ok != tot) {
        for (int r = 0; r < 3; ++r) {
            printf("lane %d:", r);
            for (int c = 0; c < 8; ++c) {
                const uint32_t w = cp[r * 8 + c];
                __half lo, hi;
                uint16_t l16 = (uint16_t)(w & 0xffff), h16 = (uint16_t)(w >> 16);
                memcpy(&lo, &l16, 2);
                memcpy(&hi, &h16, 2);
                printf(" (%.3f,%.3f)", __half2float(lo), __half2float(hi));
            }
            printf("\n   want:");
            for (int k = 0; k < 16; ++k) printf(" %.3f", Af[r * 16 + k]);
            printf("\n");
        }
    }
    // (2) D = A B^T
    double num = 0, den = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 16; ++n) {
            double s = 0;
            for (int k = 0; k < 16; ++k) s += (double)Af[m * 16 + k] * Bf[n * 16 + k];
            num += (D[m * 16 + n] - s) * (D[m * 16 + n] - s);
            den += s * s;
        }
    printf("MMA with A in TMEM (M=128, N=16, K=16): rel err %.3e\n", sqrt(num / den));
    printf("issue: A in TMEM %.1f cycles/MMA, A in smem %.1f cycles/MMA\n", cyc[0] / (8.0 * reps), cyc[1] / (8.0 * reps));
    return 0;
}
