// Prototype for the next-round NMF pass (DESIGN.md §5.1 "Next-round plan"): phase 1 of the
// row pass, A = Y+ D^T, on tcgen05 tensor cores, fp32-accurate through an fp16 hi/lo split
// (A = Yhi Dhi + Yhi Dlo + Ylo Dhi), accumulated in TMEM, read back one row per thread.
//
// Y+ is stored in HBM in UMMA core-matrix order (tile of 128 rows, chunks of 64 lambda, core
// matrices of 8 rows x 8 lambda = 128 B), so a plain cp.async.bulk lands a chunk in the
// canonical no-swizzle K-major layout.  One CTA per SM; warp 0 copies, warp 1 issues the MMAs
// (M = 128, N = 16, K = 16 per instruction), warps 2..5 drain the accumulator (double-buffered
// in TMEM) to global memory.  Reports the Y stream rate (GB/s) and checks sampled rows against
// an fp64 host reference.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tc05_phase1 tc05_phase1.cu
//   ./tc05_phase1 [rows] [Nk]
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

constexpr int TM = 128;      // rows per tile (UMMA M)
#ifndef NNV
#define NNV 16
#endif
constexpr int NN = NNV;       // UMMA N (K components padded)
constexpr int CL = 64;       // lambda per chunk
constexpr int NST = 3;       // chunk stages
constexpr int CHB = TM * CL * 2;  // bytes per hi (or lo) chunk = 16 KB

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned par) {
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(su32(b)),
        "r"(par)
        : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(b))
        : "memory");
}
// no-swizzle canonical descriptor (units of 16 B), Blackwell version bit
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version
    return d;                // base offset 0, layout type 0 (SWIZZLE_NONE)
}
// instruction descriptor: f16 x f16 -> f32, K-major A and B, N = 16, M = 128
constexpr uint32_t IDESC = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);

__device__ __forceinline__ void mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(a), "l"(b), "r"(IDESC), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b))
                 : "memory");
}

// NPASS = 2 streams every tile twice, the second stream one tile later (P1(0), P1(1), P2(0),
// P1(2), P2(1), ...), into a discarded accumulator: the L2 re-read a phase 2 would need.
#ifndef NPASS
#define NPASS 1
#endif
__device__ __forceinline__ void seq(int u, int mine, int& m, int& second) {
    if (NPASS == 1) { m = u; second = 0; return; }
    if (u == 0) { m = 0; second = 0; return; }
    if (u & 1) {
        if ((u + 1) / 2 < mine) { m = (u + 1) / 2; second = 0; }
        else { m = mine - 1; second = 1; }
    } else { m = u / 2 - 1; second = 1; }
}
// Yc: [tiles][chunks][2][CHB] (hi, lo), core-matrix order within a chunk:
//     ((pb * 8 + lb) * 8 + r) * 8 + l  for row 8 pb + r, lambda 8 lb + l of the chunk
// Dc: [2][NK/8][NN/8][8][8] (hi, lo): core matrix (lb, nb) at (lb * NN/8 + nb) * 64 halves
__global__ void __launch_bounds__(192, 1) k_phase1(const __half* __restrict__ Yc, const __half* __restrict__ Dc,
                                                 float* __restrict__ Aout, int ntiles, int nchunk) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[NST], empty[NST], accf[2], acce[2];
    __shared__ uint64_t dbar;
    __shared__ uint32_t tbase;
    const int NK = nchunk * CL;
    const int dbytes = NK * NN * 2;        // one of Dhi / Dlo
    uint8_t* Dh = sm;
    uint8_t* Dl = sm + dbytes;
    uint8_t* st = sm + 2 * dbytes;         // [NST][2][CHB]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mb_init(&full[s], 1);
            mb_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mb_init(&accf[b], 1);
            mb_init(&acce[b], 4);
        }
        mb_init(&dbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // TMEM: 2 accumulators x 16 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tbase;
    const int mine = ntiles > (int)blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (warp == 0) {
        if (lane == 0) {
            mb_expect(&dbar, 2 * dbytes);
            bulk(Dh, Dc, dbytes, &dbar);
            bulk(Dl, Dc + dbytes / 2, dbytes, &dbar);
            int s = 0;
            unsigned ph = 0;
            for (int u = 0; u < NPASS * mine; ++u) {
                int m, second;
                seq(u, mine, m, second);
                const int t = blockIdx.x + m * gridDim.x;
                for (int c = 0; c < nchunk; ++c) {
                    mb_wait(&empty[s], ph ^ 1);
                    mb_expect(&full[s], 2 * CHB);
                    const __half* src = Yc + ((size_t)t * nchunk + c) * 2 * (CHB / 2);
                    bulk(st + (size_t)s * 2 * CHB, src, 2 * CHB, &full[s]);
                    if (++s == NST) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            mb_wait(&dbar, 0);
            int s = 0;
            unsigned ph = 0;
            for (int u = 0; u < NPASS * mine; ++u) {
                int m, second;
                seq(u, mine, m, second);
                const int ab = m & 1;
                if (!second) {
                    mb_wait(&acce[ab], ((m >> 1) & 1) ^ 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                }
                const uint32_t td = second ? tmem + 32 : tmem + ab * NN;
                for (int c = 0; c < nchunk; ++c) {
                    mb_wait(&full[s], ph);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t ah = su32(st + (size_t)s * 2 * CHB), al = ah + CHB;
                    const uint32_t dh = su32(Dh), dl = su32(Dl);
#pragma unroll
                    for (int k = 0; k < CL / 16; ++k) {
                        // A: core (pb, lb) at (pb * 8 + lb) * 128 B: K step (lb) 128 B, M step (pb) 1024 B
                        const uint64_t aH = sdesc(ah + k * 256, 128, 1024), aL = sdesc(al + k * 256, 128, 1024);
                        // B: core (lb, nb) at (lb * NB + nb) * 128 B: K step NB * 128 B, N step 128 B
                        constexpr uint32_t NB = NN / 8;
                        const uint32_t boff = (uint32_t)(c * (CL / 8) + 2 * k) * NB * 128;
                        const uint64_t bH = sdesc(dh + boff, NB * 128, 128), bL = sdesc(dl + boff, NB * 128, 128);
                        const uint32_t first = (c == 0 && k == 0) ? 0u : 1u;
                        mma(td, aH, bH, first);
                        mma(td, aH, bL, 1u);
                        mma(td, aL, bH, 1u);
                    }
                    commit(&empty[s]);
                    if (++s == NST) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                if (!second) commit(&accf[ab]);
            }
        }
    } else {  // warps 2..5: TMEM lanes 32 * (warp % 4)
        const int q = warp & 3;
        for (int m = 0; m < mine; ++m) {
            const int ab = m & 1;
            mb_wait(&accf[ab], (m >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            uint32_t v[16];
            const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + ab * NN;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mb_arrive(&acce[ab]);
            const int t = blockIdx.x + m * gridDim.x;
            float4* o = reinterpret_cast<float4*>(Aout + ((size_t)t * TM + 32 * q + lane) * NN);
#pragma unroll
            for (int j = 0; j < NN / 4; ++j)
                o[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]), __uint_as_float(v[4 * j + 2]),
                                   __uint_as_float(v[4 * j + 3]));
        }
    }
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main(int argc, char** argv) {
    const long rows_req = argc > 1 ? atol(argv[1]) : (1L << 20);
    const int NKr = argc > 2 ? atoi(argv[2]) : 1600;
    const int nchunk = (NKr + CL - 1) / CL, NK = nchunk * CL;
    const int ntiles = (int)((rows_req + TM - 1) / TM);
    const long rows = (long)ntiles * TM;
    const int K = 6;
    printf("rows %ld Nk %d (padded %d) K %d tiles %d\n", rows, NKr, NK, K, ntiles);
    // inputs: Y+ in [0, 3), D in (0, 1], fp32, split into fp16 hi / lo
    std::vector<float> D((size_t)NN * NK, 0.f);
    srand(7);
    for (int k = 0; k < K; ++k)
        for (int l = 0; l < NKr; ++l) D[(size_t)k * NK + l] = 0.05f + (float)(rand() % 10000) / 10000.f;
    auto yval = [&](long p, int l) -> float {
        if (l >= NKr) return 0.f;
        uint32_t h = (uint32_t)(p * 2654435761u) ^ (uint32_t)(l * 40503u);
        h ^= h >> 13;
        h *= 0x5bd1e995u;
        h ^= h >> 15;
        return 3.f * (float)(h & 0xFFFFFF) / 16777216.f;
    };
    std::vector<__half> Yc((size_t)rows * NK * 2);
    for (long t = 0; t < ntiles; ++t)
        for (int c = 0; c < nchunk; ++c) {
            __half* base = Yc.data() + ((size_t)t * nchunk + c) * 2 * (CHB / 2);
            for (int r = 0; r < TM; ++r)
                for (int l = 0; l < CL; ++l) {
                    const float y = yval(t * TM + r, c * CL + l);
                    const __half hi = __float2half_rn(y);
                    const __half lo = __float2half_rn(y - __half2float(hi));
                    const size_t off = (((size_t)(r >> 3) * 8 + (l >> 3)) * 8 + (r & 7)) * 8 + (l & 7);
                    base[off] = hi;
                    base[CHB / 2 + off] = lo;
                }
        }
    std::vector<__half> Dc((size_t)2 * NK * NN);
    for (int n = 0; n < NN; ++n)
        for (int l = 0; l < NK; ++l) {
            const float d = D[(size_t)n * NK + l];
            const __half hi = __float2half_rn(d);
            const __half lo = __float2half_rn(d - __half2float(hi));
            const size_t off = (((size_t)(l >> 3) * (NN / 8) + (n >> 3)) * 8 + (n & 7)) * 8 + (l & 7);
            Dc[off] = hi;
            Dc[(size_t)NK * NN + off] = lo;
        }
    __half *dY, *dD;
    float* dA;
    CK(cudaMalloc(&dY, Yc.size() * 2));
    CK(cudaMalloc(&dD, Dc.size() * 2));
    CK(cudaMalloc(&dA, (size_t)rows * NN * 4));
    CK(cudaMemcpy(dY, Yc.data(), Yc.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dD, Dc.data(), Dc.size() * 2, cudaMemcpyHostToDevice));
    const size_t smem = (size_t)2 * NK * NN * 2 + (size_t)NST * 2 * CHB;
    CK(cudaFuncSetAttribute(k_phase1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    printf("smem %zu B, grid %d\n", smem, sms);
    k_phase1<<<sms, 192, smem>>>(dY, dD, dA, ntiles, nchunk);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 10;
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) k_phase1<<<sms, 192, smem>>>(dY, dD, dA, ntiles, nchunk);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double ybytes = (double)rows * NK * 4;
    printf("phase 1: %.3f ms per pass, Y stream %.1f GB/s (fp16 hi+lo = 4 B per element)\n", ms, ybytes / ms / 1e6);
    // check sampled rows against an fp64 reference from the fp32 values
    std::vector<float> A((size_t)rows * NN);
    CK(cudaMemcpy(A.data(), dA, A.size() * 4, cudaMemcpyDeviceToHost));
    double num = 0, den = 0, worst = 0;
    for (long p = 0; p < rows; p += rows / 997 + 1) {
        for (int k = 0; k < K; ++k) {
            double s = 0;
            for (int l = 0; l < NKr; ++l) s += (double)yval(p, l) * (double)D[(size_t)k * NK + l];
            const double d = (double)A[(size_t)p * NN + k] - s;
            num += d * d;
            den += s * s;
            worst = fmax(worst, fabs(d) / fabs(s));
        }
    }
    printf("sampled rel-L2 %.3e, worst rel %.3e\n", sqrt(num / den), worst);
    return 0;
}
