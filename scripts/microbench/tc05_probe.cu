// Facts the tcgen05 NMF pass depends on, measured on the B200 itself:
//  1. the TMEM layout of an M = 64 (cta_group::1, kind::f16) accumulator: which lanes /
//     columns hold D[m][n];
//  2. the no-swizzle shared-memory descriptor of an MN-major A operand (which of LBO / SBO is
//     the MN-direction stride), checked against a host product;
//  3. cudaOccupancyMaxActiveClusters for cluster sizes 1..8 at ~210 KB of dynamic smem.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tc05_probe tc05_probe.cu
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
__device__ __forceinline__ void mb_init(uint64_t* b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned par) {
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(su32(b)),
        "r"(par)
        : "memory");
}

// Test kernel: 128 threads.  A [64 x 16] (M x K) and B [N x 16] fp16 in smem, given as
// descriptors built from (lbo, sbo) for A and the K-major B layout; one MMA with M = 64 (or
// 128), N; then every warp reads its 32 lanes x NCOL columns (after a sentinel fill).
template <int M, int N, int NCOL>
__global__ void k_probe(const __half* __restrict__ Ain, int abytes, const __half* __restrict__ Bin, int bbytes,
                        uint32_t a_lbo, uint32_t a_sbo, uint32_t b_lbo, uint32_t b_sbo, int a_mn_major,
                        float* __restrict__ out) {
    __shared__ __align__(1024) __half As[128 * 64];
    __shared__ __align__(1024) __half Bs[256 * 16];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < abytes / 2; i += blockDim.x) As[i] = Ain[i];
    for (int i = tid; i < bbytes / 2; i += blockDim.x) Bs[i] = Bin[i];
    if (tid == 0) {
        mb_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tbase;
    // sentinel fill: -1 in every lane / column
    {
        uint32_t v[16];
        for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(-1.f);
        const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16);
        for (int c = 0; c < NCOL; c += 16)
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
                    ta + c),
                "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (tid == 0) {
        const uint32_t idesc = (1u << 4) | ((uint32_t)(a_mn_major ? 1 : 0) << 15) | ((uint32_t)(N >> 3) << 17) |
                               ((uint32_t)(M >> 4) << 24);
        const uint64_t ad = sdesc(su32(As), a_lbo, a_sbo);
        const uint64_t bd = sdesc(su32(Bs), b_lbo, b_sbo);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(0u));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                     : "memory");
    }
    mb_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    {
        const uint32_t ta = tmem + ((uint32_t)(32 * warp) << 16);
        for (int c = 0; c < NCOL; c += 16) {
            uint32_t v[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(ta + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int j = 0; j < 16; ++j) out[(size_t)tid * NCOL + c + j] = __uint_as_float(v[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

__global__ void k_dummy(int* p) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0 && p) p[blockIdx.x] = sm[0];
}

// K-major core-matrix layout of an R x 16 operand (R rows, 16 K): core (rg, kg) at (rg*2 + kg) * 128 B
// -> LBO (K dir) = 128, SBO (row dir) = 256.
static size_t kmaj(int r, int k) { return ((size_t)((r >> 3) * 2 + (k >> 3)) * 8 + (r & 7)) * 8 + (k & 7); }

int main() {
    int dev = 0;
    CK(cudaSetDevice(dev));
    // ---- 1. M = 64 accumulator layout: A[m][k] = (k == 0) ? m + 1 : 0, B[n][k] = (k == 0) ? (n + 1) / 64 : 0
    {
        std::vector<__half> A(64 * 16), B(16 * 16);
        for (int m = 0; m < 64; ++m)
            for (int k = 0; k < 16; ++k) A[kmaj(m, k)] = __float2half(k == 0 ? (float)(m + 1) : 0.f);
        for (int n = 0; n < 16; ++n)
            for (int k = 0; k < 16; ++k) B[kmaj(n, k)] = __float2half(k == 0 ? (float)(n + 1) / 64.f : 0.f);
        __half *dA, *dB;
        float* dO;
        CK(cudaMalloc(&dA, A.size() * 2));
        CK(cudaMalloc(&dB, B.size() * 2));
        CK(cudaMalloc(&dO, 128 * 32 * 4));
        CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
        k_probe<64, 16, 32><<<1, 128>>>(dA, (int)A.size() * 2, dB, (int)B.size() * 2, 128, 256, 128, 256, 0, dO);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        std::vector<float> O(128 * 32);
        CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
        printf("== M=64 N=16 accumulator: lane -> (m, n) of non-sentinel columns (value = (m+1)(n+1)/64)\n");
        int shown = 0;
        for (int lane = 0; lane < 128; ++lane) {
            char buf[512];
            int len = 0, any = 0;
            for (int c = 0; c < 32; ++c) {
                const float v = O[lane * 32 + c];
                if (v == -1.f) continue;
                any = 1;
                // decode: v * 64 = (m+1)(n+1)
                len += snprintf(buf + len, sizeof buf - len, " c%d=%.0f", c, v * 64.f);
                if (len > 400) break;
            }
            if (any && (shown < 200)) {
                printf("lane %3d:%s\n", lane, buf);
                ++shown;
            }
        }
        // expected from lane = m: value at column n = (m+1)(n+1)
        int ok_lane_eq_m = 1;
        for (int m = 0; m < 64; ++m)
            for (int n = 0; n < 16; ++n)
                if (O[m * 32 + n] * 64.f != (float)((m + 1) * (n + 1))) ok_lane_eq_m = 0;
        printf("layout 'lane = m, column = n' (lanes 0..63): %s\n", ok_lane_eq_m ? "YES" : "no");
        int ok_half = 1;  // lanes 32w + (m % 16) for w = m / 16
        for (int m = 0; m < 64; ++m)
            for (int n = 0; n < 16; ++n)
                if (O[(32 * (m / 16) + (m % 16)) * 32 + n] * 64.f != (float)((m + 1) * (n + 1))) ok_half = 0;
        printf("layout 'lane = 32 (m/16) + m%%16, column = n': %s\n", ok_half ? "YES" : "no");
        CK(cudaFree(dA));
        CK(cudaFree(dB));
        CK(cudaFree(dO));
    }
    // ---- 2. MN-major A (M = 64, K = 16): chunk layout [rg][lb][8 rows][8 lambda] where the MMA's
    //         M = lambda (64 = 8 groups, stride 128 B) and K = rows (16 = 2 groups, stride 1024 B).
    //         D[lambda][n] = sum_rows Y[row][lambda] V[row][n].  Try (LBO, SBO) = (128, 1024) and (1024, 128).
    {
        const int NR = 16, NL = 64, NN = 16;
        std::vector<float> Y(NR * NL), V(NR * NN);
        srand(3);
        for (auto& y : Y) y = (float)(rand() % 64) / 16.f;
        for (auto& v : V) v = (float)(rand() % 32) / 8.f;
        std::vector<__half> A(8 * 8 * 64, __float2half(0.f));  // 8 row groups (only 2 used) x 8 lambda groups
        for (int r = 0; r < NR; ++r)
            for (int l = 0; l < NL; ++l)
                A[(((size_t)(r >> 3) * 8 + (l >> 3)) * 8 + (r & 7)) * 8 + (l & 7)] = __float2half(Y[r * NL + l]);
        std::vector<__half> B(NN * 16);  // K-major B: N = 16 x K = 16 rows
        for (int n = 0; n < NN; ++n)
            for (int r = 0; r < 16; ++r) B[kmaj(n, r)] = __float2half(V[r * NN + n]);
        __half *dA, *dB;
        float* dO;
        CK(cudaMalloc(&dA, A.size() * 2));
        CK(cudaMalloc(&dB, B.size() * 2));
        CK(cudaMalloc(&dO, 128 * 32 * 4));
        CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
        const uint32_t opts[2][2] = {{128, 1024}, {1024, 128}};
        for (auto& o : opts) {
            k_probe<64, 16, 32><<<1, 128>>>(dA, (int)A.size() * 2, dB, (int)B.size() * 2, o[0], o[1], 128, 256, 1,
                                            dO);
            CK(cudaGetLastError());
            CK(cudaDeviceSynchronize());
            std::vector<float> O(128 * 32);
            CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
            // compare under both candidate accumulator layouts
            for (int lay = 0; lay < 2; ++lay) {
                double err = 0, ref = 0;
                for (int l = 0; l < NL; ++l)
                    for (int n = 0; n < NN; ++n) {
                        double s = 0;
                        for (int r = 0; r < NR; ++r) s += (double)Y[r * NL + l] * V[r * NN + n];
                        const int lane = lay == 0 ? l : 32 * (l / 16) + (l % 16);
                        const double d = O[lane * 32 + n] - s;
                        err += d * d;
                        ref += s * s;
                    }
                printf("MN-major A, LBO=%u SBO=%u, acc layout %s: rel err %.3e\n", o[0], o[1],
                       lay == 0 ? "lane=m" : "lane=32(m/16)+m%16", sqrt(err / ref));
            }
        }
        // also the K-major phase-1 view of the same chunk: M = rows (64), K = lambda (16 of them)
        CK(cudaFree(dA));
        CK(cudaFree(dB));
        CK(cudaFree(dO));
    }
    // ---- 3. cluster occupancy at ~210 KB dynamic smem
    {
        const int smem = 210 * 1024;
        CK(cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        CK(cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        int sms = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        for (int cs = 1; cs <= 16; ++cs) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cs * 64, 1, 1);
            cfg.blockDim = dim3(192, 1, 1);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int ncl = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, k_dummy, &cfg);
            printf("cluster %2d: max active clusters %d (%d SMs of %d) %s\n", cs, ncl, ncl * cs, sms,
                   e == cudaSuccess ? "" : cudaGetErrorString(e));
            (void)cudaGetLastError();
        }
    }
    return 0;
}
