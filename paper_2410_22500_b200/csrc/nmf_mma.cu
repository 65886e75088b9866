// Host side of the mma.sync NMF path (nmf_mma.cuh): input preparation (Y+ or counts into the
// block layout), plan, per-K dispatch.
#include "nmf_mma.cuh"

namespace hsnct {
namespace {

// Y+ (clamped, scaled by sigma_Y) split into fp16 hi/lo in the block layout above.  Item
// (tile, block, core matrix q, row rr), rr fastest: 32 consecutive threads write one block's
// hi and lo halves (512 contiguous bytes each); each reads 8 bins of one row.
__global__ void __launch_bounds__(256) k_mma_convert(const float* __restrict__ Y, int64_t ld, int64_t Np, int Nk,
                                                     int NB, int64_t ntiles, const unsigned* __restrict__ ymax,
                                                     uint8_t* __restrict__ Yc) {
    const float sy = pow2(mexp(__uint_as_float(*ymax)));
    const int64_t n = ntiles * NB * 32;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int rr = (int)(i & 7), q = (int)((i >> 3) & 3);
        const int64_t u = i >> 5;
        const int j = (int)(u % NB);
        const int64_t tt = u / NB;
        const int64_t r = tt * MR + (q & 1) * 8 + rr;
        const int l = 16 * j + (q >> 1) * 8;
        float v[8];
        if (r < Np && l + 8 <= Nk) {
            const float4* y = reinterpret_cast<const float4*>(Y + r * ld + l);
            const float4 a = __ldg(y), b = __ldg(y + 1);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = (r < Np && l + e < Nk) ? Y[r * ld + l + e] : 0.f;
        }
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
            hw[e] = split2(fmaxf(v[2 * e], 0.f) * sy, fmaxf(v[2 * e + 1], 0.f) * sy, lw[e]);
        uint8_t* dst = Yc + (size_t)u * BLK + q * 128 + rr * 16;
        *reinterpret_cast<uint4*>(dst) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(dst + 512) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}

// ---- counts-domain input (NEXT-1): Eq. 2 with the Appendix-A offset decoded straight into the
// block layout, Y = fp32((L[y0] - L[y]) - b) with the fp64 table L[n] = ln max(n, 1/2)
// (counts.cu, R7): the same per-element value as hsnct_counts_to_projections, and the
// two kernels below have the loop structure of k_tc_stats / k_mma_convert, so the decomposition
// from counts is bit-identical to the one from the materialised Y.
struct CountsSrc {
    const uint8_t* y;    // [Np][Nk]
    const uint8_t* y0;   // [Nr Nc][Nk]
    const float* b;      // [Nv][Nk] or null
    const double* L;     // [256] (device table)
    int64_t NrNc;
    int Nk;
};
struct CountsRow {  // the rows of y, y0 and b that row p of Y decodes from
    const uint8_t* y;
    const uint8_t* y0;
    const float* b;
};
__device__ __forceinline__ CountsRow counts_row(const CountsSrc& C, int64_t p) {
    const int64_t v = p / C.NrNc, rc = p - v * C.NrNc;
    return {C.y + p * C.Nk, C.y0 + rc * C.Nk, C.b ? C.b + v * C.Nk : nullptr};
}
__device__ __forceinline__ float decode1(const CountsRow& R, const double* Ls, int l) {
    double d = Ls[R.y0[l]] - Ls[R.y[l]];
    if (R.b) d -= (double)R.b[l];
    return (float)d;
}

// k_tc_stats (nmf_tc.cu) on decoded counts: max Y+ (bits), ||Y+||^2 per-block partials (same
// per-row order), non-finite check (b), clamped count.  One warp per row.
__global__ void __launch_bounds__(256) k_mma_counts_stats(CountsSrc C, int64_t Np, unsigned* __restrict__ ymax,
                                                          double* __restrict__ ypart, unsigned* __restrict__ status,
                                                          unsigned long long* __restrict__ nclamp) {
    __shared__ double Ls[256];
    __shared__ double red[8];
    __shared__ unsigned mred[8], cred[8];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) Ls[i] = C.L[i];
    __syncthreads();
    unsigned ncl = 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nq = (C.Nk + 3) >> 2;
    double s = 0.0;
    unsigned m = 0, bad = 0;
    for (int64_t r = (int64_t)blockIdx.x * 8 + w; r < Np; r += (int64_t)gridDim.x * 8) {
        const CountsRow R = counts_row(C, r);
        float ps = 0.f;
        for (int q = lane; q < nq; q += 32) {
            const int l = 4 * q;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float vj = l + j < C.Nk ? decode1(R, Ls, l + j) : 0.f;
                if (!isfinite(vj)) bad = ST_Y_NONFINITE;
                ncl += vj < 0.f;
                const float yp = fmaxf(vj, 0.f);
                m = max(m, __float_as_uint(yp));
                ps = fmaf(yp, yp, ps);
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
        s += (double)ps;
    }
    m = __reduce_max_sync(0xffffffffu, m);
    bad = __reduce_or_sync(0xffffffffu, bad);
    ncl = __reduce_add_sync(0xffffffffu, ncl);
    if (lane == 0) {  // (s is the same in every lane: the row sums were reduced over the warp)
        red[w] = s;
        mred[w] = m;
        cred[w] = ncl;
        if (bad) atomicOr(status, bad);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tt = 0.0;
        unsigned mm = 0;
        unsigned long long cc = 0;
        for (int j = 0; j < 8; ++j) {
            tt += red[j];
            mm = max(mm, mred[j]);
            cc += cred[j];
        }
        ypart[blockIdx.x] = tt;
        if (cc) atomicAdd(nclamp, cc);
        if (mm) atomicMax(ymax, mm);
    }
}

// k_mma_convert on decoded counts
__global__ void __launch_bounds__(256) k_mma_counts_convert(CountsSrc C, int64_t Np, int NB, int64_t ntiles,
                                                            const unsigned* __restrict__ ymax,
                                                            uint8_t* __restrict__ Yc) {
    __shared__ double Ls[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) Ls[i] = C.L[i];
    __syncthreads();
    const float sy = pow2(mexp(__uint_as_float(*ymax)));
    const int64_t n = ntiles * NB * 32;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int rr = (int)(i & 7), q = (int)((i >> 3) & 3);
        const int64_t u = i >> 5;
        const int j = (int)(u % NB);
        const int64_t tt = u / NB;
        const int64_t r = tt * MR + (q & 1) * 8 + rr;
        const int l = 16 * j + (q >> 1) * 8;
        float v[8];
        const CountsRow R = counts_row(C, r < Np ? r : 0);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = (r < Np && l + e < C.Nk) ? decode1(R, Ls, l + e) : 0.f;
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
            hw[e] = split2(fmaxf(v[2 * e], 0.f) * sy, fmaxf(v[2 * e + 1], 0.f) * sy, lw[e]);
        uint8_t* dst = Yc + (size_t)u * BLK + q * 128 + rr * 16;
        *reinterpret_cast<uint4*>(dst) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(dst + 512) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}

// blocks per warp instantiated: the smallest of these >= ceil(NB / 8)
constexpr int NBW_SET[] = {2, 4, 6, 8, 10, 13};
int nbw_of(int NB) {
    const int need = (NB + MW - 1) / MW;
    for (int v : NBW_SET)
        if (v >= need) return v;
    return 0;
}

}  // namespace

bool nmf_mma_plan(const Geometry& g, int num_sms, NmfPlan* p) {
    if (g.K > 16) return false;
    const int NB = (g.Nk + 15) / 16;
    const int nbw = nbw_of(NB);
    if (!nbw) return false;
    if (g.K > 8 && nbw > 10) return false;  // two column blocks: registers for <= 10 blocks per warp
    const size_t smem = mma_smem_bytes(nbw, g.K);
    // static part: mbarriers, the per-warp H accumulators [8 NC]^2, H / G_old / G_new, sums
    const size_t nc = (size_t)mma_nc(g.K), KK = (size_t)g.K * g.K;
    const size_t stat = 8 * (MW * MNS + MNV) + 8 * MW * 64 * nc * nc + 8 * MW * 2 + 24 * KK + 256;
    if (smem + stat + 1024 > (size_t)232448) return false;  // 227 KB per block (1 KB reserved)
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    const int64_t ntiles = (Np + MR - 1) / MR;
    // the persistent launch's D update: lambda slices of SL = ceil(Nk / nCTA) bins per CTA (dnew
    // holds 64 per component, Bsl 256 values, threads [0, K*K + K*SL) produce the outputs)
    {
        const int nC = (int)std::max<int64_t>(1, std::min<int64_t>((Np + MR - 1) / MR, (int64_t)num_sms));
        const int SL = (g.Nk + nC - 1) / nC;
        p->persist_fits = SL <= 64 && g.K * SL <= 256 && g.K * g.K + g.K * SL <= MTH;
    }
    p->mma_NB = NB;
    p->mma_NBW = nbw;
    p->mma_Npad = ntiles * MR;
    p->nblk_f = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)num_sms));
    p->nby = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms * 8, (Np + 7) / 8));
    return true;
}

cudaError_t nmf_mma_prepare(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y, int64_t ld_y,
                            unsigned* status, cudaStream_t s) {
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    cudaError_t e = nmf_tc_stats(g, p, w, Y, ld_y, status, s);
    if (e != cudaSuccess) return e;
    k_mma_convert<<<g.num_sms * 16, 256, 0, s>>>(Y, ld_y, Np, g.Nk, p.mma_NB, p.mma_Npad / MR, w.ymax,
                                                  static_cast<uint8_t*>(w.Yc));
    return cudaGetLastError();
}

cudaError_t nmf_mma_prepare_counts(const Geometry& g, const NmfPlan& p, const NmfWs& w, const DeviceTables& t,
                                   const CountsIn& cin, unsigned* status, cudaStream_t s) {
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    const CountsSrc C{cin.y, cin.y0, cin.b, t.logtab, (int64_t)g.Nr * g.Nc, g.Nk};
    cudaError_t e = cudaMemsetAsync(w.ymax, 0, 2 * sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    k_mma_counts_stats<<<p.nby, 256, 0, s>>>(C, Np, w.ymax, w.ypart, status, w.nclamp);
    k_mma_counts_convert<<<g.num_sms * 16, 256, 0, s>>>(C, Np, p.mma_NB, p.mma_Npad / MR, w.ymax,
                                                         static_cast<uint8_t*>(w.Yc));
    return cudaGetLastError();
}

cudaError_t nmf_mma_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D, int it,
                           unsigned* status, cudaStream_t s) {
    switch (g.K) {
#define M(KV) \
    case KV: return mma_launch_k<KV, false>(g, p, w, V, const_cast<float*>(D), it, 1, nullptr, nullptr, status, s);
        HSNCT_MMA_K(M)
#undef M
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t nmf_mma_persist_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D,
                                   int n_iter, double* obj, unsigned* bar, unsigned* status, cudaStream_t s) {
    switch (g.K) {
#define M(KV) \
    case KV: return mma_launch_k<KV, true>(g, p, w, V, D, 0, n_iter, obj, bar, status, s);
        HSNCT_MMA_K(M)
#undef M
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace hsnct
