// Host side of the mma.sync NMF path (nmf_mma.cuh): input preparation (Y+ or counts into the
// block layout), plan, per-K dispatch.
#include "nmf_mma.cuh"

namespace hsnct {
namespace {

// ---- input preparation: Y+ (or Eq. 2 decoded from counts) into the block layout, one pass.
// Block b takes tiles b, b + grid, ...: per tile a first sweep over its items (tile row, 8 bins)
// for max Y+, ||Y+||^2, the non-finite check and the clamped count; the tile's scale exponent
// (sigma_Y = 2^e, 2^e max < 2^14) to texp; a second sweep (L2-hot re-read) splits Y+ sigma_Y into
// fp16 hi/lo blocks.  Item (block j, core matrix q, row rr), rr fastest: 32 consecutive threads
// write one block's hi and lo halves (512 contiguous bytes each).  ||Y+||^2 partials per CUDA
// block in a fixed order (deterministic).
struct YSrc {  // fp32 Y [Np][ld]
    const float* Y;
    int64_t ld;
    __device__ void stage(double*) const {}
    __device__ void tile(int64_t) {}
    template <bool LAST>
    __device__ __forceinline__ void load8(int64_t r, int ri, int l, int64_t Np, int Nk, float (&v)[8]) const {
        (void)ri;
        if (r < Np && l + 8 <= Nk) {
            const float4* y = reinterpret_cast<const float4*>(Y + r * ld + l);
            const float4 a = LAST ? __ldcs(y) : __ldg(y), b = LAST ? __ldcs(y + 1) : __ldg(y + 1);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = (r < Np && l + e < Nk) ? Y[r * ld + l + e] : 0.f;
        }
    }
};
// uint8 counts: Y = fp32((L[y0] - L[y]) - b), L[n] = ln max(n, 1/2) in fp64 (counts.cu, DESIGN.md
// R7): the same per-element value as hsnct_counts_to_projections, so the decomposition from
// counts is bit-identical to the one from the materialised Y.
struct CSrc {
    const uint8_t* y;    // [Np][Nk]
    const uint8_t* y0;   // [Nr Nc][Nk]
    const float* b;      // [Nv][Nk] or null
    const double* Lg;    // [256] (device table)
    int64_t NrNc;
    int vec;             // N_k % 8 == 0 and y, y0 8-byte, b 16-byte aligned
    const double* L;     // the table in shared memory (stage)
    int64_t v0, rc0;     // view and (r, c) index of the current tile's first row
    __device__ void stage(double* Ls) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) Ls[i] = Lg[i];
        L = Ls;
    }
    __device__ void tile(int64_t t) {
        const int64_t r0 = t * 16;
        v0 = r0 / NrNc;
        rc0 = r0 - v0 * NrNc;
    }
    template <bool LAST>
    __device__ __forceinline__ void load8(int64_t r, int ri, int l, int64_t Np, int Nk, float (&v)[8]) const {
        int64_t rc = rc0 + ri, vv = v0;
        if (rc >= NrNc) {  // the tile crosses into the next view
            rc -= NrNc;
            ++vv;
        }
        const uint8_t* yr = y + r * Nk;
        const uint8_t* y0r = y0 + rc * Nk;
        const float* br = b ? b + vv * Nk : nullptr;
        if (vec && r < Np && l + 8 <= Nk) {  // 8-byte count loads, 16-byte offset loads
            const uint2 a = LAST ? __ldcs(reinterpret_cast<const uint2*>(yr + l)) : __ldg(reinterpret_cast<const uint2*>(yr + l));
            const uint2 o = __ldg(reinterpret_cast<const uint2*>(y0r + l));
            float bb[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            if (br) {
                const float4 b0 = __ldg(reinterpret_cast<const float4*>(br + l)), b1 = __ldg(reinterpret_cast<const float4*>(br + l) + 1);
                bb[0] = b0.x; bb[1] = b0.y; bb[2] = b0.z; bb[3] = b0.w;
                bb[4] = b1.x; bb[5] = b1.y; bb[6] = b1.z; bb[7] = b1.w;
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const unsigned ye = ((e < 4 ? a.x : a.y) >> (8 * (e & 3))) & 0xffu;
                const unsigned oe = ((e < 4 ? o.x : o.y) >> (8 * (e & 3))) & 0xffu;
                double d = L[oe] - L[ye];
                if (br) d -= (double)bb[e];
                v[e] = (float)d;
            }
            return;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            float f = 0.f;
            if (r < Np && l + e < Nk) {
                double d = L[y0r[l + e]] - L[yr[l + e]];
                if (br) d -= (double)br[l + e];
                f = (float)d;
            }
            v[e] = f;
        }
    }
};

template <class Src>
__global__ void __launch_bounds__(256) k_mma_prep(Src src, int64_t Np, int Nk, int NB, int64_t ntiles,
                                                  uint8_t* __restrict__ Yc, int* __restrict__ texp,
                                                  double* __restrict__ ypart, unsigned* __restrict__ status,
                                                  unsigned long long* __restrict__ nclamp) {
    __shared__ double Ls[256];
    __shared__ float redm[8];
    __shared__ double reds[8];
    __shared__ unsigned redc[8];
    src.stage(Ls);
    __syncthreads();
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int nit = NB * 32;
    double s = 0.0;
    unsigned ncl = 0, bad = 0;
    for (int64_t tt = blockIdx.x; tt < ntiles; tt += gridDim.x) {
        src.tile(tt);
        float m = 0.f, ps = 0.f;
        for (int i = tid; i < nit; i += 256) {
            const int rr = i & 7, q = (i >> 3) & 3, j = i >> 5;
            const int ri = (q & 1) * 8 + rr;
            float v[8];
            src.template load8<false>(tt * MR + ri, ri, 16 * j + (q >> 1) * 8, Np, Nk, v);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                if (!isfinite(v[e])) bad = ST_Y_NONFINITE;
                ncl += v[e] < 0.f;
                const float yp = fmaxf(v[e], 0.f);
                m = fmaxf(m, yp);
                ps = fmaf(yp, yp, ps);
            }
        }
        s += (double)ps;
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) redm[w] = m;
        __syncthreads();
        float tm = redm[0];
#pragma unroll
        for (int u = 1; u < 8; ++u) tm = fmaxf(tm, redm[u]);
        const int e = mexp(tm);
        const float sy = pow2(e);
        if (tid == 0) texp[tt] = e;
        for (int i = tid; i < nit; i += 256) {
            const int rr = i & 7, q = (i >> 3) & 3, j = i >> 5;
            const int ri = (q & 1) * 8 + rr;
            float v[8];
            src.template load8<true>(tt * MR + ri, ri, 16 * j + (q >> 1) * 8, Np, Nk, v);
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                hw[u] = split2(fmaxf(v[2 * u], 0.f) * sy, fmaxf(v[2 * u + 1], 0.f) * sy, lw[u]);
            uint8_t* dst = Yc + ((size_t)tt * NB + j) * BLK + q * 128 + rr * 16;
            *reinterpret_cast<uint4*>(dst) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4*>(dst + 512) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
        __syncthreads();  // redm is reused by the next tile
    }
    s = warp_sum_d(s);
    ncl = __reduce_add_sync(0xffffffffu, ncl);
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (lane == 0) {
        reds[w] = s;
        redc[w] = ncl;
        if (bad) atomicOr(status, bad);
    }
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        unsigned long long c = 0;
        for (int u = 0; u < 8; ++u) {
            t += reds[u];
            c += redc[u];
        }
        ypart[blockIdx.x] = t;
        if (c) atomicAdd(nclamp, c);
    }
}

// blocks per warp instantiated: the smallest of these >= ceil(NB / warps)
constexpr int NBW_SET[] = {2, 4, 6, 8, 10, 13};
constexpr int NBW_SET16[] = {1, 2, 3, 4, 5};
int nbw_of(int NB, int mw) {
    const int need = (NB + mw - 1) / mw;
    if (mw == MW16) {
        for (int v : NBW_SET16)
            if (v >= need) return v;
        return 0;
    }
    for (int v : NBW_SET)
        if (v >= need) return v;
    return 0;
}

}  // namespace

bool nmf_mma_plan(const Geometry& g, int num_sms, NmfPlan* p) {
    if (g.K > 16) return false;
    const int NB = (g.Nk + 15) / 16;
    // K = 9..16 (two column blocks): 8 warps with <= 10 blocks each (255 registers).  In a build with
    // -DHSNCT_MMA_MW16 (not the product library), HSNCT_MMA_MW=16 selects the 16-warp form (<= 5 blocks per warp, 128 registers, four warps per scheduler),
    // measured slower at C6 (12.1 vs 10.4 ms per iteration: the per-warp, per-tile work -- partial-A
    // exchange, operand loads, barriers -- is paid 16 times; profiles/r02/session4/ab_split.txt)
    int mw = MW;
#ifdef HSNCT_MMA_MW16  // experimental build only (build.py --variant=mw16 -DHSNCT_MMA_MW16)
    if (g.K > 8) {
        const char* e = getenv("HSNCT_MMA_MW");
        if (e && atoi(e) == 16) mw = MW16;
    }
#endif
    const int nbw = nbw_of(NB, mw);
    if (!nbw) return false;
    if (g.K > 8 && nbw > 10) return false;  // two column blocks: registers for <= 10 blocks per warp
    const size_t smem = mma_smem_bytes(nbw, g.K, mw);
    // static part: mbarriers, the H accumulators of 8 warps [8 NC]^2, H / G_old / G_new, G as
    // float, the tile's new V, sums
    const size_t nc = (size_t)mma_nc(g.K), KK = (size_t)g.K * g.K;
    const size_t stat = 8 * ((size_t)mw * MNS + MNV) + 8 * 8 * 64 * nc * nc + 8 * (size_t)mw * 2 + 24 * KK +
                        4 * 16 * (size_t)g.K + 4 * 8 * nc * MR + 256;
    if (smem + stat + 1024 > (size_t)232448) return false;  // 227 KB per block (1 KB reserved)
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    const int64_t ntiles = (Np + MR - 1) / MR;
    // the persistent launch's D update: lambda slices of SL = ceil(Nk / nCTA) bins per CTA (dnew
    // holds 64 per component, Bsl 256 values, threads [0, K*K + K*SL) produce the outputs)
    {
        const int nC = (int)std::max<int64_t>(1, std::min<int64_t>((Np + MR - 1) / MR, (int64_t)num_sms));
        const int SL = (g.Nk + nC - 1) / nC;
        p->persist_fits = SL <= 64 && g.K * SL <= 256 && g.K * g.K + g.K * SL <= mw * 32;
    }
    p->mma_NB = NB;
    p->mma_NBW = nbw;
    p->mma_MW = mw;
    p->mma_Npad = ntiles * MR;
    p->nblk_f = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)num_sms));
    p->nby = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms * 8, (Np + 7) / 8));
    return true;
}

cudaError_t nmf_mma_prepare(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y, int64_t ld_y,
                            unsigned* status, cudaStream_t s) {
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    k_mma_prep<YSrc><<<p.nby, 256, 0, s>>>(YSrc{Y, ld_y}, Np, g.Nk, p.mma_NB, p.mma_Npad / MR,
                                          static_cast<uint8_t*>(w.Yc), w.texp, w.ypart, status, w.nclamp);
    return cudaGetLastError();
}

cudaError_t nmf_mma_prepare_counts(const Geometry& g, const NmfPlan& p, const NmfWs& w, const DeviceTables& t,
                                   const CountsIn& cin, unsigned* status, cudaStream_t s) {
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    const bool vec = g.Nk % 8 == 0 && (reinterpret_cast<uintptr_t>(cin.y) & 7) == 0 &&
                     (reinterpret_cast<uintptr_t>(cin.y0) & 7) == 0 &&
                     (cin.b == nullptr || (reinterpret_cast<uintptr_t>(cin.b) & 15) == 0);
    CSrc src{cin.y, cin.y0, cin.b, t.logtab, (int64_t)g.Nr * g.Nc, vec ? 1 : 0, nullptr, 0, 0};
    k_mma_prep<CSrc><<<p.nby, 256, 0, s>>>(src, Np, g.Nk, p.mma_NB, p.mma_Npad / MR, static_cast<uint8_t*>(w.Yc),
                                          w.texp, w.ypart, status, w.nclamp);
    return cudaGetLastError();
}

cudaError_t nmf_mma_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D, int it,
                           unsigned* status, cudaStream_t s) {
#define M(KV) \
    case KV: return mma_launch_k<KV, false>(g, p, w, V, const_cast<float*>(D), it, 1, nullptr, nullptr, status, s);
#define M16(KV) \
    case KV: return mma_launch_k16<KV, false>(g, p, w, V, const_cast<float*>(D), it, 1, nullptr, nullptr, status, s);
#ifdef HSNCT_MMA_MW16
    if (p.mma_MW == MW16) {
        switch (g.K) {
            HSNCT_MMA_KHI(M16)
            default: return cudaErrorInvalidValue;
        }
    }
#endif
    switch (g.K) {
        HSNCT_MMA_K(M)
        default: return cudaErrorInvalidValue;
    }
#undef M16
#undef M
}

cudaError_t nmf_mma_persist_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D,
                                   int n_iter, double* obj, unsigned* bar, unsigned* status, cudaStream_t s) {
#define M(KV) \
    case KV: return mma_launch_k<KV, true>(g, p, w, V, D, 0, n_iter, obj, bar, status, s);
#define M16(KV) \
    case KV: return mma_launch_k16<KV, true>(g, p, w, V, D, 0, n_iter, obj, bar, status, s);
#ifdef HSNCT_MMA_MW16
    if (p.mma_MW == MW16) {
        switch (g.K) {
            HSNCT_MMA_KHI(M16)
            default: return cudaErrorInvalidValue;
        }
    }
#endif
    switch (g.K) {
        HSNCT_MMA_K(M)
        default: return cudaErrorInvalidValue;
    }
#undef M16
#undef M
}

}  // namespace hsnct
