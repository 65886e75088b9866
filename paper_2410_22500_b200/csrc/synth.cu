// Subspace expansion, Eq. 6: x^h = x^s (D^s)^T on a window
// of slices [s0, s0+ns) and bins [b0, b0+nb):
//     Xh[n][b] = sum_k X[k][s0*Nc*Nc + n] * D[k][b0 + b]
// HBM-write bound (4 B written per output, K/2 flop/B): every thread owns
// output quads along b (float4 streaming stores, evict-first), the D window
// lives in shared memory, X[k][n] is broadcast through L1.
#include <algorithm>

#include "internal.h"

namespace hsnct {
namespace {

constexpr int ST = 256;

// (x, x) * b + c on both halves: one packed FFMA2 with a broadcast scalar
__device__ __forceinline__ float2 ffma2s(float x, float2 b, float2 c) {
    float2 r;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %2};\n\t"
        "mov.b64 rb, {%3, %4};\n\t"
        "mov.b64 rc, {%5, %6};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
        "mov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(x), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}
constexpr int BCH = 512;   // max bins per block column (D window in smem <= K * 512 floats)

template <int K, bool VEC>
__global__ void __launch_bounds__(ST) k_synth(const float* __restrict__ X, const float* __restrict__ D,
                                              int64_t Nx, int Nk, int64_t n0, int64_t nn, int b0,
                                              int nb, int bcw, float* __restrict__ Xh, int64_t ld) {
    __shared__ __align__(16) float Ds[K * BCH];
    const int bc0 = blockIdx.y * bcw;                 // first bin (window-relative) of this column
    const int nbc = min(bcw, nb - bc0);
    for (int t = threadIdx.x; t < K * BCH; t += ST) {
        const int k = t / BCH, b = t - k * BCH;
        Ds[t] = (b < nbc) ? D[(int64_t)k * Nk + b0 + bc0 + b] : 0.f;
    }
    __syncthreads();
    const int nq = (nbc + 3) >> 2;
    const int64_t total = nn * nq;
    for (int64_t idx = (int64_t)blockIdx.x * ST + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * ST) {
        const int64_t n = idx / nq;
        const int q = (int)(idx - n * nq);
        float x[K];
#pragma unroll
        for (int k = 0; k < K; ++k) x[k] = __ldg(X + (int64_t)k * Nx + n0 + n);
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const float4 d = reinterpret_cast<const float4*>(Ds + k * BCH)[q];
            o.x = fmaf(x[k], d.x, o.x);
            o.y = fmaf(x[k], d.y, o.y);
            o.z = fmaf(x[k], d.z, o.z);
            o.w = fmaf(x[k], d.w, o.w);
        }
        float* dst = Xh + n * ld + bc0 + 4 * q;
        const int valid = nbc - 4 * q;
        if (VEC && valid >= 4) {
            __stcs(reinterpret_cast<float4*>(dst), o);
        } else {
            if (valid > 0) __stcs(dst + 0, o.x);
            if (valid > 1) __stcs(dst + 1, o.y);
            if (valid > 2) __stcs(dst + 2, o.z);
            if (valid > 3) __stcs(dst + 3, o.w);
        }
    }
}

// Vectorised variant (Xh 16-byte aligned, ld % 4 == 0): a warp owns 32 consecutive bin
// quads (128 bins) of a bin group and walks chunks of 32 consecutive voxels: X[k][chunk] is
// one coalesced load per k, broadcast voxel by voxel with a shuffle; each lane keeps its D
// quads in registers; packed f32x2 FMAs; one streaming 16-byte store per lane per voxel.
// Grid: (voxel-chunk blocks, bin groups).
template <int K>
__global__ void __launch_bounds__(ST) k_synth_v(const float* __restrict__ X, const float* __restrict__ D, int64_t Nx,
                                                int Nk, int64_t n0, int64_t nn, int b0, int nb,
                                                float* __restrict__ Xh, int64_t ld) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nq = (nb + 3) >> 2;
    const int nqg = (nq + 31) >> 5;                    // bin groups of 32 quads
    const int64_t nchunk = (nn + 31) >> 5;
    const int64_t nunits = nchunk * nqg;               // unit = (voxel chunk, bin group), group fastest
    const int64_t wstride = (int64_t)gridDim.x * (ST / 32);
    // this warp's X chunk, k-major, so that one broadcast LDS.128 serves four voxels
    __shared__ __align__(16) float xs[ST / 32][K][32];
    int grp = -1, q = 0;
    bool act = false, full = false;
    float4 d[K];
    for (int64_t u = (int64_t)blockIdx.x * (ST / 32) + warp; u < nunits; u += wstride) {
        const int g = (int)(u % nqg);
        const int64_t ch = u / nqg;
        if (g != grp) {  // this lane's bin quad and its D values
            grp = g;
            q = g * 32 + lane;
            act = q < nq;
            full = 4 * q + 3 < nb;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                float v[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int b = 4 * q + e;
                    v[e] = (act && b < nb) ? __ldg(D + (int64_t)k * Nk + b0 + b) : 0.f;
                }
                d[k] = make_float4(v[0], v[1], v[2], v[3]);
            }
        }
        const int64_t nb0 = ch << 5;
        const int cnt = (int)min((int64_t)32, nn - nb0);
        __syncwarp();  // the previous unit's reads of xs are done
#pragma unroll
        for (int k = 0; k < K; ++k) xs[warp][k][lane] = lane < cnt ? __ldg(X + (int64_t)k * Nx + n0 + nb0 + lane) : 0.f;
        __syncwarp();
        float* dst = Xh + nb0 * ld + 4 * q;
        for (int i = 0; i < cnt; i += 4) {
            float4 xv[K];
#pragma unroll
            for (int k = 0; k < K; ++k) xv[k] = *reinterpret_cast<const float4*>(&xs[warp][k][i]);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float2 o01 = make_float2(0.f, 0.f), o23 = make_float2(0.f, 0.f);
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const float x = j == 0 ? xv[k].x : (j == 1 ? xv[k].y : (j == 2 ? xv[k].z : xv[k].w));
                    o01 = ffma2s(x, make_float2(d[k].x, d[k].y), o01);
                    o23 = ffma2s(x, make_float2(d[k].z, d[k].w), o23);
                }
                if (act && i + j < cnt) {
                    if (full) {
                        __stcs(reinterpret_cast<float4*>(dst), make_float4(o01.x, o01.y, o23.x, o23.y));
                    } else {
                        const int valid = nb - 4 * q;
                        __stcs(dst, o01.x);
                        if (valid > 1) __stcs(dst + 1, o01.y);
                        if (valid > 2) __stcs(dst + 2, o23.x);
                    }
                }
                dst += ld;
            }
        }
    }
}

#define HSNCT_K_CASES(M) \
    M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15) M(16)

template <int K>
cudaError_t synth_k(const Geometry& g, const float* X, const float* D, int s0, int ns, int b0, int nb,
                    float* Xh, int64_t ld, cudaStream_t s, int num_sms) {
    const int64_t Nx = (int64_t)g.Nr * g.Nc * g.Nc;
    const int64_t n0 = (int64_t)s0 * g.Nc * g.Nc, nn = (int64_t)ns * g.Nc * g.Nc;
    const int ncol = (nb + BCH - 1) / BCH;
    const int bcw = (((nb + ncol - 1) / ncol) + 3) & ~3;   // equal columns, multiple of 4
    const int nq = bcw / 4;
    const int64_t per_col = nn * nq;
    const int64_t want = std::max<int64_t>(1, ((int64_t)num_sms * 8) / ncol);
    const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>(want, (per_col + ST - 1) / ST));
    dim3 grid(nblk, ncol);
    const bool vec = ((reinterpret_cast<uintptr_t>(Xh) & 15) == 0) && (ld % 4 == 0);
    if (vec) {  // one flat list of (voxel chunk, bin group) units over num_sms x 8 blocks
        const int64_t nunits = ((nn + 31) / 32) * ((nb + 127) / 128);
        const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms * 8, (nunits + 7) / 8));
        k_synth_v<K><<<(unsigned)blocks, ST, 0, s>>>(X, D, Nx, g.Nk, n0, nn, b0, nb, Xh, ld);
        return cudaGetLastError();
    }
    if (vec)
        k_synth<K, true><<<grid, ST, 0, s>>>(X, D, Nx, g.Nk, n0, nn, b0, nb, bcw, Xh, ld);
    else
        k_synth<K, false><<<grid, ST, 0, s>>>(X, D, Nx, g.Nk, n0, nn, b0, nb, bcw, Xh, ld);
    return cudaGetLastError();
}

}  // namespace

cudaError_t synthesize(const Geometry& g, const float* X, const float* D, int s0, int ns, int b0,
                       int nb, float* Xh, int64_t ld_xh, cudaStream_t s) {
    if (ns <= 0 || nb <= 0) return cudaSuccess;
    switch (g.K) {
#define M(KV) \
    case KV:  \
        return synth_k<KV>(g, X, D, s0, ns, b0, nb, Xh, ld_xh, s, g.num_sms);
        HSNCT_K_CASES(M)
#undef M
        default:
            return cudaErrorInvalidValue;
    }
}

}  // namespace hsnct
