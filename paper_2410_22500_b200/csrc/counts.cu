// Counts-domain input (NEXT-1; Eq. 2, with the Appendix-A offset, PAPER.md:
// 718-725, and the 1/2-count floor of DESIGN.md R7):
//
//   Y[p][k] = fp32( (L[y0[rc][k]] - L[y[p][k]]) - b[v][k] ),  L[n] = ln(max(n, 1/2)) in fp64,
//   p = (v N_r + r) N_c + c, rc = p mod N_r N_c, v = p div N_r N_c.
//
// The 256-entry fp64 table is built on the host with the same libm log the oracle calls, so the
// fp64 difference equals the oracle's and the single rounding makes Y bit-identical to
// fp32(oracle).  The decomposition reads 1 byte of y (plus 1/N_v byte of y0, shared by all
// views and served from L2) instead of 4 bytes of Y per element in its input preparation.
#include "internal.h"

namespace hsnct {
namespace {

__device__ __forceinline__ double warp_sum_dd(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One warp per row at a time, lanes over bin quads (the loop structure and fp32 row-sum order
// of k_yplus, so the ||Y+||^2 partials equal those of the materialised path bit for bit).
// mode 0: raw Y into out[p * ld_out + k], k < Nk.  mode 1: Y+ = max(Y, 0) into out[p * Nkp + k]
// with zero padding up to Nkp, per-block ||Y+||^2 partials in ypart, clamped count in nclamp.
// vec: y, y0 rows are 4-byte aligned (Nk % 4 == 0) and b rows 16-byte aligned.
__global__ void __launch_bounds__(256) k_counts(const uint8_t* __restrict__ y, const uint8_t* __restrict__ y0,
                                                const float* __restrict__ b, int64_t Np, int64_t NrNc, int Nk,
                                                int Nkp, const double* __restrict__ Lg, float* __restrict__ out,
                                                int64_t ld_out, int mode, int vec, double* __restrict__ ypart,
                                                unsigned* __restrict__ status,
                                                unsigned long long* __restrict__ nclamp) {
    __shared__ double L[256];
    __shared__ double red[8];
    __shared__ unsigned cred[8];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) L[i] = Lg[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t nw = (int64_t)gridDim.x * 8;
    const int nq = (mode ? Nkp : Nk + 3) >> 2;
    double s = 0.0;
    unsigned ncl = 0, bad = 0;
    for (int64_t p = (int64_t)blockIdx.x * 8 + w; p < Np; p += nw) {
        const int64_t v = p / NrNc, rc = p - v * NrNc;
        const uint8_t* yr = y + p * Nk;
        const uint8_t* y0r = y0 + rc * Nk;
        const float* br = b ? b + v * Nk : nullptr;
        float rs = 0.f;
#pragma unroll 4
        for (int q = lane; q < nq; q += 32) {
            const int l0 = 4 * q;
            unsigned yy[4] = {0, 0, 0, 0}, oo[4] = {0, 0, 0, 0};
            float bb[4] = {0.f, 0.f, 0.f, 0.f};
            if (vec && l0 + 3 < Nk) {
                const uchar4 a = __ldcs(reinterpret_cast<const uchar4*>(yr + l0));
                const uchar4 c = __ldg(reinterpret_cast<const uchar4*>(y0r + l0));
                yy[0] = a.x, yy[1] = a.y, yy[2] = a.z, yy[3] = a.w;
                oo[0] = c.x, oo[1] = c.y, oo[2] = c.z, oo[3] = c.w;
                if (br) {
                    const float4 f = __ldg(reinterpret_cast<const float4*>(br + l0));
                    bb[0] = f.x, bb[1] = f.y, bb[2] = f.z, bb[3] = f.w;
                }
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (l0 + e < Nk) {
                        yy[e] = yr[l0 + e];
                        oo[e] = y0r[l0 + e];
                        if (br) bb[e] = br[l0 + e];
                    }
            }
            float f[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                double d = L[oo[e]] - L[yy[e]];
                if (br) {
                    if (!isfinite(bb[e])) bad = ST_Y_NONFINITE;
                    d -= (double)bb[e];
                }
                f[e] = l0 + e < Nk ? (float)d : 0.f;
            }
            if (mode == 0) {
                float* o = out + p * ld_out + l0;
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (l0 + e < Nk) o[e] = f[e];
            } else {
                ncl += (f[0] < 0.f) + (f[1] < 0.f) + (f[2] < 0.f) + (f[3] < 0.f);
                float4 t = make_float4(fmaxf(f[0], 0.f), fmaxf(f[1], 0.f), fmaxf(f[2], 0.f), fmaxf(f[3], 0.f));
                rs = fmaf(t.x, t.x, fmaf(t.y, t.y, fmaf(t.z, t.z, fmaf(t.w, t.w, rs))));
                reinterpret_cast<float4*>(out + p * Nkp)[q] = t;
            }
        }
        s += (double)rs;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    if (lane == 0 && bad) atomicOr(status, bad);
    if (mode == 0) return;
    s = warp_sum_dd(s);
    ncl = __reduce_add_sync(0xffffffffu, ncl);
    if (lane == 0) {
        red[w] = s;
        cred[w] = ncl;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        unsigned long long c = 0;
        for (int i = 0; i < 8; ++i) {
            t += red[i];
            c += cred[i];
        }
        ypart[blockIdx.x] = t;
        if (c) atomicAdd(nclamp, c);
    }
}

}  // namespace

cudaError_t counts_decode(const Geometry& g, const DeviceTables& t, const CountsIn& cin, float* out, int64_t ld_out,
                          int mode, int nblk, double* ypart, unsigned long long* nclamp, cudaStream_t s) {
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc, NrNc = (int64_t)g.Nr * g.Nc;
    const int Nkp = (g.Nk + 3) & ~3;
    const bool vec = g.Nk % 4 == 0 && (reinterpret_cast<uintptr_t>(cin.y) & 3) == 0 &&
                     (reinterpret_cast<uintptr_t>(cin.y0) & 3) == 0 &&
                     (cin.b == nullptr || (reinterpret_cast<uintptr_t>(cin.b) & 15) == 0);
    k_counts<<<nblk, 256, 0, s>>>(cin.y, cin.y0, cin.b, Np, NrNc, g.Nk, Nkp, t.logtab, out, ld_out, mode, vec ? 1 : 0,
                                  ypart, t.status, nclamp);
    return cudaGetLastError();
}

}  // namespace hsnct
