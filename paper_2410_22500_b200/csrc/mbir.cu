// MBIR of the subspace sinograms (NEXT-3; Eq. 5; DESIGN.md
// R24-R26): x = argmin_{x >= 0} 1/(2 sv^2) ||y - A x||^2 + h(x), h the QGGMRF prior (q = 2) on
// the 8-neighbourhood, solved by separable-quadratic-surrogate (SQS) iterations.  Per iteration:
//
//   k_project   e = y - A x for every (slice, view, bin) and all K channels at once: the exact
//               transpose of k_backproject's linear interpolation (weight max(0, 1 - |u - c|),
//               u = x cos + y sin + (N_c - 1)/2), written as a gather so that every output is
//               one register accumulator (deterministic, no atomics).  Block = one slice and a
//               group of VB views of one orientation class; the slice is streamed through shared
//               memory in strips of R lines (rows for |cos| >= |sin|, columns otherwise) so
//               that along a line the bins of a warp read <= 3 consecutive pixels each.
//   backproject (fbp.cu, reused) g = A^T e, scaled pi/N_v (folded back out in k_sqs).
//   k_sqs       per voxel and channel: gradient and curvature of the surrogate, Jacobi step
//               x <- max(0, x - g / (dd + dp)) into the other iterate buffer.
//
// Iterates live channel-innermost, Xi[r][i][j][KP] (KP = K rounded up to even: one FFMA2 per
// channel pair), so the projector's geometry is shared by all channels as in the backprojector.
#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"

namespace hsnct {
namespace {

constexpr int PT = 512;          // projector threads (16 warps)
constexpr int PW = PT / 32;

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 r;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mov.b64 rc, {%6, %7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}

__device__ __forceinline__ void cp_async8(float* dst, const float* src, bool ok) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
}

// X[k][n] (channel-planar, n over N_r N_c^2) -> Xi[n][KP] (pad channels 0)
template <int KP>
__global__ void __launch_bounds__(256) k_to_inner(const float* __restrict__ X, int K, int64_t Nx, float* __restrict__ Xi) {
    const int64_t n = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (n >= Nx) return;
    float v[KP];
#pragma unroll
    for (int k = 0; k < KP; ++k) v[k] = k < K ? X[(int64_t)k * Nx + n] : 0.f;
#pragma unroll
    for (int k = 0; k < KP; k += 2) *reinterpret_cast<float2*>(Xi + n * KP + k) = make_float2(v[k], v[k + 1]);
}

// Xi[n][2] = (1, 0): the all-ones image of one slice (data curvature A^T A 1)
__global__ void k_ones(float2* __restrict__ Xi, int64_t n) {
    const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (t < n) Xi[t] = make_float2(1.f, 0.f);
}

// Forward projection of one slice (blockIdx.y) for the VB views of group blockIdx.x.
// groups[g][0] = orientation class (1: |cos| >= |sin|, lines = image rows, position = column;
// 0: lines = columns, position = row); groups[g][1 + s] = view of slot s or -1.
// Warp w serves view slot w / WPV and the 32*CPT bins starting at (w % WPV) 32 CPT; lane l owns
// bins base + 32 m + l, m < CPT.  Per line L and bin c the pixels with |u - c| < 1 lie in
// (pc - 1/|a|, pc + 1/|a|), pc the position where u = c, a the position's coefficient
// (|a| >= 1/sqrt 2): at most three consecutive positions, from ceil(pc - 1/|a| - 1e-3).
// Every staged line carries PPAD zero positions on both sides and p0 is clamped to
// [-PPAD, Nc + PPAD - 3], so the three taps never leave the strip and need no bounds test
// (a clamped p0 lies >= 1 position away from the bin: weight 0).
// Strip layout: row class [line][PPAD + pos][KP] (a line = one contiguous image row);
// column class [PPAD + pos][line][KP] (per image row, the strip's columns are contiguous), the
// position pitch padded to an odd number of 8-byte words (bank spread of a warp's taps).
// mode 0: out = E[r][v][c][Kc] = y - A x (y = Y[((v Nr + r) Nc + c) K + k], or -A x if Y is
//         NULL), channels K..Kc-1 zero; osc * sum of e^2 is added to *obj (nullable).
// mode 1: out = P[((v Nr + r) Nc + c) K + k] = (A x), the layout of V.
constexpr int PPAD = 4;
__host__ __device__ inline int col_pitch(int R, int KP) { return R * KP + (((R * KP / 2) & 1) ? 0 : 2); }
__host__ __device__ inline int strip_floats(int R, int Nc, int KP) {
    return max(R * (Nc + 2 * PPAD) * KP, (Nc + 2 * PPAD) * col_pitch(R, KP));
}

template <int KP, int CPT>
__global__ void __launch_bounds__(PT, 1) k_project(const float* __restrict__ Xi, int Nr, int Nc, int Nv,
                                                   const int* __restrict__ groups, int VB, int R,
                                                   const float* __restrict__ cos_t, const float* __restrict__ sin_t,
                                                   const float* __restrict__ Y, int K, int mode,
                                                   float* __restrict__ out, int Kc, double* obj, double osc) {
    extern __shared__ __align__(16) float xs[];  // [2][strip_floats]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int r = blockIdx.y;
    const int* grp = groups + blockIdx.x * (VB + 1);
    const int rowcls = grp[0];
    const int WPV = (Nc + 32 * CPT - 1) / (32 * CPT);
    const int slot = warp / WPV;
    const int v = slot < VB ? grp[1 + slot] : -1;
    const int cbase = (warp % WPV) * 32 * CPT + lane;
    const float half = 0.5f * (float)(Nc - 1);
    float a = 1.f, b = 0.f, inv = 0.f, ra = 0.f;
    if (v >= 0) {
        const float cs = cos_t[v], sn = sin_t[v];
        a = rowcls ? cs : sn;  // coefficient of the position along the line
        b = rowcls ? sn : cs;  // coefficient of the line index
        inv = 1.f / a;
        ra = fabsf(inv);
    }
    const float* Xr = Xi + (int64_t)r * Nc * Nc * KP;
    const int SF = strip_floats(R, Nc, KP);
    // element (line l, position p) of a strip at l * sL + (p + PPAD) * sP floats
    const int sL = rowcls ? (Nc + 2 * PPAD) * KP : KP;
    const int sP = rowcls ? KP : col_pitch(R, KP);
    const int nchk = (Nc + R - 1) / R;

    // zero padding positions of both buffers (never written by the copies)
    for (int t = tid; t < 2 * R * 2 * PPAD * (KP / 2); t += PT) {
        const int e2 = t % (KP / 2), q = t / (KP / 2);
        const int pp = q % (2 * PPAD), lq = q / (2 * PPAD), l = lq % R, bf = lq / R;
        const int p = pp < PPAD ? pp - PPAD : Nc + pp - PPAD;
        *reinterpret_cast<float2*>(xs + bf * SF + l * sL + (p + PPAD) * sP + 2 * e2) = make_float2(0.f, 0.f);
    }

    // strip ck (lines ck*R .. ck*R+nl-1) into buffer bf, 8-byte copies
    auto stage = [&](int ck, int bf) {
        float* dst = xs + bf * SF;
        const int L0 = ck * R, nl = min(R, Nc - L0);
        if (rowcls) {
            for (int l = 0; l < nl; ++l) {
                const float* src = Xr + (int64_t)(L0 + l) * Nc * KP;
                float* d = dst + l * sL + PPAD * KP;
                for (int e = tid; e < Nc * KP / 2; e += PT) cp_async8(d + 2 * e, src + 2 * e, true);
            }
        } else {
            for (int p = warp; p < Nc; p += PW) {
                const float* src = Xr + ((int64_t)p * Nc + L0) * KP;
                float* d = dst + (p + PPAD) * sP;
                for (int e = lane; e < nl * KP / 2; e += 32) cp_async8(d + 2 * e, src + 2 * e, true);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    float2 acc[CPT][KP / 2];
#pragma unroll
    for (int m = 0; m < CPT; ++m)
#pragma unroll
        for (int q = 0; q < KP / 2; ++q) acc[m][q] = make_float2(0.f, 0.f);

    stage(0, 0);
    for (int ck = 0; ck < nchk; ++ck) {
        const int bf = ck & 1;
        if (ck + 1 < nchk) {
            stage(ck + 1, bf ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        if (v >= 0) {
            const float* strip = xs + bf * SF + PPAD * sP;
            const int nl = min(R, Nc - ck * R);
            for (int l = 0; l < nl; ++l) {
                const float t = fmaf((float)(ck * R + l) - half, b, half);
                const float* line = strip + l * sL;
#pragma unroll
                for (int m = 0; m < CPT; ++m) {
                    const float c = (float)(cbase + 32 * m);
                    const float pc = fmaf(c - t, inv, half);
                    const int p0 = min(max((int)ceilf(pc - ra - 1e-3f), -PPAD), Nc + PPAD - 3);
                    float u = fmaf((float)p0 - half, a, t) - c;  // u(p0) - c, then + a per tap
                    const float* px = line + p0 * sP;
#pragma unroll
                    for (int q3 = 0; q3 < 3; ++q3) {
                        const float w = fmaxf(0.f, 1.f - fabsf(u));
                        u += a;
#pragma unroll
                        for (int q = 0; q < KP / 2; ++q)
                            acc[m][q] = ffma2(make_float2(w, w), *reinterpret_cast<const float2*>(px + q3 * sP + 2 * q),
                                              acc[m][q]);
                    }
                }
            }
        }
        __syncthreads();  // buffer bf is refilled by the next iteration's prefetch
    }

    double sq = 0.0;
    if (v >= 0) {
#pragma unroll
        for (int m = 0; m < CPT; ++m) {
            const int c = cbase + 32 * m;
            if (c >= Nc) break;
            const int64_t prow = ((int64_t)v * Nr + r) * Nc + c;
            if (mode == 0) {
                float* e = out + (((int64_t)r * Nv + v) * Nc + c) * Kc;
#pragma unroll
                for (int k = 0; k < KP; ++k) {
                    if (k >= K) break;
                    const float ax = (k & 1) ? acc[m][k >> 1].y : acc[m][k >> 1].x;
                    const float ev = (Y ? Y[prow * K + k] : 0.f) - ax;
                    e[k] = ev;
                    sq += (double)ev * ev;
                }
                for (int k = K; k < Kc; ++k) e[k] = 0.f;
            } else {
#pragma unroll
                for (int k = 0; k < KP; ++k) {
                    if (k >= K) break;
                    out[prow * K + k] = (k & 1) ? acc[m][k >> 1].y : acc[m][k >> 1].x;
                }
            }
        }
    }
    if (obj) {
        __shared__ double red[PW];
#pragma unroll
        for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) red[warp] = sq;
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int w = 0; w < PW; ++w) s += red[w];
            atomicAdd(obj, s * osc);
        }
    }
}

__device__ __forceinline__ float lg2a(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float ex2a(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct SqsParams {
    float gs;       // -1/sv^2 * N_v/pi: data gradient = gs * G (G = (pi/N_v) A^T e)
    float ds;       // -1/sv^2 * N_v/pi: data curvature = ds * G1 (G1 = (pi/N_v) A^T (-A 1))
    float c0;       // w(0) = 1 / (sx^p (T sx)^(2-p))
    float k2;       // (2 - p) / p
    float e;        // 2 - p (exponent of u)
    float inv_tsx;  // 1 / (T sx)
    float rho_s;    // c0 / p: rho(d) = rho_s d^2 / (1 + u)
    float b1, b2;   // edge and diagonal neighbour weights
};

// Jacobi SQS step of every voxel n of the N_r slices, all channels.  update = 0: only the prior
// term of the objective at Xc (added to *obj).  Xout (nullable): also write the new iterate
// channel-planar X[k][n] (the last iteration).
template <int KP>
__global__ void __launch_bounds__(256) k_sqs(const float* __restrict__ Xc, const float* __restrict__ G,
                                             const float* __restrict__ G1, float* __restrict__ Xn,
                                             float* __restrict__ Xout, int K, int Nc, int64_t Nx, SqsParams sp,
                                             double* obj, int update, unsigned* status) {
    const int64_t n = (int64_t)blockIdx.x * 256 + threadIdx.x;
    double prior = 0.0;
    if (n < Nx) {
        const int64_t pl = n % ((int64_t)Nc * Nc);
        const int i = (int)(pl / Nc), j = (int)(pl % Nc);
        float x0[KP], g[KP], dk[KP];
#pragma unroll
        for (int q = 0; q < KP; q += 2) {
            const float2 t = *reinterpret_cast<const float2*>(Xc + n * KP + q);
            x0[q] = t.x;
            x0[q + 1] = t.y;
        }
        const float dd = update ? sp.ds * G1[pl] : 0.f;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            g[k] = (update && k < K) ? sp.gs * G[(int64_t)k * Nx + n] : 0.f;
            dk[k] = dd;
        }
        float pr = 0.f;
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
            const int di = nb < 3 ? -1 : (nb < 5 ? 0 : 1);
            const int dj = (nb == 0 || nb == 3 || nb == 5) ? -1 : ((nb == 1 || nb == 6) ? 0 : 1);
            const int i2 = i + di, j2 = j + dj;
            if (i2 < 0 || i2 >= Nc || j2 < 0 || j2 >= Nc) continue;
            const float bw = (di != 0 && dj != 0) ? sp.b2 : sp.b1;
            const float* xn = Xc + (n + (int64_t)di * Nc + dj) * KP;
            const bool fwd = nb >= 4;  // (0,+1), (+1,-1), (+1,0), (+1,+1): each unordered pair once
#pragma unroll
            for (int q = 0; q < KP; q += 2) {
                const float2 t = *reinterpret_cast<const float2*>(xn + q);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int k = q + h;
                    if (k >= K) break;
                    const float d = x0[k] - (h ? t.y : t.x);
                    const float u = sp.e == 0.f ? 1.f : ex2a(sp.e * lg2a(fabsf(d) * sp.inv_tsx));
                    const float rr = 1.f / (1.f + u);
                    const float w = sp.c0 * rr * fmaf(sp.k2, rr, 1.f);
                    g[k] = fmaf(bw * w, d, g[k]);
                    dk[k] = fmaf(2.f * bw, w, dk[k]);
                    if (obj && fwd) pr = fmaf(bw * sp.rho_s * d * d, rr, pr);
                }
            }
        }
        prior = pr;
        if (update) {
            float xv[KP];
            bool fin = true;
#pragma unroll
            for (int k = 0; k < KP; ++k) {
                const float t = x0[k] - g[k] / dk[k];
                fin &= k >= K || isfinite(t);
                xv[k] = k < K ? fmaxf(0.f, t) : 0.f;
            }
            if (!fin) atomicOr(status, ST_NUMERIC);
#pragma unroll
            for (int q = 0; q < KP; q += 2)
                *reinterpret_cast<float2*>(Xn + n * KP + q) = make_float2(xv[q], xv[q + 1]);
            if (Xout) {
#pragma unroll
                for (int k = 0; k < KP; ++k)
                    if (k < K) Xout[(int64_t)k * Nx + n] = xv[k];
            }
        }
    }
    if (obj) {
        __shared__ double red[8];
#pragma unroll
        for (int o = 16; o; o >>= 1) prior += __shfl_xor_sync(0xffffffffu, prior, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = prior;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s = 0.0;
            for (int w = 0; w < 8; ++w) s += red[w];
            atomicAdd(obj, s);
        }
    }
}

}  // namespace

// ------------------------------------------------------------------------ host side

int mbir_kp(int K) { return (K + 1) & ~1; }
int mbir_cpt(int K) { return mbir_kp(K) <= 8 ? 4 : 2; }

MbirGroups mbir_groups(const Geometry& g, const float* cs, const float* sn) {
    MbirGroups G;
    const int cpt = mbir_cpt(g.K);
    const int wpv = (g.Nc + 32 * cpt - 1) / (32 * cpt);
    G.vb = std::max(1, PW / wpv);
    for (int cls = 1; cls >= 0; --cls) {
        std::vector<int> vs;
        for (int v = 0; v < g.Nv; ++v)
            if ((std::fabs(cs[v]) >= std::fabs(sn[v])) == (cls == 1)) vs.push_back(v);
        for (size_t s = 0; s < vs.size(); s += G.vb) {
            G.table.push_back(cls);
            for (int q = 0; q < G.vb; ++q) G.table.push_back(s + q < vs.size() ? vs[s + q] : -1);
            ++G.ng;
        }
    }
    return G;
}

static int strip_lines(int Nc, int KP) { return std::max(1, std::min(16, 24576 / ((Nc + 2 * PPAD) * KP))); }

template <int KP, int CPT>
static cudaError_t project_k(const Geometry& g, const DeviceTables& t, const float* Xi, int Nr, int K,
                             const float* Y, int mode, float* out, int Kc, double* obj, double osc, cudaStream_t s) {
    const int R = strip_lines(g.Nc, KP);
    const size_t smem = (size_t)2 * strip_floats(R, g.Nc, KP) * sizeof(float);
    static SmemAttr attr;
    cudaError_t e = ensure_smem((const void*)k_project<KP, CPT>, (int)smem, attr);
    if (e != cudaSuccess) return e;
    dim3 grid(t.mbir_ng, Nr);
    k_project<KP, CPT><<<grid, PT, smem, s>>>(Xi, Nr, g.Nc, g.Nv, t.mbir_groups, t.mbir_vb, R, t.cos_t, t.sin_t, Y,
                                             K, mode, out, Kc, obj, osc);
    return cudaGetLastError();
}

cudaError_t mbir_project(const Geometry& g, const DeviceTables& t, const float* Xi, int Nr, int K, const float* Y,
                         int mode, float* out, int Kc, double* obj, double osc, cudaStream_t s) {
    const int KP = mbir_kp(K);
    if (mbir_cpt(g.K) == 4) {
        switch (KP) {
            case 2: return project_k<2, 4>(g, t, Xi, Nr, K, Y, mode, out, Kc, obj, osc, s);
            case 4: return project_k<4, 4>(g, t, Xi, Nr, K, Y, mode, out, Kc, obj, osc, s);
            case 6: return project_k<6, 4>(g, t, Xi, Nr, K, Y, mode, out, Kc, obj, osc, s);
            case 8: return project_k<8, 4>(g, t, Xi, Nr, K, Y, mode, out, Kc, obj, osc, s);
            default: return cudaErrorInvalidValue;
        }
    }
    switch (KP) {
        case 2: return project_k<2, 2>(g, t, Xi, Nr, K, Y, mode, out, Kc, obj, osc, s);
        case 10: return project_k<10, 2>(g, t, Xi, Nr, K, Y, mode, out, Kc, obj, osc, s);
        case 12: return project_k<12, 2>(g, t, Xi, Nr, K, Y, mode, out, Kc, obj, osc, s);
        case 14: return project_k<14, 2>(g, t, Xi, Nr, K, Y, mode, out, Kc, obj, osc, s);
        case 16: return project_k<16, 2>(g, t, Xi, Nr, K, Y, mode, out, Kc, obj, osc, s);
        default: return cudaErrorInvalidValue;
    }
}

template <int KP>
static cudaError_t to_inner_k(const float* X, int K, int64_t Nx, float* Xi, cudaStream_t s) {
    k_to_inner<KP><<<(unsigned)((Nx + 255) / 256), 256, 0, s>>>(X, K, Nx, Xi);
    return cudaGetLastError();
}

cudaError_t mbir_to_inner(const float* X, int K, int64_t Nx, float* Xi, cudaStream_t s) {
    switch (mbir_kp(K)) {
        case 2: return to_inner_k<2>(X, K, Nx, Xi, s);
        case 4: return to_inner_k<4>(X, K, Nx, Xi, s);
        case 6: return to_inner_k<6>(X, K, Nx, Xi, s);
        case 8: return to_inner_k<8>(X, K, Nx, Xi, s);
        case 10: return to_inner_k<10>(X, K, Nx, Xi, s);
        case 12: return to_inner_k<12>(X, K, Nx, Xi, s);
        case 14: return to_inner_k<14>(X, K, Nx, Xi, s);
        case 16: return to_inner_k<16>(X, K, Nx, Xi, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t mbir_ones(float* Xi1, int Nc, cudaStream_t s) {
    const int64_t n = (int64_t)Nc * Nc;
    k_ones<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(reinterpret_cast<float2*>(Xi1), n);
    return cudaGetLastError();
}

template <int KP>
static cudaError_t sqs_k(const float* Xc, const float* G, const float* G1, float* Xn, float* Xout, int K, int Nc,
                         int64_t Nx, const SqsParams& sp, double* obj, int update, unsigned* status, cudaStream_t s) {
    k_sqs<KP><<<(unsigned)((Nx + 255) / 256), 256, 0, s>>>(Xc, G, G1, Xn, Xout, K, Nc, Nx, sp, obj, update, status);
    return cudaGetLastError();
}

cudaError_t mbir_sqs(const Geometry& g, const MbirPrm& prm, const float* Xc, const float* G, const float* G1,
                     float* Xn, float* Xout, double* obj, int update, unsigned* status, cudaStream_t s) {
    const double sv = prm.sigma_v, sx = prm.sigma_x, p = prm.p, T = prm.T;
    SqsParams sp;
    const double iv = 1.0 / (sv * sv), bp = (double)g.Nv / M_PI;
    sp.gs = (float)(-iv * bp);
    sp.ds = (float)(-iv * bp);
    const double c0 = 1.0 / (std::pow(sx, p) * std::pow(T * sx, 2.0 - p));
    sp.c0 = (float)c0;
    sp.k2 = (float)((2.0 - p) / p);
    sp.e = (float)(2.0 - p);
    sp.inv_tsx = (float)(1.0 / (T * sx));
    sp.rho_s = (float)(c0 / p);
    const double b1 = 1.0 / (4.0 + 4.0 / std::sqrt(2.0));
    sp.b1 = (float)b1;
    sp.b2 = (float)(b1 / std::sqrt(2.0));
    const int64_t Nx = (int64_t)g.Nr * g.Nc * g.Nc;
    switch (mbir_kp(g.K)) {
        case 2: return sqs_k<2>(Xc, G, G1, Xn, Xout, g.K, g.Nc, Nx, sp, obj, update, status, s);
        case 4: return sqs_k<4>(Xc, G, G1, Xn, Xout, g.K, g.Nc, Nx, sp, obj, update, status, s);
        case 6: return sqs_k<6>(Xc, G, G1, Xn, Xout, g.K, g.Nc, Nx, sp, obj, update, status, s);
        case 8: return sqs_k<8>(Xc, G, G1, Xn, Xout, g.K, g.Nc, Nx, sp, obj, update, status, s);
        case 10: return sqs_k<10>(Xc, G, G1, Xn, Xout, g.K, g.Nc, Nx, sp, obj, update, status, s);
        case 12: return sqs_k<12>(Xc, G, G1, Xn, Xout, g.K, g.Nc, Nx, sp, obj, update, status, s);
        case 14: return sqs_k<14>(Xc, G, G1, Xn, Xout, g.K, g.Nc, Nx, sp, obj, update, status, s);
        case 16: return sqs_k<16>(Xc, G, G1, Xn, Xout, g.K, g.Nc, Nx, sp, obj, update, status, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace hsnct
