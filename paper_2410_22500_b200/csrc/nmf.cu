// Subspace extraction, Eq. 4, by Lee-Seung multiplicative
// updates (R1-R3: V half first, denominators floored at 1e-30) on
// Y+ = max(Y, 0) (R6).  One iteration is three kernels:
//
//   k_vstep   row pass:    A = Y+ D^T (fp32 FFMA, lanes over lambda, warp-reduced),
//                          V <- V .* A ./ max(V G, 1e-30)  (row-local, fp64 update math)
//   k_bpart   column pass: per row-chunk partials of B = V^T Y+ and H = V^T V
//   k_dupdate D update:    B, H reduced in a fixed order, D <- D .* B ./ max(H D, 1e-30),
//                          G = D D^T for the next row pass, objective terms (fp64)
//
// Everything is deterministic: static schedules, fixed-order reductions, no
// floating-point atomics (the only atomics are integer status / ticket words).
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace hsnct {
namespace {

constexpr int VT = 256;        // row-pass threads
constexpr int VW = VT / 32;    // row-pass warps
constexpr int RPW = 4;         // rows per warp step
constexpr int BT_MAX = 128;    // column-pass threads (one lambda quad each)
constexpr int BROWS = 32;      // V rows staged per column-pass sub-chunk
// default plan: the FFMA row pass everywhere -- the tcgen05 pass measured 0.53 of HBM at
// C3 / C5 against the persistent FFMA kernel's 0.72 (profiles/r02/tc/)
constexpr int64_t TC_MIN_ROWS = INT64_MAX;
// The mma.sync row pass (one launch per iteration + k_dred) against the persistent FFMA kernel,
// per iteration (scripts/tc_perf.py, profiles/r02/mma/): C1 19.6 vs 12.7 us, C2 59.2 vs 46.8 us
// (its fixed per-iteration cost dominates below ~25 tiles per SM), C3 1.83 vs 2.39 ms, C4 3.94 vs
// 5.47 ms, C5 8.35 vs 11.03 ms.  The slice-reduced C3-C5 shapes of the parity tests (61-65K rows)
// take the same kernel as the full ones.
constexpr int64_t MMA_MIN_ROWS = 60000;

// two independent fp32 FMAs in one packed instruction (fma.rn.f32x2): same rounding as FFMA
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    float2 r;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\t"
        "mov.b64 rb, {%4, %5};\n\t"
        "mov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
        "mov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}

__device__ __forceinline__ float4 ld4(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
}

// Zero the columns >= Nk of a quad starting at l0 (padding may hold anything).
__device__ __forceinline__ void mask_quad(float4& y, int l0, int Nk) {
    if (l0 + 3 >= Nk) {
        if (l0 + 0 >= Nk) y.x = 0.f;
        if (l0 + 1 >= Nk) y.y = 0.f;
        if (l0 + 2 >= Nk) y.z = 0.f;
        if (l0 + 3 >= Nk) y.w = 0.f;
    }
}

__device__ __forceinline__ bool finite4(const float4& y) {
    return isfinite(y.x) && isfinite(y.y) && isfinite(y.z) && isfinite(y.w);
}

__device__ __forceinline__ float4 clamp0(float4 y) {
    y.x = fmaxf(y.x, 0.f);
    y.y = fmaxf(y.y, 0.f);
    y.z = fmaxf(y.z, 0.f);
    y.w = fmaxf(y.w, 0.f);
    return y;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ unsigned warp_or(unsigned v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------------------ G init
// G = D0 D0^T (fp64), thread t -> output t % K^2, lambda residue class t / K^2,
// classes combined in a fixed order.  Also validates D0 (finite, >= 0).
template <int K>
__global__ void __launch_bounds__(256) k_gram_init(const float* __restrict__ D, int Nk,
                                                   double* __restrict__ Gd,
                                                   unsigned* __restrict__ status) {
    constexpr int KK = K * K;
    constexpr int NG = 256 / KK;
    __shared__ double part[NG][KK];
    unsigned bad = 0;
    for (int i = threadIdx.x; i < K * Nk; i += blockDim.x) {
        const float d = D[i];
        if (!(isfinite(d) && d >= 0.f)) bad = ST_INIT_BAD;
    }
    bad = warp_or(bad);
    if (bad && (threadIdx.x & 31) == 0) atomicOr(status, bad);
    if ((int)threadIdx.x < NG * KK) {
        const int o = threadIdx.x % KK, gg = threadIdx.x / KK;
        const int a = o / K, b = o - (o / K) * K;
        double s = 0.0;
        for (int l = gg; l < Nk; l += NG) s = fma((double)D[(int64_t)a * Nk + l], (double)D[(int64_t)b * Nk + l], s);
        part[gg][o] = s;
    }
    __syncthreads();
    if ((int)threadIdx.x < KK) {
        double s = 0.0;
        for (int gg = 0; gg < NG; ++gg) s += part[gg][threadIdx.x];
        Gd[threadIdx.x] = s;
    }
}

// ---------------------------------------------------------------- row pass
template <int K, bool FIRST>
__global__ void __launch_bounds__(VT) k_vstep(const float* __restrict__ Y, int64_t ld, int64_t Np,
                                              int Nk, int Nkp, float* __restrict__ V,
                                              const float* __restrict__ D,
                                              const double* __restrict__ Gd,
                                              double* __restrict__ vpart,
                                              unsigned* __restrict__ status,
                                              unsigned long long* __restrict__ nclamp) {
    extern __shared__ __align__(16) float Ds[];  // [K][Nkp], zero padded
    unsigned ncl = 0;
    __shared__ double Gs[K * K];
    __shared__ double red[2][VW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < K * Nkp; i += VT) {
        const int k = i / Nkp, l = i - k * Nkp;
        Ds[i] = (l < Nk) ? D[(int64_t)k * Nk + l] : 0.f;
    }
    for (int i = tid; i < K * K; i += VT) Gs[i] = Gd[i];
    __syncthreads();

    const int nq = Nkp >> 2;
    double vdotA = 0.0, ysq = 0.0;
    unsigned bad = 0;
    const int64_t nwarps = (int64_t)gridDim.x * VW;
    for (int64_t grp = (int64_t)blockIdx.x * VW + warp; grp * RPW < Np; grp += nwarps) {
        const int64_t r0 = grp * RPW;
        const float* yrow[RPW];
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) yrow[rr] = Y + min(r0 + rr, Np - 1) * ld;
        float acc[RPW][K];
        float ys[RPW];
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) {
            ys[rr] = 0.f;
#pragma unroll
            for (int k = 0; k < K; ++k) acc[rr][k] = 0.f;
        }
        for (int q = lane; q < nq; q += 32) {
            const int l0 = q * 4;
            float4 y[RPW];
#pragma unroll
            for (int rr = 0; rr < RPW; ++rr) {
                y[rr] = ld4(yrow[rr] + l0);
                mask_quad(y[rr], l0, Nk);
                if (FIRST) {
                    if (!finite4(y[rr])) bad |= ST_Y_NONFINITE;
                    if (r0 + rr < Np)
                        ncl += (y[rr].x < 0.f) + (y[rr].y < 0.f) + (y[rr].z < 0.f) + (y[rr].w < 0.f);
                }
                y[rr] = clamp0(y[rr]);
                if (FIRST) {
                    ys[rr] = fmaf(y[rr].x, y[rr].x, ys[rr]);
                    ys[rr] = fmaf(y[rr].y, y[rr].y, ys[rr]);
                    ys[rr] = fmaf(y[rr].z, y[rr].z, ys[rr]);
                    ys[rr] = fmaf(y[rr].w, y[rr].w, ys[rr]);
                }
            }
            // rows in pairs: one packed FMA per (row pair, component, bin), the same per-row
            // summation order as scalar FFMA
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const float4 d = reinterpret_cast<const float4*>(Ds + k * Nkp)[q];
#pragma unroll
                for (int rr = 0; rr < RPW; rr += 2) {
                    float2 a = make_float2(acc[rr][k], acc[rr + 1][k]);
                    a = fma2(make_float2(y[rr].x, y[rr + 1].x), make_float2(d.x, d.x), a);
                    a = fma2(make_float2(y[rr].y, y[rr + 1].y), make_float2(d.y, d.y), a);
                    a = fma2(make_float2(y[rr].z, y[rr + 1].z), make_float2(d.z, d.z), a);
                    a = fma2(make_float2(y[rr].w, y[rr + 1].w), make_float2(d.w, d.w), a);
                    acc[rr][k] = a.x;
                    acc[rr + 1][k] = a.y;
                }
            }
        }
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                float a = acc[rr][k];
#pragma unroll
                for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                acc[rr][k] = a;
            }
        }
#pragma unroll
        for (int rr = 0; rr < RPW; ++rr) {
            const int64_t r = r0 + rr;
            if (FIRST && r < Np) ysq += (double)ys[rr];
            if (lane == rr && r < Np) {
                float* vr = V + r * K;
                double v[K];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const float vk = vr[k];
                    if (FIRST && !(isfinite(vk) && vk >= 0.f)) bad |= ST_INIT_BAD;
                    v[k] = (double)vk;
                }
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    double vg = 0.0;
#pragma unroll
                    for (int j = 0; j < K; ++j) vg = fma(v[j], Gs[j * K + k], vg);
                    const double a = (double)acc[rr][k];
                    const float vn = (float)(v[k] * a / fmax(vg, 1e-30));
                    if (!isfinite(vn)) bad |= ST_NUMERIC;
                    vr[k] = vn;
                    vdotA += (double)vn * a;
                }
            }
        }
    }
    if (FIRST) {
        ncl = __reduce_add_sync(0xffffffffu, ncl);
        if (lane == 0 && ncl) atomicAdd(nclamp, (unsigned long long)ncl);
    }
    // block reduction of the fp64 partials (fixed order)
    vdotA = warp_sum(vdotA);
    ysq = warp_sum(ysq);
    bad = warp_or(bad);
    if (lane == 0) {
        red[0][warp] = vdotA;
        red[1][warp] = ysq;
        if (bad) atomicOr(status, bad);
    }
    __syncthreads();
    if (tid == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int w = 0; w < VW; ++w) {
            s0 += red[0][w];
            s1 += red[1][w];
        }
        vpart[2 * blockIdx.x + 0] = s0;
        vpart[2 * blockIdx.x + 1] = s1;
    }
}

// ------------------------------------------------------------- column pass
template <int K>
__global__ void __launch_bounds__(BT_MAX) k_bpart(const float* __restrict__ Y, int64_t ld, int64_t Np,
                                                  int Nk, int Nkp, const float* __restrict__ V,
                                                  int64_t rpc, float* __restrict__ Bpart,
                                                  double* __restrict__ Hpart) {
    __shared__ float Vs[BROWS * K];
    const int tid = threadIdx.x;
    const int q = blockIdx.y * blockDim.x + tid;
    const int nq = Nkp >> 2;
    const bool qv = q < nq;
    const int l0 = q * 4;
    const int64_t rb0 = (int64_t)blockIdx.x * rpc;
    const int64_t re = min(Np, rb0 + rpc);
    constexpr int HPT = (K * K + 31) / 32;  // H outputs per thread (blockDim >= 32)
    const bool do_h = blockIdx.y == 0;
    float2 axy[K], azw[K];  // B partial of the quad: bins (l0, l0+1) and (l0+2, l0+3), packed FMAs
#pragma unroll
    for (int k = 0; k < K; ++k) axy[k] = azw[k] = make_float2(0.f, 0.f);
    double h[HPT];
#pragma unroll
    for (int j = 0; j < HPT; ++j) h[j] = 0.0;
    for (int64_t rb = rb0; rb < re; rb += BROWS) {
        const int nr = (int)min((int64_t)BROWS, re - rb);
        __syncthreads();
        for (int i = tid; i < nr * K; i += blockDim.x) Vs[i] = V[rb * K + i];
        __syncthreads();
        if (qv) {
            const float* yp = Y + rb * ld + l0;
            int i = 0;
            for (; i + 4 <= nr; i += 4) {
                float4 y[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    y[u] = ld4(yp + (int64_t)(i + u) * ld);
                    mask_quad(y[u], l0, Nk);
                    y[u] = clamp0(y[u]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const float v = Vs[(i + u) * K + k];
                        axy[k] = fma2(make_float2(v, v), make_float2(y[u].x, y[u].y), axy[k]);
                        azw[k] = fma2(make_float2(v, v), make_float2(y[u].z, y[u].w), azw[k]);
                    }
                }
            }
            for (; i < nr; ++i) {
                float4 y = ld4(yp + (int64_t)i * ld);
                mask_quad(y, l0, Nk);
                y = clamp0(y);
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const float v = Vs[i * K + k];
                    axy[k] = fma2(make_float2(v, v), make_float2(y.x, y.y), axy[k]);
                    azw[k] = fma2(make_float2(v, v), make_float2(y.z, y.w), azw[k]);
                }
            }
        }
        if (do_h) {
#pragma unroll
            for (int j = 0; j < HPT; ++j) {
                const int t = tid + j * (int)blockDim.x;
                if (t < K * K) {
                    const int ha = t / K, hb = t - (t / K) * K;
                    double hs = 0.0;
                    for (int i = 0; i < nr; ++i) hs = fma((double)Vs[i * K + ha], (double)Vs[i * K + hb], hs);
                    h[j] += hs;
                }
            }
        }
    }
    if (qv) {
#pragma unroll
        for (int k = 0; k < K; ++k)
            reinterpret_cast<float4*>(Bpart + ((int64_t)blockIdx.x * K + k) * Nkp)[q] =
                make_float4(axy[k].x, axy[k].y, azw[k].x, azw[k].y);
    }
    if (do_h) {
#pragma unroll
        for (int j = 0; j < HPT; ++j) {
            const int t = tid + j * (int)blockDim.x;
            if (t < K * K) Hpart[(int64_t)blockIdx.x * K * K + t] = h[j];
        }
    }
}

// Fixed-order block reduction of one double per thread (result valid in thread 0).
__device__ __forceinline__ double block_sum(double v, double* sh) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
    return s;
}

// ------------------------------------------------------------- D update v2
// Two-stage fixed-order reduction of the P per-CTA partials, spread over a
// (ceil(N_k/32) x DG2) grid so that the reads of the partials are issued by
// many SMs at once:
//   block (bx, by): B partial sums for lambdas [32 bx, 32 bx + 32) over the chunks
//                   c = by*8 + w (mod 8*DG2) (warp w), and an H partial over the
//                   chunks c = by + DG2*m; written as level-2 partials.
//   last of the DG2 blocks of column bx: B, H in a fixed order, D update for its
//                   32 lambdas, <B, D_new> and (D_new D_new^T) partials.
//   last column block overall: G for the next row pass and the objective terms.
// BT: type of the B partials -- float (per-CTA partials of one GPU) or double (the sums of a
// sharded decomposition, already reduced over CTAs and ranks: P = 1)
template <int K, typename BT = float>
__global__ void __launch_bounds__(256) k_dred(const BT* __restrict__ Bpart,
                                              const double* __restrict__ Hpart, int P, int PH, int Nk, int Nkp,
                                              float* __restrict__ D, double* __restrict__ Gd,
                                              const double* __restrict__ vpart, int nblk_v,
                                              const double* __restrict__ ypart, int nby,
                                              double* __restrict__ L2B, double* __restrict__ L2H,
                                              double* __restrict__ dpart, double* __restrict__ Gpart,
                                              double* __restrict__ ysq_store, int first,
                                              double* __restrict__ obj2,
                                              unsigned* __restrict__ colcnt,
                                              unsigned* __restrict__ counter,
                                              unsigned* __restrict__ status) {
    constexpr int KK = K * K;
    constexpr int NS = (256 / KK) > 0 ? (256 / KK) : 1;
    __shared__ double bw[8][K][32];
    __shared__ double hs[NS][KK];
    __shared__ double Hs[KK];
    __shared__ double dsm[K][32];
    __shared__ double red[8];
    __shared__ double sc[4];
    __shared__ int flag;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int bx = blockIdx.x, by = blockIdx.y, nbx = gridDim.x;
    const int l = bx * 32 + lane;
    // ---- stage A: level-2 partials
    {
        double acc[K];
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = 0.0;
        if (l < Nk) {
            for (int c = by * 8 + w; c < P; c += 8 * DG2) {
#pragma unroll
                for (int k = 0; k < K; ++k) acc[k] += (double)__ldcg(Bpart + ((int64_t)c * K + k) * Nkp + l);
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) bw[w][k][lane] = acc[k];
    }
    for (int t = tid; t < KK * NS; t += 256) {
        const int o = t % KK, sub = t / KK;
        double s = 0.0;
        for (int c = by + DG2 * sub; c < PH; c += DG2 * NS) s += __ldcg(Hpart + (int64_t)c * KK + o);
        hs[sub][o] = s;
    }
    __syncthreads();
    for (int t = tid; t < K * 32; t += 256) {
        const int k = t / 32, ln = t % 32;
        double s = 0.0;
        for (int ww = 0; ww < 8; ++ww) s += bw[ww][k][ln];
        L2B[(((int64_t)bx * DG2 + by) * K + k) * 32 + ln] = s;
    }
    for (int o = tid; o < KK; o += 256) {
        double s = 0.0;
        for (int sub = 0; sub < NS; ++sub) s += hs[sub][o];
        L2H[((int64_t)bx * DG2 + by) * KK + o] = s;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) flag = (atomicAdd(colcnt + bx, 1u) == DG2 - 1);
    __syncthreads();
    if (!flag) return;
    __threadfence();
    // ---- column finalize (last of the DG2 blocks of column bx)
    for (int o = tid; o < KK; o += 256) {
        double s = 0.0;
        for (int yy = 0; yy < DG2; ++yy) s += __ldcg(L2H + ((int64_t)bx * DG2 + yy) * KK + o);
        Hs[o] = s;
    }
    __syncthreads();
    unsigned bad = 0;
    double bd = 0.0;
    if (w == 0) {
        if (l < Nk) {
            double B[K], d[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                double s = 0.0;
                for (int yy = 0; yy < DG2; ++yy) s += __ldcg(L2B + (((int64_t)bx * DG2 + yy) * K + k) * 32 + lane);
                B[k] = s;
                d[k] = (double)D[(int64_t)k * Nk + l];
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {
                double hd = 0.0;
#pragma unroll
                for (int j = 0; j < K; ++j) hd = fma(Hs[k * K + j], d[j], hd);
                const float dn = (float)(d[k] * B[k] / fmax(hd, 1e-30));
                if (!isfinite(dn)) bad |= ST_NUMERIC;
                D[(int64_t)k * Nk + l] = dn;
                dsm[k][lane] = (double)dn;
                bd += B[k] * (double)dn;
            }
        } else {
#pragma unroll
            for (int k = 0; k < K; ++k) dsm[k][lane] = 0.0;
        }
        bd = warp_sum(bd);
        bad = warp_or(bad);
        if (lane == 0) {
            dpart[bx] = bd;
            if (bad) atomicOr(status, bad);
        }
    }
    __syncthreads();
    for (int t = tid; t < KK; t += 256) {
        const int a = t / K, b = t - (t / K) * K;
        double s = 0.0;
        for (int u = 0; u < 32; ++u) s = fma(dsm[a][u], dsm[b][u], s);
        Gpart[(int64_t)bx * KK + t] = s;
    }
    if (tid == 0) colcnt[bx] = 0u;
    __threadfence();
    __syncthreads();
    if (tid == 0) flag = (atomicAdd(counter, 1u) == (unsigned)nbx - 1);
    __syncthreads();
    if (!flag) return;
    __threadfence();
    // ---- global finalize: objective terms and G for the next row pass
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    for (int i = tid; i < nblk_v; i += 256) {
        v0 += __ldcg(vpart + 2 * i);
        v1 += __ldcg(vpart + 2 * i + 1);
    }
    if (first)
        for (int i = tid; i < nby; i += 256) v1 += __ldcg(ypart + i);
    for (int i = tid; i < nbx; i += 256) v2 += __ldcg(dpart + i);
    const double va = block_sum(v0, red);
    const double ysq_new = block_sum(v1, red);
    const double bdot = block_sum(v2, red);
    if (tid == 0) {
        double ysq;
        if (first) {
            ysq = ysq_new;
            *ysq_store = ysq;
            if (!(ysq > 0.0)) atomicOr(status, (unsigned)ST_Y_ALLZERO);
        } else {
            ysq = *ysq_store;
        }
        double hg_old = 0.0;
        for (int t = 0; t < KK; ++t) hg_old += Hs[t] * Gd[t];
        sc[0] = ysq;
        sc[1] = va;
        sc[2] = bdot;
        sc[3] = hg_old;
    }
    __syncthreads();
    for (int t = tid; t < KK * NS; t += 256) {
        const int o = t % KK, sub = t / KK;
        double s = 0.0;
        for (int i = sub; i < nbx; i += NS) s += __ldcg(Gpart + (int64_t)i * KK + o);
        hs[sub][o] = s;
    }
    __syncthreads();
    for (int o = tid; o < KK; o += 256) {
        double s = 0.0;
        for (int sub = 0; sub < NS; ++sub) s += hs[sub][o];
        Gd[o] = s;
    }
    __syncthreads();
    if (tid == 0) {
        double hg_new = 0.0;
        for (int t = 0; t < KK; ++t) hg_new += Hs[t] * Gd[t];
        if (obj2) {
            obj2[0] = sc[0] - 2.0 * sc[1] + sc[3];
            obj2[1] = sc[0] - 2.0 * sc[2] + hg_new;
        }
        *counter = 0u;
    }
}

// ------------------------------------------------------ sharded decomposition (NEXT-4)
// The per-CTA partials of one row pass reduced in a fixed order into red (fp64):
//   red[k*Nk + l] = sum_c Bpart[c][k][l],  red[K*Nk + o] = sum_c Hpart[c][o],
//   red[K*Nk + KK] = sum_c vpart[2c] (<V_new, A>),
//   red[K*Nk + KK + 1] = sum_c vpart[2c+1] + sum_b ypart[b] (||Y+||^2; used on the first iteration)
// Grid: ceil(K*Nk / 256) blocks over (k, l); block 0 also reduces H and the scalars.
template <int K>
__global__ void __launch_bounds__(256) k_red_local(const float* __restrict__ Bpart, int P, int Nk, int Nkp,
                                                   const double* __restrict__ Hpart, int PH,
                                                   const double* __restrict__ vpart, int nvp,
                                                   const double* __restrict__ ypart, int nby,
                                                   double* __restrict__ red) {
    constexpr int KK = K * K;
    __shared__ double sred[8];
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i < K * Nk) {
        const int k = i / Nk, l = i - k * Nk;
        double s = 0.0;
        for (int c = 0; c < P; ++c) s += (double)__ldcg(Bpart + ((int64_t)c * K + k) * Nkp + l);
        red[i] = s;
    }
    if (blockIdx.x == 0) {
        for (int o = threadIdx.x; o < KK; o += 256) {
            double s = 0.0;
            for (int c = 0; c < PH; ++c) s += __ldcg(Hpart + (int64_t)c * KK + o);
            red[K * Nk + o] = s;
        }
        double v0 = 0.0, v1 = 0.0;
        for (int c = threadIdx.x; c < nvp; c += 256) {
            v0 += __ldcg(vpart + 2 * c);
            v1 += __ldcg(vpart + 2 * c + 1);
        }
        for (int b = threadIdx.x; b < nby; b += 256) v1 += __ldcg(ypart + b);
        const double a = block_sum(v0, sred);
        const double y = block_sum(v1, sred);
        if (threadIdx.x == 0) {
            red[K * Nk + KK] = a;
            red[K * Nk + KK + 1] = y;
        }
    }
}

// ------------------------------------------------------------ K dispatch
#define HSNCT_K_CASES(M) \
    M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15) M(16)

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }
int64_t Np_(const Geometry& g) { return (int64_t)g.Nv * g.Nr * g.Nc; }

}  // namespace

NmfPlan nmf_plan(const Geometry& g, int num_sms) {
    NmfPlan p{};
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    p.Nkp = (g.Nk + 3) & ~3;
    p.nbx = (g.Nk + 31) / 32;
    p.fused = nmf_fused_plan(g, num_sms, &p);
    {  // HSNCT_NMF=twopass: the two-pass kernels (k_vstep + k_bpart + k_dred) on any shape
        const char* nm = getenv("HSNCT_NMF");
        if (nm && strcmp(nm, "twopass") == 0) p.fused = false;
    }
    const char* np_env = getenv("HSNCT_NO_PERSIST");
    p.persist = p.fused && p.persist_fits && !(np_env && np_env[0] == '1');
    // tcgen05 row pass: HSNCT_NMF=tc / ffma forces the choice; by default the plan takes the
    // kernel that measured faster on the shape (TC_MIN_ROWS)
    {
        const char* nm = getenv("HSNCT_NMF");
        const bool force_tc = nm && strcmp(nm, "tc") == 0, force_ffma = nm && strcmp(nm, "ffma") == 0;
        const bool want = force_tc || (!force_ffma && Np >= TC_MIN_ROWS);
        NmfPlan q = p;
        if (want && nmf_tc_plan(g, num_sms, &q)) {
            p = q;
            p.tc = true;
            p.fused = false;
            p.persist = false;
            p.nby = num_sms * 8;
        }
    }
    // mma.sync row pass (nmf_mma.cu): the default from MMA_MIN_ROWS rows (K <= 8, N_k <= 1664);
    // HSNCT_NMF=mma forces it, =ffma / =twopass / =tc exclude it
    {
        const char* nm = getenv("HSNCT_NMF");
        const bool force_mma = nm && strcmp(nm, "mma") == 0;
        const bool want = force_mma || (!nm && Np >= MMA_MIN_ROWS) || (nm && nm[0] == '\0' && Np >= MMA_MIN_ROWS);
        NmfPlan q = p;
        if (want && !p.tc && (p.fused || force_mma) && nmf_mma_plan(g, num_sms, &q)) {
            p = q;
            p.mma = true;
            p.fused = false;
            // all iterations in one cooperative launch unless HSNCT_NO_PERSIST=1
            p.persist = p.persist_fits && !(np_env && np_env[0] == '1');
        }
    }
    // two-pass fallback (very long spectra, or HSNCT_NMF=twopass)
    p.smem_v = (size_t)g.K * p.Nkp * sizeof(float);
    int occ = (int)std::max<size_t>(1, std::min<size_t>(4, (200u * 1024u) / std::max<size_t>(p.smem_v + 4096, 1)));
    const int64_t groups = (Np + VW * RPW - 1) / (VW * RPW);
    p.nblk_v = (int)std::max<int64_t>(1, std::min<int64_t>(groups, (int64_t)num_sms * occ));
    const int nq = p.Nkp / 4;
    p.nlam_blk = (nq + BT_MAX - 1) / BT_MAX;
    const int per = (nq + p.nlam_blk - 1) / p.nlam_blk;
    p.bthreads = std::max(32, ((per + 31) / 32) * 32);
    // row chunks of the column pass: ~8 blocks of up to 128 threads per SM in flight (it streams
    // Y from HBM with a long dependent loop per thread; 2 per SM measured 12% warps active)
    const int64_t want = std::max<int64_t>(1, ((int64_t)num_sms * 8) / p.nlam_blk);
    p.nchunk = (int)std::max<int64_t>(1, std::min<int64_t>(want, (Np + BROWS - 1) / BROWS));
    p.rows_per_chunk = (Np + p.nchunk - 1) / p.nchunk;
    p.nchunk = (int)((Np + p.rows_per_chunk - 1) / p.rows_per_chunk);
    if (p.nchunk < 1) p.nchunk = 1;
    p.P = p.tc ? p.tc_ncl : p.mma ? p.nblk_f : p.fused ? p.PB : p.nchunk;
    p.PH = p.tc ? TC_CLUSTER * p.tc_ncl : p.mma ? p.nblk_f : p.fused ? p.PB : p.nchunk;
    p.nvp = p.tc ? TC_CLUSTER * p.tc_ncl : p.mma ? p.nblk_f : p.fused ? p.PB : p.nblk_v;
    return p;
}

size_t nmf_ws_bytes(const Geometry& g, const NmfPlan& p) {
    const size_t KK = (size_t)g.K * g.K;
    size_t b = 0;
    b += align256(KK * sizeof(double));                               // Gd
    b += align256((size_t)p.nvp * 2 * sizeof(double));                // vpart
    b += align256((size_t)std::max(p.nbx, p.nblk_f) * sizeof(double));        // dpart
    b += align256((size_t)std::max(p.nbx, p.nblk_f) * KK * sizeof(double));   // Gpart
    b += align256(sizeof(double));                                    // ysq
    b += align256((size_t)p.PH * KK * sizeof(double));                // Hpart
    const size_t bstride = p.Nkp;
    b += align256((size_t)p.P * g.K * bstride * sizeof(float));       // Bpart
    b += align256((size_t)p.nbx * DG2 * g.K * 32 * sizeof(double));   // L2B
    b += align256((size_t)p.nbx * DG2 * KK * sizeof(double));         // L2H
    if (p.fused) {
        b += align256((size_t)Np_(g) * bstride * sizeof(float));      // Yp (fp32)
        b += align256((size_t)p.nby * sizeof(double));                // ypart
    }
    if (p.tc) {
        b += align256((size_t)p.tc_Npad * p.tc_Nk16 * 4);             // Yc: fp16 hi + lo per element
        b += align256((size_t)p.nby * sizeof(double));                // ypart
        b += align256(2 * sizeof(unsigned));                          // ymax, max row norm
    }
    if (p.mma) {
        b += align256((size_t)p.mma_Npad * p.mma_NB * 16 * 4);        // Yc: fp16 hi + lo per element
        b += align256((size_t)p.nby * sizeof(double));                // ypart
        b += align256((size_t)(p.mma_Npad / 16) * sizeof(int));      // texp: per-tile scale exponents
    }
    return b;
}

NmfWs nmf_ws_carve(const Geometry& g, const NmfPlan& p, void* ws) {
    const size_t KK = (size_t)g.K * g.K;
    char* c = static_cast<char*>(ws);
    NmfWs w{};
    auto take = [&](size_t bytes) {
        char* r = c;
        c += align256(bytes);
        return r;
    };
    w.Gd = (double*)take(KK * sizeof(double));
    w.vpart = (double*)take((size_t)p.nvp * 2 * sizeof(double));
    w.dpart = (double*)take((size_t)std::max(p.nbx, p.nblk_f) * sizeof(double));
    w.Gpart = (double*)take((size_t)std::max(p.nbx, p.nblk_f) * KK * sizeof(double));
    w.ysq = (double*)take(sizeof(double));
    w.Hpart = (double*)take((size_t)p.PH * KK * sizeof(double));
    const size_t bstride = p.Nkp;
    w.Bpart = (float*)take((size_t)p.P * g.K * bstride * sizeof(float));
    w.L2B = (double*)take((size_t)p.nbx * DG2 * g.K * 32 * sizeof(double));
    w.L2H = (double*)take((size_t)p.nbx * DG2 * KK * sizeof(double));
    if (p.fused) {
        w.Yp = (float*)take((size_t)Np_(g) * bstride * sizeof(float));
        w.ypart = (double*)take((size_t)p.nby * sizeof(double));
    }
    if (p.tc) {
        w.Yc = take((size_t)p.tc_Npad * p.tc_Nk16 * 4);
        w.ypart = (double*)take((size_t)p.nby * sizeof(double));
        w.ymax = (unsigned*)take(2 * sizeof(unsigned));
    }
    if (p.mma) {
        w.Yc = take((size_t)p.mma_Npad * p.mma_NB * 16 * 4);
        w.ypart = (double*)take((size_t)p.nby * sizeof(double));
        w.texp = (int*)take((size_t)(p.mma_Npad / 16) * sizeof(int));
    }
    return w;
}

int nmf_init_launches(const NmfPlan& p) { return p.tc ? 3 : (p.fused || p.mma) ? 2 : 1; }

cudaError_t nmf_launch_init(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y, int64_t ld_y,
                            const float* D, unsigned* status, cudaStream_t s, const DeviceTables* t,
                            const CountsIn* cin) {
    if (cin && !p.fused && !p.mma) return cudaErrorInvalidValue;  // the caller decodes into a Y buffer instead
    if (p.mma && cin) {
        cudaError_t e = nmf_mma_prepare_counts(g, p, w, *t, *cin, status, s);
        if (e != cudaSuccess) return e;
    } else if (p.tc) {
        cudaError_t e = nmf_tc_prepare(g, p, w, Y, ld_y, status, s);
        if (e != cudaSuccess) return e;
    } else if (p.mma) {
        cudaError_t e = nmf_mma_prepare(g, p, w, Y, ld_y, status, s);
        if (e != cudaSuccess) return e;
    } else if (p.fused && cin) {  // Y+ decoded from the counts (NEXT-1), same partials as k_yplus
        cudaError_t e = counts_decode(g, *t, *cin, w.Yp, p.Nkp, 1, p.nby, w.ypart, w.nclamp, s);
        if (e != cudaSuccess) return e;
    } else if (p.fused) {
        cudaError_t e = nmf_yplus_launch(g, p, w, Y, ld_y, status, s);
        if (e != cudaSuccess) return e;
    }
    switch (g.K) {
#define M(KV)                                                               \
    case KV:                                                                \
        k_gram_init<KV><<<1, 256, 0, s>>>(D, g.Nk, w.Gd, status);           \
        break;
        HSNCT_K_CASES(M)
#undef M
        default:
            return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <int K>
static cudaError_t iter_k(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y,
                          int64_t ld, float* V, float* D, int it, double* obj2,
                          unsigned* status, unsigned* counter, cudaStream_t s) {
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    const bool first = it == 0;
    if (p.tc) {
        cudaError_t e = nmf_tc_launch(g, p, w, V, D, it, status, s);
        if (e != cudaSuccess) return e;
    } else if (p.mma) {
        cudaError_t e = nmf_mma_launch(g, p, w, V, D, it, status, s);
        if (e != cudaSuccess) return e;
    } else if (p.fused) {
        cudaError_t e = nmf_fused_launch(g, p, w, V, D, it, status, s);
        if (e != cudaSuccess) return e;
    } else {
        static SmemAttr attr_f, attr_n;  // per K instantiation, per device
        cudaError_t e = first ? ensure_smem((const void*)k_vstep<K, true>, (int)p.smem_v, attr_f)
                              : ensure_smem((const void*)k_vstep<K, false>, (int)p.smem_v, attr_n);
        if (e != cudaSuccess) return e;
        if (first)
            k_vstep<K, true><<<p.nblk_v, VT, p.smem_v, s>>>(Y, ld, Np, g.Nk, p.Nkp, V, D, w.Gd, w.vpart, status,
                                                            w.nclamp);
        else
            k_vstep<K, false><<<p.nblk_v, VT, p.smem_v, s>>>(Y, ld, Np, g.Nk, p.Nkp, V, D, w.Gd, w.vpart, status,
                                                             w.nclamp);
        dim3 gb(p.nchunk, p.nlam_blk);
        k_bpart<K><<<gb, p.bthreads, 0, s>>>(Y, ld, Np, g.Nk, p.Nkp, V, p.rows_per_chunk, w.Bpart, w.Hpart);
    }
    dim3 gd(p.nbx, DG2);
    k_dred<K><<<gd, 256, 0, s>>>(w.Bpart, w.Hpart, p.P, p.PH, g.Nk, p.Nkp, D, w.Gd, w.vpart, p.nvp,
                                 w.ypart, (p.fused || p.tc || p.mma) ? p.nby : 0, w.L2B,
                                 w.L2H, w.dpart, w.Gpart, w.ysq, first ? 1 : 0, obj2, counter + 1,
                                 counter, status);
    return cudaGetLastError();
}

int nmf_launches_per_iter(const NmfPlan& p) { return (p.fused || p.tc || p.mma) ? 2 : 3; }

// ------------------------------------------------------ sharded decomposition (NEXT-4)
size_t nmf_red_size(const Geometry& g) { return (size_t)g.K * g.Nk + (size_t)g.K * g.K + 2; }

template <int K>
static cudaError_t shard_rowpass_k(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y, int64_t ld,
                                   float* V, const float* D, int it, double* red, unsigned* status, cudaStream_t s) {
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    const bool first = it == 0;
    if (p.tc) {
        cudaError_t e = nmf_tc_launch(g, p, w, V, D, it, status, s);
        if (e != cudaSuccess) return e;
    } else if (p.mma) {
        cudaError_t e = nmf_mma_launch(g, p, w, V, D, it, status, s);
        if (e != cudaSuccess) return e;
    } else if (p.fused) {
        cudaError_t e = nmf_fused_launch(g, p, w, V, D, it, status, s);
        if (e != cudaSuccess) return e;
    } else {
        static SmemAttr attr_f, attr_n;
        cudaError_t e = first ? ensure_smem((const void*)k_vstep<K, true>, (int)p.smem_v, attr_f)
                              : ensure_smem((const void*)k_vstep<K, false>, (int)p.smem_v, attr_n);
        if (e != cudaSuccess) return e;
        if (first)
            k_vstep<K, true><<<p.nblk_v, VT, p.smem_v, s>>>(Y, ld, Np, g.Nk, p.Nkp, V, D, w.Gd, w.vpart, status,
                                                            w.nclamp);
        else
            k_vstep<K, false><<<p.nblk_v, VT, p.smem_v, s>>>(Y, ld, Np, g.Nk, p.Nkp, V, D, w.Gd, w.vpart, status,
                                                             w.nclamp);
        dim3 gb(p.nchunk, p.nlam_blk);
        k_bpart<K><<<gb, p.bthreads, 0, s>>>(Y, ld, Np, g.Nk, p.Nkp, V, p.rows_per_chunk, w.Bpart, w.Hpart);
    }
    const bool yp = p.fused || p.tc || p.mma;
    k_red_local<K><<<(K * g.Nk + 255) / 256, 256, 0, s>>>(w.Bpart, p.P, g.Nk, p.Nkp, w.Hpart, p.PH, w.vpart, p.nvp,
                                                          yp ? w.ypart : nullptr, yp ? p.nby : 0, red);
    return cudaGetLastError();
}

template <int K>
static cudaError_t shard_dupdate_k(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* D, const double* red,
                                   int it, double* obj2, unsigned* status, unsigned* counter, cudaStream_t s) {
    constexpr int KK = K * K;
    dim3 gd(p.nbx, DG2);
    // the global sums as one "partial": B [K][N_k] (stride N_k), H, {<V, A>, ||Y+||^2}
    k_dred<K, double><<<gd, 256, 0, s>>>(red, red + (size_t)K * g.Nk, 1, 1, g.Nk, g.Nk, D, w.Gd,
                                         red + (size_t)K * g.Nk + KK, 1, nullptr, 0, w.L2B, w.L2H, w.dpart,
                                         w.Gpart, w.ysq, it == 0 ? 1 : 0, obj2, counter + 1, counter, status);
    return cudaGetLastError();
}

cudaError_t nmf_shard_rowpass(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y, int64_t ld_y,
                              float* V, const float* D, int it, double* red, unsigned* status, cudaStream_t s) {
    switch (g.K) {
#define M(KV) \
    case KV:  \
        return shard_rowpass_k<KV>(g, p, w, Y, ld_y, V, D, it, red, status, s);
        HSNCT_K_CASES(M)
#undef M
        default:
            return cudaErrorInvalidValue;
    }
}

cudaError_t nmf_shard_dupdate(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* D, const double* red,
                              int it, double* obj2, unsigned* status, unsigned* counter, cudaStream_t s) {
    switch (g.K) {
#define M(KV) \
    case KV:  \
        return shard_dupdate_k<KV>(g, p, w, D, red, it, obj2, status, counter, s);
        HSNCT_K_CASES(M)
#undef M
        default:
            return cudaErrorInvalidValue;
    }
}

std::string nmf_plan_desc(const Geometry& g, const NmfPlan& p) {
    char b[256];
    if (p.tc)
        snprintf(b, sizeof b, "tc k_nmf_tc<K=%d> cluster=%d grid=%d ring=%d+%dx%d-bin bins/CTA=%d..%d +k_dred", g.K,
                 TC_CLUSTER, TC_CLUSTER * p.tc_ncl, p.tc_R, p.tc_R2, p.tc_rg.W, p.tc_rg.L[TC_CLUSTER - 1],
                 p.tc_rg.L[0]);
    else if (p.mma)
        snprintf(b, sizeof b, "mma k_nmf_mma<K=%d,NBW=%d,PERSIST=%d%s> grid=%d 16-row tiles, %d blocks/row%s", g.K,
                 p.mma_NBW, p.persist ? 1 : 0, p.mma_MW == 16 ? ",MW=16" : "", p.nblk_f, p.mma_NB,
                 p.persist ? "" : " +k_dred");
    else if (p.persist)
        snprintf(b, sizeof b, "persist k_nmf_persist<K=%d,LP=%d,NBG=%d,NGRP=%d> grid=%d", g.K, p.LP, p.nbuf,
                 p.ngrp, p.nblk_f);
    else if (p.fused)
        snprintf(b, sizeof b, "fused k_nmf_fused<K=%d,LP=%d,NBG=%d,NGRP=%d>+k_dred grid=%d", g.K, p.LP, p.nbuf,
                 p.ngrp, p.nblk_f);
    else
        snprintf(b, sizeof b, "twopass k_vstep<K=%d>+k_bpart+k_dred grid=%d", g.K, p.nblk_v);
    return b;
}

cudaError_t nmf_launch_iter(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y,
                            int64_t ld_y, float* V, float* D, int it, double* obj2,
                            unsigned* status, unsigned* counter, cudaStream_t s) {
    switch (g.K) {
#define M(KV) \
    case KV:  \
        return iter_k<KV>(g, p, w, Y, ld_y, V, D, it, obj2, status, counter, s);
        HSNCT_K_CASES(M)
#undef M
        default:
            return cudaErrorInvalidValue;
    }
}

}  // namespace hsnct
