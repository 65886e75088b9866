// Fused single-pass Lee-Seung iteration: one read of Y+ per iteration.
//
// Input is Y+ = max(Y, 0) materialised once per decompose call by k_yplus
// (compact rows of Nkp floats, zero padding), so the hot loop carries no clamp,
// mask or branch.  One persistent CTA per SM streams 8-row tiles through a ring
// of NBUF shared-memory buffers filled by cp.async.bulk (one bulk copy per tile,
// completion on an mbarrier).  The CTA is warp-specialised:
//
//   compute warps  2 groups x 4 warps.  Group g owns rows 4g..4g+3 of every tile;
//                  thread t of a group owns the lambda pairs 2(t + 128 i), i < LP, for
//                  the whole kernel, with the matching columns of the CTA's partial
//                  B = V^T Y+ in registers.
//                    phase 1 (tile j):   part[r][k] = sum_l Y+[r][l] D[k][l] (D from smem)
//                                        -> warp transpose-reduce -> red[], arrive part
//                    phase 2 (tile j-1): B[k][l] += V_new[r][k] Y+[r][l]     -> arrive empty
//   reducer warp   per tile: fixed-order sum of the 4 warp partials of each row,
//                  V[r][k] <- V[r][k] A[r][k] / max(sum_j V[r][j] G[j][k], 1e-30),
//                  H += V_new^T V_new, <V_new, A>; arrive vn; then refills the ring.
//
// The V update of tile j overlaps phase 2 of tile j-1, so the compute warps never
// wait on it.  Per-CTA partials (B per group, H, <V_new, A>) are reduced in a fixed
// order by k_dred.  Deterministic: static schedule, fixed reduction trees.
#pragma once
#include <algorithm>

#include "internal.h"

namespace hsnct {
namespace {

constexpr int RG = 4;              // rows per tile (= rows per compute-group step)
constexpr int NG = 2;              // compute groups (alternate tiles)
constexpr int GW = 4;              // warps per group
constexpr int CW = NG * GW;        // compute warps
constexpr int TG = GW * 32;        // threads per group
constexpr int NTHREADS = (CW + NG) * 32;   // + one reducer/producer warp per group

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// Orders this thread's prior generic-proxy shared-memory accesses (ring reads)
// before its subsequent bulk copies into the same buffers.
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Generic -> async proxy ordering for global memory (V rows written by the
// previous iteration are read by this iteration's bulk copies).
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Fixed-order block reduction of one double per thread (result valid in thread 0).
__device__ __forceinline__ double block_sum_d(double v, double* sh) {
    v = warp_sum_d(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += sh[w];
    __syncthreads();
    return s;
}

// Warp transpose-reduce of N values per lane.  On return the lane holds
// tr_nout(N) values; value j is the warp sum of original index tr_base(lane) + j.
// Halving steps (while the count is even) exchange half of the values; the rest
// are plain butterflies, after which lanes that differ only in those butterfly
// bits hold identical values (the lane with zero bits there writes them).
__host__ __device__ constexpr int tr_nout(int n, int o = 16) {
    return o == 0 ? n : (n % 2 == 0 ? tr_nout(n / 2, o / 2) : tr_nout(n, o / 2));
}
__host__ __device__ constexpr unsigned tr_bfly(int n, int o = 16) {
    return o == 0 ? 0u : (n % 2 == 0 ? tr_bfly(n / 2, o / 2) : ((unsigned)o | tr_bfly(n, o / 2)));
}
template <int O, int n>
__device__ __forceinline__ void tr_step(float* v, int lane) {
    if constexpr (O == 0) {
        return;
    } else if constexpr (n % 2 == 0) {
        const bool up = (lane & O) != 0;
#pragma unroll
        for (int j = 0; j < n / 2; ++j) {
            const float send = up ? v[j] : v[j + n / 2];
            const float keep = up ? v[j + n / 2] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, O);
        }
        tr_step<O / 2, n / 2>(v, lane);
    } else {
#pragma unroll
        for (int j = 0; j < n; ++j) v[j] += __shfl_xor_sync(0xffffffffu, v[j], O);
        tr_step<O / 2, n>(v, lane);
    }
}
template <int N>
__device__ __forceinline__ int tr_base(int lane) {
    int b = 0, n = N;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        if (n % 2 == 0) {
            if (lane & o) b += n / 2;
            n /= 2;
        }
    }
    return b;
}

// Y+ = max(Y, 0) into compact rows of Nkp floats (padding = 0); flags non-finite
// Y (the clamp would hide NaN); per-block ||Y+||^2 partials (fp64).
__global__ void __launch_bounds__(256) k_yplus(const float* __restrict__ Y, int64_t ld, int64_t Np, int Nk,
                                               int Nkp, float* __restrict__ Yp, double* __restrict__ ypart,
                                               unsigned* __restrict__ status) {
    __shared__ double red[8];
    const int nq = Nkp >> 2;
    const int64_t total = Np * nq;
    double s = 0.0;
    unsigned bad = 0;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = idx / nq;
        const int q = (int)(idx - p * nq);
        const int l0 = 4 * q;
        float4 y = __ldcs(reinterpret_cast<const float4*>(Y + p * ld + l0));
        if (l0 + 3 >= Nk) {
            if (l0 + 0 >= Nk) y.x = 0.f;
            if (l0 + 1 >= Nk) y.y = 0.f;
            if (l0 + 2 >= Nk) y.z = 0.f;
            if (l0 + 3 >= Nk) y.w = 0.f;
        }
        if (!(isfinite(y.x) && isfinite(y.y) && isfinite(y.z) && isfinite(y.w))) bad = ST_Y_NONFINITE;
        y.x = fmaxf(y.x, 0.f);
        y.y = fmaxf(y.y, 0.f);
        y.z = fmaxf(y.z, 0.f);
        y.w = fmaxf(y.w, 0.f);
        s += (double)(y.x * y.x + y.y * y.y) + (double)(y.z * y.z + y.w * y.w);
        reinterpret_cast<float4*>(Yp + p * Nkp)[q] = y;
    }
    s = warp_sum_d(s);
#pragma unroll
    for (int o = 16; o; o >>= 1) bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        red[w] = s;
        if (bad) atomicOr(status, bad);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
        ypart[blockIdx.x] = t;
    }
}

template <int K, int LP, int NBUF>
struct FusedShared {
    static constexpr int GK = RG * K;
    static constexpr int KP = (K + 3) & ~3;
    static constexpr int KK = K * K;
    uint64_t full[NBUF], empty[NBUF], partb[NG], vnb[NG];
    float red[NG][GW][GK];
    __align__(16) float Vn[NG][RG][KP];
    float Gs[KK];
    double hs[NG][KK];
    double vs[NG];
    unsigned bad;
};

// One pass over this CTA's tiles (tile j = blockIdx.x + j*gridDim.x, RG rows each)
// with the current D (smem Ds) and G (sh.Gs).  Tiles alternate between the two
// compute groups; a group runs phase 1, waits for its reducer warp's V update of
// that tile, runs phase 2 and releases the buffer while the other group computes.
// On return (all threads), the CTA's partials are written: B (groups combined in a
// fixed order) to Bout[K][Nkp], H to Hout[K*K], <V_new, A> to *vout.
template <int K, int LP, int NBUF>
__device__ __forceinline__ void tile_pass(const float* __restrict__ Yp, int64_t Np, int Nkp,
                                          float* __restrict__ V, float* ring, const float* Ds,
                                          FusedShared<K, LP, NBUF>& sh, float* __restrict__ Bout,
                                          double* __restrict__ Hout, double* __restrict__ vout,
                                          bool first) {
    constexpr int GK = RG * K;
    constexpr int KP = (K + 3) & ~3;
    constexpr int DS = 2 * TG * LP;
    constexpr int KK = K * K;
    // keep the tile in registers between the phases when it fits the 168-register budget
    constexpr bool YREG = (2 * RG * LP + 2 * K * LP + RG * K) <= 120;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntiles = (Np + RG - 1) / RG;
    const int64_t nmine = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const size_t tile_floats = (size_t)RG * Nkp + RG * K;  // Y+ rows, then the old V rows

    if (tid == 0) {
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&sh.full[b], 1);
            mbar_init(&sh.empty[b], TG);
        }
        for (int g = 0; g < NG; ++g) {
            mbar_init(&sh.partb[g], TG);
            mbar_init(&sh.vnb[g], 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    float2 bacc[K][LP];
    if (warp < CW) {
        // ======================= compute warps =======================
        const int g = warp / GW;
        const int wg = warp - g * GW;
        const int t = tid - g * TG;
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int i = 0; i < LP; ++i) bacc[k][i] = make_float2(0.f, 0.f);
        const float* dbase = Ds + 2 * t;
        int64_t kth = 0;  // this group's tile count
        for (int64_t j = g; j < nmine; j += NG, ++kth) {
            const int b = (int)(j % NBUF);
            mbar_wait(&sh.full[b], (unsigned)((j / NBUF) & 1));
            const float* yb = ring + (size_t)b * tile_floats + 2 * t;
            // YREG: the tile's Y+ values owned by this thread go to registers and the
            // buffer is released at once (deeper prefetch, phase 2 without smem reads);
            // otherwise phase 2 re-reads the buffer and releases it afterwards.
            float2 y[YREG ? LP : 1][RG];
            if constexpr (YREG) {
#pragma unroll
                for (int i = 0; i < LP; ++i)
#pragma unroll
                    for (int r = 0; r < RG; ++r)
                        y[i][r] = *reinterpret_cast<const float2*>(yb + (size_t)r * Nkp + 2 * TG * i);
                mbar_arrive(&sh.empty[b]);
            }
            // ---- phase 1
            float part[GK];
#pragma unroll
            for (int x = 0; x < GK; ++x) part[x] = 0.f;
#pragma unroll
            for (int i = 0; i < LP; ++i) {
                float2 yy[RG];
#pragma unroll
                for (int r = 0; r < RG; ++r)
                    yy[r] = YREG ? y[YREG ? i : 0][r]
                                 : *reinterpret_cast<const float2*>(yb + (size_t)r * Nkp + 2 * TG * i);
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const float2 d = *reinterpret_cast<const float2*>(dbase + k * DS + 2 * TG * i);
#pragma unroll
                    for (int r = 0; r < RG; ++r)
                        part[r * K + k] = fmaf(yy[r].x, d.x, fmaf(yy[r].y, d.y, part[r * K + k]));
                }
            }
            tr_step<16, GK>(part, lane);
            if (((unsigned)lane & tr_bfly(GK)) == 0) {
                const int base = tr_base<GK>(lane);
#pragma unroll
                for (int x = 0; x < tr_nout(GK); ++x) sh.red[g][wg][base + x] = part[x];
            }
            mbar_arrive(&sh.partb[g]);
            // ---- phase 2 (after the reducer's V update of this tile)
            mbar_wait(&sh.vnb[g], (unsigned)(kth & 1));
#pragma unroll
            for (int r = 0; r < RG; ++r) {
                float vr[KP];
#pragma unroll
                for (int q = 0; q < KP / 4; ++q) {
                    const float4 v4 = reinterpret_cast<const float4*>(&sh.Vn[g][r][0])[q];
                    vr[4 * q + 0] = v4.x;
                    vr[4 * q + 1] = v4.y;
                    vr[4 * q + 2] = v4.z;
                    vr[4 * q + 3] = v4.w;
                }
#pragma unroll
                for (int i = 0; i < LP; ++i) {
                    const float2 yv = YREG ? y[YREG ? i : 0][r]
                                           : *reinterpret_cast<const float2*>(yb + (size_t)r * Nkp + 2 * TG * i);
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        bacc[k][i].x = fmaf(vr[k], yv.x, bacc[k][i].x);
                        bacc[k][i].y = fmaf(vr[k], yv.y, bacc[k][i].y);
                    }
                }
            }
            if constexpr (!YREG) mbar_arrive(&sh.empty[b]);
        }
    } else {
        // =============== reducer / producer warp of group g (tiles j = g mod NG) ===============
        const int g = warp - CW;
        auto issue = [&](int64_t jj) {
            const int b = (int)(jj % NBUF);
            const int64_t r0 = (blockIdx.x + jj * gridDim.x) * RG;
            const int nv = (int)min((int64_t)RG, Np - r0);
            const unsigned bytes = (unsigned)(nv * Nkp * sizeof(float));
            const unsigned vbytes = nv == RG ? (unsigned)(RG * K * sizeof(float)) : 0u;  // 16K bytes
            mbar_expect_tx(&sh.full[b], bytes + vbytes);
            float* slot = ring + (size_t)b * tile_floats;
            bulk_g2s(slot, Yp + r0 * Nkp, bytes, &sh.full[b]);
            if (vbytes) bulk_g2s(slot + (size_t)RG * Nkp, V + r0 * K, vbytes, &sh.full[b]);
        };
        if (lane == 0) {
            fence_proxy_async_global();
            fence_proxy_async();
            for (int64_t jj = g; jj < min((int64_t)NBUF, nmine); jj += NG) issue(jj);
        }
        double vdotA = 0.0;
        double hacc[(KK + 31) / 32];
#pragma unroll
        for (int x = 0; x < (KK + 31) / 32; ++x) hacc[x] = 0.0;
        unsigned bad = 0;
        int64_t kth = 0;
        for (int64_t j = g; j < nmine; j += NG, ++kth) {
            const int64_t r0 = (blockIdx.x + j * gridDim.x) * RG;
            const int nv = (int)min((int64_t)RG, Np - r0);
            const int b = (int)(j % NBUF);
            mbar_wait(&sh.full[b], (unsigned)((j / NBUF) & 1));
            const float* vslot = ring + (size_t)b * tile_floats + (size_t)RG * Nkp;
            float vo_all[(GK + 31) / 32][K];
            float vo_me[(GK + 31) / 32];
#pragma unroll
            for (int u = 0; u < (GK + 31) / 32; ++u) {
                const int s = lane + 32 * u;
                const int r = (s < GK ? s : 0) / K;
#pragma unroll
                for (int jj = 0; jj < K; ++jj)
                    vo_all[u][jj] = nv == RG ? vslot[r * K + jj] : ((r < nv) ? V[(r0 + r) * K + jj] : 0.f);
                vo_me[u] = vo_all[u][s < GK ? s - r * K : 0];
            }
            mbar_wait(&sh.partb[g], (unsigned)(kth & 1));
            float vnew[(GK + 31) / 32], aval[(GK + 31) / 32];
#pragma unroll
            for (int u = 0; u < (GK + 31) / 32; ++u) {
                const int s = lane + 32 * u;
                vnew[u] = 0.f;
                aval[u] = 0.f;
                if (s < GK) {
                    const int r = s / K, k = s - (s / K) * K;
                    float a = 0.f;
#pragma unroll
                    for (int w = 0; w < GW; ++w) a += sh.red[g][w][s];
                    float vg = 0.f;
#pragma unroll
                    for (int jj = 0; jj < K; ++jj) vg = fmaf(vo_all[u][jj], sh.Gs[jj * K + k], vg);
                    float vn = __fdiv_rn(vo_me[u] * a, fmaxf(vg, 1e-30f));
                    if (r >= nv) vn = 0.f;
                    vnew[u] = vn;
                    aval[u] = a;
                    sh.Vn[g][r][k] = vn;
                }
            }
            __syncwarp();
            mbar_arrive(&sh.vnb[g]);
            // off the compute warps' critical path: V store, checks, objective, H, refill
#pragma unroll
            for (int u = 0; u < (GK + 31) / 32; ++u) {
                const int s = lane + 32 * u;
                if (s < GK && s / K < nv) {
                    if (first && !(isfinite(vo_me[u]) && vo_me[u] >= 0.f)) bad |= ST_INIT_BAD;
                    if (!isfinite(vnew[u])) bad |= ST_NUMERIC;
                    V[r0 * K + s] = vnew[u];
                    vdotA += (double)vnew[u] * (double)aval[u];
                }
            }
#pragma unroll
            for (int x = 0; x < (KK + 31) / 32; ++x) {
                const int tt = lane + 32 * x;
                if (tt < KK) {
                    const int a = tt / K, c = tt - (tt / K) * K;
                    double s = 0.0;
#pragma unroll
                    for (int r = 0; r < RG; ++r) s = fma((double)sh.Vn[g][r][a], (double)sh.Vn[g][r][c], s);
                    hacc[x] += s;
                }
            }
            // refill.  YREG: the group released tile j's buffer before arriving on
            // part(j).  Otherwise: its previous tile j - NG was released before part(j).
            const int64_t m = YREG ? j : j - NG;
            if (m >= 0 && m + NBUF < nmine) {
                mbar_wait(&sh.empty[m % NBUF], (unsigned)((m / NBUF) & 1));
                if (lane == 0) {
                    fence_proxy_async();
                    issue(m + NBUF);
                }
            }
        }
        vdotA = warp_sum_d(vdotA);
#pragma unroll
        for (int o = 16; o; o >>= 1) bad |= __shfl_xor_sync(0xffffffffu, bad, o);
        if (lane == 0) {
            sh.vs[g] = vdotA;
            if (bad) atomicOr(&sh.bad, bad);
        }
#pragma unroll
        for (int x = 0; x < (KK + 31) / 32; ++x) {
            const int tt = lane + 32 * x;
            if (tt < KK) sh.hs[g][tt] = hacc[x];
        }
    }
    // ---- CTA partials: group 1's B through smem (the ring is idle now), fixed order 0 + 1
    __syncthreads();
    float* scratch = ring;  // [K][DS]
    if (warp >= GW && warp < CW) {
        const int t = tid - TG;
#pragma unroll
        for (int i = 0; i < LP; ++i)
#pragma unroll
            for (int k = 0; k < K; ++k)
                *reinterpret_cast<float2*>(scratch + k * DS + 2 * (t + TG * i)) = bacc[k][i];
    }
    __syncthreads();
    if (warp < GW) {
        const int t = tid;
#pragma unroll
        for (int i = 0; i < LP; ++i) {
            const int l0 = 2 * (t + TG * i);
            if (l0 < Nkp) {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const float2 o = *reinterpret_cast<const float2*>(scratch + k * DS + l0);
                    *reinterpret_cast<float2*>(Bout + (int64_t)k * Nkp + l0) =
                        make_float2(bacc[k][i].x + o.x, bacc[k][i].y + o.y);
                }
            }
        }
    }
    for (int o = tid; o < KK; o += NTHREADS) Hout[o] = sh.hs[0][o] + sh.hs[1][o];
    if (tid == 0) *vout = sh.vs[0] + sh.vs[1];
    __syncthreads();  // scratch (ring) reads done before any reuse
}

// Stage D (zero padded to DS columns) and G into shared memory.
template <int K, int LP, int NBUF>
__device__ __forceinline__ void stage_dg(const float* __restrict__ D, int Nk, const double* Gsrc, float* Ds,
                                         FusedShared<K, LP, NBUF>& sh) {
    constexpr int DS = 2 * TG * LP;
    for (int i = threadIdx.x; i < K * DS; i += NTHREADS) {
        const int k = i / DS, l = i - k * DS;
        Ds[i] = (l < Nk) ? __ldcg(D + (int64_t)k * Nk + l) : 0.f;
    }
    for (int i = threadIdx.x; i < K * K; i += NTHREADS) sh.Gs[i] = (float)Gsrc[i];
}

template <int K, int LP, int NBUF>
__global__ void __launch_bounds__(NTHREADS, 1) k_nmf_fused(const float* __restrict__ Yp, int64_t Np, int Nk,
                                                           int Nkp, float* __restrict__ V,
                                                           const float* __restrict__ D,
                                                           const double* __restrict__ Gd,
                                                           float* __restrict__ Bpart,
                                                           double* __restrict__ Hpart,
                                                           double* __restrict__ vpart, int first,
                                                           unsigned* __restrict__ status) {
    constexpr int DS = 2 * TG * LP;
    __shared__ FusedShared<K, LP, NBUF> sh;
    extern __shared__ __align__(128) float smem[];
    const size_t tile_floats = (size_t)RG * Nkp + RG * K;
    float* ring = smem;                              // [NBUF][tile] + slack DS
    float* Ds = smem + NBUF * tile_floats + DS;      // [K][DS]
    for (size_t i = threadIdx.x; i < NBUF * tile_floats + DS; i += NTHREADS) ring[i] = 0.f;
    if (threadIdx.x == 0) sh.bad = 0u;
    stage_dg<K, LP, NBUF>(D, Nk, Gd, Ds, sh);
    __syncthreads();
    tile_pass<K, LP, NBUF>(Yp, Np, Nkp, V, ring, Ds, sh, Bpart + (int64_t)blockIdx.x * K * Nkp,
                           Hpart + (int64_t)blockIdx.x * K * K, vpart + 2 * (int64_t)blockIdx.x, first != 0);
    if (threadIdx.x == 0) {
        vpart[2 * (int64_t)blockIdx.x + 1] = 0.0;
        if (sh.bad) atomicOr(status, sh.bad);
    }
}

// Software grid barrier for a cooperative launch (all CTAs co-resident).
__device__ __forceinline__ void grid_sync(unsigned* count, unsigned* gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = *(volatile unsigned*)gen;
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            *(volatile unsigned*)count = 0u;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            unsigned cur;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(gen) : "memory");
                if (cur == g) __nanosleep(64);
            } while (cur == g);
        }
        __threadfence();
    }
    __syncthreads();
}

struct PersistArgs {
    const float* Yp;
    int64_t Np;
    int Nk, Nkp, n_iter;
    float* V;
    float* D;
    double* Gd;      // [KK] in: G(D0); out: G(D_n)
    float* Bpart;    // [nCTA][K][Nkp]
    double* Hpart;   // [nCTA][KK]
    double* vpart;   // [nCTA][2]
    double* dpart;   // [nCTA]
    double* Gpart;   // [nCTA][KK]
    const double* ypart;
    int nby;
    double* ysq;
    double* obj;     // [2 n_iter] or null
    unsigned* bar;   // [2] barrier count, generation
    unsigned* status;
};

// All n_iter Lee-Seung iterations in one cooperative launch.  Per iteration:
//   tile_pass -> grid barrier -> D update of this CTA's lambda slice (B, H reduced
//   over the CTA partials in a fixed order) -> grid barrier -> G_new from the slice
//   partials (every CTA, same fixed order), objective (CTA 0), D restaged.
template <int K, int LP, int NBUF>
__global__ void __launch_bounds__(NTHREADS, 1) k_nmf_persist(PersistArgs A) {
    constexpr int DS = 2 * TG * LP;
    constexpr int KK = K * K;
    __shared__ FusedShared<K, LP, NBUF> sh;
    __shared__ double Hs[KK], Gold[KK], Gnew[KK];
    __shared__ double gacc[NTHREADS];
    __shared__ double sc[4];
    extern __shared__ __align__(128) float smem[];
    const int tid = threadIdx.x;
    const int nC = gridDim.x, c = blockIdx.x;
    const size_t tile_floats = (size_t)RG * A.Nkp + RG * K;
    float* ring = smem;
    float* Ds = smem + NBUF * tile_floats + DS;
    for (size_t i = tid; i < NBUF * tile_floats + DS; i += NTHREADS) ring[i] = 0.f;
    for (int i = tid; i < KK; i += NTHREADS) Gold[i] = A.Gd[i];
    if (tid == 0) sh.bad = 0u;
    stage_dg<K, LP, NBUF>(A.D, A.Nk, Gold, Ds, sh);
    __syncthreads();
    // lambda slice of this CTA for the D update
    const int SL = (A.Nk + nC - 1) / nC;
    const int l0 = c * SL, l1 = min(A.Nk, l0 + SL);
    const int nsl = max(0, l1 - l0);
    double ysq = 0.0;
    for (int it = 0; it < A.n_iter; ++it) {
        tile_pass<K, LP, NBUF>(A.Yp, A.Np, A.Nkp, A.V, ring, Ds, sh, A.Bpart + (int64_t)c * K * A.Nkp,
                               A.Hpart + (int64_t)c * KK, A.vpart + 2 * (int64_t)c, it == 0);
        grid_sync(A.bar, A.bar + 1);
        // ---- H = sum_c Hpart[c] (fixed order: residue classes, then classes in order)
        {
            constexpr int NQ = NTHREADS / KK > 0 ? NTHREADS / KK : 1;
            if (tid < NQ * KK) {
                const int o = tid % KK, q = tid / KK;
                double s = 0.0;
                for (int cc = q; cc < nC; cc += NQ) s += __ldcg(A.Hpart + (int64_t)cc * KK + o);
                gacc[tid] = s;
            }
            __syncthreads();
            for (int o = tid; o < KK; o += NTHREADS) {
                double s = 0.0;
                for (int q = 0; q < NQ; ++q) s += gacc[q * KK + o];
                Hs[o] = s;
            }
            __syncthreads();
        }
        // ---- B for the slice (K x nsl outputs over nC partials), D update, slice partials
        {
            const int nout = K * nsl;
            const int NQ = nout > 0 ? max(1, NTHREADS / nout) : 1;
            if (nout > 0 && tid < NQ * nout) {
                const int o = tid % nout, q = tid / nout;
                const int k = o / nsl, l = l0 + (o - (o / nsl) * nsl);
                double s = 0.0;
                for (int cc = q; cc < nC; cc += NQ)
                    s += (double)__ldcg(A.Bpart + ((int64_t)cc * K + k) * A.Nkp + l);
                gacc[tid] = s;
            }
            __syncthreads();
            double bd = 0.0;
            float dn[K];
            unsigned bad = 0;
            if (tid < nsl) {
                const int l = l0 + tid;
                double B[K], d[K];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    double s = 0.0;
                    for (int q = 0; q < NQ; ++q) s += gacc[q * nout + k * nsl + tid];
                    B[k] = s;
                    d[k] = (double)__ldcg(A.D + (int64_t)k * A.Nk + l);
                }
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    double hd = 0.0;
#pragma unroll
                    for (int jj = 0; jj < K; ++jj) hd = fma(Hs[k * K + jj], d[jj], hd);
                    dn[k] = (float)(d[k] * B[k] / fmax(hd, 1e-30));
                    if (!isfinite(dn[k])) bad |= ST_NUMERIC;
                    bd += B[k] * (double)dn[k];
                }
            }
            __syncthreads();  // all reads of the old D slice done
            if (tid < nsl) {
#pragma unroll
                for (int k = 0; k < K; ++k) A.D[(int64_t)k * A.Nk + l0 + tid] = dn[k];
                if (bad) atomicOr(A.status, bad);
            }
            // slice partials: <B, D_new> and D_new D_new^T (fixed order over the slice)
            gacc[tid] = (tid < nsl) ? bd : 0.0;
            __syncthreads();
            if (tid == 0) {
                double s = 0.0;
                for (int u = 0; u < nsl; ++u) s += gacc[u];
                A.dpart[c] = s;
            }
            __syncthreads();
            if (tid < nsl) {
#pragma unroll
                for (int k = 0; k < K; ++k) ring[k * 64 + tid] = dn[k];  // ring idle: slice staging
            }
            __syncthreads();
            for (int o = tid; o < KK; o += NTHREADS) {
                const int a = o / K, b = o - (o / K) * K;
                double s = 0.0;
                for (int u = 0; u < nsl; ++u) s = fma((double)ring[a * 64 + u], (double)ring[b * 64 + u], s);
                A.Gpart[(int64_t)c * KK + o] = s;
            }
        }
        grid_sync(A.bar, A.bar + 1);
        // ---- G_new (every CTA, same fixed order), objective (CTA 0), restage D
        {
            constexpr int NQ = NTHREADS / KK > 0 ? NTHREADS / KK : 1;
            if (tid < NQ * KK) {
                const int o = tid % KK, q = tid / KK;
                double s = 0.0;
                for (int cc = q; cc < nC; cc += NQ) s += __ldcg(A.Gpart + (int64_t)cc * KK + o);
                gacc[tid] = s;
            }
            __syncthreads();
            for (int o = tid; o < KK; o += NTHREADS) {
                double s = 0.0;
                for (int q = 0; q < NQ; ++q) s += gacc[q * KK + o];
                Gnew[o] = s;
            }
            __syncthreads();
        }
        if (c == 0) {
            double v0 = 0.0, v1 = 0.0, v2 = 0.0;
            for (int i = tid; i < nC; i += NTHREADS) {
                v0 += __ldcg(A.vpart + 2 * i);
                v2 += __ldcg(A.dpart + i);
            }
            if (it == 0)
                for (int i = tid; i < A.nby; i += NTHREADS) v1 += __ldcg(A.ypart + i);
            const double va = block_sum_d(v0, gacc);
            const double ysq_new = block_sum_d(v1, gacc);
            const double bdot = block_sum_d(v2, gacc);
            if (tid == 0) {
                if (it == 0) {
                    ysq = ysq_new;
                    *A.ysq = ysq;
                    if (!(ysq > 0.0)) atomicOr(A.status, (unsigned)ST_Y_ALLZERO);
                }
                double hg_old = 0.0, hg_new = 0.0;
                for (int t = 0; t < KK; ++t) {
                    hg_old += Hs[t] * Gold[t];
                    hg_new += Hs[t] * Gnew[t];
                }
                if (A.obj) {
                    A.obj[2 * it] = ysq - 2.0 * va + hg_old;
                    A.obj[2 * it + 1] = ysq - 2.0 * bdot + hg_new;
                }
            }
        }
        for (int o = tid; o < KK; o += NTHREADS) Gold[o] = Gnew[o];
        __syncthreads();
        stage_dg<K, LP, NBUF>(A.D, A.Nk, Gold, Ds, sh);
        __syncthreads();
    }
    if (c == 0)
        for (int o = tid; o < KK; o += NTHREADS) A.Gd[o] = Gold[o];
    if (tid == 0 && sh.bad) atomicOr(A.status, sh.bad);
}

}  // namespace

constexpr int lp_cap(int K) {
    // registers per compute thread: 2*K*LP (B columns) + RG*K (row partials) + loads
    return (160 - RG * K) / (2 * K) < 8 ? (160 - RG * K) / (2 * K) : 8;
}

template <int K, int LP, int NB>
inline cudaError_t fused_klb(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D,
                             bool first, unsigned* status, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_nmf_fused<K, LP, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
        attr = true;
    }
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    k_nmf_fused<K, LP, NB><<<p.nblk_f, NTHREADS, p.smem_f, s>>>(w.Yp, Np, g.Nk, p.Nkp, V, D, w.Gd, w.Bpart,
                                                               w.Hpart, w.vpart, first ? 1 : 0, status);
    return cudaGetLastError();
}

template <int K, int LP, int NB>
inline cudaError_t persist_klb(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D,
                               int n_iter, double* obj, unsigned* bar, unsigned* status, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_nmf_persist<K, LP, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
        attr = true;
    }
    PersistArgs A;
    A.Yp = w.Yp;
    A.Np = (int64_t)g.Nv * g.Nr * g.Nc;
    A.Nk = g.Nk;
    A.Nkp = p.Nkp;
    A.n_iter = n_iter;
    A.V = V;
    A.D = D;
    A.Gd = w.Gd;
    A.Bpart = w.Bpart;
    A.Hpart = w.Hpart;
    A.vpart = w.vpart;
    A.dpart = w.dpart;
    A.Gpart = w.Gpart;
    A.ypart = w.ypart;
    A.nby = p.nby;
    A.ysq = w.ysq;
    A.obj = obj;
    A.bar = bar;
    A.status = status;
    void* args[] = {&A};
    return cudaLaunchCooperativeKernel((const void*)k_nmf_persist<K, LP, NB>, dim3(p.nblk_f), dim3(NTHREADS), args,
                                       p.smem_f, s);
}

// (K, LP, NBUF) dispatch to a callable templated on the three
template <int K, int LP, class F>
inline cudaError_t disp_nb(const NmfPlan& p, F&& f) {
    switch (p.nbuf) {
        case 4: return f.template operator()<K, LP, 4>();
        case 6: return f.template operator()<K, LP, 6>();
        case 8: return f.template operator()<K, LP, 8>();
        default: return cudaErrorInvalidValue;
    }
}
template <int K, class F>
inline cudaError_t disp_lp(const NmfPlan& p, F&& f) {
    constexpr int C = lp_cap(K);
    switch (p.LP) {
        case 1: return disp_nb<K, 1>(p, f);
        case 2: return disp_nb<K, (2 <= C ? 2 : 1)>(p, f);
        case 3: return disp_nb<K, (3 <= C ? 3 : 1)>(p, f);
        case 4: return disp_nb<K, (4 <= C ? 4 : 1)>(p, f);
        case 5: return disp_nb<K, (5 <= C ? 5 : 1)>(p, f);
        case 6: return disp_nb<K, (6 <= C ? 6 : 1)>(p, f);
        case 7: return disp_nb<K, (7 <= C ? 7 : 1)>(p, f);
        case 8: return disp_nb<K, (8 <= C ? 8 : 1)>(p, f);
        default: return cudaErrorInvalidValue;
    }
}

// Per-K entry points, defined in nmf_fused_k<K>.cu (one translation unit per K).
template <int K>
cudaError_t fused_launch_k(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D, bool first,
                           unsigned* status, cudaStream_t s) {
    return disp_lp<K>(p, [&]<int KK, int LP, int NB>() {
        return fused_klb<KK, LP, NB>(g, p, w, V, D, first, status, s);
    });
}
template <int K>
cudaError_t persist_launch_k(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D, int n_iter,
                             double* obj, unsigned* bar, unsigned* status, cudaStream_t s) {
    return disp_lp<K>(p, [&]<int KK, int LP, int NB>() {
        return persist_klb<KK, LP, NB>(g, p, w, V, D, n_iter, obj, bar, status, s);
    });
}
#define HSNCT_FUSED_EXTERN(KV)                                                                                  \
    extern template cudaError_t fused_launch_k<KV>(const Geometry&, const NmfPlan&, const NmfWs&, float*,       \
                                                   const float*, bool, unsigned*, cudaStream_t);                \
    extern template cudaError_t persist_launch_k<KV>(const Geometry&, const NmfPlan&, const NmfWs&, float*,     \
                                                     float*, int, double*, unsigned*, unsigned*, cudaStream_t);
HSNCT_FUSED_EXTERN(1) HSNCT_FUSED_EXTERN(2) HSNCT_FUSED_EXTERN(3) HSNCT_FUSED_EXTERN(4)
HSNCT_FUSED_EXTERN(5) HSNCT_FUSED_EXTERN(6) HSNCT_FUSED_EXTERN(7) HSNCT_FUSED_EXTERN(8)

}  // namespace hsnct
