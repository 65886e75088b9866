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
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
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
__global__ void __launch_bounds__(NTHREADS, 1) k_nmf_fused(const float* __restrict__ Yp, int64_t Np, int Nk,
                                                           int Nkp, float* __restrict__ V,
                                                           const float* __restrict__ D,
                                                           const double* __restrict__ Gd,
                                                           float* __restrict__ Bpart,
                                                           double* __restrict__ Hpart,
                                                           double* __restrict__ vpart,
                                                           unsigned* __restrict__ status) {
    // Tiles are RG rows; the CTA's tile sequence j = 0, 1, 2, ... alternates between
    // the two compute groups (group j % 2).  A group runs phase 1, waits for the
    // reducer's V update of that tile, runs phase 2 and releases the buffer, while
    // the other group computes its own tile; the ring keeps NBUF - 2 tiles in flight.
    constexpr int GK = RG * K;
    constexpr int KP = (K + 3) & ~3;
    constexpr int DS = 2 * TG * LP;  // smem row stride of D (>= Nkp, zero padded)
    constexpr int KK = K * K;
    extern __shared__ __align__(128) float smem[];
    __shared__ __align__(8) uint64_t full[NBUF], empty[NBUF], partb[NG], vnb[NG];
    __shared__ float red[NG][GW][GK];
    __shared__ __align__(16) float Vn[NG][RG][KP];
    __shared__ float Gs[KK];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ntiles = (Np + RG - 1) / RG;
    const int64_t nmine = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const size_t tile_floats = (size_t)RG * Nkp + RG * K;   // Y+ rows, then the old V rows
    float* ring = smem;                                  // [NBUF][RG*Nkp + RG*K] + slack DS
    float* Ds = smem + NBUF * tile_floats + DS;          // [K][DS]

    for (size_t i = tid; i < NBUF * tile_floats + DS; i += NTHREADS) ring[i] = 0.f;
    for (int i = tid; i < K * DS; i += NTHREADS) {
        const int k = i / DS, l = i - k * DS;
        Ds[i] = (l < Nk) ? D[(int64_t)k * Nk + l] : 0.f;
    }
    for (int i = tid; i < KK; i += NTHREADS) Gs[i] = (float)Gd[i];
    for (int i = tid; i < NG * RG * KP; i += NTHREADS) (&Vn[0][0][0])[i] = 0.f;
    if (tid == 0) {
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&empty[b], TG);
        }
        for (int g = 0; g < NG; ++g) {
            mbar_init(&partb[g], TG);
            mbar_init(&vnb[g], 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp < CW) {
        // ======================= compute warps =======================
        const int g = warp / GW;
        const int wg = warp - g * GW;
        const int t = tid - g * TG;
        float2 bacc[K][LP];
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int i = 0; i < LP; ++i) bacc[k][i] = make_float2(0.f, 0.f);
        const float* dbase = Ds + 2 * t;
        int64_t kth = 0;  // this group's tile count
        for (int64_t j = g; j < nmine; j += NG, ++kth) {
            const int b = (int)(j % NBUF);
            mbar_wait(&full[b], (unsigned)((j / NBUF) & 1));
            const float* yb = ring + (size_t)b * tile_floats + 2 * t;
            // ---- phase 1
            float part[GK];
#pragma unroll
            for (int x = 0; x < GK; ++x) part[x] = 0.f;
#pragma unroll
            for (int i = 0; i < LP; ++i) {
                float2 y[RG];
#pragma unroll
                for (int r = 0; r < RG; ++r)
                    y[r] = *reinterpret_cast<const float2*>(yb + (size_t)r * Nkp + 2 * TG * i);
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const float2 d = *reinterpret_cast<const float2*>(dbase + k * DS + 2 * TG * i);
#pragma unroll
                    for (int r = 0; r < RG; ++r)
                        part[r * K + k] = fmaf(y[r].x, d.x, fmaf(y[r].y, d.y, part[r * K + k]));
                }
            }
            tr_step<16, GK>(part, lane);
            if (((unsigned)lane & tr_bfly(GK)) == 0) {
                const int base = tr_base<GK>(lane);
#pragma unroll
                for (int x = 0; x < tr_nout(GK); ++x) red[g][wg][base + x] = part[x];
            }
            mbar_arrive(&partb[g]);
            // ---- phase 2 (after the reducer's V update of this tile)
            mbar_wait(&vnb[g], (unsigned)(kth & 1));
            float vr[RG][KP];
#pragma unroll
            for (int r = 0; r < RG; ++r) {
#pragma unroll
                for (int q = 0; q < KP / 4; ++q) {
                    const float4 v4 = reinterpret_cast<const float4*>(&Vn[g][r][0])[q];
                    vr[r][4 * q + 0] = v4.x;
                    vr[r][4 * q + 1] = v4.y;
                    vr[r][4 * q + 2] = v4.z;
                    vr[r][4 * q + 3] = v4.w;
                }
            }
#pragma unroll
            for (int i = 0; i < LP; ++i) {
                float2 y[RG];
#pragma unroll
                for (int r = 0; r < RG; ++r)
                    y[r] = *reinterpret_cast<const float2*>(yb + (size_t)r * Nkp + 2 * TG * i);
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    float2 a = bacc[k][i];
#pragma unroll
                    for (int r = 0; r < RG; ++r) {
                        a.x = fmaf(vr[r][k], y[r].x, a.x);
                        a.y = fmaf(vr[r][k], y[r].y, a.y);
                    }
                    bacc[k][i] = a;
                }
            }
            mbar_arrive(&empty[b]);
        }
        // CTA partial of B for this group
#pragma unroll
        for (int i = 0; i < LP; ++i) {
            const int l0 = 2 * (t + TG * i);
            if (l0 < Nkp) {
#pragma unroll
                for (int k = 0; k < K; ++k)
                    *reinterpret_cast<float2*>(Bpart + (((int64_t)blockIdx.x * NG + g) * K + k) * Nkp + l0) =
                        bacc[k][i];
            }
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
            mbar_expect_tx(&full[b], bytes + vbytes);
            float* slot = ring + (size_t)b * tile_floats;
            bulk_g2s(slot, Yp + r0 * Nkp, bytes, &full[b]);
            if (vbytes) bulk_g2s(slot + (size_t)RG * Nkp, V + r0 * K, vbytes, &full[b]);
        };
        if (lane == 0) {
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
            mbar_wait(&full[b], (unsigned)((j / NBUF) & 1));
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
            mbar_wait(&partb[g], (unsigned)(kth & 1));
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
                    for (int w = 0; w < GW; ++w) a += red[g][w][s];
                    float vg = 0.f;
#pragma unroll
                    for (int jj = 0; jj < K; ++jj) vg = fmaf(vo_all[u][jj], Gs[jj * K + k], vg);
                    float vn = __fdiv_rn(vo_me[u] * a, fmaxf(vg, 1e-30f));
                    if (r >= nv) vn = 0.f;
                    vnew[u] = vn;
                    aval[u] = a;
                    Vn[g][r][k] = vn;
                }
            }
            __syncwarp();
            mbar_arrive(&vnb[g]);
            // off the compute warps' critical path: V store, checks, objective, H, refill
#pragma unroll
            for (int u = 0; u < (GK + 31) / 32; ++u) {
                const int s = lane + 32 * u;
                if (s < GK && s / K < nv) {
                    if (j < NG && !(isfinite(vo_me[u]) && vo_me[u] >= 0.f)) bad |= ST_INIT_BAD;
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
                    for (int r = 0; r < RG; ++r) s = fma((double)Vn[g][r][a], (double)Vn[g][r][c], s);
                    hacc[x] += s;
                }
            }
            // refill: this group's previous tile (j - NG) was released before part(j)
            if (j >= NG && j - NG + NBUF < nmine) {
                const int64_t m = j - NG;
                mbar_wait(&empty[m % NBUF], (unsigned)((m / NBUF) & 1));
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
            vpart[2 * ((int64_t)blockIdx.x * NG + g)] = vdotA;
            vpart[2 * ((int64_t)blockIdx.x * NG + g) + 1] = 0.0;
            if (bad) atomicOr(status, bad);
        }
#pragma unroll
        for (int x = 0; x < (KK + 31) / 32; ++x) {
            const int tt = lane + 32 * x;
            if (tt < KK) Hpart[((int64_t)blockIdx.x * NG + g) * KK + tt] = hacc[x];
        }
    }
}

}  // namespace

// ------------------------------------------------------------------- host side
constexpr int lp_cap(int K) {
    // registers per compute thread: 2*K*LP (B columns) + RG*K (row partials) + loads
    return (160 - RG * K) / (2 * K) < 8 ? (160 - RG * K) / (2 * K) : 8;
}

static int nbuf_for(int Nkp, int LP, int K) {
    const size_t tile = ((size_t)RG * Nkp + RG * K) * sizeof(float);
    const size_t fixed = (size_t)(2 * TG * LP) * sizeof(float) * (1 + K);
    for (int nb = 8; nb >= 4; nb -= 2)   // even: reducer g refills only group-g tiles
        if (nb * tile + fixed <= 205 * 1024) return nb;
    return 0;
}

bool nmf_fused_plan(const Geometry& g, int num_sms, NmfPlan* p) {
    if (g.K > 8) return false;
    const int Nkp = (g.Nk + 3) & ~3;
    const int pairs = (g.Nk + 1) / 2;
    const int LP = (pairs + TG - 1) / TG;
    if (LP > lp_cap(g.K)) return false;
    const int nbuf = nbuf_for(Nkp, LP, g.K);
    if (nbuf < 4) return false;
    p->LP = LP;
    p->nbuf = nbuf;
    p->fthreads = NTHREADS;
    p->smem_f = ((size_t)nbuf * (RG * Nkp + RG * g.K) + (size_t)2 * TG * LP * (1 + g.K)) * sizeof(float);
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    const int64_t ntiles = (Np + RG - 1) / RG;
    p->nblk_f = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)num_sms));
    p->PB = p->nblk_f * NG;
    p->nby = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms * 8, (Np * (Nkp / 4) + 255) / 256));
    return true;
}

template <int K, int LP, int NB>
static cudaError_t fused_klb(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D,
                             unsigned* status, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_nmf_fused<K, LP, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
        attr = true;
    }
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    k_nmf_fused<K, LP, NB><<<p.nblk_f, NTHREADS, p.smem_f, s>>>(w.Yp, Np, g.Nk, p.Nkp, V, D, w.Gd, w.Bpart,
                                                               w.Hpart, w.vpart, status);
    return cudaGetLastError();
}

template <int K, int LP>
static cudaError_t fused_kl(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D,
                            unsigned* status, cudaStream_t s) {
    switch (p.nbuf) {
        case 4: return fused_klb<K, LP, 4>(g, p, w, V, D, status, s);
        case 6: return fused_klb<K, LP, 6>(g, p, w, V, D, status, s);
        case 8: return fused_klb<K, LP, 8>(g, p, w, V, D, status, s);
        default: return cudaErrorInvalidValue;
    }
}

template <int K>
static cudaError_t fused_k(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D,
                           unsigned* status, cudaStream_t s) {
    constexpr int C = lp_cap(K);
    switch (p.LP) {
        case 1: return fused_kl<K, 1>(g, p, w, V, D, status, s);
        case 2: return fused_kl<K, (2 <= C ? 2 : 1)>(g, p, w, V, D, status, s);
        case 3: return fused_kl<K, (3 <= C ? 3 : 1)>(g, p, w, V, D, status, s);
        case 4: return fused_kl<K, (4 <= C ? 4 : 1)>(g, p, w, V, D, status, s);
        case 5: return fused_kl<K, (5 <= C ? 5 : 1)>(g, p, w, V, D, status, s);
        case 6: return fused_kl<K, (6 <= C ? 6 : 1)>(g, p, w, V, D, status, s);
        case 7: return fused_kl<K, (7 <= C ? 7 : 1)>(g, p, w, V, D, status, s);
        case 8: return fused_kl<K, (8 <= C ? 8 : 1)>(g, p, w, V, D, status, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t nmf_yplus_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y, int64_t ld_y,
                             unsigned* status, cudaStream_t s) {
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    k_yplus<<<p.nby, 256, 0, s>>>(Y, ld_y, Np, g.Nk, p.Nkp, w.Yp, w.ypart, status);
    return cudaGetLastError();
}

cudaError_t nmf_fused_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D,
                             unsigned* status, cudaStream_t s) {
    switch (g.K) {
        case 1: return fused_k<1>(g, p, w, V, D, status, s);
        case 2: return fused_k<2>(g, p, w, V, D, status, s);
        case 3: return fused_k<3>(g, p, w, V, D, status, s);
        case 4: return fused_k<4>(g, p, w, V, D, status, s);
        case 5: return fused_k<5>(g, p, w, V, D, status, s);
        case 6: return fused_k<6>(g, p, w, V, D, status, s);
        case 7: return fused_k<7>(g, p, w, V, D, status, s);
        case 8: return fused_k<8>(g, p, w, V, D, status, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace hsnct
