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

#include "internal.h"

namespace hsnct {
namespace {

constexpr int VT = 256;        // row-pass threads
constexpr int VW = VT / 32;    // row-pass warps
constexpr int RPW = 4;         // rows per warp step
constexpr int BT_MAX = 128;    // column-pass threads (one lambda quad each)
constexpr int BROWS = 32;      // V rows staged per column-pass sub-chunk
constexpr int DT = 256;        // D-update threads (one lambda each)

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
template <int K>
__global__ void __launch_bounds__(256) k_gram_init(const float* __restrict__ D, int Nk,
                                                   double* __restrict__ Gd,
                                                   unsigned* __restrict__ status) {
    __shared__ double part[256];
    unsigned bad = 0;
    for (int i = threadIdx.x; i < K * Nk; i += blockDim.x) {
        float d = D[i];
        if (!(isfinite(d) && d >= 0.f)) bad = ST_INIT_BAD;
    }
    bad = warp_or(bad);
    if (bad && (threadIdx.x & 31) == 0) atomicOr(status, bad);
    for (int t = 0; t < K * K; ++t) {
        const int a = t / K, b = t % K;
        double s = 0.0;
        for (int l = threadIdx.x; l < Nk; l += blockDim.x)
            s += (double)D[(int64_t)a * Nk + l] * (double)D[(int64_t)b * Nk + l];
        part[threadIdx.x] = s;
        __syncthreads();
        for (int w = blockDim.x / 2; w > 0; w >>= 1) {
            if ((int)threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) Gd[t] = part[0];
        __syncthreads();
    }
}

// ---------------------------------------------------------------- row pass
template <int K, bool FIRST>
__global__ void __launch_bounds__(VT) k_vstep(const float* __restrict__ Y, int64_t ld, int64_t Np,
                                              int Nk, int Nkp, float* __restrict__ V,
                                              const float* __restrict__ D,
                                              const double* __restrict__ Gd,
                                              double* __restrict__ vpart,
                                              unsigned* __restrict__ status) {
    extern __shared__ __align__(16) float Ds[];  // [K][Nkp], zero padded
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
                }
                y[rr] = clamp0(y[rr]);
                if (FIRST) {
                    ys[rr] = fmaf(y[rr].x, y[rr].x, ys[rr]);
                    ys[rr] = fmaf(y[rr].y, y[rr].y, ys[rr]);
                    ys[rr] = fmaf(y[rr].z, y[rr].z, ys[rr]);
                    ys[rr] = fmaf(y[rr].w, y[rr].w, ys[rr]);
                }
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const float4 d = reinterpret_cast<const float4*>(Ds + k * Nkp)[q];
#pragma unroll
                for (int rr = 0; rr < RPW; ++rr) {
                    float a = acc[rr][k];
                    a = fmaf(y[rr].x, d.x, a);
                    a = fmaf(y[rr].y, d.y, a);
                    a = fmaf(y[rr].z, d.z, a);
                    a = fmaf(y[rr].w, d.w, a);
                    acc[rr][k] = a;
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
    const bool do_h = blockIdx.y == 0 && tid < K * K;
    const int ha = tid / K, hb = tid - (tid / K) * K;
    float4 acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    double h = 0.0;
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
                        acc[k].x = fmaf(v, y[u].x, acc[k].x);
                        acc[k].y = fmaf(v, y[u].y, acc[k].y);
                        acc[k].z = fmaf(v, y[u].z, acc[k].z);
                        acc[k].w = fmaf(v, y[u].w, acc[k].w);
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
                    acc[k].x = fmaf(v, y.x, acc[k].x);
                    acc[k].y = fmaf(v, y.y, acc[k].y);
                    acc[k].z = fmaf(v, y.z, acc[k].z);
                    acc[k].w = fmaf(v, y.w, acc[k].w);
                }
            }
        }
        if (do_h) {
            double hs = 0.0;
            for (int i = 0; i < nr; ++i) hs = fma((double)Vs[i * K + ha], (double)Vs[i * K + hb], hs);
            h += hs;
        }
    }
    if (qv) {
#pragma unroll
        for (int k = 0; k < K; ++k)
            reinterpret_cast<float4*>(Bpart + ((int64_t)blockIdx.x * K + k) * Nkp)[q] = acc[k];
    }
    if (do_h) Hpart[(int64_t)blockIdx.x * K * K + tid] = h;
}

// ---------------------------------------------------------------- D update
template <int K>
__global__ void __launch_bounds__(DT) k_dupdate(const float* __restrict__ Bpart,
                                                const double* __restrict__ Hpart, int nchunk, int Nk,
                                                int Nkp, float* __restrict__ D, double* __restrict__ Gd,
                                                const double* __restrict__ vpart, int nblk_v,
                                                double* __restrict__ dpart, double* __restrict__ Gpart,
                                                double* __restrict__ ysq_store, int first,
                                                double* __restrict__ obj2,
                                                unsigned* __restrict__ counter,
                                                unsigned* __restrict__ status) {
    __shared__ double Hs[K * K];
    __shared__ double dsm[K][DT];
    __shared__ double red[DT / 32];
    __shared__ int is_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int t = tid; t < K * K; t += DT) {
        double s = 0.0;
        for (int c = 0; c < nchunk; ++c) s += Hpart[(int64_t)c * K * K + t];
        Hs[t] = s;
    }
    __syncthreads();
    const int l = blockIdx.x * DT + tid;
    double bd = 0.0;
    unsigned bad = 0;
    if (l < Nk) {
        double B[K], d[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = 0.0;
            for (int c = 0; c < nchunk; ++c) s += (double)Bpart[((int64_t)c * K + k) * Nkp + l];
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
            dsm[k][tid] = (double)dn;
            bd += B[k] * (double)dn;
        }
    } else {
#pragma unroll
        for (int k = 0; k < K; ++k) dsm[k][tid] = 0.0;
    }
    bd = warp_sum(bd);
    bad = warp_or(bad);
    if (lane == 0) {
        red[warp] = bd;
        if (bad) atomicOr(status, bad);
    }
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < DT / 32; ++w) s += red[w];
        dpart[blockIdx.x] = s;
    }
    // per-block partial of G_new = D_new D_new^T (fixed order over this block's lambdas)
    for (int t = tid; t < K * K; t += DT) {
        const int a = t / K, b = t - (t / K) * K;
        double s = 0.0;
        for (int u = 0; u < DT; ++u) s = fma(dsm[a][u], dsm[b][u], s);
        Gpart[(int64_t)blockIdx.x * K * K + t] = s;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) is_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    // ---- last block: objective terms and G for the next row pass
    __shared__ double sc[4];
    if (tid == 0) {
        double ysq;
        if (first) {
            ysq = 0.0;
            for (int i = 0; i < nblk_v; ++i) ysq += __ldcg(vpart + 2 * i + 1);
            *ysq_store = ysq;
            if (!(ysq > 0.0)) atomicOr(status, (unsigned)ST_Y_ALLZERO);
        } else {
            ysq = *ysq_store;
        }
        double va = 0.0, bdot = 0.0;
        for (int i = 0; i < nblk_v; ++i) va += __ldcg(vpart + 2 * i);
        for (int i = 0; i < (int)gridDim.x; ++i) bdot += __ldcg(dpart + i);
        double hg_old = 0.0;
        for (int t = 0; t < K * K; ++t) hg_old += Hs[t] * Gd[t];
        sc[0] = ysq;
        sc[1] = va;
        sc[2] = bdot;
        sc[3] = hg_old;
    }
    __syncthreads();
    for (int t = tid; t < K * K; t += DT) {
        double s = 0.0;
        for (int i = 0; i < (int)gridDim.x; ++i) s += __ldcg(Gpart + (int64_t)i * K * K + t);
        Gd[t] = s;
    }
    __syncthreads();
    if (tid == 0) {
        double hg_new = 0.0;
        for (int t = 0; t < K * K; ++t) hg_new += Hs[t] * Gd[t];
        if (obj2) {
            obj2[0] = sc[0] - 2.0 * sc[1] + sc[3];
            obj2[1] = sc[0] - 2.0 * sc[2] + hg_new;
        }
        *counter = 0u;
    }
}

// ------------------------------------------------------------ K dispatch
#define HSNCT_K_CASES(M) \
    M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15) M(16)

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

}  // namespace

NmfPlan nmf_plan(const Geometry& g, int num_sms) {
    NmfPlan p{};
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    p.Nkp = (g.Nk + 3) & ~3;
    p.smem_v = (size_t)g.K * p.Nkp * sizeof(float);
    // row pass: 256-thread blocks, up to `occ` per SM (smem-limited), static schedule
    int occ = (int)std::max<size_t>(1, std::min<size_t>(4, (200u * 1024u) / std::max<size_t>(p.smem_v + 4096, 1)));
    const int64_t groups = (Np + VW * RPW - 1) / (VW * RPW);
    p.nblk_v = (int)std::max<int64_t>(1, std::min<int64_t>(groups, (int64_t)num_sms * occ));
    // column pass: one lambda quad per thread
    const int nq = p.Nkp / 4;
    p.nlam_blk = (nq + BT_MAX - 1) / BT_MAX;
    const int per = (nq + p.nlam_blk - 1) / p.nlam_blk;
    p.bthreads = std::max(32, ((per + 31) / 32) * 32);
    const int64_t want = std::max<int64_t>(1, ((int64_t)num_sms * 8) / p.nlam_blk);
    p.nchunk = (int)std::max<int64_t>(1, std::min<int64_t>(want, (Np + BROWS - 1) / BROWS));
    p.rows_per_chunk = (Np + p.nchunk - 1) / p.nchunk;
    p.nchunk = (int)((Np + p.rows_per_chunk - 1) / p.rows_per_chunk);
    if (p.nchunk < 1) p.nchunk = 1;
    p.nblk_d = (g.Nk + DT - 1) / DT;
    return p;
}

size_t nmf_ws_bytes(const Geometry& g, const NmfPlan& p) {
    const size_t KK = (size_t)g.K * g.K;
    size_t b = 0;
    b += align256(KK * sizeof(double));                          // Gd
    b += align256((size_t)p.nblk_v * 2 * sizeof(double));        // vpart
    b += align256((size_t)p.nblk_d * sizeof(double));            // dpart
    b += align256((size_t)p.nblk_d * KK * sizeof(double));       // Gpart
    b += align256(sizeof(double));                               // ysq
    b += align256((size_t)p.nchunk * KK * sizeof(double));       // Hpart
    b += align256((size_t)p.nchunk * g.K * p.Nkp * sizeof(float));  // Bpart
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
    w.vpart = (double*)take((size_t)p.nblk_v * 2 * sizeof(double));
    w.dpart = (double*)take((size_t)p.nblk_d * sizeof(double));
    w.Gpart = (double*)take((size_t)p.nblk_d * KK * sizeof(double));
    w.ysq = (double*)take(sizeof(double));
    w.Hpart = (double*)take((size_t)p.nchunk * KK * sizeof(double));
    w.Bpart = (float*)take((size_t)p.nchunk * g.K * p.Nkp * sizeof(float));
    return w;
}

cudaError_t nmf_launch_init(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* D,
                            unsigned* status, cudaStream_t s) {
    (void)p;
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
                          int64_t ld, float* V, float* D, bool first, double* obj2,
                          unsigned* status, unsigned* counter, cudaStream_t s) {
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    static bool attr_done = false;  // per-K instantiation
    if (!attr_done) {
        cudaFuncSetAttribute(k_vstep<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        cudaFuncSetAttribute(k_vstep<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        attr_done = true;
    }
    if (first)
        k_vstep<K, true><<<p.nblk_v, VT, p.smem_v, s>>>(Y, ld, Np, g.Nk, p.Nkp, V, D, w.Gd, w.vpart, status);
    else
        k_vstep<K, false><<<p.nblk_v, VT, p.smem_v, s>>>(Y, ld, Np, g.Nk, p.Nkp, V, D, w.Gd, w.vpart, status);
    dim3 gb(p.nchunk, p.nlam_blk);
    k_bpart<K><<<gb, p.bthreads, 0, s>>>(Y, ld, Np, g.Nk, p.Nkp, V, p.rows_per_chunk, w.Bpart, w.Hpart);
    k_dupdate<K><<<p.nblk_d, DT, 0, s>>>(w.Bpart, w.Hpart, p.nchunk, g.Nk, p.Nkp, D, w.Gd, w.vpart,
                                         p.nblk_v, w.dpart, w.Gpart, w.ysq, first ? 1 : 0,
                                         obj2, counter, status);
    return cudaGetLastError();
}

cudaError_t nmf_launch_iter(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y,
                            int64_t ld_y, float* V, float* D, bool first, double* obj2,
                            unsigned* status, unsigned* counter, cudaStream_t s) {
    switch (g.K) {
#define M(KV) \
    case KV:  \
        return iter_k<KV>(g, p, w, Y, ld_y, V, D, first, obj2, status, counter, s);
        HSNCT_K_CASES(M)
#undef M
        default:
            return cudaErrorInvalidValue;
    }
}

}  // namespace hsnct
