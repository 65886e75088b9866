// Tensor-core Lee-Seung iteration (Eq. 4; R1-R3, R20),
// K <= 8: both contractions of the fused row pass run on the tensor cores
// (mma.sync f16 -> f32) from an fp16 hi/lo split of every operand, which keeps the
// products fp32-accurate (|x - hi - lo| <= 2^-22 |x|; the dropped lo*lo term is
// below that) at the SAME 4 bytes per element of Y as fp32.
//
// Why mma.sync and not tcgen05: the V update is row-local and must see the whole
// row of Y (all N_k bins) before the B = V^T Y half can use the new V.  A tile must
// therefore hold complete rows in shared memory; tcgen05 needs M >= 64 rows
// (64 x 1600 x 4 B = 410 KB > 227 KB), mma.sync needs 16 (8 real rows + 8 zero rows
// in phase 1, K = 8 rows in phase 2).  At this shape the pass needs ~40% of the
// measured mma.sync f16 rate (555 TFLOP/s, scripts/microbench) and is HBM-bound.
//
// Input: Y+ split once per call by k_ysplit into rows of [hi(N16) | lo(N16)] halves,
// N16 = N_k rounded up to 16 (zero padded).  One persistent CTA per SM, 12 warps, a
// static schedule of 8-row tiles (CTA c: tiles c, c + nCTA, ...), visited forward in
// even iterations and backward in odd ones (L2 reuse), streamed through NSLOT
// shared-memory slots by cp.async.bulk (one copy per row into a 16-byte padded row
// pitch, so ldmatrix rows never share banks, plus one copy of the tile's old V rows).
// Warp w owns the 16-bin k-steps [w S/12, (w+1) S/12) of every row, S = N16/16.
//   registers:  its D fragments (hi, lo; loaded once per pass from D), its B = V^T Y+
//               partial (fp32, RN-added per tile), the tile's Y fragments;
//   per tile:   ldmatrix Y (hi, lo) -> slot released (the last warp out refills it);
//               phase 1: A_w = Y D^T over its bins, 3 mma m16n8k16 per k-step
//                 (hi*Dhi + hi*Dlo + lo*Dhi), rows 8..15 of the 16-row A are zero;
//               partials of the 12 warps summed in a fixed order (one named barrier);
//               V[r][k] <- V[r][k] A[r][k] / max(sum_j V[r][j] G[j][k], 1e-30)
//                 (every warp, redundantly; one stores V, one accumulates H);
//               phase 2: B[k][l] += sum_r V_new[r][k] Y+[r][l], 3 mma m16n8k8 per
//                 k-step on the transposed Y fragments (movmatrix), started from zero
//                 and added to the fp32 running partial with round-to-nearest.
// Per-CTA partials and the D update are as in the FFMA kernel (nmf_fused.cuh).
// Deterministic: static schedule, fixed reduction orders, no floating-point atomics.
#pragma once
#include <cuda_fp16.h>

#include <algorithm>

#include "internal.h"
#include "nmf_common.cuh"

namespace hsnct {
namespace {

constexpr int MR = 8;            // rows per tile
constexpr int MWARPS = 12;       // warps per CTA
constexpr int MTHREADS = MWARPS * 32;
constexpr int MVW = MWARPS - 1;  // warp that stores V / accumulates <V_new, A>
constexpr int MHW = MWARPS - 2;  // warp that accumulates H
constexpr int MSPW_MAX = 12;     // k-steps per warp supported (N16 <= 12*12*16)

__device__ __forceinline__ unsigned pack_h2(__half lo, __half hi) {
    return (unsigned)__half_as_ushort(lo) | ((unsigned)__half_as_ushort(hi) << 16);
}
// x -> (hi, lo) halves with hi = rn(x), lo = rn(x - hi); packed pairs for two values
__device__ __forceinline__ void split2(float x0, float x1, unsigned& hi, unsigned& lo) {
    const __half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
    const __half l0 = __float2half_rn(x0 - __half2float(h0)), l1 = __float2half_rn(x1 - __half2float(h1));
    hi = pack_h2(h0, h1);
    lo = pack_h2(l0, l1);
}
__device__ __forceinline__ void ldsm_x4(unsigned addr, unsigned& r0, unsigned& r1, unsigned& r2, unsigned& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(unsigned addr, unsigned& r0, unsigned& r1, unsigned& r2, unsigned& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ unsigned movm_t(unsigned a) {
    unsigned d;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
    return d;
}
// c += A(16x16, rows 8..15 zero) * B(16x8)
__device__ __forceinline__ void mma16816(float* c, unsigned a0, unsigned a2, unsigned b0, unsigned b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
// c += A(16x8) * B(8x8)
__device__ __forceinline__ void mma1688(float* c, unsigned a0, unsigned a1, unsigned b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5}, {%6}, {%0, %1, %2, %3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(b0));
}

// Y+ = max(Y, 0) split into rows of [hi(N16) | lo(N16)] halves (zero padded); flags
// non-finite Y; per-block ||Y+||^2 partials (fp64, from the fp32 values).
__global__ void __launch_bounds__(256) k_ysplit(const float* __restrict__ Y, int64_t ld, int64_t Np, int Nk,
                                                int N16, __half* __restrict__ Yh, double* __restrict__ ypart,
                                                unsigned* __restrict__ status) {
    __shared__ double red[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nq = N16 >> 2;
    const int64_t nw = (int64_t)gridDim.x * 8;
    double s = 0.0;
    unsigned bad = 0;
    for (int64_t p = (int64_t)blockIdx.x * 8 + w; p < Np; p += nw) {
        const float* src = Y + p * ld;
        uint2* dhi = reinterpret_cast<uint2*>(Yh + p * 2 * N16);
        uint2* dlo = reinterpret_cast<uint2*>(Yh + p * 2 * N16 + N16);
        float rs = 0.f;
#pragma unroll 4
        for (int q = lane; q < nq; q += 32) {
            const int l0 = 4 * q;
            float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
            if (l0 < Nk) {
                y = __ldcs(reinterpret_cast<const float4*>(src + l0));  // l0 + 3 < ld (ld % 4 == 0)
                if (l0 + 1 >= Nk) y.y = 0.f;
                if (l0 + 2 >= Nk) y.z = 0.f;
                if (l0 + 3 >= Nk) y.w = 0.f;
            }
            if (!(isfinite(y.x) && isfinite(y.y) && isfinite(y.z) && isfinite(y.w))) bad = ST_Y_NONFINITE;
            y.x = fmaxf(y.x, 0.f);
            y.y = fmaxf(y.y, 0.f);
            y.z = fmaxf(y.z, 0.f);
            y.w = fmaxf(y.w, 0.f);
            rs = fmaf(y.x, y.x, fmaf(y.y, y.y, fmaf(y.z, y.z, fmaf(y.w, y.w, rs))));
            uint2 h, l;
            split2(y.x, y.y, h.x, l.x);
            split2(y.z, y.w, h.y, l.y);
            dhi[q] = h;
            dlo[q] = l;
        }
        s += (double)rs;
    }
    s = warp_sum_d(s);
#pragma unroll
    for (int o = 16; o; o >>= 1) bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    if (lane == 0) {
        red[w] = s;
        if (bad) atomicOr(status, bad);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < 8; ++i) t += red[i];
        ypart[blockIdx.x] = t;
    }
}

struct MmaArgs {
    const __half* Yh;  // [Np][2*N16]
    int64_t Np;
    int Nk, N16, n_iter, nslot;
    float* V;
    float* D;
    double* Gd;        // [KK] in: G(D0); out: G(D_n)
    float* Bpart;      // [nCTA][K][N16]
    double* Hpart;     // [nCTA][KK]
    double* vpart;     // [nCTA][2]
    double* dpart;     // [nCTA]
    double* Gpart;     // [nCTA][KK]
    const double* ypart;
    int nby;
    double* ysq;
    double* obj;       // [2 n_iter] or null
    uint64_t* trace;   // [trace_iters][nCTA][TRACE_SLOTS] or null
    int trace_iters;
    unsigned* bar;     // grid-barrier arrival counter, zero at launch
    unsigned* status;
};

__host__ __device__ constexpr unsigned mma_row_pitch(int N16) { return 4u * (unsigned)N16 + 16u; }
__host__ __device__ constexpr unsigned mma_slot_bytes(int N16, int K) {
    return (MR * mma_row_pitch(N16) + 4u * MR * (unsigned)K + 127u) & ~127u;
}

template <int K>
struct MmaShared {
    static constexpr int KK = K * K;
    uint64_t full[8];
    uint64_t part[4];               // the 12 warps' phase-1 partials of a tile are in
    unsigned rel[8];
    float2 red[4][MWARPS][32];      // per-warp partial A fragments, by tile index mod 4
    float Vn[MWARPS][MR][8];        // each warp's copy of the tile's new V rows (for H)
    float Gs[KK];
    double Hs[KK], Gold[KK], Gnew[KK];
    double gacc[MTHREADS];
    double dred[MTHREADS / 32];
    double dnew[K * 16];            // the CTA's lambda slice of D_new (nsl <= 16 for N16 <= 2304)
    double Bsl[8 * 16];
    double vsw[MWARPS];
    unsigned bad;
};

template <int K, int SPW>
__global__ void __launch_bounds__(MTHREADS, 1) k_nmf_mma(MmaArgs A) {
    constexpr int KK = K * K;
    __shared__ MmaShared<K> sh;
    extern __shared__ __align__(128) unsigned char mslots[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;  // mma fragment row / column pair
    const int nC = gridDim.x, c = blockIdx.x;
    const int N16 = A.N16, S = N16 >> 4, NS = A.nslot;
    const unsigned RP = mma_row_pitch(N16), SB = mma_slot_bytes(N16, K);
    const int s0 = (warp * S) / MWARPS, ns = ((warp + 1) * S) / MWARPS - s0;  // this warp's k-steps
    const int64_t ntiles = (A.Np + MR - 1) / MR;
    const int64_t nmine = ntiles > c ? (ntiles - 1 - c) / nC + 1 : 0;
    const unsigned sbase = smem_u32(mslots);

    // ---- prologue (slots zeroed once: rows a partial tile does not fill stay finite)
    for (int i = tid; i < NS * (int)(SB >> 4); i += MTHREADS)
        reinterpret_cast<uint4*>(mslots)[i] = make_uint4(0u, 0u, 0u, 0u);
    fence_proxy_async();
    if (tid == 0) {
        for (int b = 0; b < NS; ++b) {
            mbar_init(&sh.full[b], 1);
            sh.rel[b] = 0u;
        }
        for (int i = 0; i < 4; ++i) mbar_init(&sh.part[i], MWARPS);
        sh.bad = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < KK; i += MTHREADS) {
        sh.Gold[i] = A.Gd[i];
        sh.Gs[i] = (float)A.Gd[i];
    }
    __syncthreads();

    auto row0 = [&](int64_t q, bool fwd) -> int64_t {
        const int64_t pos = fwd ? q : (nmine - 1 - q);
        return ((int64_t)c + pos * nC) * MR;
    };
    auto issue = [&](int b, int64_t q, bool fwd) {  // tile q of the pass into slot b
        const int64_t r0 = row0(q, fwd);
        const int nv = (int)min((int64_t)MR, A.Np - r0);
        const unsigned rowb = 4u * (unsigned)N16;
        const unsigned vbytes = nv == MR ? 4u * MR * K : 0u;
        uint64_t* bar = &sh.full[b];
        mbar_expect_tx(bar, (unsigned)nv * rowb + vbytes);
        unsigned char* slot = mslots + (size_t)b * SB;
        for (int r = 0; r < nv; ++r) bulk_g2s(slot + (size_t)r * RP, A.Yh + (r0 + r) * 2 * N16, rowb, bar);
        if (vbytes) bulk_g2s(slot + (size_t)MR * RP, A.V + r0 * K, vbytes, bar);
    };
    auto issue_head = [&](int bstart, bool fwd) {  // first NS tiles of a pass, slots bstart, bstart + 1, ...
        int b = bstart;
        for (int64_t m = 0; m < min((int64_t)NS, nmine); ++m) {
            issue(b, m, fwd);
            b = b + 1 == NS ? 0 : b + 1;
        }
    };

    // D fragments of this warp's k-steps (hi, lo), from the fp32 D (zero for k >= K, l >= Nk)
    unsigned dh[SPW][2], dl[SPW][2];
    auto load_dfrag = [&]() {
#pragma unroll
        for (int s = 0; s < SPW; ++s) {
            float v[4] = {0.f, 0.f, 0.f, 0.f};
            if (s < ns && g < K) {
                const int lb = 16 * (s0 + s) + 2 * t4;
                const float* dr = A.D + (int64_t)g * A.Nk;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int l = lb + (e & 1) + 8 * (e >> 1);
                    v[e] = l < A.Nk ? __ldcg(dr + l) : 0.f;
                }
            }
            split2(v[0], v[1], dh[s][0], dl[s][0]);
            split2(v[2], v[3], dh[s][1], dl[s][1]);
        }
    };
    load_dfrag();

    // lambda slice of this CTA for the D update
    const int SL = (A.Nk + nC - 1) / nC;
    const int l0s = min(A.Nk, c * SL), l1s = min(A.Nk, l0s + SL);
    const int nsl = max(0, l1s - l0s);
    unsigned epoch = 0;
    double ysq = 0.0;
    int64_t n0 = 0;
    int slot_b = 0;          // slot of the next tile (running over all passes) ...
    unsigned slot_ph = 0u;   // ... and its mbarrier phase
    auto stamp = [&](int it, int slot) {
        if (A.trace && tid == 0 && it < A.trace_iters) {
            uint64_t tnow;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
            A.trace[((int64_t)it * nC + c) * TRACE_SLOTS + slot] = tnow;
        }
    };
    if (tid == 0) {
        fence_proxy_async_global();
        issue_head(0, true);
    }

    for (int it = 0; it < A.n_iter; ++it) {
        const bool fwd = (it & 1) == 0, first = it == 0;
        stamp(it, 0);
        // ================================ row pass ================================
        float bt[SPW][4];
#pragma unroll
        for (int s = 0; s < SPW; ++s) bt[s][0] = bt[s][1] = bt[s][2] = bt[s][3] = 0.f;
        double vdotA = 0.0;
        constexpr int NHX = (KK + MWARPS * 32 - 1) / (MWARPS * 32);  // H entries per lane
        double hacc[NHX];
#pragma unroll
        for (int x = 0; x < NHX; ++x) hacc[x] = 0.0;
        unsigned bad = 0;
        // Software pipeline over the CTA's tiles (iteration j):
        //   phase 1 of tile j -> publish its 12 partials (split arrive) ->
        //   wait for the partials of tile j - 1 (published one iteration ago, so the wait
        //   is normally already satisfied) -> V update of tile j - 1 -> phase 2 of tile
        //   j - 1 (ldmatrix.trans rereads its slot) -> slot released, last warp refills.
        // Two slots are in use at a time; partial buffers rotate over 4 (a warp can be at
        // most three tiles ahead of another's reads).
        float rf_p[2] = {0.f, 0.f}, vo_p[2] = {0.f, 0.f};
        int nv_p = 0, b_p = 0;
        int64_t r0_p = 0;
        const int mi = lane >> 3, rr = lane & 7;
        const unsigned aoff = (unsigned)rr * RP + (mi >= 2 ? 2u * N16 : 0u) + (unsigned)(mi & 1) * 16u;
        for (int64_t j = 0; j <= nmine; ++j) {
            const bool cur = j < nmine;
            const int64_t n = n0 + j;
            const int b = slot_b;
            const unsigned ph = slot_ph;
            if (cur && ++slot_b == NS) {
                slot_b = 0;
                slot_ph ^= 1u;
            }
            const int64_t r0 = cur ? row0(j, fwd) : 0;
            const int nv = cur ? (int)min((int64_t)MR, A.Np - r0) : 0;
            float rf[2] = {0.f, 0.f}, vo[2] = {0.f, 0.f};
            if (cur) {
                mbar_wait(&sh.full[b], ph);
                // -- V-update factors for (row g, k = 2 t4, 2 t4 + 1) from the old V rows
                const float* vrow = reinterpret_cast<const float*>(mslots + (size_t)b * SB + (size_t)MR * RP) + g * K;
                float vj[K];
#pragma unroll
                for (int jj = 0; jj < K; ++jj) vj[jj] = nv == MR ? vrow[jj] : (g < nv ? A.V[(r0 + g) * K + jj] : 0.f);
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int k = 2 * t4 + e;
                    if (k < K) {
                        float vg = 0.f, vk = 0.f;
#pragma unroll
                        for (int jj = 0; jj < K; ++jj) {
                            vg = fmaf(vj[jj], sh.Gs[jj * K + k], vg);
                            if (jj == k) vk = vj[jj];
                        }
                        vo[e] = vk;
                        rf[e] = __fdiv_rn(vk, fmaxf(vg, 1e-30f));
                    }
                }
                // -- phase 1: A_w = Y+ D^T over this warp's bins.  Every warp runs SPW steps
                //    (no divergence around the .aligned ops); steps past its own reread a
                //    valid one and meet zero D fragments.
                const unsigned acur = sbase + (unsigned)b * SB + aoff;
                float a1[3][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
                for (int s = 0; s < SPW; ++s) {
                    const unsigned ks = (unsigned)(s < ns ? s0 + s : s0) * 32u;
                    unsigned y0, y1, y2, y3;
                    ldsm_x4(acur + ks, y0, y1, y2, y3);
                    mma16816(a1[0], y0, y1, dh[s][0], dh[s][1]);
                    mma16816(a1[1], y0, y1, dl[s][0], dl[s][1]);
                    mma16816(a1[2], y2, y3, dh[s][0], dh[s][1]);
                }
                const int pb = (int)(n & 3);
                sh.red[pb][warp][lane] = make_float2(a1[0][0] + (a1[1][0] + a1[2][0]), a1[0][1] + (a1[1][1] + a1[2][1]));
                __syncwarp();
                if (lane == 0) mbar_arrive(&sh.part[pb]);
            }
            if (j > 0) {
                // ---- tile p = j - 1: V update, then phase 2
                const int64_t np = n - 1;
                const int pb = (int)(np & 3);
                mbar_wait(&sh.part[pb], (unsigned)((np >> 2) & 1));
                float av[2] = {0.f, 0.f};
#pragma unroll
                for (int w = 0; w < MWARPS; ++w) {
                    const float2 p = sh.red[pb][w][lane];
                    av[0] += p.x;
                    av[1] += p.y;
                }
                float vn[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) vn[e] = (g < nv_p && 2 * t4 + e < K) ? av[e] * rf_p[e] : 0.f;
                // bookkeeping spread over the warps: warp w < MR stores row w of V_new and
                // its share of <V_new, A>; H entry tt is accumulated by warp tt % MWARPS
                if (warp < MR && g == warp) {
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int k = 2 * t4 + e;
                        if (g < nv_p && k < K) {
                            if (first && !(isfinite(vo_p[e]) && vo_p[e] >= 0.f)) bad |= ST_INIT_BAD;
                            if (!isfinite(vn[e])) bad |= ST_NUMERIC;
                            A.V[(r0_p + g) * K + k] = vn[e];
                            vdotA += (double)vn[e] * (double)av[e];
                        }
                    }
                }
                if (warp < KK) {
                    sh.Vn[warp][g][2 * t4] = vn[0];
                    sh.Vn[warp][g][2 * t4 + 1] = vn[1];
                    __syncwarp();
#pragma unroll
                    for (int x = 0; x < (KK + MWARPS * 32 - 1) / (MWARPS * 32); ++x) {
                        const int tt = warp + MWARPS * (lane + 32 * x);
                        if (tt < KK) {
                            const int a = tt / K, cc = tt - (tt / K) * K;
                            double hsum = 0.0;
#pragma unroll
                            for (int r = 0; r < MR; ++r)
                                hsum = fma((double)sh.Vn[warp][r][a], (double)sh.Vn[warp][r][cc], hsum);
                            hacc[x] += hsum;
                        }
                    }
                    __syncwarp();
                }
                // V_new as the B fragment of phase 2: (V[2t4][g], V[2t4+1][g]) hi / lo
                unsigned vh, vl;
                split2(vn[0], vn[1], vh, vl);
                vh = movm_t(vh);
                vl = movm_t(vl);
                const unsigned aprv = sbase + (unsigned)b_p * SB + aoff;
#pragma unroll
                for (int s = 0; s < SPW; ++s) {
                    const unsigned ks = (unsigned)(s < ns ? s0 + s : s0) * 32u;
                    unsigned t0, t1, t2, t3;
                    ldsm_x4_t(aprv + ks, t0, t1, t2, t3);
                    float c2[4] = {0.f, 0.f, 0.f, 0.f};
                    mma1688(c2, t0, t1, vh);
                    mma1688(c2, t0, t1, vl);
                    mma1688(c2, t2, t3, vh);
#pragma unroll
                    for (int e = 0; e < 4; ++e) bt[s][e] += c2[e];
                }
                // slot of tile p consumed: the last warp out refills it with tile p + NS
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();
                    if (atomicAdd(&sh.rel[b_p], 1u) % MWARPS == MWARPS - 1) {
                        if (j - 1 + NS < nmine) {
                            fence_proxy_async();
                            issue(b_p, j - 1 + NS, fwd);
                        }
                    }
                }
            }
            rf_p[0] = rf[0];
            rf_p[1] = rf[1];
            vo_p[0] = vo[0];
            vo_p[1] = vo[1];
            nv_p = nv;
            r0_p = r0;
            b_p = b;
        }
        n0 += nmine;
        // ---- CTA partials: B (each warp owns its bins), H, <V_new, A>
        {
            float* Bo = A.Bpart + (int64_t)c * K * N16;
#pragma unroll
            for (int s = 0; s < SPW; ++s) {
                if (s < ns) {
                    const int lb = 16 * (s0 + s) + g;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int k = 2 * t4 + (e & 1), l = lb + 8 * (e >> 1);
                        if (k < K) Bo[(int64_t)k * N16 + l] = bt[s][e];
                    }
                }
            }
        }
        vdotA = warp_sum_d(vdotA);
#pragma unroll
        for (int o = 16; o; o >>= 1) bad |= __shfl_xor_sync(0xffffffffu, bad, o);
        if (lane == 0) {
            sh.vsw[warp] = vdotA;
            if (bad) atomicOr(&sh.bad, bad);
        }
#pragma unroll
        for (int x = 0; x < NHX; ++x) {
            const int tt = warp + MWARPS * (lane + 32 * x);
            if (tt < KK) A.Hpart[(int64_t)c * KK + tt] = hacc[x];
        }
        fence_proxy_async_global();  // this thread's V stores before the next pass's bulk copies
        __syncthreads();
        if (tid == 0) {
            double v = 0.0;
            for (int w = 0; w < MWARPS; ++w) v += sh.vsw[w];
            A.vpart[2 * (int64_t)c] = v;
            A.vpart[2 * (int64_t)c + 1] = 0.0;
            if (it + 1 < A.n_iter) issue_head(slot_b, !fwd);  // head tiles of the next pass (V rows final)
        }
        stamp(it, 1);
        grid_sync(A.bar, epoch);
        stamp(it, 2);
        // <V_new, A> for the objective (last CTA), read before the second barrier (after it,
        // CTAs already in the next pass overwrite their vpart)
        double va = 0.0;
        if (c == nC - 1) {
            double v0 = 0.0;
            for (int i = tid; i < nC; i += MTHREADS) v0 += __ldcg(A.vpart + 2 * i);
            va = block_sum_all(v0, sh.dred);
        }
        // ============================== D update ==================================
        {
            const int nB = K * nsl, nout = KK + nB;
            const int NQ = max(1, MTHREADS / nout);
            if (tid < NQ * nout) {
                const int o = tid % nout, q = tid / nout;
                double s = 0.0;
                if (o < KK) {
                    const double* src = A.Hpart + o;
                    s = batched_sum(q, NQ, nC, [&](int cc) { return __ldcg(src + (int64_t)cc * KK); });
                } else {
                    const int ob = o - KK, k = ob / nsl, l = l0s + (ob - (ob / nsl) * nsl);
                    const float* src = A.Bpart + (int64_t)k * N16 + l;
                    const int64_t stride = (int64_t)K * N16;
                    s = batched_sum(q, NQ, nC, [&](int cc) { return (double)__ldcg(src + (int64_t)cc * stride); });
                }
                sh.gacc[tid] = s;
            }
            __syncthreads();
            for (int o = tid; o < nout; o += MTHREADS) {
                double s = 0.0;
                for (int q = 0; q < NQ; ++q) s += sh.gacc[q * nout + o];
                if (o < KK) sh.Hs[o] = s;
                else sh.Bsl[o - KK] = s;
            }
            __syncthreads();
        }
        {
            double bd = 0.0;
            if (tid < nsl) {
                const int l = l0s + tid;
                unsigned dbad = 0;
                double d[K];
#pragma unroll
                for (int k = 0; k < K; ++k) d[k] = (double)__ldcg(A.D + (int64_t)k * A.Nk + l);
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    double hd = 0.0;
#pragma unroll
                    for (int jj = 0; jj < K; ++jj) hd = fma(sh.Hs[k * K + jj], d[jj], hd);
                    const double B = sh.Bsl[k * nsl + tid];
                    const float dn = (float)(d[k] * B / fmax(hd, 1e-30));
                    if (!isfinite(dn)) dbad |= ST_NUMERIC;
                    bd += B * (double)dn;
                    sh.dnew[k * 16 + tid] = (double)dn;
                }
                if (dbad) atomicOr(A.status, dbad);
            }
            __syncthreads();  // all reads of the old D slice done
            if (tid < nsl) {
#pragma unroll
                for (int k = 0; k < K; ++k) A.D[(int64_t)k * A.Nk + l0s + tid] = (float)sh.dnew[k * 16 + tid];
            }
            sh.gacc[tid] = bd;
            __syncthreads();
            if (tid == 0) {
                double s = 0.0;
                for (int u = 0; u < nsl; ++u) s += sh.gacc[u];
                A.dpart[c] = s;
            }
            for (int o = tid; o < KK; o += MTHREADS) {
                const int a = o / K, b2 = o - (o / K) * K;
                double s = 0.0;
                for (int u = 0; u < nsl; ++u) s = fma(sh.dnew[a * 16 + u], sh.dnew[b2 * 16 + u], s);
                A.Gpart[(int64_t)c * KK + o] = s;
            }
        }
        stamp(it, 3);
        grid_sync(A.bar, epoch);
        // ---- G_new (every CTA, same fixed order), D fragments restaged, objective
        {
            constexpr int NQ = MTHREADS / KK > 0 ? MTHREADS / KK : 1;
            double s = 0.0;
            if (tid < NQ * KK) {
                const int o = tid % KK, q = tid / KK;
                s = batched_sum(q, NQ, nC, [&](int cc) { return __ldcg(A.Gpart + (int64_t)cc * KK + o); });
            }
            load_dfrag();
            if (tid < NQ * KK) sh.gacc[tid] = s;
            __syncthreads();
            for (int o = tid; o < KK; o += MTHREADS) {
                double tq = 0.0;
                for (int q = 0; q < NQ; ++q) tq += sh.gacc[q * KK + o];
                sh.Gnew[o] = tq;
                sh.Gs[o] = (float)tq;
            }
            __syncthreads();
        }
        if (c == nC - 1) {
            double v1 = 0.0, v2 = 0.0;
            for (int i = tid; i < nC; i += MTHREADS) v2 += __ldcg(A.dpart + i);
            if (it == 0)
                for (int i = tid; i < A.nby; i += MTHREADS) v1 += __ldcg(A.ypart + i);
            const double ysq_new = block_sum_all(v1, sh.dred);
            const double bdot = block_sum_all(v2, sh.dred);
            if (tid == 0) {
                if (it == 0) {
                    ysq = ysq_new;
                    *A.ysq = ysq;
                    if (!(ysq > 0.0)) atomicOr(A.status, (unsigned)ST_Y_ALLZERO);
                }
                double hg_old = 0.0, hg_new = 0.0;
                for (int tt = 0; tt < KK; ++tt) {
                    hg_old += sh.Hs[tt] * sh.Gold[tt];
                    hg_new += sh.Hs[tt] * sh.Gnew[tt];
                }
                if (A.obj) {
                    A.obj[2 * it] = ysq - 2.0 * va + hg_old;
                    A.obj[2 * it + 1] = ysq - 2.0 * bdot + hg_new;
                }
            }
        }
        __syncthreads();  // the objective (thread 0) has read Gold; K*K > 32 spans several warps
        for (int o = tid; o < KK; o += MTHREADS) sh.Gold[o] = sh.Gnew[o];
        __syncthreads();
        stamp(it, 4);
    }
    if (c == 0)
        for (int o = tid; o < KK; o += MTHREADS) A.Gd[o] = sh.Gold[o];
    if (tid == 0 && sh.bad) atomicOr(A.status, sh.bad);
}

}  // namespace

// ------------------------------------------------------------------ host side
inline int mma_spw(int N16) { return ((N16 >> 4) + MWARPS - 1) / MWARPS; }
inline int mma_nslot(int N16, int K) {
    const int ns = (int)((200u * 1024u) / mma_slot_bytes(N16, K));
    return std::min(8, ns);
}

template <int K, int SPW>
inline cudaError_t mma_klb(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D, int n_iter,
                           double* obj, unsigned* bar, unsigned* status, cudaStream_t s) {
    static size_t attr = 0;
    if (attr < p.smem_m) {
        cudaError_t e = cudaFuncSetAttribute(k_nmf_mma<K, SPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)p.smem_m);
        if (e != cudaSuccess) return e;
        attr = p.smem_m;
    }
    MmaArgs A;
    A.Yh = reinterpret_cast<const __half*>(w.Yp);
    A.Np = (int64_t)g.Nv * g.Nr * g.Nc;
    A.Nk = g.Nk;
    A.N16 = p.N16;
    A.n_iter = n_iter;
    A.nslot = p.nslot;
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
    A.trace = w.trace;
    A.trace_iters = w.trace_iters;
    A.bar = bar;
    A.status = status;
    void* args[] = {&A};
    cudaError_t e = cudaMemsetAsync(bar, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    return cudaLaunchCooperativeKernel((const void*)k_nmf_mma<K, SPW>, dim3(p.nblk_f), dim3(MTHREADS), args,
                                       p.smem_m, s);
}

template <int K>
cudaError_t mma_launch_k(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D, int n_iter,
                         double* obj, unsigned* bar, unsigned* status, cudaStream_t s) {
    switch (p.spw) {
#define M(SP) \
    case SP: return mma_klb<K, SP>(g, p, w, V, D, n_iter, obj, bar, status, s);
        M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12)
#undef M
        default: return cudaErrorInvalidValue;
    }
}
#define HSNCT_MMA_EXTERN(KV)                                                                                   \
    extern template cudaError_t mma_launch_k<KV>(const Geometry&, const NmfPlan&, const NmfWs&, float*, float*, \
                                                 int, double*, unsigned*, unsigned*, cudaStream_t);
HSNCT_MMA_EXTERN(1) HSNCT_MMA_EXTERN(2) HSNCT_MMA_EXTERN(3) HSNCT_MMA_EXTERN(4)
HSNCT_MMA_EXTERN(5) HSNCT_MMA_EXTERN(6) HSNCT_MMA_EXTERN(7) HSNCT_MMA_EXTERN(8)

}  // namespace hsnct
