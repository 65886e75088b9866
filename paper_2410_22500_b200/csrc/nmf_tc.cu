// Subspace extraction, Eq. 4, Lee-Seung multiplicative updates (DESIGN.md
// R1-R3): the row pass of one iteration on the 5th-generation tensor cores (tcgen05, TMEM
// accumulators, operands staged by the TMA unit).  DESIGN.md §5.1b.
//
//   For each 64-row tile R of Y+:   A_R = Y+_R D^T                       (phase 1)
//                                   V_R <- V_R .* A_R ./ max(V_R G, 1e-30)  (G = D D^T)
//                                   B  += V_R^T Y+_R,  H += V_R^T V_R      (phase 2)
//   followed by k_dred (nmf.cu): D <- D .* B ./ max(H D, 1e-30), G for the next pass, the
//   objective terms.  Y+ is read from HBM ONCE per iteration.
//
// Why a cluster.  The V update needs all N_k bins of a row before phase 2 may use the new V,
// so a tile's rows must stay on chip between the two phases; UMMA needs >= 64 rows, and 64 rows
// x 1600 bins x 4 B = 410 KB exceeds one SM's shared memory.  A cluster of NCL = 4 CTAs splits
// the bins into four ranges (the lambda range of cluster rank j is fixed for the kernel); every
// CTA streams its range of each tile into a ring of 16 KB chunk slots (64 rows x 64 bins),
// computes its partial A in TMEM, the four partials are summed through distributed shared
// memory in a fixed rank order (bitwise identical in all four CTAs), every CTA applies the
// same V update, and phase 2 runs on its resident chunks.
//
// Precision (R20).  fp32-accurate products from an fp16 hi/lo split: x = hi + lo,
// hi = fp16(s x), lo = fp16(s x - hi), |x - (hi + lo)/s| <= 2^-22 |x| for the scaled values in
// the normal range, with power-of-two scales s chosen so that s*max < 2^14: one per call for Y+
// (k_tc_stats), one per component and CTA range for D (kernel prologue), one per component and
// tile for V (the tile's own max).  Each MMA uses [hi | lo] of the small operand as its N = 16
// columns, and the large operand's hi and lo are two MMAs into the same accumulator, so all
// four partial products are summed exactly in fp32.  Tensor-core accumulation truncates, which
// biases long sums; every accumulator therefore covers one 64-bin chunk (phase 1) or one tile
// (phase 2) only, and the rest of the sums are fp32 FADD/FFMA in registers.
//
// Warp roles (192 threads, one CTA per SM):
//   warp 0   producer: cp.async.bulk of each chunk (hi and lo blocks, contiguous) into the ring
//   warp 1   MMA issuer (one thread): phase 1 of tile i, phase 2 of tile i-1 as soon as its
//            V is ready or a ring slot it holds is needed; tcgen05.commit releases the slots
//   warps 2-5 epilogue: TMEM drains, the cluster exchange of A, the V update, V in its
//            operand layout, the phase-2 drain into fp32 register accumulators of B, H = V^T V
// Deterministic: static tile schedule, fixed-order sums, no floating-point atomics.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "internal.h"
#include "tc_ptx.cuh"

namespace hsnct {
namespace {

using namespace tc;

constexpr int TR = 64;                  // rows per tile (phase-1 UMMA M = 64)
constexpr int NCL = TC_CLUSTER;         // CTAs per cluster = bin ranges
constexpr int NN = 16;                  // UMMA N: [hi k = 0..7 | lo k = 0..7]
constexpr int MAXCH = 8;                // chunks per range
constexpr int MAXR = 16;                // ring slots (upper bound)
constexpr int VOPB = 8 * 2 * 128;       // bytes of the V operand (8 row groups x 2 n groups)
constexpr int XRB = (NCL - 1) * TR * 8 * 4;  // bytes of the peers' partials of A (one tile)
// Warps: 0 producer (one lane), 1 phase-1 MMA issuer, 2 and 3 phase-2 MMA issuers (even / odd
// chunks; whole converged warps, elect.sync inside the MMA asm: ~15-20 ns per MMA), 4-7
// epilogue (TMEM lane quarter = warp % 4).  Two warps per SM sub-partition leave 255 registers.
constexpr int NTHR = 256;
constexpr int EPI0 = 128;               // first epilogue thread
constexpr uint32_t TMEM_COLS = 512;     // [0, 256): phase-1 accumulators, [256, 512): phase 2

struct TcArgs {
    const __half* Yc;       // converted Y+: [tile][range][chunk][hi | lo][row group][bin group][8][8]
    int64_t Np;
    int Nk, Nk16, Nkp;
    float* V;
    const float* D;
    const double* Gd;
    float* Bpart;           // [ncl][K][Nkp]
    double* Hpart;          // [nCTA][K*K]
    double* vpart;          // [nCTA][2]
    const unsigned* ymax;   // bits of max Y+ (k_tc_stats)
    const unsigned* ynorm;  // bits of max_r ||Y+_r||^2 (k_tc_stats)
    unsigned* status;
    int first;
    int R;                  // ring slots (phase 1; shared with phase 2 when R2 == 0)
    int R2;                 // phase-2 ring slots: 0 = phase 2 reads the phase-1 ring (chunks stay
                            // resident through the V update); > 0 = phase 2 re-streams each tile's
                            // chunks (from L2) into its own ring
    int maxch;              // chunks of the longest range (D-operand buffer)
    TcRanges rg;
    uint64_t* trace;        // diagnostics: [tile][nCTA][TRACE_SLOTS] %globaltimer stamps, or null
    int trace_tiles;
};

// Trace slots of the tcgen05 pass (hsnct_debug_trace; scripts/trace_tc.py)
enum TcStamp {
    TS_EPI_START = 0,   // epilogue: iteration start
    TS_P1_SEEN = 1,     // epilogue: phase-1 accumulator complete
    TS_X_SEEN = 2,      // epilogue: the cluster's four partials of A received
    TS_V_READY = 3,     // epilogue: V operand written (vfull)
    TS_P2_DRAINED = 4,  // epilogue: phase 2 of the previous tile drained
    TS_MMA_P1_0 = 5,    // MMA: first chunk of phase 1 landed
    TS_MMA_P1_END = 6,  // MMA: phase 1 issued (commit)
    TS_MMA_P2_0 = 7,    // MMA: phase 2 start (V ready)
    TS_MMA_P2_END = 8,  // MMA: phase 2 issued
    TS_LD_0 = 9,        // producer: first chunk copy issued
    TS_LD_END = 10,     // producer: last chunk copy issued
    TS_V_DONE = 11,     // epilogue: V update computed (before the operand writes)
};

// power-of-two scale with s * m < 2^14 (so fp16 hi <= 2^14 and no overflow); 1 for m <= 0
__host__ __device__ inline float sigma_of(float m) {
    if (!(m > 0.f) || !isfinite(m)) return 1.f;
    int E;
    frexpf(m, &E);  // m = f 2^E, f in [0.5, 1)
    const int s = min(120, max(-120, 14 - E));
    return ldexpf(1.f, s);
}

__device__ __forceinline__ void split(float x, __half& hi, __half& lo) {
    hi = __float2half_rn(x);
    lo = __float2half_rn(x - __half2float(hi));
}

// Offset (in halves) of tile t, the range starting at bin l0, chunk c (chunks of W bins).
__device__ __forceinline__ int64_t chunk_off(int64_t t, int Nk16, int l0, int c, int W) {
    return t * (int64_t)TR * Nk16 * 2 + (int64_t)TR * l0 * 2 + (int64_t)c * TR * W * 2;
}
// bin groups (of 8) in chunk c of a range of L bins
__device__ __forceinline__ int chunk_groups(int L, int c, int W) { return min(W, L - c * W) >> 3; }

template <int K>
__global__ void __launch_bounds__(NTHR, 1) k_nmf_tc(TcArgs A) {
    static_assert(K >= 1 && K <= 8, "tcgen05 pass: K <= 8");
    constexpr int KK = K * K;
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[MAXR], empty[MAXR], full2[MAXR], empty2[MAXR];
    __shared__ volatile int p1seen;     // tiles whose phase-1 chunks have all landed (re-stream mode)
    __shared__ uint64_t p1full[2], p1empty[2], vfull[2], p2full[2], p2empty[2], xfull, xempty;
    __shared__ uint32_t tbase;
    __shared__ double Gs[KK];
    __shared__ float Gf[KK];
    __shared__ unsigned dmaxb[8];
    __shared__ float invsd[8];          // 1 / (sigma_Y sigma_D[k]) of this CTA's range
    __shared__ float sv[8];             // sigma_V[k] (launch constant, from the Cauchy-Schwarz bound)
    __shared__ float svinv[8];          // 1 / (sigma_Y sigma_V[k])
    __shared__ double red[4];
    auto stamp = [&](int64_t i, int slot) {
        if (A.trace && i < A.trace_tiles)
            A.trace[((int64_t)i * gridDim.x + blockIdx.x) * TRACE_SLOTS + slot] = globaltimer();
    };

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank();
    const uint32_t cid = cluster_id(), ncl = num_clusters();
    const int W = A.rg.W;
    const int l0 = A.rg.l0[rank], L = A.rg.L[rank], nch = A.rg.nch[rank];
    const int R = A.R, R2 = A.R2;
    const int SLOTB = TR * W * 4;       // one chunk: hi + lo halves
    const int DOPC = W * 32;            // one chunk of the D operand: W/8 bin groups x 2 n groups x 128 B
    uint8_t* ring = sm;
    uint8_t* ring2 = sm + (size_t)R * SLOTB;
    uint8_t* Dop = ring2 + (size_t)R2 * SLOTB;
    uint8_t* Vop = Dop + (size_t)A.maxch * DOPC;
    float* xrecv = reinterpret_cast<float*>(Vop + 2 * VOPB);  // [NCL-1][TR][8] partials of A from the peers
    const int64_t ntiles = (A.Np + TR - 1) / TR;
    const int64_t nmine = (int64_t)cid < ntiles ? (ntiles - 1 - cid) / ncl + 1 : 0;

    // ---------------------------------------------------------------- prologue
    if (tid == 0) {
        for (int s = 0; s < R; ++s) {
            mb_init(&full[s], 1);
            mb_init(&empty[s], 1);
        }
        for (int s = 0; s < R2; ++s) {
            mb_init(&full2[s], 1);
            mb_init(&empty2[s], 1);
        }
        p1seen = 0;
        for (int b = 0; b < 2; ++b) {
            mb_init(&p1full[b], 1);
            mb_init(&p1empty[b], 4);
            mb_init(&vfull[b], 1);
            mb_init(&p2full[b], R2 ? 1 : 2);   // one commit per phase-2 issuer
            mb_init(&p2empty[b], 4);
        }
        mb_init(&xfull, 1);          // armed by expect_tx; completed by the peers' st.async bytes
        mb_init(&xempty, NCL - 1);   // the peers have read what this CTA sent them
        mb_init_fence();
    }
    if (warp == 1) tmem_alloc(&tbase, TMEM_COLS);
    if (tid < 8) dmaxb[tid] = 0u;
    for (int i = tid; i < KK; i += NTHR) {
        Gs[i] = A.Gd[i];
        Gf[i] = (float)A.Gd[i];
    }
    __syncthreads();
    // this range's max of D per component -> sigma_D
    for (int i = tid; i < K * L; i += NTHR) {
        const int k = i / L, l = l0 + (i - k * L);
        if (l < A.Nk) atomicMax(&dmaxb[k], __float_as_uint(fmaxf(A.D[(int64_t)k * A.Nk + l], 0.f)));
    }
    __syncthreads();
    const float sy = sigma_of(__uint_as_float(*A.ymax));
    if (tid < 8) {
        invsd[tid] = 1.f / (sy * sigma_of(__uint_as_float(dmaxb[tid])));
        // V_new[r,k] <= A[r,k] / G[k,k] <= ||Y+_r|| / ||D_k|| (all terms >= 0; Cauchy-Schwarz),
        // with a factor 2 for rounding: a scale that keeps every V of this pass in fp16 range
        const double bound = tid < K ? 2.0 * sqrt((double)__uint_as_float(*A.ynorm) / Gs[tid * K + tid]) : 0.0;
        const float s = sigma_of((float)fmin(bound, 3.0e38));
        sv[tid] = s;
        svinv[tid] = 1.f / (sy * s);
    }
    // D operand (phase-1 B, K-major): chunk c, element (n, bin l) at
    // ((l/8)*2 + n/8)*64 + (n%8)*8 + l%8 halves; n < 8: hi of component n, n >= 8: lo
    {
        __half* dop = reinterpret_cast<__half*>(Dop);
        for (int i = tid; i < nch * W * 8; i += NTHR) {
            const int c = i / (W * 8), r2 = i - c * (W * 8);
            const int l = r2 >> 3, k = r2 & 7;
            const int lam = l0 + c * W + l;
            __half hi = __float2half_rn(0.f), lo = hi;
            if (k < K && c * W + l < L && lam < A.Nk)
                split(A.D[(int64_t)k * A.Nk + lam] * sigma_of(__uint_as_float(dmaxb[k])), hi, lo);
            __half* base = dop + (size_t)c * (DOPC / 2) + (size_t)(l >> 3) * 128 + (l & 7);
            base[(0 * 64) + k * 8] = hi;   // n = k       (n group 0)
            base[(1 * 64) + k * 8] = lo;   // n = 8 + k   (n group 1)
        }
    }
    fence_proxy_async();
    fence_before();
    __syncthreads();
    cluster_sync();  // every CTA's barriers are initialised before any remote arrive
    fence_after();
    const uint32_t tmem = tbase;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            // streamed once: evict first; re-streamed by phase 2 from L2: default (LRU) policy
            const uint64_t pol = R2 ? policy_evict_normal() : policy_evict_first();
            int64_t seq = 0;
            for (int64_t i = 0; i < nmine; ++i) {
                const int64_t t = cid + i * ncl;
                for (int c = 0; c < nch; ++c, ++seq) {
                    const int s = (int)(seq % R);
                    mb_wait(&empty[s], (unsigned)(((seq / R) & 1) ^ 1));
                    if (c == 0) stamp(i, TS_LD_0);
                    if (c == nch - 1) stamp(i, TS_LD_END);
                    const unsigned bytes = 2048u * (unsigned)chunk_groups(L, c, W);
                    mb_expect_tx(&full[s], bytes);
                    bulk_g2s_hint(ring + (size_t)s * SLOTB, A.Yc + chunk_off(t, A.Nk16, l0, c, W), bytes, &full[s], pol);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ phase-1 MMA issuer (whole warp)
        constexpr uint32_t ID1 = idesc_f16(64, NN, false);  // A = Y+ tile (64 rows), K-major over bins
        const uint32_t ring_a = __shfl_sync(0xffffffffu, smem_u32(ring), 0);
        const uint32_t dop_a = __shfl_sync(0xffffffffu, smem_u32(Dop), 0);
        const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
        int64_t seq = 0;
        for (int64_t i = 0; i < nmine; ++i) {
            const int p = (int)(i & 1);
            if (i >= 2) mb_wait(&p1empty[p], (unsigned)(((i - 2) >> 1) & 1));
            fence_after();
            for (int c = 0; c < nch; ++c, ++seq) {
                const int s = (int)(seq % R);
                mb_wait(&full[s], (unsigned)((seq / R) & 1));
                fence_after();
                if (c == 0 && lane == 0) stamp(i, TS_MMA_P1_0);
                const uint32_t w = (uint32_t)chunk_groups(L, c, W);
                const uint32_t a = ring_a + (uint32_t)s * SLOTB;
                const uint32_t d = tm + (uint32_t)p * 128u + (uint32_t)c * NN;
                const uint64_t ah = sdesc(a, 128u, w * 128u), al = sdesc(a + 1024u * w, 128u, w * 128u);
                const uint64_t bd = sdesc(dop_a + (uint32_t)c * DOPC, 256u, 128u);
                // descriptor start addresses advance in 16-byte units: +256 B (A), +512 B (B) per K-step
                for (uint32_t ks = 0; ks < w / 2; ++ks) {
                    mma_f16_warp(d, ah + ks * 16u, bd + ks * 32u, ID1, ks > 0 ? 1u : 0u);
                    mma_f16_warp(d, al + ks * 16u, bd + ks * 32u, ID1, 1u);
                }
                if (R2) mma_commit_warp(&empty[s]);  // phase 2 re-streams: free the slot now
            }
            if (R2 && lane == 0) p1seen = (int)(i + 1);  // every chunk of tile i has landed (is in L2)
            mma_commit_warp(&p1full[p]);
            if (lane == 0) stamp(i, TS_MMA_P1_END);
        }
    } else if (warp == 3 && R2) {
        // ------------------------------------------------------------ phase-2 re-stream producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();  // second and last read of these bytes
            int64_t seq = 0;
            for (int64_t i = 0; i < nmine; ++i) {
                while (p1seen <= (int)i) __nanosleep(64);
                const int64_t t = cid + i * ncl;
                for (int c = 0; c < nch; ++c, ++seq) {
                    const int s = (int)(seq % R2);
                    mb_wait(&empty2[s], (unsigned)(((seq / R2) & 1) ^ 1));
                    const unsigned bytes = 2048u * (unsigned)chunk_groups(L, c, W);
                    mb_expect_tx(&full2[s], bytes);
                    bulk_g2s_hint(ring2 + (size_t)s * SLOTB, A.Yc + chunk_off(t, A.Nk16, l0, c, W), bytes, &full2[s], pol);
                }
            }
        }
    } else if (warp == 2 || warp == 3) {
        // ------------------------------------------------------------ phase-2 MMA issuers (whole warps)
        constexpr uint32_t ID2 = idesc_f16(128, NN, true);  // A = Y+ tile^T (128 bins), MN-major
        const uint32_t ring_a = __shfl_sync(0xffffffffu, smem_u32(ring), 0);
        const uint32_t vop_a = __shfl_sync(0xffffffffu, smem_u32(Vop), 0);
        const uint32_t ring2_a = __shfl_sync(0xffffffffu, smem_u32(ring2), 0);
        const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
        const int c0 = warp - 2;           // chunk parity of this issuer (two issuers when resident)
        const int cstep = R2 ? 1 : 2;      // one issuer (warp 2) when phase 2 re-streams
        for (int64_t i = 0; i < nmine; ++i) {
            const int p = (int)(i & 1);
            mb_wait(&vfull[p], (unsigned)((i >> 1) & 1));
            if (i >= 2) mb_wait(&p2empty[p], (unsigned)(((i - 2) >> 1) & 1));
            fence_after();
            if (lane == 0 && c0 == 0) stamp(i, TS_MMA_P2_0);
            const uint64_t vb = sdesc(vop_a + (uint32_t)p * VOPB, 256u, 128u);
            for (int c = c0; c < nch; c += cstep) {
                const int64_t seq = i * nch + c;
                const int s = (int)(seq % (R2 ? R2 : R));
                if (R2) {
                    mb_wait(&full2[s], (unsigned)((seq / R2) & 1));
                    fence_after();
                }
                const uint32_t w = (uint32_t)chunk_groups(L, c, W);
                const uint32_t a = (R2 ? ring2_a : ring_a) + (uint32_t)s * SLOTB;
                const uint32_t d = tm + 256u + (uint32_t)p * 128u + (uint32_t)c * NN;
                const uint64_t ah = sdesc(a, w * 128u, 128u), al = sdesc(a + 1024u * w, w * 128u, 128u);
                const uint32_t kst = (2u * w * 128u) >> 4;  // K-step (16 rows = 2 row groups), 16-B units
#pragma unroll
                for (uint32_t ks = 0; ks < TR / 16; ++ks) {
                    mma_f16_warp(d, ah + ks * kst, vb + ks * 32u, ID2, ks > 0 ? 1u : 0u);
                    mma_f16_warp(d, al + ks * kst, vb + ks * 32u, ID2, 1u);
                }
                mma_commit_warp(R2 ? &empty2[s] : &empty[s]);  // the slot is free once these MMAs have read it
            }
            mma_commit_warp(&p2full[p]);
            if (lane == 0 && c0 == 0) stamp(i, TS_MMA_P2_END);
        }
    } else if (warp >= 4 && warp < 8) {
        // ------------------------------------------------------------ epilogue (warps 4-7)
        const int q = warp & 3;            // TMEM lane quarter
        const int e = tid - EPI0;
        const bool act = lane < 16;        // phase-1 (M = 64) rows 16q .. 16q+15 live in lanes 0..15
        const int row = 16 * q + lane;
        const uint32_t toff = tmem + ((uint32_t)(32 * q) << 16);
        constexpr int KT = K * (K + 1) / 2;  // upper triangle of H
        float bacc[MAXCH][K];                // B partial: bin l0 + c W + 32 q + lane (phase-2 M = 128 lanes)
#pragma unroll
        for (int c = 0; c < MAXCH; ++c)
#pragma unroll
            for (int k = 0; k < K; ++k) bacc[c][k] = 0.f;
        double hrow[KT];  // this thread's rows' share of H = V^T V (owner tiles), fp64
#pragma unroll
        for (int u = 0; u < KT; ++u) hrow[u] = 0.0;
        double vdot = 0.0;
        unsigned bad = 0;
        const uint32_t xr_a = smem_u32(xrecv);
        float svi[K], svs[K], isd[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            svi[k] = svinv[k];
            svs[k] = sv[k];
            isd[k] = invsd[k];
        }
        auto drain2 = [&](int64_t j) {
            const int pp = (int)(j & 1);
            mb_wait(&p2full[pp], (unsigned)((j >> 1) & 1));
            fence_after();
#pragma unroll
            for (int c0 = 0; c0 < MAXCH; c0 += 2) {
                if (c0 < nch) {
                    float v[32];
                    tmem_ld32(toff + 256u + (uint32_t)pp * 128u + (uint32_t)c0 * NN, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int u = 0; u < 2; ++u)
                        if (c0 + u < nch) {
#pragma unroll
                            for (int k = 0; k < K; ++k)
                                bacc[c0 + u][k] = fmaf(v[16 * u + k] + v[16 * u + 8 + k], svi[k], bacc[c0 + u][k]);
                        }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mb_arrive(&p2empty[pp]);
        };
        // V_old of the next tile, prefetched one tile ahead (its latency is off the chain)
        float vold[K];
        auto load_vold = [&](int64_t i) {
            const int64_t grow = (cid + i * ncl) * TR + row;
            const bool valid = act && i < nmine && grow < A.Np;
#pragma unroll
            for (int k = 0; k < K; ++k) vold[k] = valid ? __ldcg(A.V + grow * K + k) : 0.f;
        };
        load_vold(0);
        for (int64_t i = 0; i < nmine; ++i) {
            const int p = (int)(i & 1);
            const int64_t t = cid + i * ncl;
            const int64_t grow = t * TR + row;
            const bool valid = act && grow < A.Np;
            // arm the receive barrier for this tile's three peer partials (its previous phase,
            // tile i-1, completed when that tile was received)
            if (e == 0) {
                stamp(i, TS_EPI_START);
                mb_expect_tx(&xfull, (unsigned)XRB);
            }
            // ---- phase-1 drain: partial A of this CTA's bin range, chunks summed in order
            mb_wait(&p1full[p], (unsigned)((i >> 1) & 1));
            fence_after();
            if (e == 0) stamp(i, TS_P1_SEEN);
            float a[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = 0.f;
#pragma unroll
            for (int c0 = 0; c0 < MAXCH; c0 += 2) {
                if (c0 < nch) {
                    float v[32];
                    tmem_ld32(toff + (uint32_t)p * 128u + (uint32_t)c0 * NN, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int u = 0; u < 2; ++u)
                        if (c0 + u < nch) {
#pragma unroll
                            for (int k = 0; k < K; ++k) a[k] += v[u * 16 + k] + v[u * 16 + 8 + k];
                        }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mb_arrive(&p1empty[p]);
#pragma unroll
            for (int k = 0; k < K; ++k) a[k] *= isd[k];
            // ---- push the partial to the three peers (st.async, tx-counted on their xfull),
            //      once they have read what this CTA sent them for the previous tile
            if (i >= 1) mb_wait(&xempty, (unsigned)((i - 1) & 1));
            if (act) {
                const float4 a0 = make_float4(a[0], a[1], a[2], a[3]), a1 = make_float4(a[4], a[5], a[6], a[7]);
#pragma unroll
                for (int dr = 1; dr < NCL; ++dr) {
                    const uint32_t r = (rank + (uint32_t)dr) % NCL;     // destination
                    const int j = NCL - 1 - dr;                          // its slot for this source
                    const uint32_t off = xr_a + (uint32_t)(((j * TR) + row) * 8 * sizeof(float));
                    const uint32_t bar = mapa(smem_u32(&xfull), r);
                    st_async4(mapa(off, r), a0, bar);
                    st_async4(mapa(off + 16u, r), a1, bar);
                }
            }
            mb_wait(&xfull, (unsigned)(i & 1));
            if (e == 0) stamp(i, TS_X_SEEN);
            // ---- A summed over the cluster in rank order 0..NCL-1 (identical in every CTA),
            //      then the V update (fp32; G = D D^T of the D this pass uses)
            float vn[K];
#pragma unroll
            for (int k = 0; k < K; ++k) vn[k] = 0.f;
            float As[8];
            if (act) {
#pragma unroll
                for (int k = 0; k < 8; ++k) As[k] = 0.f;
#pragma unroll
                for (int src = 0; src < NCL; ++src) {
                    float4 u0, u1;
                    if (src == (int)rank) {
                        u0 = make_float4(a[0], a[1], a[2], a[3]);
                        u1 = make_float4(a[4], a[5], a[6], a[7]);
                    } else {
                        const int j = (src - (int)rank - 1 + NCL) % NCL;
                        const float4* xp = reinterpret_cast<const float4*>(xrecv + ((size_t)j * TR + row) * 8);
                        u0 = xp[0];
                        u1 = xp[1];
                    }
                    As[0] += u0.x; As[1] += u0.y; As[2] += u0.z; As[3] += u0.w;
                    As[4] += u1.x; As[5] += u1.y; As[6] += u1.z; As[7] += u1.w;
                }
                if (valid) {
#pragma unroll
                    for (int k = 0; k < K; ++k)
                        if (A.first && !(isfinite(vold[k]) && vold[k] >= 0.f)) bad |= ST_INIT_BAD;
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        float vg = 0.f;
#pragma unroll
                        for (int j2 = 0; j2 < K; ++j2) vg = fmaf(vold[j2], Gf[j2 * K + k], vg);
                        vn[k] = vold[k] * As[k] * __frcp_rn(fmaxf(vg, 1e-30f));
                        if (!isfinite(vn[k])) bad |= ST_NUMERIC;
                    }
                }
                if (e == 0) stamp(i, TS_V_DONE);
                // V operand (phase-2 B, K-major over rows): element (n, row r) at
                // ((r/8)*2 + n/8)*64 + (n%8)*8 + r%8 halves; scaled by the launch's sigma_V
                __half* vop = reinterpret_cast<__half*>(Vop + (size_t)p * VOPB) + (size_t)(row >> 3) * 128 + (row & 7);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    __half hi = __float2half_rn(0.f), lo = hi;
                    if (k < K) split(vn[k] * svs[k], hi, lo);
                    vop[k * 8] = hi;
                    vop[64 + k * 8] = lo;
                }
            }
            load_vold(i + 1);
            fence_proxy_async();
            named_bar(1, 128);
            if (e == 0) {
                mb_arrive(&vfull[p]);
                stamp(i, TS_V_READY);
                // every row thread has read the peers' partials: tell the senders (pure signal)
                for (int dr = 1; dr < NCL; ++dr) mb_arrive_remote_relaxed(mapa(smem_u32(&xempty), (rank + (uint32_t)dr) % NCL));
            }
            // the owner CTA of the tile stores V and accumulates <V_new, A> and H (fp64, per row)
            if ((int)(i % NCL) == (int)rank && valid) {
                int u = 0;
#pragma unroll
                for (int ka = 0; ka < K; ++ka) {
                    A.V[grow * K + ka] = vn[ka];
                    vdot += (double)vn[ka] * (double)As[ka];
#pragma unroll
                    for (int kb = ka; kb < K; ++kb, ++u) hrow[u] = fma((double)vn[ka], (double)vn[kb], hrow[u]);
                }
            }
            // ---- phase-2 drain of the previous tile
            if (i >= 1) {
                drain2(i - 1);
                if (e == 0) stamp(i - 1, TS_P2_DRAINED);
            }
        }
        if (nmine >= 1) drain2(nmine - 1);
        // ---- outputs: this CTA's bin range of the cluster's B partial, H and <V, A> partials
#pragma unroll
        for (int c = 0; c < MAXCH; ++c) {
            const int lam = c * W + 32 * q + lane;
            if (c < nch && 32 * q + lane < chunk_groups(L, c, W) * 8 && l0 + lam < A.Nk) {
#pragma unroll
                for (int k = 0; k < K; ++k) A.Bpart[((int64_t)cid * K + k) * A.Nkp + l0 + lam] = bacc[c][k];
            }
        }
        // H: the 64 row threads' fp64 partials summed in a fixed order (scratch: the idle ring;
        // every MMA has completed -- the last drain waited for the last commit)
        double* hs = reinterpret_cast<double*>(ring);
        if (act) {
#pragma unroll
            for (int u = 0; u < KT; ++u) hs[(size_t)row * KT + u] = hrow[u];
        }
        // <V_new, A> partial: fixed-order warp then block sum
#pragma unroll
        for (int o = 16; o; o >>= 1) vdot += __shfl_xor_sync(0xffffffffu, vdot, o);
        if (lane == 0) red[q] = vdot;
        bad = __reduce_or_sync(0xffffffffu, bad);
        if (lane == 0 && bad) atomicOr(A.status, bad);
        named_bar(1, 128);
        if (e < KK) {
            const int ha = e / K, hb = e - (e / K) * K;
            const int lo_ = min(ha, hb), hi_ = max(ha, hb);
            const int u = lo_ * K - lo_ * (lo_ - 1) / 2 + (hi_ - lo_);
            double s = 0.0;
            for (int r = 0; r < TR; ++r) s += hs[(size_t)r * KT + u];
            A.Hpart[(int64_t)blockIdx.x * KK + e] = s;
        }
        if (e == 0) {
            A.vpart[2 * (int64_t)blockIdx.x] = (red[0] + red[1]) + (red[2] + red[3]);
            A.vpart[2 * (int64_t)blockIdx.x + 1] = 0.0;
        }
    }
    // ---------------------------------------------------------------- teardown
    fence_before();
    __syncthreads();
    cluster_sync();  // no CTA leaves while a peer may still write into it or arrive on its barriers
    fence_after();
    if (warp == 1) tmem_dealloc(tmem, TMEM_COLS);
}

// ------------------------------------------------------------ input preparation
// Pass 1: max(Y+) and max_r ||Y+_r||^2 (as float bits; order-independent, so deterministic),
// ||Y+||^2 partials per block (fixed order), non-finite check.  One warp per row.
__global__ void __launch_bounds__(256) k_tc_stats(const float* __restrict__ Y, int64_t ld, int64_t Np, int Nk,
                                                  unsigned* __restrict__ ymax, unsigned* __restrict__ ynorm,
                                                  double* __restrict__ ypart, unsigned* __restrict__ status,
                                                  unsigned long long* __restrict__ nclamp) {
    __shared__ double red[8];
    __shared__ unsigned mred[8], nred[8], cred[8];
    unsigned ncl = 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nq = (Nk + 3) >> 2;
    double s = 0.0;
    unsigned m = 0, nm = 0, bad = 0;
    for (int64_t r = (int64_t)blockIdx.x * 8 + w; r < Np; r += (int64_t)gridDim.x * 8) {
        const float* y = Y + r * ld;
        float ps = 0.f;
        for (int q = lane; q < nq; q += 32) {
            const int l = 4 * q;
            float v[4];
            if (l + 4 <= Nk) {
                const float4 u = __ldg(reinterpret_cast<const float4*>(y + l));
                v[0] = u.x; v[1] = u.y; v[2] = u.z; v[3] = u.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) v[j] = l + j < Nk ? y[l + j] : 0.f;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (!isfinite(v[j])) bad = ST_Y_NONFINITE;
                ncl += v[j] < 0.f;
                const float yp = fmaxf(v[j], 0.f);
                m = max(m, __float_as_uint(yp));
                ps = fmaf(yp, yp, ps);
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
        nm = max(nm, __float_as_uint(ps));
        s += (double)ps;
    }
    m = __reduce_max_sync(0xffffffffu, m);
    bad = __reduce_or_sync(0xffffffffu, bad);
    ncl = __reduce_add_sync(0xffffffffu, ncl);
    if (lane == 0) {
        red[w] = s;
        mred[w] = m;
        nred[w] = nm;
        cred[w] = ncl;
        if (bad) atomicOr(status, bad);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        unsigned mm = 0, nn = 0;
        unsigned long long c = 0;
        for (int j = 0; j < 8; ++j) {
            t += red[j];
            mm = max(mm, mred[j]);
            nn = max(nn, nred[j]);
            c += cred[j];
        }
        ypart[blockIdx.x] = t;
        if (c) atomicAdd(nclamp, c);
        if (mm) atomicMax(ymax, mm);
        if (nn) atomicMax(ynorm, nn);
    }
}

// Pass 2: Y+ scaled by sigma_Y and split into fp16 hi/lo in the chunked UMMA core-matrix layout.
// Item (tile t, row group rg, bin group g, row rr), rr fastest: 8 consecutive threads write one
// 128-byte core matrix row block (coalesced), each reading 8 bins of its row.
__global__ void __launch_bounds__(256) k_tc_convert(const float* __restrict__ Y, int64_t ld, int64_t Np, int Nk,
                                                    int Nk16, TcRanges rg, const unsigned* __restrict__ ymax,
                                                    __half* __restrict__ Yc) {
    const float sy = sigma_of(__uint_as_float(*ymax));
    const int G8 = Nk16 >> 3;
    const int64_t ntiles = (Np + TR - 1) / TR;
    const int64_t n = ntiles * 8 * G8 * 8;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int rr = (int)(i & 7);
        int64_t u = i >> 3;
        const int g = (int)(u % G8);
        u /= G8;
        const int rgi = (int)(u & 7);
        const int64_t t = u >> 3;
        const int64_t r = t * TR + rgi * 8 + rr;
        const int l = g * 8;
        float v[8];
        if (r < Np && l + 8 <= Nk) {
            const float4* y = reinterpret_cast<const float4*>(Y + r * ld + l);
            const float4 a = __ldg(y), b = __ldg(y + 1);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = (r < Np && l + j < Nk) ? Y[r * ld + l + j] : 0.f;
        }
        // bin range j, chunk c, bin group within the chunk
        int j = 0;
#pragma unroll
        for (int jj = 1; jj < NCL; ++jj)
            if (l >= rg.l0[jj]) j = jj;
        const int loc = l - rg.l0[j];
        const int c = loc / rg.W, lb = (loc - c * rg.W) >> 3;
        const int w = chunk_groups(rg.L[j], c, rg.W);
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            __half h0, l0_, h1, l1;
            split(fmaxf(v[2 * q], 0.f) * sy, h0, l0_);
            split(fmaxf(v[2 * q + 1], 0.f) * sy, h1, l1);
            hw[q] = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
            lw[q] = (uint32_t)__half_as_ushort(l0_) | ((uint32_t)__half_as_ushort(l1) << 16);
        }
        __half* dst = Yc + chunk_off(t, Nk16, rg.l0[j], c, rg.W) + (int64_t)((rgi * w + lb) * 8 + rr) * 8;
        *reinterpret_cast<uint4*>(dst) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(dst + 512 * w) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}

size_t tc_smem_bytes(int R, int W, int maxch) {  // R: all ring slots (phase 1 + phase 2)
    return (size_t)R * TR * W * 4 + (size_t)maxch * W * 32 + 2 * VOPB + XRB;
}

template <int K>
cudaError_t tc_launch_k(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D, int it,
                        unsigned* status, cudaStream_t s) {
    static SmemAttr attr;
    cudaError_t e = ensure_smem((const void*)k_nmf_tc<K>, (int)p.tc_smem, attr);
    if (e != cudaSuccess) return e;
    TcArgs A;
    A.Yc = reinterpret_cast<const __half*>(w.Yc);
    A.Np = (int64_t)g.Nv * g.Nr * g.Nc;
    A.Nk = g.Nk;
    A.Nk16 = p.tc_Nk16;
    A.Nkp = p.Nkp;
    A.V = V;
    A.D = D;
    A.Gd = w.Gd;
    A.Bpart = w.Bpart;
    A.Hpart = w.Hpart;
    A.vpart = w.vpart;
    A.ymax = w.ymax;
    A.ynorm = w.ymax + 1;
    A.status = status;
    A.first = it == 0 ? 1 : 0;
    A.R = p.tc_R;
    A.R2 = p.tc_R2;
    A.maxch = p.tc_maxch;
    A.rg = p.tc_rg;
    A.trace = w.trace;
    A.trace_tiles = w.trace ? w.trace_iters : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(NCL * p.tc_ncl, 1, 1);
    cfg.blockDim = dim3(NTHR, 1, 1);
    cfg.dynamicSmemBytes = p.tc_smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = NCL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_nmf_tc<K>, A);
}

template <int K>
int tc_max_clusters(size_t smem) {
    static SmemAttr attr;
    if (ensure_smem((const void*)k_nmf_tc<K>, (int)smem, attr) != cudaSuccess) return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(NCL * 64, 1, 1);
    cfg.blockDim = dim3(NTHR, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = NCL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, k_nmf_tc<K>, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    return n;
}

#define HSNCT_TC_K(M) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8)

}  // namespace

bool nmf_tc_plan(const Geometry& g, int num_sms, NmfPlan* p) {
    (void)num_sms;
    if (g.K > 8) return false;
    const int Nk16 = (g.Nk + 15) & ~15;
    const int n16 = Nk16 / 16;
    if (n16 < NCL) return false;  // every CTA needs a non-empty bin range
    TcRanges rg{};
    int acc = 0, Lmax = 0;
    for (int j = 0; j < NCL; ++j) {
        const int cnt = n16 / NCL + (j < n16 % NCL ? 1 : 0);
        rg.l0[j] = 16 * acc;
        rg.L[j] = 16 * cnt;
        acc += cnt;
        Lmax = std::max(Lmax, rg.L[j]);
    }
    // chunk width: the one whose ring holds the most whole tiles of the longest range (the
    // ring must hold one tile while the next streams in)
    // 227 KB per block minus the driver's 1 KB and at most 2 KB of static shared memory
    const size_t budget = (size_t)232448 - 3072;
    int bestW = 0, bestR = 0;
    double best = 0.0;
    for (int W = 64; W <= 128; W += 16) {
        const int nch = (Lmax + W - 1) / W;
        if (nch > MAXCH) continue;
        int R = MAXR;
        while (R > 0 && tc_smem_bytes(R, W, nch) > budget) --R;
        if (R < nch + 1) continue;
        const double depth = (double)R / nch;
        if (depth > best + 1e-9) {
            best = depth;
            bestW = W;
            bestR = R;
        }
    }
    if (!bestW) return false;
    rg.W = bestW;
    int maxch = 0;
    for (int j = 0; j < NCL; ++j) {
        rg.nch[j] = (rg.L[j] + bestW - 1) / bestW;
        maxch = std::max(maxch, rg.nch[j]);
    }
    const size_t smem = tc_smem_bytes(bestR, bestW, maxch);
    int ncl = 0;
    switch (g.K) {
#define M(KV) \
    case KV: ncl = tc_max_clusters<KV>(smem); break;
        HSNCT_TC_K(M)
#undef M
        default: return false;
    }
    if (ncl < 1) return false;
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    const int64_t ntiles = (Np + TR - 1) / TR;
    p->tc_ncl = (int)std::max<int64_t>(1, std::min<int64_t>(ncl, ntiles));
    // Default: each tile's chunks stay resident in one ring through the V update.
    // HSNCT_TC_RESTREAM=1: phase 2 re-streams them from L2 into a second ring (the phase-1 ring
    // takes half the slots rounded up); measured slower (L2 latency doubles under the 2x L2
    // traffic)
    const char* rs = getenv("HSNCT_TC_RESTREAM");
    const bool restream = rs && rs[0] == '1' && bestR - (bestR + 1) / 2 >= maxch;
    p->tc_R = restream ? (bestR + 1) / 2 : bestR;
    p->tc_R2 = restream ? bestR - p->tc_R : 0;
    p->tc_maxch = maxch;
    p->tc_smem = smem;
    p->tc_rg = rg;
    p->tc_Nk16 = Nk16;
    p->tc_Npad = ntiles * TR;
    return true;
}

cudaError_t nmf_tc_prepare(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y, int64_t ld_y,
                           unsigned* status, cudaStream_t s) {
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    cudaError_t e = cudaMemsetAsync(w.ymax, 0, 2 * sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    k_tc_stats<<<p.nby, 256, 0, s>>>(Y, ld_y, Np, g.Nk, w.ymax, w.ymax + 1, w.ypart, status, w.nclamp);
    k_tc_convert<<<g.num_sms * 16, 256, 0, s>>>(Y, ld_y, Np, g.Nk, p.tc_Nk16, p.tc_rg, w.ymax,
                                                  reinterpret_cast<__half*>(w.Yc));
    return cudaGetLastError();
}

cudaError_t nmf_tc_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D, int it,
                          unsigned* status, cudaStream_t s) {
    switch (g.K) {
#define M(KV) \
    case KV: return tc_launch_k<KV>(g, p, w, V, D, it, status, s);
        HSNCT_TC_K(M)
#undef M
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace hsnct
