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
// the bins into four ranges (the bin range of cluster rank j is fixed for the kernel); every
// CTA streams its range of each tile into a ring of 128-bin chunk slots (64 rows x 128 bins),
// computes its partial A in TMEM, the four partials are summed in a fixed rank order (pushed
// to the peers with st.async; bitwise identical in all four CTAs), every CTA applies the same
// V update, and phase 2 runs on the tile's data.
//
// Why TMEM holds the tile for phase 2.  Keeping the chunks in shared memory until phase 2
// (round 2's first version) leaves room for two tiles, and the ~3 us between a tile's last
// chunk landing and its phase-2 MMAs completing (cluster exchange, V update, MMAs) drained the
// ring every tile (0.53 of HBM).  Here each chunk is stored in transposed
// core-matrix order (8 rows of one bin contiguous): phase 1 reads it as an MN-major operand,
// tcgen05.cp then copies it into TMEM with the bins on the 128 lanes -- exactly phase 2's A
// operand (Y+^T, M = 128 bins, K = rows) -- and the shared-memory slot is free again.  TMEM
// (512 columns) holds one tile's Y+^T (256) and the phase-1 / phase-2 accumulators (256).
//
// Precision (R20).  fp32-accurate products from an fp16 hi/lo split: x = hi + lo,
// hi = fp16(s x), lo = fp16(s x - hi), |x - (hi + lo)/s| <= 2^-22 |x| for the scaled values in
// the normal range, with power-of-two scales s chosen so that s*max < 2^14: one per call for Y+
// (k_tc_stats), one per component and CTA range for D (kernel prologue), one per component
// for V (the launch's Cauchy-Schwarz bound).  Each MMA uses [hi | lo] of the small operand as
// its N = 16 columns, and the large operand's hi and lo are two MMAs into the same accumulator,
// so all four partial products are summed.  Tensor-core accumulation truncates, which biases
// long sums; every accumulator therefore covers one chunk (phase 1) or one tile (phase 2), and
// the rest of the sums are fp32 FADD/FFMA in registers.
//
// Warps (256 threads, one CTA per SM): 0 producer (cp.async.bulk of each chunk), 1 phase-1 MMA
// issuer + tcgen05.cp, 2 and 3 phase-2 MMA issuers (even / odd bin blocks), 4-7 epilogue (TMEM
// drains, the A exchange, the V update, V in operand layout, B in fp32 registers, H = V^T V).
// The issuers are whole converged warps (elect.sync inside the asm) so that descriptor math
// stays warp-uniform: ~15-20 ns per MMA instead of ~60-80 from one divergent lane.
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
constexpr int CW = 128;                 // bins per chunk = phase-2 M = TMEM lanes
constexpr int MAXCH = 4;                // chunks per range (TMEM: 64 columns of Y+^T each)
constexpr int NB = 16;                  // chunks in flight (mbarrier pairs of the byte ring)
constexpr uint32_t COL_P1 = 256, COL_P2 = 384;  // TMEM: [0,256) Y+^T, P1 / P2 accumulators (2 parities)
constexpr int VOPB = 8 * 2 * 128;       // bytes of the V operand (8 row groups x 2 n groups)
constexpr int XRB = (NCL - 1) * TR * 8 * 4;  // bytes of the peers' partials of A (one tile)
constexpr int NTHR = 256;
constexpr int EPI0 = 128;               // first epilogue thread
constexpr uint32_t TMEM_COLS = 512;

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
    int R;                  // bytes of the chunk ring (chunks packed at their real size, FIFO)
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
    __shared__ uint64_t full[NB], empty[NB];
    __shared__ uint32_t choff[NB];      // byte offset in the ring of the chunk using barrier pair b
    __shared__ uint64_t ydone, yfree;   // tile's Y+^T copied into TMEM / phase 2 done reading it
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
    const uint32_t RB = (uint32_t)A.R;  // ring bytes
    const int DOPC = W * 32;            // one chunk of the D operand: W/8 bin groups x 2 n groups x 128 B
    uint8_t* ring = sm;
    uint8_t* Dop = sm + RB;             // (the tail chunk's TMEM copy may read past the ring into Dop)
    uint8_t* Vop = Dop + (size_t)A.maxch * DOPC;
    float* xrecv = reinterpret_cast<float*>(Vop + 2 * VOPB);  // [NCL-1][TR][8] partials of A from the peers
    const int64_t ntiles = (A.Np + TR - 1) / TR;
    const int64_t nmine = (int64_t)cid < ntiles ? (ntiles - 1 - cid) / ncl + 1 : 0;

    // ---------------------------------------------------------------- prologue
    if (tid == 0) {
        for (int s = 0; s < NB; ++s) {
            mb_init(&full[s], 1);
            mb_init(&empty[s], 1);
        }
        mb_init(&ydone, 1);
        mb_init(&yfree, 2);  // one commit per phase-2 issuer
        for (int b = 0; b < 2; ++b) {
            mb_init(&p1full[b], 1);
            mb_init(&p1empty[b], 4);
            mb_init(&vfull[b], 1);
            mb_init(&p2full[b], 2);   // one commit per phase-2 issuer
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
        // Byte ring: chunks (32 KB, and the range's short tail) are packed FIFO at their real
        // size, so the ring holds two whole tiles; a chunk is released (empty[b]) once its
        // phase-1 MMAs and its copy into TMEM have completed, in order.
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();  // streamed once per iteration
            uint32_t start[NB];                         // ring offset of the in-flight chunks
            uint32_t head = 0;
            int64_t seq = 0, oldest = 0;                // oldest chunk not yet known to be released
            auto release_oldest = [&]() {
                mb_wait(&empty[oldest % NB], (unsigned)((oldest / NB) & 1));
                ++oldest;
            };
            for (int64_t i = 0; i < nmine; ++i) {
                const int64_t t = cid + i * ncl;
                for (int c = 0; c < nch; ++c, ++seq) {
                    const uint32_t bytes = 2048u * (uint32_t)chunk_groups(L, c, W);
                    uint32_t at;
                    for (;;) {
                        if (seq - oldest >= NB) {
                            release_oldest();
                            continue;
                        }
                        if (oldest == seq) head = 0;  // ring empty: restart at its base
                        const uint32_t tail = oldest < seq ? start[oldest % NB] : head;
                        if (oldest == seq || head > tail) {  // free: [head, RB) and [0, tail)
                            if (head + bytes <= RB) { at = head; break; }
                            if (bytes <= tail) { at = 0; break; }
                        } else if (head + bytes <= tail) {   // free: [head, tail)
                            at = head;
                            break;
                        }
                        release_oldest();
                    }
                    start[seq % NB] = at;
                    head = at + bytes;
                    const int b = (int)(seq % NB);
                    if (c == 0) stamp(i, TS_LD_0);
                    if (c == nch - 1) stamp(i, TS_LD_END);
                    choff[b] = at;  // published to the consumers by the expect_tx arrive (release)
                    mb_expect_tx(&full[b], bytes);
                    bulk_g2s_hint(ring + at, A.Yc + chunk_off(t, A.Nk16, l0, c, W), bytes, &full[b], pol);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ phase-1 MMA issuer + copy to TMEM
        constexpr uint32_t ID1 = idesc_f16(64, NN, true);  // A = Y+ tile (64 rows), MN-major (rows contiguous)
        const uint32_t ring_a = __shfl_sync(0xffffffffu, smem_u32(ring), 0);
        const uint32_t dop_a = __shfl_sync(0xffffffffu, smem_u32(Dop), 0);
        const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
        for (int64_t i = 0; i < nmine; ++i) {
            const int p = (int)(i & 1);
            if (i >= 2) mb_wait(&p1empty[p], (unsigned)(((i - 2) >> 1) & 1));
            fence_after();
            for (int c = 0; c < nch; ++c) {
                const int64_t seq = i * nch + c;
                const int s = (int)(seq % NB);
                mb_wait(&full[s], (unsigned)((seq / NB) & 1));
                fence_after();
                if (c == 0 && lane == 0) stamp(i, TS_MMA_P1_0);
                const uint32_t w = (uint32_t)chunk_groups(L, c, W);
                const uint32_t a = ring_a + choff[s];
                const uint32_t d = tm + COL_P1 + (uint32_t)p * 64u + (uint32_t)c * NN;
                // MN-major A: LBO = bin-group stride (K), SBO = row-group stride (M); K-step = 2 bin groups
                const uint64_t ah = sdesc(a, 1024u, 128u), al = sdesc(a + 1024u * w, 1024u, 128u);
                const uint64_t bd = sdesc(dop_a + (uint32_t)c * DOPC, 256u, 128u);
                for (uint32_t ks = 0; ks < w / 2; ++ks) {
                    mma_f16_warp(d, ah + ks * 128u, bd + ks * 32u, ID1, ks > 0 ? 1u : 0u);
                    mma_f16_warp(d, al + ks * 128u, bd + ks * 32u, ID1, 1u);
                }
            }
            mma_commit_warp(&p1full[p]);
            if (lane == 0) stamp(i, TS_MMA_P1_END);
            // Y+^T of this tile into TMEM (after phase 2 of the previous tile has read its copy);
            // every chunk is a 128-bin block: 4 row blocks x (hi, lo) copies of 128 lanes x 256 bits
            if (i >= 1) mb_wait(&yfree, (unsigned)((i - 1) & 1));
            fence_after();
            for (int c = 0; c < nch; ++c) {
                const int64_t seq = i * nch + c;
                const int s = (int)(seq % NB);
                const uint32_t w = (uint32_t)chunk_groups(L, c, W);
                const uint32_t a = ring_a + choff[s];
#pragma unroll
                for (uint32_t hl = 0; hl < 2; ++hl)
#pragma unroll
                    for (uint32_t kb = 0; kb < TR / 16; ++kb)
                        tmem_cp_128x256b_warp(tm + (uint32_t)c * 64u + hl * 32u + kb * 8u,
                                              sdesc(a + hl * 1024u * w + kb * 256u, 128u, 1024u));
                mma_commit_warp(&empty[s]);  // the slot is free once its MMAs and copies completed
            }
            mma_commit_warp(&ydone);
        }
    } else if (warp == 2 || warp == 3) {
        // ------------------------------------------------------------ phase-2 MMA issuers (A = Y+^T in TMEM)
        constexpr uint32_t ID2 = idesc_f16(128, NN, false);  // A from TMEM: 128 bins x 16 rows per MMA
        const uint32_t vop_a = __shfl_sync(0xffffffffu, smem_u32(Vop), 0);
        const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
        const int c0 = warp - 2;  // bin blocks of this issuer: even / odd
        for (int64_t i = 0; i < nmine; ++i) {
            const int p = (int)(i & 1);
            mb_wait(&vfull[p], (unsigned)((i >> 1) & 1));
            mb_wait(&ydone, (unsigned)(i & 1));
            if (i >= 2) mb_wait(&p2empty[p], (unsigned)(((i - 2) >> 1) & 1));
            fence_after();
            if (lane == 0 && c0 == 0) stamp(i, TS_MMA_P2_0);
            const uint64_t vb = sdesc(vop_a + (uint32_t)p * VOPB, 256u, 128u);
            for (int c = c0; c < nch; c += 2) {
                const uint32_t d = tm + COL_P2 + (uint32_t)p * 64u + (uint32_t)c * NN;
#pragma unroll
                for (uint32_t ks = 0; ks < TR / 16; ++ks) {
                    mma_f16_tmem_warp(d, tm + (uint32_t)c * 64u + ks * 8u, vb + ks * 32u, ID2, ks > 0 ? 1u : 0u);
                    mma_f16_tmem_warp(d, tm + (uint32_t)c * 64u + 32u + ks * 8u, vb + ks * 32u, ID2, 1u);
                }
            }
            mma_commit_warp(&p2full[p]);
            mma_commit_warp(&yfree);
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
        float bacc[MAXCH][K];                // B partial: bin l0 + c CW + 32 q + lane (phase-2 M = 128 lanes)
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
                    tmem_ld32(toff + COL_P2 + (uint32_t)pp * 64u + (uint32_t)c0 * NN, v);
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
        // V_old prefetched two tiles ahead: under full HBM load a global read takes ~3 us, about
        // one tile period, so a one-tile prefetch left the V update waiting on it
        float vold[K], vnext[K];
        auto load_v = [&](int64_t i, float (&dst)[K]) {
            const int64_t grow = (cid + i * ncl) * TR + row;
            const bool valid = act && i < nmine && grow < A.Np;
#pragma unroll
            for (int k = 0; k < K; ++k) dst[k] = valid ? __ldcg(A.V + grow * K + k) : 0.f;
        };
        load_v(0, vold);
        load_v(1, vnext);
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
                    tmem_ld32(toff + COL_P1 + (uint32_t)p * 64u + (uint32_t)c0 * NN, v);
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
#pragma unroll
            for (int k = 0; k < K; ++k) vold[k] = vnext[k];
            load_v(i + 2, vnext);
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

// Pass 2: Y+ scaled by sigma_Y and split into fp16 hi/lo, per chunk in TRANSPOSED core-matrix
// order: [hi | lo][bin group lg][row group rg][8 bins][8 rows] (8 consecutive tile rows of one
// bin are 16 contiguous bytes).  Phase 1 reads a chunk as an MN-major operand (M = rows) and
// tcgen05.cp copies it into TMEM with the bins on the lanes (phase 2's A = Y+^T).
// Item (tile t, row group rg, global bin group G, bin l8), l8 fastest: a warp reads 32
// consecutive bins of each of 8 rows (coalesced) and writes 16 bytes per thread.
__global__ void __launch_bounds__(256) k_tc_convert(const float* __restrict__ Y, int64_t ld, int64_t Np, int Nk,
                                                    int Nk16, TcRanges rg, const unsigned* __restrict__ ymax,
                                                    __half* __restrict__ Yc) {
    const float sy = sigma_of(__uint_as_float(*ymax));
    const int G8 = Nk16 >> 3;
    const int64_t ntiles = (Np + TR - 1) / TR;
    const int64_t n = ntiles * 8 * G8 * 8;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int l8 = (int)(i & 7);
        int64_t u = i >> 3;
        const int G = (int)(u % G8);
        u /= G8;
        const int rgi = (int)(u & 7);
        const int64_t t = u >> 3;
        const int l = G * 8 + l8;
        const int64_t r0 = t * TR + rgi * 8;
        float v[8];
#pragma unroll
        for (int r8 = 0; r8 < 8; ++r8) v[r8] = (r0 + r8 < Np && l < Nk) ? __ldg(Y + (r0 + r8) * ld + l) : 0.f;
        // bin range j, chunk c, bin group within the chunk
        int j = 0;
#pragma unroll
        for (int jj = 1; jj < NCL; ++jj)
            if (l >= rg.l0[jj]) j = jj;
        const int loc = l - rg.l0[j];
        const int c = loc / rg.W, lg = (loc - c * rg.W) >> 3;
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
        __half* dst = Yc + chunk_off(t, Nk16, rg.l0[j], c, rg.W) + (int64_t)((lg * 8 + rgi) * 8 + l8) * 8;
        *reinterpret_cast<uint4*>(dst) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(dst + 512 * w) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}

size_t tc_smem_bytes(int ring_bytes, int W, int maxch) {
    return (size_t)ring_bytes + (size_t)maxch * W * 32 + 2 * VOPB + XRB;
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
    // 128-bin chunks: one chunk = one block of 128 TMEM lanes of Y+^T
    const size_t budget = (size_t)232448 - 3072;  // 227 KB minus the driver's 1 KB and <= 2 KB static
    const int bestW = CW;
    const int maxch0 = (Lmax + CW - 1) / CW;
    if (maxch0 > MAXCH) return false;
    // the rest of the shared memory is the byte ring (16-byte granular); it must hold a tile
    const int bestR = (int)((budget - tc_smem_bytes(0, bestW, maxch0)) & ~(size_t)15);
    if (bestR < maxch0 * TR * CW * 4) return false;
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
    p->tc_R = bestR;
    p->tc_R2 = 0;
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
