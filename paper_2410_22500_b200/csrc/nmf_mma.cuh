// Subspace extraction, Eq. 4, Lee-Seung multiplicative updates (DESIGN.md
// R1-R3): the row pass of one iteration on the tensor cores through warp-level mma.sync
// (m16n8k16, fp16 operands, fp32 accumulators).  DESIGN.md §5.1c.
//
//   For each 16-row tile R of Y+:   A_R = Y+_R D^T                           (phase 1)
//                                   V_R <- V_R .* A_R ./ max(V_R G, 1e-30)   (G = D D^T)
//                                   B  += V_R^T Y+_R,  H += V_R^T V_R        (phase 2)
//   followed by k_dred (nmf.cu): the D update, G for the next pass, the objective terms.
//
// Why mma.sync and not tcgen05 here.  The V update is row-local and needs all N_k bins of a
// row before phase 2 may use the new V, so a tile must stay on chip through a dependency
// chain (phase 1 -> cross-warp sum -> V update -> phase 2).  UMMA needs >= 64-row tiles, which
// do not fit one SM at N_k = 1600 (DESIGN.md §5.1b measured the 4-CTA-cluster version at 0.53
// of HBM).  m16n8k16 works on 16-row tiles: 16 x 1600 x 4 B = 100 KB, so the tile is split over
// the CTA's 8 warps by bin range, each warp streams its own 13 KB chunk of every tile into a
// private two-slot ring (cp.async.bulk, one mbarrier per slot, refilled by the warp itself),
// the warp's D operand and its columns of B^T stay in registers for the whole pass, and the
// chain per tile is short (two MMA sweeps of 13 blocks and a 256-thread barrier).  The pass
// issues ~0.05 warp instructions per Y+ element against ~0.46 for the FFMA kernel (§5.1).
//
// Y+ layout (prepared once per call by k_mma_convert): per tile t and 16-bin block j one
// contiguous 1 KB block [hi 512 B | lo 512 B], each half the four 8x8 core matrices in
// ldmatrix.x4 order (rows 0-7 bins 0-7, rows 8-15 bins 0-7, rows 0-7 bins 8-15, rows 8-15
// bins 8-15), rows of 16 B.  ldmatrix.x4 reads a block as the phase-1 A operand (row-major,
// M = rows, K = bins) and ldmatrix.x4.trans as the phase-2 A operand (Y+^T: M = bins, K =
// rows); both conflict-free (32 lanes x 16 contiguous bytes).
//
// Precision (R20): the same fp16 hi/lo split as the tcgen05 pass: x = (hi + lo)/s,
// |error| <= 2^-22 |x| in the normal range, power-of-two scales s with s max < 2^14 -- one per
// 16-row tile for Y+ (k_mma_prep), one per component and warp (bin range) for D, one per
// component and tile for V.  Three MMAs per block (hi.hi + hi.lo + lo.hi; lo.lo is below 2^-22);
// a column block with <= 4 components (K <= 4; the second block at K = 9..12) is packed as
// interleaved hi/lo columns and takes two (PK below).  Phase-1
// accumulators run over one warp's 13 blocks; phase-2 accumulators cover one block of one tile
// and are added to the fp32 register sums with their scale (FFMA), so no tensor-core sum is
// longer than 39 MMAs.  Cross-warp and cross-CTA sums are fp32 / fp64 in a fixed order:
// deterministic.
#pragma once
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "internal.h"
#include "nmf_common.cuh"

namespace hsnct {
namespace {

constexpr int MR = 16;          // rows per tile (the MMA's M in phase 1, its K in phase 2)
constexpr int MW = 8;           // warps per CTA = bin ranges of a tile
constexpr int MTH = MW * 32;
constexpr int MNS = 2;          // ring slots per warp
constexpr int MNV = 4;          // ring slots of the old-V rows (issued MNV - 1 tiles ahead)
constexpr int BLK = 1024;       // bytes of one 16 x 16 block (hi + lo)

struct MmaArgs {
    const uint8_t* Yc;    // [ntiles][NB][BLK]
    int64_t Np;
    int Nk, Nkp, NB;      // NB = ceil(Nk / 16) blocks per tile
    float* V;
    float* D;             // read (and, PERSIST, updated in place)
    double* Gd;           // G(D) in; PERSIST: G(D_n) out
    float* Bpart;         // [nCTA][K][Nkp]
    double* Hpart;        // [nCTA][K*K]
    double* vpart;        // [nCTA][2]
    const int* texp;      // [ntiles] exponent of each tile's Y+ scale sigma_Y = 2^texp (k_mma_prep)
    unsigned* status;
    int it;               // iteration index (one pass per launch)
    // persistent launch: all n_iter iterations with the D update between passes
    int n_iter;
    double* dpart;        // [nCTA] <B, D_new> slice partials
    double* Gpart;        // [nCTA][K*K] slice partials of D_new D_new^T
    const double* ypart;  // [nby] ||Y+||^2 partials
    int nby;
    double* ysq;
    double* obj;          // [2 n_iter] or null
    unsigned* bar;        // grid-barrier arrival counter, zero at launch
};

// exponent e of the power-of-two scale 2^e with 2^e m < 2^14 (fp16 hi <= 2^14, no overflow):
// m = f 2^E, f in [0.5, 1) -> e = 14 - E, clamped to [-120, 120]; 0 for m <= 0 or non-finite.
// (Bit arithmetic; subnormal m gives E <= -126, i.e. the clamp.)
__device__ __forceinline__ int mexp(float m) {
    if (!(m > 0.f) || !isfinite(m)) return 0;
    const int be = (int)(__float_as_uint(m) >> 23);
    if (be == 0) return 120;
    return min(120, max(-120, 14 - (be - 126)));
}
__device__ __forceinline__ float pow2(int e) { return __int_as_float((127 + e) << 23); }  // |e| <= 126

// {x0, x1} -> fp16 hi pair (return) and lo pair (lo); x0 in the low half
__device__ __forceinline__ uint32_t split2(float x0, float x1, uint32_t& lo) {
    const __half h0 = __float2half_rn(x0), h1 = __float2half_rn(x1);
    const __half l0 = __float2half_rn(x0 - __half2float(h0)), l1 = __float2half_rn(x1 - __half2float(h1));
    lo = (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
    return (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void ldsm4(uint32_t (&r)[4], unsigned addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm4t(uint32_t (&r)[4], unsigned addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
// d += a b  (m16n8k16, row.col, f16 x f16 -> f32)
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Column blocks of 8 components: NC = 1 (K <= 8) or 2 (K = 9..16)
__host__ __device__ constexpr int mma_nc(int K) { return (K + 7) / 8; }
// Warps per CTA (= bin ranges of a tile): 8, or 16 (MW16: two column blocks with half the blocks
// per warp, so that the per-warp state fits 128 registers and four warps share a scheduler)
constexpr int MW16 = 16;
// Partial-A buffers: two (a warp may write tile m + 1's partials while others still read tile
// m's), one with 16 warps (the V update's second barrier already orders them; shared memory)
__host__ __device__ constexpr int mma_nrb(int mw) { return mw == MW16 ? 1 : 2; }
// Dynamic shared memory: ring [mw][MNS][NBW*BLK] | old V rows [MNV][MR*K] | partial A
// [nrb][mw][NC][32 reader lanes][4]
__host__ __device__ constexpr size_t mma_vrows_off(int NBW, int mw = MW) { return (size_t)mw * MNS * NBW * BLK; }
__host__ __device__ constexpr size_t mma_red_off(int NBW, int K, int mw = MW) {
    return mma_vrows_off(NBW, mw) + (((size_t)MNV * MR * K * 4 + 15) & ~(size_t)15);
}
__host__ __device__ constexpr size_t mma_smem_bytes(int NBW, int K, int mw = MW) {
    return mma_red_off(NBW, K, mw) + (size_t)mma_nrb(mw) * mw * mma_nc(K) * 128 * 4;
}

// The row pass (one iteration's V half-step and the B, H, <V_new, A> partials of each CTA) and,
// with PERSIST, all n_iter iterations in one cooperative launch with the D half-step between
// passes (grid barriers; the same fixed-order reductions as k_nmf_persist, nmf_fused.cuh).
// Tiles: CTA c owns c, c + nCTA, ... (forward in even iterations, backward in odd ones, so the
// tiles a pass ends with -- the ones most likely still in L2 -- start the next).
// Warp w owns the blocks [w NB / 8, (w + 1) NB / 8) of every tile; tile m's V store, H and
// <V_new, A> terms are taken by warp m % 8 (every warp holds the whole new V of the tile).
// Components: NC column blocks of 8 (K = 9..16: every MMA of the pass and every per-lane
// V-update value twice, once per block).
template <int K, int NBW, bool PERSIST, int MWT = 8>
__global__ void __launch_bounds__(MWT * 32, 1) k_nmf_mma(MmaArgs A) {
    static_assert(K >= 1 && K <= 16, "two n8 column blocks at most");
    static_assert(MWT == 8 || (MWT == MW16 && mma_nc(K) == 2), "8 warps, or 16 with two column blocks");
    constexpr int MW = MWT, MTH = MWT * 32;  // (shadow the 8-warp constants)
    constexpr int MHW = 8;                   // warps that own tiles' H / <V, A> terms (m % 8)
    constexpr int NRB = mma_nrb(MWT);
    constexpr int NC = mma_nc(K);
    // DISTV: the V update computed once per tile (warp w: components w and w + 8, lane: row
    // lane % 16) and shared through shared memory with a second barrier, instead of redundantly in
    // every warp (C5: 2.7% per iteration in steady state, fewer instructions under the power cap).
    // HSNCT_MMA_NODISTV builds the redundant version (A/B).
#ifdef HSNCT_MMA_NODISTV
    constexpr bool DISTV = false;
#else
    constexpr bool DISTV = true;
#endif
    static_assert(DISTV || MWT == 8, "16 warps: the per-tile V update only");
    // PK (K = 1..4 and 9..12): the last column block (PB) holds at most four components and
    // carries them -- PK0 = 8 PB onwards; below for K = 9..12 -- as interleaved hi/lo
    // column pairs (column 2i: hi of component 8 + i, column 2i + 1: lo), so one MMA gives the
    // hi.hi and hi.lo products and a second one lo.hi (+ lo.lo): 5 MMAs per block and phase
    // instead of 6, half the second block's accumulators and D-operand registers.  Lane (g, t)
    // then holds component 8 + t of that block (the two columns' sum), rows / bins g and g + 8.
    // (K <= 4: 2 MMAs per block and phase instead of 3.)
    constexpr int PB = NC - 1, PK0 = 8 * PB;
    constexpr bool PK = DISTV && K - PK0 <= 4;
    constexpr int KK = K * K;
    constexpr int HW = 64 * NC * NC;  // per-warp H accumulators [2 NC values][NC column blocks][32 lanes]
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t full[MW][MNS];
    __shared__ uint64_t vfull[MNV];
    __shared__ double hsh[MHW][HW];
    __shared__ double vsh[MW];
    __shared__ double Hs[KK], Gold[KK], Gnew[KK];
    __shared__ double red8[MW];
    __shared__ float Gf[(NC == 1 && !DISTV) ? 1 : 16 * K];  // G as float [j][16] (the V update's V G)
    // DISTV: the tile's new V as the phase-2 B operand, split once by the V update's threads:
    // [component][t][vh0, vh1, vl0, vl1] (one 16-byte load per lane and column block), and the
    // exponents of the per-component scales sigma_V (zero for components >= K)
    __shared__ __align__(16) uint32_t vfrag_s[DISTV ? 8 * NC * 16 : 4];
    __shared__ __align__(8) int ev_s[DISTV ? 8 * NC : 2];
    __shared__ __align__(8) uint32_t vpk_s[PK ? 64 : 2];  // PK: packed block [column][t][b0, b1]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int c = blockIdx.x, nC = gridDim.x;
    const size_t slotb = (size_t)NBW * BLK;
    uint8_t* ring = smem;
    float* vrows = reinterpret_cast<float*>(smem + mma_vrows_off(NBW, MW));
    float* red = reinterpret_cast<float*>(smem + mma_red_off(NBW, K, MW));
    const int jb = warp * A.NB / MW, nb = (warp + 1) * A.NB / MW - jb;
    const int64_t ntiles = (A.Np + MR - 1) / MR;
    const int64_t nmine = ntiles > c ? (ntiles - 1 - c) / nC + 1 : 0;
    if (tid == 0) {
        for (int w = 0; w < MW; ++w)
            for (int s = 0; s < MNS; ++s) mbar_init(&full[w][s], 1);
        for (int s = 0; s < MNV; ++s) mbar_init(&vfull[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < KK; i += MTH) Gold[i] = A.Gd[i];
    __syncthreads();
    uint8_t* myring = ring + (size_t)warp * MNS * slotb;
    const unsigned ringw = smem_u32(myring);
    auto tile_of = [&](int64_t q, bool fw) { return (int64_t)c + (fw ? q : nmine - 1 - q) * nC; };
    // lane 0: this warp's chunk of tile q (pass direction fw) into slot s (0 bytes: completes the
    // phase, warps without blocks)
    auto issue_y = [&](int s, int64_t q, bool fw) {
        const unsigned bytes = (unsigned)nb * BLK;
        mbar_expect_tx(&full[warp][s], bytes);
        if (bytes)
            bulk_g2s(myring + (size_t)s * slotb, A.Yc + ((size_t)tile_of(q, fw) * A.NB + jb) * BLK, bytes,
                     &full[warp][s]);
    };
    // warp 0 lane 0: old V rows of tile q into V slot s (full tiles; the ragged one only arrives)
    auto issue_v = [&](int s, int64_t q, bool fw) {
        const int64_t r0 = tile_of(q, fw) * MR;
        if (r0 + MR <= A.Np) {
            mbar_expect_tx(&vfull[s], (unsigned)(MR * K * 4));
            bulk_g2s(vrows + (size_t)s * MR * K, A.V + r0 * K, (unsigned)(MR * K * 4), &vfull[s]);
        } else {
            mbar_arrive_cta(&vfull[s]);
        }
    };
    // phase-2 ldmatrix.trans: lanes 8i..8i+7 address core matrix (0, 2, 1, 3)[i]
    const unsigned toff = (unsigned)((((lane >> 3) == 1) ? 2 : ((lane >> 3) == 2) ? 1 : (lane >> 3)) * 128 +
                                     (lane & 7) * 16);
    // partial-A exchange: the reader lane L = 4 k + u takes rows 2u, 2u+1, 2u+8, 2u+9 of component
    // k (of a column block) as one float4 at slot L ^ (k >> 1) (conflict-free reads, 2-way writes).
    // Writer offsets of this lane's accumulator values (A[g][2t], A[g][2t+1], A[g+8][2t],
    // A[g+8][2t+1] of each column block):
    const int wsl0 = 8 * t + ((g >> 1) ^ t), wsl1 = 8 * t + 4 + ((g >> 1) ^ t);
    const int wo0 = 4 * wsl0 + (g & 1), wo1 = 4 * wsl1 + (g & 1);
    const int rsl = lane ^ (g >> 1);  // this lane's read slot (k = g, u = t)
    if (warp < MHW)
        for (int i = lane; i < HW; i += 32) hsh[warp][i] = 0.0;
    if constexpr (DISTV) {
        for (int i = tid; i < 8 * NC * 16; i += MTH) vfrag_s[i] = 0u;
        for (int i = tid; i < 8 * NC; i += MTH) ev_s[i] = 0;
        if constexpr (PK)
            for (int i = tid; i < 64; i += MTH) vpk_s[i] = 0u;
    }

    // D update slice of this CTA (PERSIST)
    const int SL = (A.Nk + nC - 1) / nC;
    const int l0s = min(A.Nk, c * SL), nsl = max(0, min(A.Nk, l0s + SL) - l0s);
    unsigned epoch = 0;
    double ysq = 0.0;
    int64_t n0 = 0;  // running tile count of this CTA (mbarrier slots and phases)
    const int it_end = PERSIST ? A.n_iter : A.it + 1;
    for (int it = PERSIST ? 0 : A.it; it < it_end; ++it) {
        const bool fwd = (it & 1) == 0;
        const bool first = it == 0;
        if (!PERSIST || it == 0) {  // head tiles (later passes: issued at the end of the previous one)
            if (lane == 0) {
                for (int64_t q = 0; q < min((int64_t)MNS, nmine); ++q) issue_y((int)((n0 + q) % MNS), q, fwd);
                if (warp == 0)
                    for (int64_t q = 0; q < min((int64_t)MNV, nmine); ++q) issue_v((int)((n0 + q) % MNV), q, fwd);
            }
        }
        // columns g (+ 8) of G (the V update's V G) and this warp's D operand (B of phase 1:
        // K = bins, N = components) as fp16 hi/lo, in registers for the pass.  D and G change
        // between the passes of a persistent launch: L2 loads (__ldcg), G from shared memory.
        // (NC = 2: from a float copy in shared memory, to save the registers)
        float gcol[NC == 1 ? K : 1];
        if constexpr (NC == 1 && !DISTV) {
#pragma unroll
            for (int j = 0; j < K; ++j) gcol[j] = g < K ? (float)Gold[j * K + g] : 0.f;
        } else {
            for (int i = tid; i < 16 * K; i += MTH) Gf[i] = i % 16 < K ? (float)Gold[(i / 16) * K + i % 16] : 0.f;
            __syncthreads();
        }
        uint32_t dh[NBW][NC][2], dl[NBW][NC][2];
        float invA[NC][2];  // 1 / sigma_D[k] for this lane's output columns k = 2t, 2t + 1 (+ 8 nc)
#pragma unroll
        for (int nc = 0; nc < NC; ++nc) {
            const int kd = (PK && nc == PB) ? PK0 + (g >> 1) : g + 8 * nc;
            float dv[NBW][4];
            float mx = 0.f;
#pragma unroll
            for (int j = 0; j < NBW; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int l = 16 * (jb + j) + 2 * t + (e & 1) + (e >> 1) * 8;
                    dv[j][e] = (j < nb && kd < K && l < A.Nk) ? __ldcg(A.D + (int64_t)kd * A.Nk + l) : 0.f;
                    mx = fmaxf(mx, fabsf(dv[j][e]));
                }
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const int ed = mexp(mx);
            const float sd = pow2(ed);
#pragma unroll
            for (int j = 0; j < NBW; ++j) {
                dh[j][nc][0] = split2(dv[j][0] * sd, dv[j][1] * sd, dl[j][nc][0]);
                dh[j][nc][1] = split2(dv[j][2] * sd, dv[j][3] * sd, dl[j][nc][1]);
                if (PK && nc == PB && (g & 1)) {  // odd column: the lo part (dl of the block is unused)
                    dh[j][nc][0] = dl[j][nc][0];
                    dh[j][nc][1] = dl[j][nc][1];
                }
            }
            invA[nc][0] = pow2(-__shfl_sync(0xffffffffu, ed, 8 * t));  // (x 1 / sigma_Y of the tile)
            invA[nc][1] = pow2(-__shfl_sync(0xffffffffu, ed, 8 * t + 4));
        }

        float bacc[NBW][NC][4];
#pragma unroll
        for (int j = 0; j < NBW; ++j)
#pragma unroll
            for (int nc = 0; nc < NC; ++nc)
#pragma unroll
                for (int e = 0; e < 4; ++e) bacc[j][nc][e] = 0.f;
        double vdotA = 0.0;
        unsigned bad = 0;
        int ety = nmine > 0 ? __ldg(A.texp + tile_of(0, fwd)) : 0;  // tile scale exponent (k_mma_prep)

        for (int64_t m = 0; m < nmine; ++m) {
            const int64_t n = n0 + m;
            const int s = (int)(n % MNS);
            const unsigned par = (unsigned)((n / MNS) & 1);
            const int sv4 = (int)(n % MNV);
            const int64_t tile = tile_of(m, fwd), r0 = tile * MR;
            const int nv = (int)min((int64_t)MR, A.Np - r0);
            const float isy = pow2(-ety);  // 1 / sigma_Y of the tile
            // the next tile's exponent, one tile ahead (an L2 load's latency exceeds phase 1)
            ety = m + 1 < nmine ? __ldg(A.texp + tile_of(m + 1, fwd)) : 0;
            mbar_wait(&full[warp][s], par);
            const unsigned sb = ringw + (unsigned)(s * slotb);
            // ---- phase 1: this warp's partial A = Y+_R D^T over its blocks.  Straight-line code
            //      over NBW blocks: blocks j >= nb re-read the last block with a zero D operand (no
            //      branches between the MMAs, so the compiler can overlap the blocks' latencies)
            float a0[NC][4], a1[NC][4], a2[NC][4];
#pragma unroll
            for (int nc = 0; nc < NC; ++nc)
#pragma unroll
                for (int e = 0; e < 4; ++e) a0[nc][e] = a1[nc][e] = a2[nc][e] = 0.f;
            if (nb > 0) {
#pragma unroll
                for (int j = 0; j < NBW; ++j) {
                    // (only the last block is skipped when the warp has fewer: a branch per block
                    // would serialise the sweeps; C6 -2.4% per iteration, C5 neutral)
                    if (j == NBW - 1 && nb < NBW) break;
                    const unsigned ba = sb + (unsigned)min(j, nb - 1) * BLK;
                    uint32_t yh[4], yl[4];
                    ldsm4(yh, ba + lane * 16);
                    ldsm4(yl, ba + 512 + lane * 16);
#pragma unroll
                    for (int nc = 0; nc < NC; ++nc) {
                        if (PK && nc == PB) {  // columns (hi, lo) of components PK0..PK0 + 3
                            mma16816(a0[nc], yh, dh[j][nc][0], dh[j][nc][1]);
                            mma16816(a1[nc], yl, dh[j][nc][0], dh[j][nc][1]);
                            continue;
                        }
                        mma16816(a0[nc], yh, dh[j][nc][0], dh[j][nc][1]);
                        mma16816(a1[nc], yh, dl[j][nc][0], dl[j][nc][1]);
                        // (NC = 2: both small products in one accumulator, for the registers)
                        mma16816(NC == 1 ? a2[nc] : a1[nc], yl, dh[j][nc][0], dh[j][nc][1]);
                    }
                }
            }
#pragma unroll
            for (int nc = 0; nc < NC; ++nc) {
                float* rb = red + (size_t)(((n & (NRB - 1)) * MW + warp) * NC + nc) * 128;
                const float i0 = invA[nc][0] * isy, i1 = invA[nc][1] * isy;
                if (PK && nc == PB) {
                    // component kk = t of the block, rows g and g + 8: the reader's slot of (kk, row)
                    const int wp = (((4 * t + (g >> 1)) ^ (t >> 1)) << 2) + (g & 1);
                    rb[wp] = ((a0[nc][0] + a0[nc][1]) + (a1[nc][0] + a1[nc][1])) * i0;
                    rb[wp + 2] = ((a0[nc][2] + a0[nc][3]) + (a1[nc][2] + a1[nc][3])) * i0;
                    continue;
                }
                rb[wo0] = (a0[nc][0] + (a1[nc][0] + a2[nc][0])) * i0;
                rb[wo1] = (a0[nc][1] + (a1[nc][1] + a2[nc][1])) * i1;
                rb[wo0 + 2] = (a0[nc][2] + (a1[nc][2] + a2[nc][2])) * i0;
                rb[wo1 + 2] = (a0[nc][3] + (a1[nc][3] + a2[nc][3])) * i1;
            }
            // V G and the old V of this lane's (row, component) pairs -- before the barrier, so no
            // warp can still be reading old V rows of a ragged tile (global memory) once the
            // tile's owner warp stores the new ones
            float vg[NC][4], vo[NC][4];
            if constexpr (DISTV) {
                // old V rows of a ragged tile into its (unused) V slot, read after the barrier
                if (nv < MR && warp == 0) {
                    float* vs = vrows + (size_t)sv4 * MR * K;
                    for (int i = lane; i < nv * K; i += 32) vs[i] = A.V[r0 * K + i];
                }
            } else {
                mbar_wait(&vfull[sv4], (unsigned)((n / MNV) & 1));
                const float* vr = nv == MR ? vrows + (size_t)sv4 * MR * K : A.V + r0 * K;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int r = 2 * t + (e & 1) + (e >> 1) * 8;
                    float vrow[K];
#pragma unroll
                    for (int j = 0; j < K; ++j) vrow[j] = r < nv ? vr[r * K + j] : 0.f;
#pragma unroll
                    for (int nc = 0; nc < NC; ++nc) {
                        const int kd = g + 8 * nc;
                        float x = 0.f, v0 = 0.f;
#pragma unroll
                        for (int j = 0; j < K; ++j) {
                            if constexpr (NC == 1) x = fmaf(vrow[j], gcol[j], x);
                            else x = fmaf(vrow[j], Gf[j * 16 + kd], x);
                            if (j == kd) v0 = vrow[j];
                        }
                        vg[nc][e] = x;
                        vo[nc][e] = kd < K ? v0 : 0.f;
                    }
                }
            }
            named_bar(1, MTH);
            // every warp has read the old V of tile m - 1: its V slot takes tile m + MNV - 1
            if (warp == 0 && lane == 0 && m >= 1 && m + MNV - 1 < nmine)
                issue_v((int)((n + MNV - 1) % MNV), m + MNV - 1, fwd);
            // ---- V update (every warp, redundantly): lane (g, t) -> components g (+ 8), rows 2t,
            //      2t+1, 2t+8, 2t+9 -- exactly its part of the phase-2 B operand
            float av[NC][4], vn[NC][4];
            uint32_t vh0[NC], vh1[NC], vl0[NC], vl1[NC];
            int evs[NC];
            float invB[NC][2], ivB[NC][2];
            if constexpr (DISTV) {
                mbar_wait(&vfull[sv4], (unsigned)((n / MNV) & 1));
                // component, tile row (16 warps: the half-warps sum warps 0-7 and 8-15's partials)
                const int k = MW == MW16 ? warp : warp + 8 * (lane >> 4), r = lane & 15;
                if (k < K) {
                    const int kk = k & 7, u = (r & 7) >> 1, e = (r & 1) + 2 * (r >> 3);
                    const float* rd = red + (size_t)((n & (NRB - 1)) * MW * NC + (k >> 3)) * 128 + ((4 * kk + u) ^ (kk >> 1)) * 4 + e;
                    if constexpr (MW == MW16) rd += (lane >> 4) * 8 * NC * 128;
                    float a = rd[0];
#pragma unroll
                    for (int w = 1; w < 8; ++w) a += rd[w * NC * 128];
                    if constexpr (MW == MW16) a += __shfl_xor_sync(0xffffffffu, a, 16);
                    const float* vr = vrows + (size_t)sv4 * MR * K + r * K;
                    float x = 0.f, v0 = 0.f;
                    if (r < nv) {
#pragma unroll
                        for (int j = 0; j < K; ++j) {
                            const float vj = vr[j];
                            x = fmaf(vj, Gf[j * 16 + k], x);
                            if (j == k) v0 = vj;
                        }
                    }
                    const float vnk = a * (v0 * rcp_approx(fmaxf(x, 1e-30f)));
                    {   // sigma_V of the component over the tile's 16 rows (this half-warp), hi/lo split
                        const unsigned hm = (lane & 16) ? 0xffff0000u : 0x0000ffffu;
                        float vmax = fabsf(vnk);
#pragma unroll
                        for (int o = 1; o < 16; o <<= 1) vmax = fmaxf(vmax, __shfl_xor_sync(hm, vmax, o));
                        const int ev = mexp(vmax);
                        const float xs = vnk * pow2(ev);
                        const __half hh = __float2half_rn(xs);
                        const __half hl = __float2half_rn(xs - __half2float(hh));
                        // row r = 2 t + i (+ 8): half i of word (r >> 3) (hi) / 2 + (r >> 3) (lo)
                        __half* fr = reinterpret_cast<__half*>(vfrag_s) + ((k * 4 + u) * 4 + (r >> 3)) * 2 + (r & 1);
                        fr[0] = hh;
                        fr[4] = hl;
                        if (r == 0) ev_s[k] = ev;
                        if constexpr (PK) {
                            if (k >= PK0) {  // packed block: column 2 (k - PK0) hi, 2 (k - PK0) + 1 lo
                                __half* fp = reinterpret_cast<__half*>(vpk_s) +
                                             (((2 * (k - PK0)) * 4 + u) * 2 + (r >> 3)) * 2 + (r & 1);
                                fp[0] = hh;
                                fp[16] = hl;
                            }
                        }
                    }
                    if (r < nv && (MW == 8 || lane < 16)) {
                        if (first && !(isfinite(v0) && v0 >= 0.f)) bad |= ST_INIT_BAD;
                        if (!isfinite(vnk)) bad |= ST_NUMERIC;
                        A.V[(r0 + r) * K + k] = vnk;
                        vdotA += (double)(vnk * a);
                    }
                }
                named_bar(2, MTH);
            }
#pragma unroll
            for (int nc = 0; nc < NC; ++nc) {
              if (PK && nc == PB) {
                // packed block: this lane's column g (hi or lo of component PK0 + g / 2); the outputs
                // (columns 2t, 2t + 1) belong to component PK0 + t
                const uint2 f = *reinterpret_cast<const uint2*>(&vpk_s[lane * 2]);
                vh0[nc] = f.x;
                vh1[nc] = f.y;
                invB[nc][0] = isy * pow2(-ev_s[PK0 + t]);
              } else if constexpr (DISTV) {
                const uint4 f = *reinterpret_cast<const uint4*>(&vfrag_s[(8 * nc * 4 + lane) * 4]);
                vh0[nc] = f.x;
                vh1[nc] = f.y;
                vl0[nc] = f.z;
                vl1[nc] = f.w;
                evs[nc] = ev_s[g + 8 * nc];
                const int2 e2 = *reinterpret_cast<const int2*>(&ev_s[2 * t + 8 * nc]);
                ivB[nc][0] = pow2(-e2.x);  // 1 / sigma_V[k], k = 2t (+ 8 nc)
                ivB[nc][1] = pow2(-e2.y);
                invB[nc][0] = isy * ivB[nc][0];
                invB[nc][1] = isy * ivB[nc][1];
              } else {
                const float4* rd =
                    reinterpret_cast<const float4*>(red + (size_t)(((n & 1) * MW) * NC + nc) * 128) + rsl;
                float4 s4 = rd[0];
#pragma unroll
                for (int w = 1; w < MW; ++w) {
                    const float4 q = rd[w * NC * 32];
                    s4.x += q.x;
                    s4.y += q.y;
                    s4.z += q.z;
                    s4.w += q.w;
                }
                av[nc][0] = s4.x;
                av[nc][1] = s4.y;
                av[nc][2] = s4.z;
                av[nc][3] = s4.w;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    // V / max(VG, 1e-30) by the approximate reciprocal (the divisor is a normal
                    // number; 1 ulp); rows and components outside the tile have vo = 0
                    vn[nc][e] = av[nc][e] * (vo[nc][e] * rcp_approx(fmaxf(vg[nc][e], 1e-30f)));
                }
                float vmax = 0.f;
#pragma unroll
                for (int e = 0; e < 4; ++e) vmax = fmaxf(vmax, fabsf(vn[nc][e]));
                vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, 1));
                vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, 2));
                const int ev = mexp(vmax);
                const float sv = pow2(ev);
                vh0[nc] = split2(vn[nc][0] * sv, vn[nc][1] * sv, vl0[nc]);
                vh1[nc] = split2(vn[nc][2] * sv, vn[nc][3] * sv, vl1[nc]);
                evs[nc] = ev;
                ivB[nc][0] = pow2(-__shfl_sync(0xffffffffu, ev, 8 * t));  // 1 / sigma_V[k], k = 2t (+ 8 nc)
                ivB[nc][1] = pow2(-__shfl_sync(0xffffffffu, ev, 8 * t + 4));
                invB[nc][0] = isy * ivB[nc][0];
                invB[nc][1] = isy * ivB[nc][1];
              }
            }
            if (warp == (int)(m % MHW)) {  // this tile's V store, <V_new, A>, H += V_new^T V_new
                float va = 0.f;
                if constexpr (!DISTV)
#pragma unroll
                for (int nc = 0; nc < NC; ++nc)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int r = 2 * t + (e & 1) + (e >> 1) * 8, kd = g + 8 * nc;
                        if (kd < K && r < nv) {
                            if (first && !(isfinite(vo[nc][e]) && vo[nc][e] >= 0.f)) bad |= ST_INIT_BAD;
                            if (!isfinite(vn[nc][e])) bad |= ST_NUMERIC;
                            A.V[(r0 + r) * K + kd] = vn[nc][e];
                            va = fmaf(vn[nc][e], av[nc][e], va);
                        }
                    }
                if constexpr (!DISTV) vdotA += (double)va;
                uint32_t vp0 = 0u, vp1 = 0u;
                if constexpr (PK) {  // H needs block PB component-per-column: the unpacked fragments
                    vp0 = vh0[PB];
                    vp1 = vh1[PB];
                    const uint4 f = *reinterpret_cast<const uint4*>(&vfrag_s[(PK0 * 4 + lane) * 4]);
                    vh0[PB] = f.x;
                    vh1[PB] = f.y;
                    vl0[PB] = f.z;
                    vl1[PB] = f.w;
                    evs[PB] = ev_s[g + PK0];
                    const int2 e2 = *reinterpret_cast<const int2*>(&ev_s[2 * t + PK0]);
                    ivB[PB][0] = pow2(-e2.x);
                    ivB[PB][1] = pow2(-e2.y);
                }
                // H on the tensor core: A operand V^T (rows g, g + 8: this lane's B-operand
                // fragments of column blocks 0 and 1), B operand V (column block nb2):
                // C[g (+8)][2t + i + 8 nb2] = sum_r V[r][.] V[r][.], scaled by sigma_V sigma_V
                const uint32_t ah[4] = {vh0[0], NC > 1 ? vh0[NC - 1] : 0u, vh1[0], NC > 1 ? vh1[NC - 1] : 0u};
                const uint32_t al[4] = {vl0[0], NC > 1 ? vl0[NC - 1] : 0u, vl1[0], NC > 1 ? vl1[NC - 1] : 0u};
#pragma unroll
                for (int nb2 = 0; nb2 < NC; ++nb2) {
                    float hc[4] = {0.f, 0.f, 0.f, 0.f};
                    mma16816(hc, ah, vh0[nb2], vh1[nb2]);
                    mma16816(hc, ah, vl0[nb2], vl1[nb2]);
                    mma16816(hc, al, vh0[nb2], vh1[nb2]);
#pragma unroll
                    for (int q = 0; q < (NC > 1 ? 4 : 2); ++q) {  // rows g (q < 2), g + 8 (q >= 2)
                        const float ir = pow2(-evs[q >> 1 < NC ? q >> 1 : 0]);
                        double& hd = hsh[warp][(q * NC + nb2) * 32 + lane];  // lane-major: conflict-free
                        hd += (double)(hc[q] * (ir * ivB[nb2][q & 1]));
                    }
                }
                if constexpr (PK) {  // back to the packed block for phase 2
                    vh0[PB] = vp0;
                    vh1[PB] = vp1;
                }
            }
            // ---- phase 2: B^T[l][k] += sum_r Y+[r][l] V_new[r][k] over this warp's blocks (blocks
            //      j >= nb accumulate a copy of the last block into columns that are never stored)
            if (nb > 0) {
#pragma unroll
                for (int j = 0; j < NBW; ++j) {
                    if (j == NBW - 1 && nb < NBW) break;
                    const unsigned ba = sb + (unsigned)min(j, nb - 1) * BLK + toff;
                    uint32_t th[4], tl[4];
                    ldsm4t(th, ba);
                    ldsm4t(tl, ba + 512);
#pragma unroll
                    for (int nc = 0; nc < NC; ++nc) {
                        float cc[4] = {0.f, 0.f, 0.f, 0.f};
                        if (PK && nc == PB) {  // bins g, g + 8 of component PK0 + t: hi and lo columns summed
                            mma16816(cc, th, vh0[nc], vh1[nc]);
                            mma16816(cc, tl, vh0[nc], vh1[nc]);
                            bacc[j][nc][0] = fmaf(cc[0] + cc[1], invB[nc][0], bacc[j][nc][0]);
                            bacc[j][nc][2] = fmaf(cc[2] + cc[3], invB[nc][0], bacc[j][nc][2]);
                            continue;
                        }
                        mma16816(cc, th, vh0[nc], vh1[nc]);
                        mma16816(cc, th, vl0[nc], vl1[nc]);
                        mma16816(cc, tl, vh0[nc], vh1[nc]);
                        bacc[j][nc][0] = fmaf(cc[0], invB[nc][0], bacc[j][nc][0]);
                        bacc[j][nc][1] = fmaf(cc[1], invB[nc][1], bacc[j][nc][1]);
                        bacc[j][nc][2] = fmaf(cc[2], invB[nc][0], bacc[j][nc][2]);
                        bacc[j][nc][3] = fmaf(cc[3], invB[nc][1], bacc[j][nc][3]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0 && m + MNS < nmine) {
                fence_proxy_async();  // this warp's ldmatrix reads of the slot before the refill
                issue_y(s, m + MNS, fwd);
            }
        }
        n0 += nmine;
        // the next pass's head tiles (reverse direction: the tiles just streamed, likely in L2)
        if (PERSIST && it + 1 < it_end) {
            __syncwarp();
            if (lane == 0) {
                fence_proxy_async();
                for (int64_t q = 0; q < min((int64_t)MNS, nmine); ++q) issue_y((int)((n0 + q) % MNS), q, !fwd);
            }
        }

        // ---- this CTA's partials: B [K][Nkp] (lambda < Nk), H, <V_new, A> (warps summed in order)
        float* Bo = A.Bpart + (int64_t)c * K * A.Nkp;
#pragma unroll
        for (int j = 0; j < NBW; ++j) {
            if (j < nb) {
                const int l = 16 * (jb + j) + g;
#pragma unroll
                for (int nc = 0; nc < NC; ++nc) {
                    if (PK && nc == PB) {
                        if (PK0 + t < K) {
                            if (l < A.Nk) Bo[(int64_t)(PK0 + t) * A.Nkp + l] = bacc[j][nc][0];
                            if (l + 8 < A.Nk) Bo[(int64_t)(PK0 + t) * A.Nkp + l + 8] = bacc[j][nc][2];
                        }
                        continue;
                    }
                    const int k0 = 2 * t + 8 * nc;
                    if (k0 < K) {
                        if (l < A.Nk) Bo[(int64_t)k0 * A.Nkp + l] = bacc[j][nc][0];
                        if (l + 8 < A.Nk) Bo[(int64_t)k0 * A.Nkp + l + 8] = bacc[j][nc][2];
                    }
                    if (k0 + 1 < K) {
                        if (l < A.Nk) Bo[(int64_t)(k0 + 1) * A.Nkp + l] = bacc[j][nc][1];
                        if (l + 8 < A.Nk) Bo[(int64_t)(k0 + 1) * A.Nkp + l + 8] = bacc[j][nc][3];
                    }
                }
            }
        }
        vdotA = warp_sum_d(vdotA);
        bad = __reduce_or_sync(0xffffffffu, bad);
        if (lane == 0) {
            vsh[warp] = vdotA;
            if (bad) atomicOr(A.status, bad);
        }
        if (PERSIST) fence_proxy_async_global();  // this thread's V stores before the next bulk copies
        __syncthreads();
        if (tid < KK) {
            const int ka = tid / K, kb = tid - (tid / K) * K;
            double h = 0.0;
            // H[ka][kb] is the sum of lane 4 (ka % 8) + (kb % 8) / 2's value q = 2 (ka / 8) + kb % 2,
            // column block kb / 8
            const int hi = ((2 * (ka >> 3) + (kb & 1)) * NC + (kb >> 3)) * 32 + 4 * (ka & 7) + ((kb & 7) >> 1);
            for (int w = 0; w < MHW; ++w) h += hsh[w][hi];
            A.Hpart[(int64_t)c * KK + tid] = h;
        }
        if (tid == 0) {
            double v = 0.0;
            for (int w = 0; w < MW; ++w) v += vsh[w];
            A.vpart[2 * (int64_t)c] = v;
            A.vpart[2 * (int64_t)c + 1] = 0.0;
        }
        __syncthreads();  // hsh read before it is cleared for the next pass
        if (warp < MHW)
            for (int i = lane; i < HW; i += 32) hsh[warp][i] = 0.0;
        if constexpr (PERSIST) {
            // the next pass's old-V head rows (written by this pass: generic stores, fenced above)
            if (it + 1 < it_end && tid == 0) {
                fence_proxy_async();
                for (int64_t q = 0; q < min((int64_t)MNV, nmine); ++q) issue_v((int)((n0 + q) % MNV), q, !fwd);
            }
            // ---- D half-step (k_nmf_persist's fixed-order scheme): grid barrier -> H and this
            //      CTA's lambda slice of B over the nC partials -> D update of the slice, <B, D_new>
            //      and D_new D_new^T slice partials -> grid barrier -> G_new, objective
            double* gacc = reinterpret_cast<double*>(red);  // the partial-A buffers are idle here
            double* Bsl = gacc + MTH;                        // [K * nsl]  (<= 256)
            double* dnew = Bsl + 256;                        // [K][64] (the buffers hold >= 1024 NC doubles)
            grid_sync(A.bar, epoch);
            const bool objcta = c == nC - 1 && (A.obj || it == 0);
            double va = 0.0;
            if (objcta) {
                double v0 = 0.0;
                for (int i = tid; i < nC; i += MTH) v0 += __ldcg(A.vpart + 2 * i);
                va = block_sum_all(v0, red8);
            }
            {
                const int nB = K * nsl, nout = KK + nB;
                const int NQ = max(1, MTH / nout);
                if (tid < NQ * nout) {
                    const int o = tid % nout, q = tid / nout;
                    double sacc = 0.0;
                    if (o < KK) {
                        const double* src = A.Hpart + o;
                        sacc = batched_sum(q, NQ, nC, [&](int cc) { return __ldcg(src + (int64_t)cc * KK); });
                    } else {
                        const int ob = o - KK, k = ob / nsl, l = l0s + (ob - (ob / nsl) * nsl);
                        const float* src = A.Bpart + (int64_t)k * A.Nkp + l;
                        const int64_t stride = (int64_t)K * A.Nkp;
                        sacc = batched_sum(q, NQ, nC, [&](int cc) { return (double)__ldcg(src + (int64_t)cc * stride); });
                    }
                    gacc[tid] = sacc;
                }
                __syncthreads();
                for (int o = tid; o < nout; o += MTH) {
                    double sacc = 0.0;
                    for (int q = 0; q < NQ; ++q) sacc += gacc[q * nout + o];
                    if (o < KK) Hs[o] = sacc;
                    else Bsl[o - KK] = sacc;
                }
                __syncthreads();
            }
            {
                double bd = 0.0;
                if (tid < nsl) {
                    const int l = l0s + tid;
                    unsigned bd_bad = 0;
                    double d[K];
#pragma unroll
                    for (int k = 0; k < K; ++k) d[k] = (double)__ldcg(A.D + (int64_t)k * A.Nk + l);  // D_old
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        double hd = 0.0;
#pragma unroll
                        for (int jj = 0; jj < K; ++jj) hd = fma(Hs[k * K + jj], d[jj], hd);
                        const double B = Bsl[k * nsl + tid];
                        const float dn = (float)(d[k] * B / fmax(hd, 1e-30));
                        if (!isfinite(dn)) bd_bad |= ST_NUMERIC;
                        bd += B * (double)dn;
                        A.D[(int64_t)k * A.Nk + l] = dn;
                        dnew[k * 64 + tid] = (double)dn;
                    }
                    if (bd_bad) atomicOr(A.status, bd_bad);
                }
                gacc[tid] = bd;
                __syncthreads();
                if (tid == 0) {
                    double sacc = 0.0;
                    for (int u = 0; u < nsl; ++u) sacc += gacc[u];
                    A.dpart[c] = sacc;
                }
                for (int o = tid; o < KK; o += MTH) {
                    const int a = o / K, b = o - (o / K) * K;
                    double sacc = 0.0;
                    for (int u = 0; u < nsl; ++u) sacc = fma(dnew[a * 64 + u], dnew[b * 64 + u], sacc);
                    A.Gpart[(int64_t)c * KK + o] = sacc;
                }
            }
            grid_sync(A.bar, epoch);
            {
                constexpr int NQ = MTH / KK > 0 ? MTH / KK : 1;
                double sacc = 0.0;
                if (tid < NQ * KK) {
                    const int o = tid % KK, q = tid / KK;
                    sacc = batched_sum(q, NQ, nC, [&](int cc) { return __ldcg(A.Gpart + (int64_t)cc * KK + o); });
                    gacc[tid] = sacc;
                }
                __syncthreads();
                for (int o = tid; o < KK; o += MTH) {
                    double tq = 0.0;
                    for (int q = 0; q < NQ; ++q) tq += gacc[q * KK + o];
                    Gnew[o] = tq;
                }
                __syncthreads();
            }
            if (objcta) {  // the objective trace (and the Y+ = 0 check)
                double v1 = 0.0, v2 = 0.0;
                for (int i = tid; i < nC; i += MTH) v2 += __ldcg(A.dpart + i);
                if (it == 0)
                    for (int i = tid; i < A.nby; i += MTH) v1 += __ldcg(A.ypart + i);
                const double ysq_new = block_sum_all(v1, red8);
                const double bdot = block_sum_all(v2, red8);
                if (tid == 0) {
                    if (it == 0) {
                        ysq = ysq_new;
                        *A.ysq = ysq;
                        if (!(ysq > 0.0)) atomicOr(A.status, (unsigned)ST_Y_ALLZERO);
                    }
                    double hg_old = 0.0, hg_new = 0.0;
                    for (int q = 0; q < KK; ++q) {
                        hg_old += Hs[q] * Gold[q];
                        hg_new += Hs[q] * Gnew[q];
                    }
                    if (A.obj) {
                        A.obj[2 * it] = ysq - 2.0 * va + hg_old;
                        A.obj[2 * it + 1] = ysq - 2.0 * bdot + hg_new;
                    }
                }
            }
            __syncthreads();  // the objective (thread 0) has read Gold
            for (int o = tid; o < KK; o += MTH) Gold[o] = Gnew[o];
            __syncthreads();
        }
    }
    if (PERSIST && c == 0)
        for (int o = tid; o < KK; o += MTH) A.Gd[o] = Gold[o];
}

template <int K, int NBW, bool PERSIST, int MWT = 8>
cudaError_t mma_klb(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D, int it, int n_iter,
                    double* obj, unsigned* bar, unsigned* status, cudaStream_t s) {
    static SmemAttr attr;
    constexpr int MTH = MWT * 32;
    const size_t smem = mma_smem_bytes(NBW, K, MWT);
    cudaError_t e = ensure_smem((const void*)k_nmf_mma<K, NBW, PERSIST, MWT>, (int)smem, attr);
    if (e != cudaSuccess) return e;
    MmaArgs A{};
    A.Yc = static_cast<const uint8_t*>(w.Yc);
    A.Np = (int64_t)g.Nv * g.Nr * g.Nc;
    A.Nk = g.Nk;
    A.Nkp = p.Nkp;
    A.NB = p.mma_NB;
    A.V = V;
    A.D = D;
    A.Gd = w.Gd;
    A.Bpart = w.Bpart;
    A.Hpart = w.Hpart;
    A.vpart = w.vpart;
    A.texp = w.texp;
    A.status = status;
    A.it = it;
    A.n_iter = n_iter;
    A.dpart = w.dpart;
    A.Gpart = w.Gpart;
    A.ypart = w.ypart;
    A.nby = p.nby;
    A.ysq = w.ysq;
    A.obj = obj;
    A.bar = bar;
    if (!PERSIST) {
        k_nmf_mma<K, NBW, false, MWT><<<p.nblk_f, MTH, smem, s>>>(A);
        return cudaGetLastError();
    }
    e = cudaMemsetAsync(bar, 0, sizeof(unsigned), s);  // grid-barrier arrival counter
    if (e != cudaSuccess) return e;
    void* args[] = {&A};
    return cudaLaunchCooperativeKernel((const void*)k_nmf_mma<K, NBW, true, MWT>, dim3(p.nblk_f), dim3(MTH), args, smem,
                                       s);
}

}  // namespace

// Per-K launchers (instantiated in nmf_mma_lo.cu, K <= 8, and nmf_mma_hi.cu, K = 9..16).
template <int K, bool PERSIST>
cudaError_t mma_launch_k(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D, int it, int n_iter,
                         double* obj, unsigned* bar, unsigned* status, cudaStream_t s) {
    switch (p.mma_NBW) {
#define C(NB) \
    case NB: return mma_klb<K, NB, PERSIST>(g, p, w, V, D, it, n_iter, obj, bar, status, s);
        C(2) C(4) C(6) C(8) C(10)
        case 13:
            if constexpr (mma_nc(K) == 1) return mma_klb<K, 13, PERSIST>(g, p, w, V, D, it, n_iter, obj, bar, status, s);
            return cudaErrorInvalidValue;
#undef C
        default: return cudaErrorInvalidValue;
    }
}

// K = 9..16 on 16 warps (plan.mma_MW = 16; instantiated in nmf_mma_hi16.cu): <= 5 blocks per warp
template <int K, bool PERSIST>
cudaError_t mma_launch_k16(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D, int it,
                           int n_iter, double* obj, unsigned* bar, unsigned* status, cudaStream_t s) {
    switch (p.mma_NBW) {
#define C(NB) \
    case NB: return mma_klb<K, NB, PERSIST, MW16>(g, p, w, V, D, it, n_iter, obj, bar, status, s);
        C(1) C(2) C(3) C(4) C(5)
#undef C
        default: return cudaErrorInvalidValue;
    }
}

#define HSNCT_MMA_EXTERN(KV)                                                                                  \
    extern template cudaError_t mma_launch_k<KV, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*,  \
                                                        float*, int, int, double*, unsigned*, unsigned*,         \
                                                        cudaStream_t);                                           \
    extern template cudaError_t mma_launch_k<KV, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*,   \
                                                       float*, int, int, double*, unsigned*, unsigned*,          \
                                                       cudaStream_t);
#define HSNCT_MMA16_EXTERN(KV)                                                                                \
    extern template cudaError_t mma_launch_k16<KV, false>(const Geometry&, const NmfPlan&, const NmfWs&, float*, \
                                                          float*, int, int, double*, unsigned*, unsigned*,       \
                                                          cudaStream_t);                                         \
    extern template cudaError_t mma_launch_k16<KV, true>(const Geometry&, const NmfPlan&, const NmfWs&, float*,  \
                                                         float*, int, int, double*, unsigned*, unsigned*,        \
                                                         cudaStream_t);
#define HSNCT_MMA_KHI(M) M(9) M(10) M(11) M(12) M(13) M(14) M(15) M(16)
HSNCT_MMA_KHI(HSNCT_MMA16_EXTERN)
#define HSNCT_MMA_K(M) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15) M(16)
HSNCT_MMA_K(HSNCT_MMA_EXTERN)

}  // namespace hsnct
