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
// call for Y+, one per component and warp (bin range) for D, one per component and tile for
// V.  Three MMAs per block (hi.hi + hi.lo + lo.hi; lo.lo is below 2^-22).  Phase-1
// accumulators run over one warp's 13 blocks; phase-2 accumulators cover one block of one tile
// and are added to the fp32 register sums with their scale (FFMA), so no tensor-core sum is
// longer than 39 MMAs.  Cross-warp and cross-CTA sums are fp32 / fp64 in a fixed order:
// deterministic.
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
    const unsigned* ymax; // bits of max Y+ (k_tc_stats)
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

// Dynamic shared memory: ring [MW][MNS][NBW*BLK] | old V rows [MNV][MR*K] | partial A
// [2][MW][32 reader lanes][4]
__host__ __device__ constexpr size_t mma_vrows_off(int NBW) { return (size_t)MW * MNS * NBW * BLK; }
__host__ __device__ constexpr size_t mma_red_off(int NBW, int K) {
    return mma_vrows_off(NBW) + (((size_t)MNV * MR * K * 4 + 15) & ~(size_t)15);
}
__host__ __device__ constexpr size_t mma_smem_bytes(int NBW, int K) {
    return mma_red_off(NBW, K) + (size_t)2 * MW * 128 * 4;
}

// The row pass (one iteration's V half-step and the B, H, <V_new, A> partials of each CTA) and,
// with PERSIST, all n_iter iterations in one cooperative launch with the D half-step between
// passes (grid barriers; the same fixed-order reductions as k_nmf_persist, nmf_fused.cuh).
// Tiles: CTA c owns c, c + nCTA, ... (forward in even iterations, backward in odd ones, so the
// tiles a pass ends with -- the ones most likely still in L2 -- start the next).
// Warp w owns the blocks [w NB / 8, (w + 1) NB / 8) of every tile; tile m's V store, H and
// <V_new, A> terms are taken by warp m % 8 (every warp holds the whole new V of the tile).
template <int K, int NBW, bool PERSIST>
__global__ void __launch_bounds__(MTH, 1) k_nmf_mma(MmaArgs A) {
    static_assert(K >= 1 && K <= 8, "one n8 column block");
    constexpr int KK = K * K;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t full[MW][MNS];
    __shared__ uint64_t vfull[MNV];
    __shared__ double hsh[MW][64];
    __shared__ double vsh[MW];
    __shared__ double Hs[KK], Gold[KK], Gnew[KK];
    __shared__ double red8[MW];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int c = blockIdx.x, nC = gridDim.x;
    const size_t slotb = (size_t)NBW * BLK;
    uint8_t* ring = smem;
    float* vrows = reinterpret_cast<float*>(smem + mma_vrows_off(NBW));
    float* red = reinterpret_cast<float*>(smem + mma_red_off(NBW, K));
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
    const int ey = mexp(__uint_as_float(*A.ymax));
    const float sy = pow2(ey), isy = pow2(-ey);
    // phase-2 ldmatrix.trans: lanes 8i..8i+7 address core matrix (0, 2, 1, 3)[i]
    const unsigned toff = (unsigned)((((lane >> 3) == 1) ? 2 : ((lane >> 3) == 2) ? 1 : (lane >> 3)) * 128 +
                                     (lane & 7) * 16);
    // partial-A exchange: the reader lane L = 4 k + u takes rows 2u, 2u+1, 2u+8, 2u+9 of component
    // k as one float4 at slot L ^ (k >> 1) (conflict-free reads, 2-way writes).  Writer offsets of
    // this lane's four accumulator values (A[g][2t], A[g][2t+1], A[g+8][2t], A[g+8][2t+1]):
    const int wsl0 = 8 * t + ((g >> 1) ^ t), wsl1 = 8 * t + 4 + ((g >> 1) ^ t);
    const int wo0 = 4 * wsl0 + (g & 1), wo1 = 4 * wsl1 + (g & 1);
    const int rsl = lane ^ (g >> 1);  // this lane's read slot (k = g, u = t)

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
        // column g of G (the V update's V G) and this warp's D operand (B of phase 1: K = bins,
        // N = components) as fp16 hi/lo, in registers for the pass.  D and G change between the
        // passes of a persistent launch: L2 loads (__ldcg), G from shared memory.
        float gcol[K];
#pragma unroll
        for (int j = 0; j < K; ++j) gcol[j] = g < K ? (float)Gold[j * K + g] : 0.f;
        uint32_t dh[NBW][2], dl[NBW][2];
        float invA0, invA1;  // 1 / (sigma_Y sigma_D[k]) for this lane's output columns k = 2t, 2t + 1
        {
            float dv[NBW][4];
            float mx = 0.f;
#pragma unroll
            for (int j = 0; j < NBW; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int l = 16 * (jb + j) + 2 * t + (e & 1) + (e >> 1) * 8;
                    dv[j][e] = (j < nb && g < K && l < A.Nk) ? __ldcg(A.D + (int64_t)g * A.Nk + l) : 0.f;
                    mx = fmaxf(mx, fabsf(dv[j][e]));
                }
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const int ed = mexp(mx);
            const float sd = pow2(ed);
#pragma unroll
            for (int j = 0; j < NBW; ++j) {
                dh[j][0] = split2(dv[j][0] * sd, dv[j][1] * sd, dl[j][0]);
                dh[j][1] = split2(dv[j][2] * sd, dv[j][3] * sd, dl[j][1]);
            }
            invA0 = isy * pow2(-__shfl_sync(0xffffffffu, ed, 8 * t));
            invA1 = isy * pow2(-__shfl_sync(0xffffffffu, ed, 8 * t + 4));
        }

        float bacc[NBW][4];
#pragma unroll
        for (int j = 0; j < NBW; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) bacc[j][e] = 0.f;
        double vdotA = 0.0;
        double hacc0 = 0.0, hacc1 = 0.0;
        unsigned bad = 0;

        for (int64_t m = 0; m < nmine; ++m) {
            const int64_t n = n0 + m;
            const int s = (int)(n % MNS);
            const unsigned par = (unsigned)((n / MNS) & 1);
            const int sv4 = (int)(n % MNV);
            const int64_t r0 = tile_of(m, fwd) * MR;
            const int nv = (int)min((int64_t)MR, A.Np - r0);
            mbar_wait(&full[warp][s], par);
            const unsigned sb = ringw + (unsigned)(s * slotb);
            // ---- phase 1: this warp's partial A = Y+_R D^T over its blocks.  Straight-line code
            //      over NBW blocks: blocks j >= nb re-read the last block with a zero D operand (no
            //      branches between the MMAs, so the compiler can overlap the blocks' latencies)
            float a0[4] = {0.f, 0.f, 0.f, 0.f}, a1[4] = {0.f, 0.f, 0.f, 0.f}, a2[4] = {0.f, 0.f, 0.f, 0.f};
            if (nb > 0) {
#pragma unroll
                for (int j = 0; j < NBW; ++j) {
                    const unsigned ba = sb + (unsigned)min(j, nb - 1) * BLK;
                    uint32_t yh[4], yl[4];
                    ldsm4(yh, ba + lane * 16);
                    ldsm4(yl, ba + 512 + lane * 16);
                    mma16816(a0, yh, dh[j][0], dh[j][1]);
                    mma16816(a1, yh, dl[j][0], dl[j][1]);
                    mma16816(a2, yl, dh[j][0], dh[j][1]);
                }
            }
            {
                float* rb = red + (size_t)((n & 1) * MW + warp) * 128;
                rb[wo0] = (a0[0] + (a1[0] + a2[0])) * invA0;
                rb[wo1] = (a0[1] + (a1[1] + a2[1])) * invA1;
                rb[wo0 + 2] = (a0[2] + (a1[2] + a2[2])) * invA0;
                rb[wo1 + 2] = (a0[3] + (a1[3] + a2[3])) * invA1;
            }
            // V G and the old V of this lane's four (row, component) pairs -- before the barrier, so
            // no warp can still be reading old V rows of a ragged tile (global memory) once the
            // tile's owner warp stores the new ones
            mbar_wait(&vfull[sv4], (unsigned)((n / MNV) & 1));
            float vg[4], vo[4];
            {
                const float* vr = nv == MR ? vrows + (size_t)sv4 * MR * K : A.V + r0 * K;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int r = 2 * t + (e & 1) + (e >> 1) * 8;
                    float x = 0.f, v0 = 0.f;
                    if (g < K && r < nv) {
#pragma unroll
                        for (int j = 0; j < K; ++j) x = fmaf(vr[r * K + j], gcol[j], x);
                        v0 = vr[r * K + g];
                    }
                    vg[e] = x;
                    vo[e] = v0;
                }
            }
            named_bar(1, MTH);
            // every warp has read the old V of tile m - 1: its V slot takes tile m + MNV - 1
            if (warp == 0 && lane == 0 && m >= 1 && m + MNV - 1 < nmine)
                issue_v((int)((n + MNV - 1) % MNV), m + MNV - 1, fwd);
            // ---- V update (every warp, redundantly): lane (g, t) -> component g, rows 2t, 2t+1,
            //      2t+8, 2t+9 -- exactly its part of the phase-2 B operand
            float av[4];
            {
                const float4* rd = reinterpret_cast<const float4*>(red + (size_t)((n & 1) * MW) * 128) + rsl;
                float4 s4 = rd[0];
#pragma unroll
                for (int w = 1; w < MW; ++w) {
                    const float4 q = rd[w * 32];
                    s4.x += q.x;
                    s4.y += q.y;
                    s4.z += q.z;
                    s4.w += q.w;
                }
                av[0] = s4.x;
                av[1] = s4.y;
                av[2] = s4.z;
                av[3] = s4.w;
            }
            float vn[4];
            float vmax = 0.f;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                // V / max(VG, 1e-30) by the approximate reciprocal (the divisor is a normal number;
                // 1 ulp); rows and components outside the tile have vo = 0
                vn[e] = av[e] * (vo[e] * rcp_approx(fmaxf(vg[e], 1e-30f)));
                vmax = fmaxf(vmax, fabsf(vn[e]));
            }
            vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, 1));
            vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, 2));
            const int ev = mexp(vmax);
            const float sv = pow2(ev);
            uint32_t vl0, vl1;
            const uint32_t vh0 = split2(vn[0] * sv, vn[1] * sv, vl0);
            const uint32_t vh1 = split2(vn[2] * sv, vn[3] * sv, vl1);
            const int ev0 = __shfl_sync(0xffffffffu, ev, 8 * t), ev1 = __shfl_sync(0xffffffffu, ev, 8 * t + 4);
            const float ivB0 = pow2(-ev0), ivB1 = pow2(-ev1);  // 1 / sigma_V[k], k = 2t, 2t + 1
            const float invB0 = isy * ivB0, invB1 = isy * ivB1;
            if (warp == (int)(m % MW)) {  // this tile's V store, <V_new, A>, H += V_new^T V_new
                float va = 0.f;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int r = 2 * t + (e & 1) + (e >> 1) * 8;
                    if (g < K && r < nv) {
                        if (first && !(isfinite(vo[e]) && vo[e] >= 0.f)) bad |= ST_INIT_BAD;
                        if (!isfinite(vn[e])) bad |= ST_NUMERIC;
                        A.V[(r0 + r) * K + g] = vn[e];
                        va = fmaf(vn[e], av[e], va);
                    }
                }
                vdotA += (double)va;
                // H on the tensor core: A operand V^T (its fragments are this lane's B operand),
                // C[g][2t + i] = sum_r V[r][g] V[r][2t + i], scaled by sigma_V[g] sigma_V[2t + i]
                const uint32_t ah[4] = {vh0, 0u, vh1, 0u}, al[4] = {vl0, 0u, vl1, 0u};
                float hc[4] = {0.f, 0.f, 0.f, 0.f};
                mma16816(hc, ah, vh0, vh1);
                mma16816(hc, ah, vl0, vl1);
                mma16816(hc, al, vh0, vh1);
                const float ivg = pow2(-ev);
                hacc0 += (double)(hc[0] * (ivg * ivB0));
                hacc1 += (double)(hc[1] * (ivg * ivB1));
            }
            // ---- phase 2: B^T[l][k] += sum_r Y+[r][l] V_new[r][k] over this warp's blocks (blocks
            //      j >= nb accumulate a copy of the last block into columns that are never stored)
            if (nb > 0) {
#pragma unroll
                for (int j = 0; j < NBW; ++j) {
                    const unsigned ba = sb + (unsigned)min(j, nb - 1) * BLK + toff;
                    uint32_t th[4], tl[4];
                    ldsm4t(th, ba);
                    ldsm4t(tl, ba + 512);
                    float cc[4] = {0.f, 0.f, 0.f, 0.f};
                    mma16816(cc, th, vh0, vh1);
                    mma16816(cc, th, vl0, vl1);
                    mma16816(cc, tl, vh0, vh1);
                    bacc[j][0] = fmaf(cc[0], invB0, bacc[j][0]);
                    bacc[j][1] = fmaf(cc[1], invB1, bacc[j][1]);
                    bacc[j][2] = fmaf(cc[2], invB0, bacc[j][2]);
                    bacc[j][3] = fmaf(cc[3], invB1, bacc[j][3]);
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
                const int k0 = 2 * t;
                if (k0 < K) {
                    if (l < A.Nk) Bo[(int64_t)k0 * A.Nkp + l] = bacc[j][0];
                    if (l + 8 < A.Nk) Bo[(int64_t)k0 * A.Nkp + l + 8] = bacc[j][2];
                }
                if (k0 + 1 < K) {
                    if (l < A.Nk) Bo[(int64_t)(k0 + 1) * A.Nkp + l] = bacc[j][1];
                    if (l + 8 < A.Nk) Bo[(int64_t)(k0 + 1) * A.Nkp + l + 8] = bacc[j][3];
                }
            }
        }
        hsh[warp][g * 8 + 2 * t] = hacc0;
        hsh[warp][g * 8 + 2 * t + 1] = hacc1;
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
            for (int w = 0; w < MW; ++w) h += hsh[w][ka * 8 + kb];
            A.Hpart[(int64_t)c * KK + tid] = h;
        }
        if (tid == 0) {
            double v = 0.0;
            for (int w = 0; w < MW; ++w) v += vsh[w];
            A.vpart[2 * (int64_t)c] = v;
            A.vpart[2 * (int64_t)c + 1] = 0.0;
        }
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
            double* dnew = Bsl + 256;                        // [K][64]
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

// Y+ (clamped, scaled by sigma_Y) split into fp16 hi/lo in the block layout above.  Item
// (tile, block, core matrix q, row rr), rr fastest: 32 consecutive threads write one block's
// hi and lo halves (512 contiguous bytes each); each reads 8 bins of one row.
__global__ void __launch_bounds__(256) k_mma_convert(const float* __restrict__ Y, int64_t ld, int64_t Np, int Nk,
                                                     int NB, int64_t ntiles, const unsigned* __restrict__ ymax,
                                                     uint8_t* __restrict__ Yc) {
    const float sy = pow2(mexp(__uint_as_float(*ymax)));
    const int64_t n = ntiles * NB * 32;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int rr = (int)(i & 7), q = (int)((i >> 3) & 3);
        const int64_t u = i >> 5;
        const int j = (int)(u % NB);
        const int64_t tt = u / NB;
        const int64_t r = tt * MR + (q & 1) * 8 + rr;
        const int l = 16 * j + (q >> 1) * 8;
        float v[8];
        if (r < Np && l + 8 <= Nk) {
            const float4* y = reinterpret_cast<const float4*>(Y + r * ld + l);
            const float4 a = __ldg(y), b = __ldg(y + 1);
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = (r < Np && l + e < Nk) ? Y[r * ld + l + e] : 0.f;
        }
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
            hw[e] = split2(fmaxf(v[2 * e], 0.f) * sy, fmaxf(v[2 * e + 1], 0.f) * sy, lw[e]);
        uint8_t* dst = Yc + (size_t)u * BLK + q * 128 + rr * 16;
        *reinterpret_cast<uint4*>(dst) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(dst + 512) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}

// ---- counts-domain input (NEXT-1): Eq. 2 with the Appendix-A offset decoded straight into the
// block layout, Y = fp32((L[y0] - L[y]) - b) with the fp64 table L[n] = ln max(n, 1/2)
// (counts.cu, R7): the same per-element value as hsnct_counts_to_projections, and the
// two kernels below have the loop structure of k_tc_stats / k_mma_convert, so the decomposition
// from counts is bit-identical to the one from the materialised Y.
struct CountsSrc {
    const uint8_t* y;    // [Np][Nk]
    const uint8_t* y0;   // [Nr Nc][Nk]
    const float* b;      // [Nv][Nk] or null
    const double* L;     // [256] (device table)
    int64_t NrNc;
    int Nk;
};
struct CountsRow {  // the rows of y, y0 and b that row p of Y decodes from
    const uint8_t* y;
    const uint8_t* y0;
    const float* b;
};
__device__ __forceinline__ CountsRow counts_row(const CountsSrc& C, int64_t p) {
    const int64_t v = p / C.NrNc, rc = p - v * C.NrNc;
    return {C.y + p * C.Nk, C.y0 + rc * C.Nk, C.b ? C.b + v * C.Nk : nullptr};
}
__device__ __forceinline__ float decode1(const CountsRow& R, const double* Ls, int l) {
    double d = Ls[R.y0[l]] - Ls[R.y[l]];
    if (R.b) d -= (double)R.b[l];
    return (float)d;
}

// k_tc_stats (nmf_tc.cu) on decoded counts: max Y+ (bits), ||Y+||^2 per-block partials (same
// per-row order), non-finite check (b), clamped count.  One warp per row.
__global__ void __launch_bounds__(256) k_mma_counts_stats(CountsSrc C, int64_t Np, unsigned* __restrict__ ymax,
                                                          double* __restrict__ ypart, unsigned* __restrict__ status,
                                                          unsigned long long* __restrict__ nclamp) {
    __shared__ double Ls[256];
    __shared__ double red[8];
    __shared__ unsigned mred[8], cred[8];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) Ls[i] = C.L[i];
    __syncthreads();
    unsigned ncl = 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nq = (C.Nk + 3) >> 2;
    double s = 0.0;
    unsigned m = 0, bad = 0;
    for (int64_t r = (int64_t)blockIdx.x * 8 + w; r < Np; r += (int64_t)gridDim.x * 8) {
        const CountsRow R = counts_row(C, r);
        float ps = 0.f;
        for (int q = lane; q < nq; q += 32) {
            const int l = 4 * q;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float vj = l + j < C.Nk ? decode1(R, Ls, l + j) : 0.f;
                if (!isfinite(vj)) bad = ST_Y_NONFINITE;
                ncl += vj < 0.f;
                const float yp = fmaxf(vj, 0.f);
                m = max(m, __float_as_uint(yp));
                ps = fmaf(yp, yp, ps);
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
        s += (double)ps;
    }
    m = __reduce_max_sync(0xffffffffu, m);
    bad = __reduce_or_sync(0xffffffffu, bad);
    ncl = __reduce_add_sync(0xffffffffu, ncl);
    if (lane == 0) {  // (s is the same in every lane: the row sums were reduced over the warp)
        red[w] = s;
        mred[w] = m;
        cred[w] = ncl;
        if (bad) atomicOr(status, bad);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tt = 0.0;
        unsigned mm = 0;
        unsigned long long cc = 0;
        for (int j = 0; j < 8; ++j) {
            tt += red[j];
            mm = max(mm, mred[j]);
            cc += cred[j];
        }
        ypart[blockIdx.x] = tt;
        if (cc) atomicAdd(nclamp, cc);
        if (mm) atomicMax(ymax, mm);
    }
}

// k_mma_convert on decoded counts
__global__ void __launch_bounds__(256) k_mma_counts_convert(CountsSrc C, int64_t Np, int NB, int64_t ntiles,
                                                            const unsigned* __restrict__ ymax,
                                                            uint8_t* __restrict__ Yc) {
    __shared__ double Ls[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) Ls[i] = C.L[i];
    __syncthreads();
    const float sy = pow2(mexp(__uint_as_float(*ymax)));
    const int64_t n = ntiles * NB * 32;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int rr = (int)(i & 7), q = (int)((i >> 3) & 3);
        const int64_t u = i >> 5;
        const int j = (int)(u % NB);
        const int64_t tt = u / NB;
        const int64_t r = tt * MR + (q & 1) * 8 + rr;
        const int l = 16 * j + (q >> 1) * 8;
        float v[8];
        const CountsRow R = counts_row(C, r < Np ? r : 0);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = (r < Np && l + e < C.Nk) ? decode1(R, Ls, l + e) : 0.f;
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
            hw[e] = split2(fmaxf(v[2 * e], 0.f) * sy, fmaxf(v[2 * e + 1], 0.f) * sy, lw[e]);
        uint8_t* dst = Yc + (size_t)u * BLK + q * 128 + rr * 16;
        *reinterpret_cast<uint4*>(dst) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(dst + 512) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
}

template <int K, int NBW, bool PERSIST>
cudaError_t mma_klb(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D, int it, int n_iter,
                    double* obj, unsigned* bar, unsigned* status, cudaStream_t s) {
    static SmemAttr attr;
    const size_t smem = mma_smem_bytes(NBW, K);
    cudaError_t e = ensure_smem((const void*)k_nmf_mma<K, NBW, PERSIST>, (int)smem, attr);
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
    A.ymax = w.ymax;
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
        k_nmf_mma<K, NBW, false><<<p.nblk_f, MTH, smem, s>>>(A);
        return cudaGetLastError();
    }
    e = cudaMemsetAsync(bar, 0, sizeof(unsigned), s);  // grid-barrier arrival counter
    if (e != cudaSuccess) return e;
    void* args[] = {&A};
    return cudaLaunchCooperativeKernel((const void*)k_nmf_mma<K, NBW, true>, dim3(p.nblk_f), dim3(MTH), args, smem,
                                       s);
}

// blocks per warp instantiated: the smallest of these >= ceil(NB / 8)
constexpr int NBW_SET[] = {2, 4, 6, 8, 10, 13};
int nbw_of(int NB) {
    const int need = (NB + MW - 1) / MW;
    for (int v : NBW_SET)
        if (v >= need) return v;
    return 0;
}

template <int K, bool PERSIST>
cudaError_t mma_launch_k(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D, int it, int n_iter,
                         double* obj, unsigned* bar, unsigned* status, cudaStream_t s) {
    switch (p.mma_NBW) {
#define C(NB) \
    case NB: return mma_klb<K, NB, PERSIST>(g, p, w, V, D, it, n_iter, obj, bar, status, s);
        C(2) C(4) C(6) C(8) C(10) C(13)
#undef C
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

bool nmf_mma_plan(const Geometry& g, int num_sms, NmfPlan* p) {
    if (g.K > 8) return false;
    const int NB = (g.Nk + 15) / 16;
    const int nbw = nbw_of(NB);
    if (!nbw) return false;
    const size_t smem = mma_smem_bytes(nbw, g.K);
    if (smem + 6144 > (size_t)232448) return false;  // 227 KB per block with the static part
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    const int64_t ntiles = (Np + MR - 1) / MR;
    // the persistent launch's D update: lambda slices of SL = ceil(Nk / nCTA) bins per CTA (dnew
    // holds 64 per component, Bsl 256 values, threads [0, K*K + K*SL) produce the outputs)
    {
        const int nC = (int)std::max<int64_t>(1, std::min<int64_t>((Np + MR - 1) / MR, (int64_t)num_sms));
        const int SL = (g.Nk + nC - 1) / nC;
        p->persist_fits = SL <= 64 && g.K * SL <= 256 && g.K * g.K + g.K * SL <= MTH;
    }
    p->mma_NB = NB;
    p->mma_NBW = nbw;
    p->mma_Npad = ntiles * MR;
    p->nblk_f = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)num_sms));
    p->nby = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms * 8, (Np + 7) / 8));
    return true;
}

cudaError_t nmf_mma_prepare(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y, int64_t ld_y,
                            unsigned* status, cudaStream_t s) {
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    cudaError_t e = nmf_tc_stats(g, p, w, Y, ld_y, status, s);
    if (e != cudaSuccess) return e;
    k_mma_convert<<<g.num_sms * 16, 256, 0, s>>>(Y, ld_y, Np, g.Nk, p.mma_NB, p.mma_Npad / MR, w.ymax,
                                                  static_cast<uint8_t*>(w.Yc));
    return cudaGetLastError();
}

cudaError_t nmf_mma_prepare_counts(const Geometry& g, const NmfPlan& p, const NmfWs& w, const DeviceTables& t,
                                   const CountsIn& cin, unsigned* status, cudaStream_t s) {
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    const CountsSrc C{cin.y, cin.y0, cin.b, t.logtab, (int64_t)g.Nr * g.Nc, g.Nk};
    cudaError_t e = cudaMemsetAsync(w.ymax, 0, 2 * sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    k_mma_counts_stats<<<p.nby, 256, 0, s>>>(C, Np, w.ymax, w.ypart, status, w.nclamp);
    k_mma_counts_convert<<<g.num_sms * 16, 256, 0, s>>>(C, Np, p.mma_NB, p.mma_Npad / MR, w.ymax,
                                                         static_cast<uint8_t*>(w.Yc));
    return cudaGetLastError();
}

cudaError_t nmf_mma_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D, int it,
                           unsigned* status, cudaStream_t s) {
    switch (g.K) {
#define M(KV) \
    case KV: return mma_launch_k<KV, false>(g, p, w, V, const_cast<float*>(D), it, 1, nullptr, nullptr, status, s);
        M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8)
#undef M
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t nmf_mma_persist_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D,
                                   int n_iter, double* obj, unsigned* bar, unsigned* status, cudaStream_t s) {
    switch (g.K) {
#define M(KV) \
    case KV: return mma_launch_k<KV, true>(g, p, w, V, D, 0, n_iter, obj, bar, status, s);
        M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8)
#undef M
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace hsnct
