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
    const float* D;
    const double* Gd;
    float* Bpart;         // [nCTA][K][Nkp]
    double* Hpart;        // [nCTA][K*K]
    double* vpart;        // [nCTA][2]
    const unsigned* ymax; // bits of max Y+ (k_tc_stats)
    unsigned* status;
    int it;
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

// One row pass (one iteration's V half-step and the B, H, <V_new, A> partials of this CTA).
// Tiles: CTA c owns c, c + nCTA, ... (forward in even iterations, backward in odd ones).
// Warp w owns the blocks [w NB / 8, (w + 1) NB / 8) of every tile; tile m's V store, H and
// <V_new, A> terms are taken by warp m % 8 (every warp holds the whole new V of the tile).
template <int K, int NBW>
__global__ void __launch_bounds__(MTH, 1) k_nmf_mma(MmaArgs A) {
    static_assert(K >= 1 && K <= 8, "one n8 column block");
    constexpr int KK = K * K;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t full[MW][MNS];
    __shared__ uint64_t vfull[MNV];
    __shared__ double hsh[MW][64];
    __shared__ double vsh[MW];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int c = blockIdx.x, nC = gridDim.x;
    const size_t slotb = (size_t)NBW * BLK;
    uint8_t* ring = smem;
    float* vrows = reinterpret_cast<float*>(smem + mma_vrows_off(NBW));
    float* red = reinterpret_cast<float*>(smem + mma_red_off(NBW, K));
    const int jb = warp * A.NB / MW, nb = (warp + 1) * A.NB / MW - jb;
    const int64_t ntiles = (A.Np + MR - 1) / MR;
    const int64_t nmine = ntiles > c ? (ntiles - 1 - c) / nC + 1 : 0;
    const bool fwd = (A.it & 1) == 0;
    auto tile_of = [&](int64_t q) { return (int64_t)c + (fwd ? q : nmine - 1 - q) * nC; };
    if (tid == 0) {
        for (int w = 0; w < MW; ++w)
            for (int s = 0; s < MNS; ++s) mbar_init(&full[w][s], 1);
        for (int s = 0; s < MNV; ++s) mbar_init(&vfull[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint8_t* myring = ring + (size_t)warp * MNS * slotb;
    const unsigned ringw = smem_u32(myring);
    auto issue_y = [&](int s, int64_t q) {  // lane 0: this warp's chunk of tile q into slot s
        const unsigned bytes = (unsigned)nb * BLK;
        mbar_expect_tx(&full[warp][s], bytes);  // 0 bytes (nb = 0): completes the phase
        if (bytes) bulk_g2s(myring + (size_t)s * slotb, A.Yc + ((size_t)tile_of(q) * A.NB + jb) * BLK, bytes,
                            &full[warp][s]);
    };
    auto issue_v = [&](int64_t q) {  // warp 0 lane 0: old V rows of tile q (full tiles; else arrive)
        const int s = (int)(q % MNV);
        const int64_t r0 = tile_of(q) * MR;
        if (r0 + MR <= A.Np) {
            mbar_expect_tx(&vfull[s], (unsigned)(MR * K * 4));
            bulk_g2s(vrows + (size_t)s * MR * K, A.V + r0 * K, (unsigned)(MR * K * 4), &vfull[s]);
        } else {
            mbar_arrive_cta(&vfull[s]);
        }
    };
    if (lane == 0) {
        for (int64_t q = 0; q < min((int64_t)MNS, nmine); ++q) issue_y((int)q, q);
        if (warp == 0)
            for (int64_t q = 0; q < min((int64_t)MNV, nmine); ++q) issue_v(q);
    }

    // column g of G (the V update's V G) in registers
    float gcol[K];
#pragma unroll
    for (int j = 0; j < K; ++j) gcol[j] = g < K ? (float)A.Gd[j * K + g] : 0.f;
    // ---- this warp's D operand (B of phase 1: K = bins, N = components), hi/lo, in registers
    const int ey = mexp(__uint_as_float(*A.ymax));
    const float sy = pow2(ey), isy = pow2(-ey);
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
                dv[j][e] = (j < nb && g < K && l < A.Nk) ? __ldg(A.D + (int64_t)g * A.Nk + l) : 0.f;
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
    const bool first = A.it == 0;
    // phase-2 ldmatrix.trans: lanes 8i..8i+7 address core matrix (0, 2, 1, 3)[i]
    const unsigned toff = (unsigned)((((lane >> 3) == 1) ? 2 : ((lane >> 3) == 2) ? 1 : (lane >> 3)) * 128 +
                                     (lane & 7) * 16);
    // partial-A exchange: the reader lane L = 4 k + u takes rows 2u, 2u+1, 2u+8, 2u+9 of component
    // k as one float4 at slot L ^ (k >> 1) (conflict-free reads, 2-way writes).  Writer offsets of
    // this lane's four accumulator values (A[g][2t], A[g][2t+1], A[g+8][2t], A[g+8][2t+1]):
    const int wsl0 = 8 * t + ((g >> 1) ^ t), wsl1 = 8 * t + 4 + ((g >> 1) ^ t);
    const int wo0 = 4 * wsl0 + (g & 1), wo1 = 4 * wsl1 + (g & 1);
    const int rsl = lane ^ (g >> 1);  // this lane's read slot (k = g, u = t)

    for (int64_t m = 0; m < nmine; ++m) {
        const int s = (int)(m % MNS);
        const unsigned par = (unsigned)((m / MNS) & 1);
        const int64_t r0 = tile_of(m) * MR;
        const int nv = (int)min((int64_t)MR, A.Np - r0);
        mbar_wait(&full[warp][s], par);
        const unsigned sb = ringw + (unsigned)(s * slotb);
        // ---- phase 1: this warp's partial A = Y+_R D^T over its blocks.  Straight-line code over
        //      NBW blocks: blocks j >= nb re-read the last block with a zero D operand (no
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
            float* rb = red + (size_t)((m & 1) * MW + warp) * 128;
            rb[wo0] = (a0[0] + (a1[0] + a2[0])) * invA0;
            rb[wo1] = (a0[1] + (a1[1] + a2[1])) * invA1;
            rb[wo0 + 2] = (a0[2] + (a1[2] + a2[2])) * invA0;
            rb[wo1 + 2] = (a0[3] + (a1[3] + a2[3])) * invA1;
        }
        // V G and the old V of this lane's four (row, component) pairs -- before the barrier, so
        // no warp can still be reading old V rows of a ragged tile (global memory) once the
        // tile's owner warp stores the new ones
        mbar_wait(&vfull[m % MNV], (unsigned)((m / MNV) & 1));
        float vg[4], vo[4];
        {
            const float* vr = nv == MR ? vrows + (size_t)(m % MNV) * MR * K : A.V + r0 * K;
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
        // every warp has finished the V update of tile m - 1: its old-V slot takes tile m + MNV - 1
        if (warp == 0 && lane == 0 && m >= 1 && m + MNV - 1 < nmine) issue_v(m + MNV - 1);
        // ---- V update (every warp, redundantly): lane (g, t) -> component g, rows 2t, 2t+1,
        //      2t+8, 2t+9 -- exactly its part of the phase-2 B operand
        float av[4];
        {
            const float4* rd = reinterpret_cast<const float4*>(red + (size_t)((m & 1) * MW) * 128) + rsl;
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
            const int r = 2 * t + (e & 1) + (e >> 1) * 8;
            // V / max(VG, 1e-30) by the approximate reciprocal (the divisor is a normal number;
            // 1 ulp); rows and components outside the tile have vo = 0
            (void)r;
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
            issue_y(s, m + MNS);
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

template <int K, int NBW>
cudaError_t mma_klb(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D, int it,
                    unsigned* status, cudaStream_t s) {
    static SmemAttr attr;
    const size_t smem = mma_smem_bytes(NBW, K);
    cudaError_t e = ensure_smem((const void*)k_nmf_mma<K, NBW>, (int)smem, attr);
    if (e != cudaSuccess) return e;
    MmaArgs A;
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
    k_nmf_mma<K, NBW><<<p.nblk_f, MTH, smem, s>>>(A);
    return cudaGetLastError();
}

// blocks per warp instantiated: the smallest of these >= ceil(NB / 8)
constexpr int NBW_SET[] = {2, 4, 8, 13};
int nbw_of(int NB) {
    const int need = (NB + MW - 1) / MW;
    for (int v : NBW_SET)
        if (v >= need) return v;
    return 0;
}

template <int K>
cudaError_t mma_launch_k(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D, int it,
                         unsigned* status, cudaStream_t s) {
    switch (p.mma_NBW) {
        case 2: return mma_klb<K, 2>(g, p, w, V, D, it, status, s);
        case 4: return mma_klb<K, 4>(g, p, w, V, D, it, status, s);
        case 8: return mma_klb<K, 8>(g, p, w, V, D, it, status, s);
        case 13: return mma_klb<K, 13>(g, p, w, V, D, it, status, s);
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
    if (smem + 2048 > (size_t)232448) return false;  // 227 KB per block with the static part
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    const int64_t ntiles = (Np + MR - 1) / MR;
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

cudaError_t nmf_mma_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D, int it,
                           unsigned* status, cudaStream_t s) {
    switch (g.K) {
#define M(KV) \
    case KV: return mma_launch_k<KV>(g, p, w, V, D, it, status, s);
        M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8)
#undef M
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace hsnct
