// Fused single-pass Lee-Seung iteration (Eq. 4; R1-R3):
// one read of Y+ per iteration serves both contractions.
//
// Input is Y+ = max(Y, 0) materialised once per decompose call by k_yplus
// (compact rows of Nkp floats, zero padding), so the hot loop carries no clamp,
// mask or ld.  One persistent CTA per SM; CTA c owns the 4-row tiles
// c, c + nCTA, c + 2 nCTA, ... (a static schedule, identical every iteration),
// visited forward in even iterations and backward in odd ones, so the tiles a CTA
// finishes an iteration with -- the ones most likely still in L2 -- are the first
// it reads in the next.
//
// The CTA is NGRP = 3 compute groups of 4 warps.  Group g takes every third tile
// of the CTA's sequence and runs its own pipeline:
//   * its tiles arrive by cp.async.bulk (4 Y+ rows + the 4 old V rows, one
//     mbarrier per ring slot, NBG slots per group); the last warp to release a slot
//     refills it, so no thread ever waits to issue a copy;
//   * thread t of the group owns the lambda pairs 2(t + 128 i), i < LP, for the
//     whole kernel, with the matching columns of the group's partial B = V^T Y+ in
//     registers;
//   * phase 1: part[r][k] = sum_l Y+[r][l] D[k][l] (D from smem, packed f32x2 FMA
//     when registers allow), warp transpose-reduce -> smem; named barrier;
//     warp 0 sums the 4 warp partials in a fixed order and updates
//     V[r][k] <- V[r][k] A[r][k] / max(sum_j V[r][j] G[j][k], 1e-30); named barrier;
//     warp 0 stores V and accumulates <V_new, A>, warp 1 accumulates H += V_new^T V_new
//     (fp64); phase 2: B[k][l] += V_new[r][k] Y+[r][l] (packed f32x2 FMA).
// While one group sits in its V-update barrier the other two keep the SM's four
// schedulers busy.  Per-CTA partials (B: groups combined in the fixed order
// (g0 + g1) + g2; H; <V_new, A>) are reduced in a fixed order by the D update.
// Deterministic: static schedule, fixed reduction trees, no floating-point atomics.
#pragma once
#include <algorithm>

#include "internal.h"
#include "nmf_common.cuh"

namespace hsnct {
namespace {

constexpr int RG = 4;              // rows per tile
constexpr int GW = 4;              // warps per group
constexpr int TG = GW * 32;        // threads per group
constexpr int NTHREADS = 3 * TG;   // default CTA size (3 groups); 4 groups when registers allow
// Warp of group g that stores V / accumulates H: (g + 3) % 4 and (g + 2) % 4, never the warp
// g % 4 that carries the ragged last lambda pairs (see the slot rotation in Pass::run).

// d = a * b + c on both halves (one packed FFMA2 on sm_100a), each half rounded
// exactly like fmaf.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\t"
        "mov.b64 rb, {%4, %5};\n\t"
        "mov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
        "mov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
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
template <int N, int O0 = 16>
__device__ __forceinline__ int tr_base(int lane) {
    int b = 0, n = N;
#pragma unroll
    for (int o = O0; o; o >>= 1) {
        if (n % 2 == 0) {
            if (lane & o) b += n / 2;
            n /= 2;
        }
    }
    return b;
}

// Y+ = max(Y, 0) into compact rows of Nkp floats (padding = 0); flags non-finite
// Y (the clamp would hide NaN); per-block ||Y+||^2 partials (fp64).  One warp per
// row at a time, lanes over lambda quads.
__global__ void __launch_bounds__(256) k_yplus(const float* __restrict__ Y, int64_t ld, int64_t Np, int Nk,
                                               int Nkp, float* __restrict__ Yp, double* __restrict__ ypart,
                                               unsigned* __restrict__ status,
                                               unsigned long long* __restrict__ nclamp) {
    __shared__ double red[8];
    __shared__ unsigned cred[8];
    unsigned ncl = 0;
    const int nq = Nkp >> 2;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t nw = (int64_t)gridDim.x * 8;
    double s = 0.0;
    unsigned bad = 0;
    for (int64_t p = (int64_t)blockIdx.x * 8 + w; p < Np; p += nw) {
        const float4* src = reinterpret_cast<const float4*>(Y + p * ld);
        float4* dst = reinterpret_cast<float4*>(Yp + p * Nkp);
        float rs = 0.f;
#pragma unroll 4
        for (int q = lane; q < nq; q += 32) {
            float4 y = __ldcs(src + q);
            const int l0 = 4 * q;
            if (l0 + 3 >= Nk) {
                if (l0 + 0 >= Nk) y.x = 0.f;
                if (l0 + 1 >= Nk) y.y = 0.f;
                if (l0 + 2 >= Nk) y.z = 0.f;
                if (l0 + 3 >= Nk) y.w = 0.f;
            }
            if (!(isfinite(y.x) && isfinite(y.y) && isfinite(y.z) && isfinite(y.w))) bad = ST_Y_NONFINITE;
            ncl += (y.x < 0.f) + (y.y < 0.f) + (y.z < 0.f) + (y.w < 0.f);
            y.x = fmaxf(y.x, 0.f);
            y.y = fmaxf(y.y, 0.f);
            y.z = fmaxf(y.z, 0.f);
            y.w = fmaxf(y.w, 0.f);
            rs = fmaf(y.x, y.x, fmaf(y.y, y.y, fmaf(y.z, y.z, fmaf(y.w, y.w, rs))));
            dst[q] = y;
        }
        s += (double)rs;
    }
    s = warp_sum_d(s);
#pragma unroll
    for (int o = 16; o; o >>= 1) bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    ncl = __reduce_add_sync(0xffffffffu, ncl);
    if (lane == 0) {
        red[w] = s;
        cred[w] = ncl;
        if (bad) atomicOr(status, bad);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        unsigned long long c = 0;
        for (int i = 0; i < 8; ++i) {
            t += red[i];
            c += cred[i];
        }
        ypart[blockIdx.x] = t;
        if (c) atomicAdd(nclamp, c);
    }
}

template <int K, int NBG, int NGRP>
struct FusedShared {
    static constexpr int GK = RG * K;
    static constexpr int KP = (K + 3) & ~3;
    static constexpr int KK = K * K;
    uint64_t full[NGRP][NBG];
    uint64_t part[NGRP][2];   // a group's four warp partials of a tile are in (pipelined schedule)
    unsigned rel[NGRP][NBG];
    float red[NGRP][2][GW][GK];               // per-warp row partials, by tile parity
    __align__(16) float Vn[NGRP][GW][RG][KP];  // each warp's copy of the tile's new V rows
    float Gs[KK];
    double hs[NGRP][KK];
    double vs[NGRP];
    unsigned bad;
};

// Dynamic shared memory layout (floats):
//   ring  [NGRP][NBG][tile]  tile = RG*Nkp Y+ values + RG*K old V values; between
//                            passes (no copy in flight) it is the group-combine scratch
//   Ds    [Nkp][KD]          D transposed (lambda-major, KD = K rounded up to even, zero
//                            padded), in 16-byte chunks swizzled per lambda pair (ds_index)
//   Bsl   [SCR/2] doubles    the CTA's lambda slice of B in the D update
// No thread reads past column Nkp of a row (the last lambda pair is guarded).
constexpr int SCR = 8 * 64;
__host__ __device__ constexpr size_t tile_floats_of(int Nkp, int K) { return (size_t)RG * Nkp + (size_t)RG * K; }

// D in shared memory, lambda-major: the 2*KD values of lambda pair p (D[0..KD)[2p],
// D[0..KD)[2p+1]) are C = KD/2 consecutive 16-byte chunks, chunk j stored at slot
// j ^ swz(p).  A thread reads its pair's chunks with LDS.128; the XOR swizzle makes the 8
// lanes of each quarter-warp hit distinct 16-byte bank groups when C is even (odd C is
// conflict-free as is).
template <int K>
struct DLayout {
    static constexpr int KD = (K + 1) & ~1;
    static constexpr int C = KD / 2;   // float4 chunks per lambda pair
    __host__ __device__ static constexpr int swz(int p) {
        return C == 2 ? ((p >> 2) & 1) : (C == 4 ? ((p >> 1) & 3) : 0);
    }
    // float index of D[k][l] (k < KD)
    __device__ static __forceinline__ int index(int l, int k) {
        const int p = l >> 1, f = (l & 1) * KD + k;
        return ((p * C + ((f >> 2) ^ swz(p))) << 2) + (f & 3);
    }
};

template <int K, int LP, int NBG, int NGRP>
struct Pass {
    static constexpr int GK = RG * K;
    static constexpr int NE = (GK + 31) / 32;  // (tile row, component) elements per lane in the V update
    static constexpr int KP = (K + 3) & ~3;
    static constexpr int KK = K * K;
    static constexpr int DS = 2 * TG * LP;
    using Sh = FusedShared<K, NBG, NGRP>;
    static constexpr int NTH = NGRP * TG;
    // pipelined group schedule (phase 2 of tile m - 1 overlaps the partial-sum wait of tile m)
    // when each group has a third ring slot to prefetch into
    static constexpr bool PIPE = NBG >= 3;
    // warps none of whose lanes has a last lambda pair skip that slot (a warp-uniform branch).
    // Three groups only: at four (128 registers) the branch measured slower than multiplying
    // zeros (C2 49.1 -> 50.0 us per iteration), at three it pays with the slot rotation.
    static constexpr bool SKIP = NGRP == 3;
    // lane-dependent phase-1 row order, select-free first two steps of the transpose-reduce
    // (three groups: C4 6.34 -> 6.22 ms; at four groups' 128 registers it spilled, C2 +7%)
    static constexpr bool RSWAP = NGRP == 3;
    // four groups: only the first halving select-free (C2 48.3 -> 47.5 us; both halvings spilled)
    static constexpr bool RSWAP1 = NGRP == 4;

    const float* __restrict__ Yp;
    int64_t Np;
    int Nkp;
    float* __restrict__ V;
    float* ring;
    const float* Ds;
    Sh& sh;
    int64_t nmine;   // tiles of this CTA
    size_t tf;       // floats per tile
    bool rotate;     // rotate the lambda slots per group (see run)
    bool l2pf;       // L2 prefetch of the tile after the one being refilled

    __device__ __forceinline__ int64_t count_g(int g) const {
        return nmine > g ? (nmine - 1 - g) / NGRP + 1 : 0;
    }
    __device__ __forceinline__ int64_t row0(int64_t q, bool fwd) const {
        const int64_t pos = fwd ? q : (nmine - 1 - q);
        return ((int64_t)blockIdx.x + pos * (int64_t)gridDim.x) * RG;
    }
    // Row step between consecutive tiles of one group in a pass (direction fwd).
    __device__ __forceinline__ int64_t rstride(bool fwd) const {
        return (fwd ? (int64_t)1 : (int64_t)-1) * NGRP * (int64_t)gridDim.x * RG;
    }
    // Copy the tile starting at row r0 (4 Y+ rows, then its 4 old V rows) into slot b of group g.
    __device__ __forceinline__ void issue(int g, int b, int64_t r0) const {
        const int nv = (int)min((int64_t)RG, Np - r0);
        const unsigned bytes = (unsigned)(nv * Nkp * sizeof(float));
        const unsigned vbytes = nv == RG ? (unsigned)(RG * K * sizeof(float)) : 0u;  // 16K bytes
        uint64_t* bar = &sh.full[g][b];
        mbar_expect_tx(bar, bytes + vbytes);
        float* slot = ring + (size_t)(g * NBG + b) * tf;
        bulk_g2s(slot, Yp + r0 * Nkp, bytes, bar);
        if (vbytes) bulk_g2s(slot + (size_t)RG * Nkp, V + r0 * K, vbytes, bar);
    }
    // Leader of group g: the first NBG tiles of a pass (running group tile counter n0).
    __device__ __forceinline__ void issue_head(int g, int64_t n0, bool fwd) const {
        const int64_t c = count_g(g);
        int b = (int)(n0 % NBG);
        int64_t r0 = row0(g, fwd);
        for (int64_t m = 0; m < min((int64_t)NBG, c); ++m) {
            issue(g, b, r0);
            b = b + 1 == NBG ? 0 : b + 1;
            r0 += rstride(fwd);
        }
    }

    // One pass over this CTA's tiles with the current D (Ds) and G (sh.Gs).
    // n0: running group tile counter at the start of the pass (mbarrier phases).
    // If !prefetched the pass issues its own head tiles; if next >= 0 the head tiles
    // of the next pass (direction next_fwd) are issued once this pass is done.
    // On return (all threads): Bout[K][Nkp], Hout[KK], *vout written.
    __device__ void run(int64_t n0, bool first, bool fwd, bool prefetched, bool prefetch_next, bool next_fwd,
                        float* __restrict__ Bout, double* __restrict__ Hout, double* __restrict__ vout) const {
        const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
        const int g = warp / GW, wg = warp - g * GW, t = tid - g * TG;
        // lambda-slot index of this thread: the warps of group g take the slots rotated by g,
        // so the warp that carries the ragged last lambda pairs (slots < 32) is warp g % GW --
        // a different SM sub-partition for every group (warp w runs on sub-partition w % 4)
        const int rot = rotate ? g % GW : 0;
        const int tl = ((wg - rot + GW) % GW) * 32 + lane;
        const int VWARP = (rot + GW - 1) % GW, HWARP = (rot + GW - 2) % GW;
        const int64_t cnt = count_g(g);
        if (!prefetched) {
            if (t == 0) {
                fence_proxy_async_global();
                fence_proxy_async();
                issue_head(g, n0, fwd);
            }
        }
        const bool lastok = 2 * (tl + TG * (LP - 1)) < Nkp;  // last lambda pair inside the row
        // warp-uniform: some lane of this warp has its last lambda pair inside the row (the
        // other warps skip the last slot instead of multiplying zeros)
        const bool wlast = 2 * (tl - lane + TG * (LP - 1)) < Nkp;
        float2 bacc[K][LP];
#pragma unroll
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int i = 0; i < LP; ++i) bacc[k][i] = make_float2(0.f, 0.f);
        using DL = DLayout<K>;
        constexpr int KD = DL::KD, C = DL::C;
        double vdotA = 0.0;
        double hacc[(KK + 31) / 32];
#pragma unroll
        for (int x = 0; x < (KK + 31) / 32; ++x) hacc[x] = 0.0;
        unsigned bad = 0;
        const unsigned fullb = smem_u32(&sh.full[g][0]), partb = smem_u32(&sh.part[g][0]);
        const int rsw = ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1);  // phase-1 row swap (see the reduction)
        // running slot / mbarrier phase / first row of the group's current tile (no 64-bit
        // division or multiply per tile)
        int b = (int)(n0 % NBG);
        unsigned ph = (unsigned)((n0 / NBG) & 1);
        const int64_t rs = rstride(fwd);
        int64_t r0 = row0(g, fwd);
        // tile of the previous iteration (PIPE: its phase 2 runs in this iteration)
        int b_prev = 0;
        int64_t r0_prev = 0;

        // ---- phase 1 of the tile in slot `bb` (rows from r0t): V-update factor, row partials,
        //      warp transpose-reduce, partials published in red[parity of the running count]
        // ---- V-update factor of the tile in slot `bb` (lanes < GK; run between publishing the
        //      row partials and waiting for the group's, so it fills the barrier wait)
        auto vfactor = [&](int bb, int64_t r0t, int nvt, float (&rfac)[NE], float (&vome)[NE]) {
            const float* slot = ring + (size_t)(g * NBG + bb) * tf;
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                const int s = lane + 32 * e;
                rfac[e] = 0.f;
                vome[e] = 0.f;
                if (s < GK) {  // V[r][k] / max(sum_j V[r][j] G[j][k], 1e-30) from the old V rows
                    const int r = s / K, k = s - (s / K) * K;
                    float vg = 0.f;
                    if (nvt == RG) {  // warp-uniform: every tile but the ragged last one
                        const float* vrow = slot + (size_t)RG * Nkp + r * K;
#pragma unroll
                        for (int j = 0; j < K; ++j) vg = fmaf(vrow[j], sh.Gs[j * K + k], vg);
                        vome[e] = vrow[k];
                    } else {
                        const bool in = r < nvt;
#pragma unroll
                        for (int j = 0; j < K; ++j) vg = fmaf(in ? V[(r0t + r) * K + j] : 0.f, sh.Gs[j * K + k], vg);
                        vome[e] = in ? V[(r0t + r) * K + k] : 0.f;
                    }
                    rfac[e] = __fdividef(vome[e], fmaxf(vg, 1e-30f));  // 2 ulp, no slow path (vg >= 1e-30)
                }
            }
        };
        // (WV: the V-update factor first, in the same lambda -- the three-group schedule, whose
        //  code generation is sensitive to this order)
        auto phase1 = [&]<bool WV>(int bb, int64_t ncount, int64_t r0t, int nvt, float (&rfac)[NE], float (&vome)[NE]) {
            if constexpr (WV) vfactor(bb, r0t, nvt, rfac, vome);
            const float* slot = ring + (size_t)(g * NBG + bb) * tf;
            const float* yb = slot + 2 * tl;
            // p2[r][kp] = (A[r][2kp], A[r][2kp+1]) partials; per lambda one packed FFMA2
            // per (r, k pair) with Y+[r][lambda] broadcast and (D[2kp][l], D[2kp+1][l])
            float2 p2[RG][KD / 2];
#pragma unroll
            for (int r = 0; r < RG; ++r)
#pragma unroll
                for (int kp = 0; kp < KD / 2; ++kp) p2[r][kp] = make_float2(0.f, 0.f);
#pragma unroll
            for (int i = 0; i < LP; ++i) {
                if (SKIP && i == LP - 1 && !wlast) break;
                const bool ok = (i < LP - 1) || lastok;
                const int pp = tl + TG * i;  // lambda pair
                float2 yy[RG];
#pragma unroll
                for (int r = 0; r < RG; ++r)
                    yy[r] = ok ? *reinterpret_cast<const float2*>(yb + (size_t)(RSWAP ? r ^ rsw : (RSWAP1 ? r ^ (rsw & 2) : r)) * Nkp + 2 * TG * i)
                               : make_float2(0.f, 0.f);
                float dd[2 * KD];
#pragma unroll
                for (int j = 0; j < C; ++j) {
                    const float4 q4 = ok ? reinterpret_cast<const float4*>(Ds)[pp * C + (j ^ DL::swz(pp))]
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
                    dd[4 * j + 0] = q4.x;
                    dd[4 * j + 1] = q4.y;
                    dd[4 * j + 2] = q4.z;
                    dd[4 * j + 3] = q4.w;
                }
#pragma unroll
                for (int r = 0; r < RG; ++r)
#pragma unroll
                    for (int kp = 0; kp < KD / 2; ++kp) {
                        p2[r][kp] = ffma2(make_float2(yy[r].x, yy[r].x), make_float2(dd[2 * kp], dd[2 * kp + 1]),
                                          p2[r][kp]);
                        p2[r][kp] = ffma2(make_float2(yy[r].y, yy[r].y),
                                          make_float2(dd[KD + 2 * kp], dd[KD + 2 * kp + 1]), p2[r][kp]);
                    }
            }
            float part[GK];
#pragma unroll
            for (int r = 0; r < RG; ++r)
#pragma unroll
                for (int k = 0; k < K; ++k) part[r * K + k] = (k & 1) ? p2[r][k >> 1].y : p2[r][k >> 1].x;
            const int par = (int)(ncount & 1);
            if constexpr (RSWAP) {
                // local row r of this lane is tile row r ^ rsw, so the two row halvings (lane bits
                // 16 and 8) need no select: every lane keeps its local rows 0 (,1) and sends the
                // others; afterwards it holds the K partials of tile row rsw, reduced over k below
#pragma unroll
                for (int j = 0; j < GK / 2; ++j) part[j] += __shfl_xor_sync(0xffffffffu, part[j + GK / 2], 16);
#pragma unroll
                for (int j = 0; j < K; ++j) part[j] += __shfl_xor_sync(0xffffffffu, part[j + K], 8);
                tr_step<4, K>(part, lane);
                if (((unsigned)lane & tr_bfly(K, 4)) == 0) {
                    const int base = rsw * K + tr_base<K, 4>(lane);
#pragma unroll
                    for (int x = 0; x < tr_nout(K, 4); ++x) sh.red[g][par][wg][base + x] = part[x];
                }
            } else if constexpr (RSWAP1) {
#pragma unroll
                for (int j = 0; j < GK / 2; ++j) part[j] += __shfl_xor_sync(0xffffffffu, part[j + GK / 2], 16);
                tr_step<8, GK / 2>(part, lane);
                if (((unsigned)lane & tr_bfly(GK / 2, 8)) == 0) {
                    const int base = (rsw & 2) * K + tr_base<GK / 2, 8>(lane);
#pragma unroll
                    for (int x = 0; x < tr_nout(GK / 2, 8); ++x) sh.red[g][par][wg][base + x] = part[x];
                }
            } else {
                tr_step<16, GK>(part, lane);
                if (((unsigned)lane & tr_bfly(GK)) == 0) {
                    const int base = tr_base<GK>(lane);
#pragma unroll
                    for (int x = 0; x < tr_nout(GK); ++x) sh.red[g][par][wg][base + x] = part[x];
                }
            }
        };
        // ---- V update of the tile (every warp redundantly, lane s -> (r, k)) once the group's
        //      partials are in; new V rows to this warp's Vn copy, V store, <V_new, A>, H
        auto vupdate = [&](int64_t r0t, int nvt, int64_t ncount, const float (&rfac)[NE], const float (&vome)[NE]) {
            const int par = (int)(ncount & 1);
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                const int s = lane + 32 * e;
                if (s < GK) {
                    float a = 0.f;
#pragma unroll
                    for (int w = 0; w < GW; ++w) a += sh.red[g][par][w][s];
                    float vn = a * rfac[e];
                    if (s / K >= nvt) vn = 0.f;
                    sh.Vn[g][wg][s / K][s - (s / K) * K] = vn;
                    if (wg == VWARP && s / K < nvt) {
                        if (first && !(isfinite(vome[e]) && vome[e] >= 0.f)) bad |= ST_INIT_BAD;
                        if (!isfinite(vn)) bad |= ST_NUMERIC;
                        V[r0t * K + s] = vn;
                        vdotA += (double)vn * (double)a;
                    }
                }
            }
            __syncwarp();
            if (wg == HWARP) {
#pragma unroll
                for (int x = 0; x < (KK + 31) / 32; ++x) {
                    const int tt = lane + 32 * x;
                    if (tt < KK) {
                        const int a = tt / K, c = tt - (tt / K) * K;
                        double hs = 0.0;
#pragma unroll
                        for (int r = 0; r < RG; ++r)
                            hs = fma((double)sh.Vn[g][wg][r][a], (double)sh.Vn[g][wg][r][c], hs);
                        hacc[x] += hs;
                    }
                }
            }
        };
        // ---- phase 2 of the tile in slot `bb` with this warp's Vn copy: B[k][l] += V_new[r][k] Y+[r][l];
        //      then the slot is released (the last warp out refills it with the tile NBG ahead)
        auto phase2 = [&](int bb, int64_t r0t, bool refill) {
            const float* yb = ring + (size_t)(g * NBG + bb) * tf + 2 * tl;
#pragma unroll
            for (int r = 0; r < RG; ++r) {
                float vr[KP];
#pragma unroll
                for (int qq = 0; qq < KP / 4; ++qq) {
                    const float4 v4 = reinterpret_cast<const float4*>(&sh.Vn[g][wg][r][0])[qq];
                    vr[4 * qq + 0] = v4.x;
                    vr[4 * qq + 1] = v4.y;
                    vr[4 * qq + 2] = v4.z;
                    vr[4 * qq + 3] = v4.w;
                }
#pragma unroll
                for (int i = 0; i < LP; ++i) {
                    if (SKIP && i == LP - 1 && !wlast) break;
                    const bool ok = (i < LP - 1) || lastok;
                    const float2 yv = ok ? *reinterpret_cast<const float2*>(yb + (size_t)r * Nkp + 2 * TG * i)
                                         : make_float2(0.f, 0.f);
#pragma unroll
                    for (int k = 0; k < K; ++k) bacc[k][i] = ffma2(make_float2(vr[k], vr[k]), yv, bacc[k][i]);
                }
            }
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                // monotone counter: every use of a slot adds GW, so the last warp of a
                // use sees old % GW == GW - 1 (no reset, no race with the next use)
                if (atomicAdd(&sh.rel[g][bb], 1u) % GW == GW - 1) {
                    if (refill) {
                        fence_proxy_async();
                        issue(g, bb, r0t + NBG * rs);
                        // and warm L2 with the tile after it (a third tile in flight per group
                        // without a third shared-memory slot)
                        const int64_t rp = r0t + (NBG + 1) * rs;
                        if (l2pf && rp >= 0 && rp + RG <= Np) bulk_prefetch_l2(Yp + rp * Nkp, (unsigned)(RG * Nkp * sizeof(float)));
                    }
                }
            }
        };

        if constexpr (PIPE) {
            // iteration m: phase 1 of tile m, publish its partials (split arrive), phase 2 of
            // tile m - 1 (its V rows were updated last iteration), then wait for tile m's
            // partials and update its V rows.  Two slots in use, NBG - 2 >= 1 prefetching.
            for (int64_t m = 0; m <= cnt; ++m) {
                const bool cur = m < cnt;
                const int64_t n = n0 + m;
                const int nv = cur ? (int)min((int64_t)RG, Np - r0) : 0;
                float rfac[NE] = {}, vome[NE] = {};
                if (cur) {
                    mbar_wait_s(fullb + 8u * (unsigned)b, ph);
                    phase1.template operator()<false>(b, n, r0, nv, rfac, vome);
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cta(&sh.part[g][n & 1]);
                    vfactor(b, r0, nv, rfac, vome);
                }
                if (m > 0) phase2(b_prev, r0_prev, m - 1 + NBG < cnt);
                if (!cur) break;
                mbar_wait_s(partb + 8u * (unsigned)(n & 1), (unsigned)((n >> 1) & 1));
                vupdate(r0, nv, n, rfac, vome);
                b_prev = b;
                r0_prev = r0;
                r0 += rs;
                if (++b == NBG) {
                    b = 0;
                    ph ^= 1u;
                }
            }
        } else {
            for (int64_t m = 0; m < cnt; ++m, r0 += rs) {
                const int64_t n = n0 + m;
                const int nv = (int)min((int64_t)RG, Np - r0);
                mbar_wait_s(fullb + 8u * (unsigned)b, ph);
                float rfac[NE], vome[NE];
                if constexpr (true) {
                    // split barrier: publish the partials, compute the V-update factor while the
                    // group's other warps finish (C2: 49.4 -> 48.2 us per iteration; with three
                    // groups it pays once the reduction is select-free, C4 6.19 -> 6.13 ms)
                    phase1.template operator()<false>(b, n, r0, nv, rfac, vome);
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cta(&sh.part[g][n & 1]);
                    vfactor(b, r0, nv, rfac, vome);
                    mbar_wait_s(partb + 8u * (unsigned)(n & 1), (unsigned)((n >> 1) & 1));
                } else {  // (the named-barrier schedule, kept for reference)
                    phase1.template operator()<true>(b, n, r0, nv, rfac, vome);
                    named_bar(1 + g, TG);
                }
                vupdate(r0, nv, n, rfac, vome);
                phase2(b, r0, m + NBG < cnt);
                if (++b == NBG) {
                    b = 0;
                    ph ^= 1u;
                }
            }
        }
        (void)b_prev;
        (void)r0_prev;
        // ---- per-group partials to smem
        if (wg == VWARP) {
            vdotA = warp_sum_d(vdotA);
#pragma unroll
            for (int o = 16; o; o >>= 1) bad |= __shfl_xor_sync(0xffffffffu, bad, o);
            if (lane == 0) {
                sh.vs[g] = vdotA;
                if (bad) atomicOr(&sh.bad, bad);
            }
        } else if (wg == HWARP) {
#pragma unroll
            for (int x = 0; x < (KK + 31) / 32; ++x) {
                const int tt = lane + 32 * x;
                if (tt < KK) sh.hs[g][tt] = hacc[x];
            }
        }
        __syncthreads();
        // ---- CTA partial of B: groups added in order, one k at a time through the idle ring
        float* comb = ring;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (g > 0) {
#pragma unroll
                for (int i = 0; i < LP; ++i)
                    *reinterpret_cast<float2*>(comb + (g - 1) * DS + 2 * (tl + TG * i)) = bacc[k][i];
            }
            __syncthreads();
            if (g == 0) {
#pragma unroll
                for (int i = 0; i < LP; ++i) {
                    const int l0 = 2 * (tl + TG * i);
                    if (l0 < Nkp) {
                        float2 o = bacc[k][i];
#pragma unroll
                        for (int gg = 1; gg < NGRP; ++gg) {
                            const float2 og = *reinterpret_cast<const float2*>(comb + (gg - 1) * DS + l0);
                            o.x += og.x;
                            o.y += og.y;
                        }
                        *reinterpret_cast<float2*>(Bout + (int64_t)k * Nkp + l0) = o;
                    }
                }
            }
            __syncthreads();
        }
        for (int o = tid; o < KK; o += NTH) {
            double h = sh.hs[0][o];
            for (int gg = 1; gg < NGRP; ++gg) h += sh.hs[gg][o];
            Hout[o] = h;
        }
        if (tid == 0) {
            double v = sh.vs[0];
            for (int gg = 1; gg < NGRP; ++gg) v += sh.vs[gg];
            *vout = v;
        }
        // ---- head tiles of the next pass (ring idle again; V rows are final)
        fence_proxy_async_global();  // this thread's V stores before the next bulk copies
        __syncthreads();
        if (prefetch_next && t == 0) {
            fence_proxy_async();
            issue_head(g, n0 + cnt, next_fwd);
        }
    }
};

// Shared prologue: mbarriers, release counters, zeroed ring + slack.
template <int K, int NBG, int NGRP>
__device__ __forceinline__ void fused_prologue(FusedShared<K, NBG, NGRP>& sh, float* ring, size_t ring_floats) {
    for (size_t i = threadIdx.x; i < ring_floats; i += blockDim.x) ring[i] = 0.f;
    if (threadIdx.x == 0) {
        for (int g = 0; g < NGRP; ++g) {
            mbar_init(&sh.part[g][0], GW);
            mbar_init(&sh.part[g][1], GW);
        }
        for (int g = 0; g < NGRP; ++g)
            for (int b = 0; b < NBG; ++b) {
                mbar_init(&sh.full[g][b], 1);
                sh.rel[g][b] = 0u;
            }
        sh.bad = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_proxy_async();  // zero fill (generic) before the first bulk copies (async)
}

// Stage D (lambda-major, swizzled, zero padded; DLayout) and G into shared memory.
// Global reads are coalesced (row-major D); the shared-memory writes scatter.
template <int K>
__device__ __forceinline__ void stage_dg(const float* __restrict__ D, int Nk, int Nkp, const double* Gsrc, float* Ds,
                                         float* Gs) {
    using DL = DLayout<K>;
    constexpr int KD = DL::KD;
#pragma unroll 4
    for (int i = threadIdx.x; i < KD * Nkp; i += blockDim.x) {
        const int k = i / Nkp, l = i - k * Nkp;
        Ds[DL::index(l, k)] = (k < K && l < Nk) ? __ldcg(D + (int64_t)k * Nk + l) : 0.f;
    }
    for (int i = threadIdx.x; i < K * K; i += blockDim.x) Gs[i] = (float)Gsrc[i];
}

// One iteration's row pass per launch (fallback when a cooperative launch is refused).
template <int K, int LP, int NBG, int NGRP>
__global__ void __launch_bounds__(NGRP * TG, 1) k_nmf_fused(const float* __restrict__ Yp, int64_t Np, int Nk,
                                                           int Nkp, float* __restrict__ V,
                                                           const float* __restrict__ D,
                                                           const double* __restrict__ Gd,
                                                           float* __restrict__ Bpart,
                                                           double* __restrict__ Hpart,
                                                           double* __restrict__ vpart, int it, int rotate,
                                                           unsigned* __restrict__ status) {
    using P = Pass<K, LP, NBG, NGRP>;
    constexpr int DS = P::DS;
    __shared__ FusedShared<K, NBG, NGRP> sh;
    extern __shared__ __align__(128) float smem[];
    const size_t tf = tile_floats_of(Nkp, K);
    const size_t ring_floats = (size_t)NGRP * NBG * tf;
    float* ring = smem;
    float* Ds = smem + max(ring_floats, (size_t)(NGRP - 1) * DS);  // the ring doubles as the B-combine scratch
    fused_prologue<K, NBG, NGRP>(sh, ring, ring_floats);
    stage_dg<K>(D, Nk, Nkp, Gd, Ds, sh.Gs);
    __syncthreads();
    const int64_t ntiles = (Np + RG - 1) / RG;
    const int64_t nmine = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    P pass{Yp, Np, Nkp, V, ring, Ds, sh, nmine, tf, (rotate & 1) != 0, (rotate & 2) != 0};
    pass.run(0, it == 0, (it & 1) == 0, false, false, false, Bpart + (int64_t)blockIdx.x * K * Nkp,
             Hpart + (int64_t)blockIdx.x * K * K, vpart + 2 * (int64_t)blockIdx.x);
    if (threadIdx.x == 0) {
        vpart[2 * (int64_t)blockIdx.x + 1] = 0.0;
        if (sh.bad) atomicOr(status, sh.bad);
    }
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
    double* Gpart;   // [nCTA][KK] slice partials of D_new D_new^T
    const double* ypart;
    int nby;
    double* ysq;
    double* obj;     // [2 n_iter] or null
    uint64_t* trace; // [trace_iters][nCTA][TRACE_SLOTS] or null (diagnostics)
    int trace_iters;
    unsigned* bar;   // arrival counter, zero at launch
    unsigned* status;
    int rotate;      // bit 0: rotate the lambda slots per group; bit 1: L2 prefetch
};

// All n_iter Lee-Seung iterations in one cooperative launch.  Per iteration:
//   pass (the next pass's head tiles are issued as soon as it ends) -> grid barrier
//   -> H and this CTA's lambda slice of B reduced over the CTA partials in a fixed
//   order (one sweep of loads), D update of the slice, <B, D_new> slice partial ->
//   grid barrier -> D restaged, G_new = D_new D_new^T from the staged D (every CTA,
//   same fixed order, fp64), objective (last CTA, which has the fewest tiles).
template <int K, int LP, int NBG, int NGRP>
__global__ void __launch_bounds__(NGRP * TG, 1) k_nmf_persist(PersistArgs A) {
    using P = Pass<K, LP, NBG, NGRP>;
    constexpr int NTH = NGRP * TG;
    constexpr int DS = P::DS;
    constexpr int KK = K * K;
    __shared__ FusedShared<K, NBG, NGRP> sh;
    __shared__ double Hs[KK], Gold[KK], Gnew[KK];
    __shared__ double gacc[NTH];
    __shared__ double red[NTH / 32];
    __shared__ double dnew[K * 64];   // the CTA's lambda slice of D_new (nsl <= 64)
    extern __shared__ __align__(128) float smem[];
    const int tid = threadIdx.x;
    const int nC = gridDim.x, c = blockIdx.x;
    const size_t tf = tile_floats_of(A.Nkp, K);
    const size_t ring_floats = (size_t)NGRP * NBG * tf;
    float* ring = smem;
    float* Ds = smem + max(ring_floats, (size_t)(NGRP - 1) * DS);  // the ring doubles as the B-combine scratch
    double* Bsl = reinterpret_cast<double*>(Ds + (size_t)DLayout<K>::KD * A.Nkp);  // [SCR/2] B slice (fp64)
    fused_prologue<K, NBG, NGRP>(sh, ring, ring_floats);
    for (int i = tid; i < KK; i += NTH) Gold[i] = A.Gd[i];
    __syncthreads();
    stage_dg<K>(A.D, A.Nk, A.Nkp, Gold, Ds, sh.Gs);
    __syncthreads();
    const int64_t ntiles = (A.Np + RG - 1) / RG;
    const int64_t nmine = ntiles > c ? (ntiles - 1 - c) / nC + 1 : 0;
    P pass{A.Yp, A.Np, A.Nkp, A.V, ring, Ds, sh, nmine, tf, (A.rotate & 1) != 0, (A.rotate & 2) != 0};
    const int g = tid / TG;
    const int64_t cnt = pass.count_g(g);
    // lambda slice of this CTA for the D update
    const int SL = (A.Nk + nC - 1) / nC;
    const int l0 = min(A.Nk, c * SL), l1 = min(A.Nk, l0 + SL);
    const int nsl = max(0, l1 - l0);
    const bool dvec = (A.Nk % 4 == 0) && ((reinterpret_cast<uintptr_t>(A.D) & 15) == 0);
    unsigned epoch = 0;
    double ysq = 0.0;
    int64_t n0 = 0;
    auto stamp = [&](int it, int slot) {
        if (A.trace && tid == 0 && it < A.trace_iters) {
            uint64_t tnow;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
            A.trace[((int64_t)it * nC + c) * TRACE_SLOTS + slot] = tnow;
        }
    };
    for (int it = 0; it < A.n_iter; ++it) {
        const bool fwd = (it & 1) == 0;
        stamp(it, 0);
        pass.run(n0, it == 0, fwd, it > 0, it + 1 < A.n_iter, !fwd, A.Bpart + (int64_t)c * K * A.Nkp,
                 A.Hpart + (int64_t)c * KK, A.vpart + 2 * (int64_t)c);
        n0 += cnt;
        stamp(it, 1);
        grid_sync(A.bar, epoch);
        stamp(it, 2);
        // <V_new, A> for the objective (last CTA): read between the two barriers -- after the
        // second one, CTAs already in the next pass overwrite their vpart
        const bool objcta = c == nC - 1 && (A.obj || it == 0);
        double va = 0.0;
        if (objcta) {
            double v0 = 0.0;
            for (int i = tid; i < nC; i += NTH) v0 += __ldcg(A.vpart + 2 * i);
            va = block_sum_all(v0, red);
        }
        // ---- H (KK outputs) and the B slice (K x nsl outputs) over the nC partials
        {
            const int nB = K * nsl, nout = KK + nB;
            const int NQ = max(1, NTH / nout);
            if (tid < NQ * nout) {
                const int o = tid % nout, q = tid / nout;
                double s = 0.0;
                if (o < KK) {
                    const double* src = A.Hpart + o;
                    s = batched_sum(q, NQ, nC, [&](int cc) { return __ldcg(src + (int64_t)cc * KK); });
                } else {
                    const int ob = o - KK, k = ob / nsl, l = l0 + (ob - (ob / nsl) * nsl);
                    const float* src = A.Bpart + (int64_t)k * A.Nkp + l;
                    const int64_t stride = (int64_t)K * A.Nkp;
                    s = batched_sum(q, NQ, nC, [&](int cc) { return (double)__ldcg(src + (int64_t)cc * stride); });
                }
                gacc[tid] = s;
            }
            __syncthreads();
            for (int o = tid; o < nout; o += NTH) {
                double s = 0.0;
                for (int q = 0; q < NQ; ++q) s += gacc[q * nout + o];
                if (o < KK) Hs[o] = s;
                else Bsl[o - KK] = s;
            }
            __syncthreads();
        }
        stamp(it, 5);
        // ---- D update of the slice, <B, D_new> slice partial (fixed order)
        {
            double bd = 0.0;
            if (tid < nsl) {
                const int l = l0 + tid;
                unsigned bad = 0;
                double d[K];
#pragma unroll
                for (int k = 0; k < K; ++k) d[k] = (double)Ds[DLayout<K>::index(l, k)];  // = D_old
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    double hd = 0.0;
#pragma unroll
                    for (int jj = 0; jj < K; ++jj) hd = fma(Hs[k * K + jj], d[jj], hd);
                    const double B = Bsl[k * nsl + tid];
                    const float dn = (float)(d[k] * B / fmax(hd, 1e-30));
                    if (!isfinite(dn)) bad |= ST_NUMERIC;
                    bd += B * (double)dn;
                    A.D[(int64_t)k * A.Nk + l] = dn;
                    dnew[k * 64 + tid] = (double)dn;
                }
                if (bad) atomicOr(A.status, bad);
            }
            gacc[tid] = bd;
            __syncthreads();
            if (tid == 0) {
                double s = 0.0;
                for (int u = 0; u < nsl; ++u) s += gacc[u];
                A.dpart[c] = s;
            }
            // slice partial of G_new = D_new D_new^T (fixed order over the slice)
            for (int o = tid; o < KK; o += NTH) {
                const int a = o / K, b = o - (o / K) * K;
                double s = 0.0;
                for (int u = 0; u < nsl; ++u) s = fma(dnew[a * 64 + u], dnew[b * 64 + u], s);
                A.Gpart[(int64_t)c * KK + o] = s;
            }
        }
        stamp(it, 6);
        stamp(it, 3);
        grid_sync(A.bar, epoch);
        // ---- G_new from the slice partials (every CTA, same fixed order; its loads are
        //      issued together with the D restage), objective (last CTA)
        {
            constexpr int NQ = NTH / KK > 0 ? NTH / KK : 1;
            double s = 0.0;
            if (tid < NQ * KK) {
                const int o = tid % KK, q = tid / KK;
                s = batched_sum(q, NQ, nC, [&](int cc) { return __ldcg(A.Gpart + (int64_t)cc * KK + o); });
            }
            using DL = DLayout<K>;
            if (dvec) {
                const int nq = A.Nk >> 2;
#pragma unroll 8
                for (int i = tid; i < K * nq; i += NTH) {
                    const int k = i / nq, l = 4 * (i - k * nq);
                    const float4 v = __ldcg(reinterpret_cast<const float4*>(A.D) + i);
                    Ds[DL::index(l + 0, k)] = v.x;
                    Ds[DL::index(l + 1, k)] = v.y;
                    Ds[DL::index(l + 2, k)] = v.z;
                    Ds[DL::index(l + 3, k)] = v.w;
                }
            } else {
#pragma unroll 8
                for (int i = tid; i < K * A.Nk; i += NTH) {
                    const int k = i / A.Nk, l = i - k * A.Nk;
                    Ds[DL::index(l, k)] = __ldcg(A.D + i);
                }
            }
            if (tid < NQ * KK) gacc[tid] = s;
            __syncthreads();
            for (int o = tid; o < KK; o += NTH) {
                double t = 0.0;
                for (int q = 0; q < NQ; ++q) t += gacc[q * KK + o];
                Gnew[o] = t;
                sh.Gs[o] = (float)t;
            }
            __syncthreads();
        }
        stamp(it, 7);
        if (objcta) {  // the objective trace (and the Y+ = 0 check)
            double v1 = 0.0, v2 = 0.0;
            for (int i = tid; i < nC; i += NTH) v2 += __ldcg(A.dpart + i);
            if (it == 0)
                for (int i = tid; i < A.nby; i += NTH) v1 += __ldcg(A.ypart + i);
            const double ysq_new = block_sum_all(v1, red);
            const double bdot = block_sum_all(v2, red);
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
        __syncthreads();  // the objective (thread 0) has read Gold; K*K > 32 spans several warps
        for (int o = tid; o < KK; o += NTH) Gold[o] = Gnew[o];
        __syncthreads();
        stamp(it, 4);
    }
    if (c == 0)
        for (int o = tid; o < KK; o += NTH) A.Gd[o] = Gold[o];
    if (tid == 0 && sh.bad) atomicOr(A.status, sh.bad);
}

}  // namespace

// Largest LP (lambda pairs per thread) the register budget allows for K.
// The register file is split over the 4 SM sub-partitions (16K each), so the budget is set
// by warps per sub-partition: 3 (12 warps, three groups) -> 168, 4 (16 warps) -> 128.
// Budget for the B columns (2*K*LP) + row partials (RG*KD), the rest is loads/addresses.
constexpr int lp_cap(int K) {
    return (150 - RG * ((K + 1) & ~1)) / (2 * K) < 8 ? (150 - RG * ((K + 1) & ~1)) / (2 * K) : 8;
}
// four groups (16 warps, 128 registers) when the per-thread state fits
__host__ __device__ constexpr bool fits4(int K, int LP) { return 2 * K * LP + RG * ((K + 1) & ~1) <= 64; }

// dynamic smem bytes of the fused kernels
inline size_t fused_smem_bytes(int Nkp, int K, int LP, int NBG, int NGRP) {
    const size_t DS = (size_t)2 * TG * LP;
    const size_t ring = (size_t)NGRP * NBG * tile_floats_of(Nkp, K);
    return (std::max(ring, (size_t)(NGRP - 1) * DS) + (size_t)((K + 1) & ~1) * Nkp + SCR) * sizeof(float);
}

template <int K, int LP, int NB, int NG>
inline cudaError_t fused_klb(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D,
                             int it, unsigned* status, cudaStream_t s) {
    static SmemAttr attr;  // dynamic smem the kernel is allowed, per device (static + dynamic <= 227 KB)
    cudaError_t e = ensure_smem((const void*)k_nmf_fused<K, LP, NB, NG>, (int)p.smem_f, attr);
    if (e != cudaSuccess) return e;
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    k_nmf_fused<K, LP, NB, NG><<<p.nblk_f, NG * TG, p.smem_f, s>>>(w.Yp, Np, g.Nk, p.Nkp, V, D, w.Gd, w.Bpart,
                                                                  w.Hpart, w.vpart, it, (p.rotate ? 1 : 0) | (p.l2pf ? 2 : 0), status);
    return cudaGetLastError();
}

template <int K, int LP, int NB, int NG>
inline cudaError_t persist_klb(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D,
                               int n_iter, double* obj, unsigned* bar, unsigned* status, cudaStream_t s) {
    static SmemAttr attr;
    cudaError_t e0 = ensure_smem((const void*)k_nmf_persist<K, LP, NB, NG>, (int)p.smem_f, attr);
    if (e0 != cudaSuccess) return e0;
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
    A.trace = w.trace;
    A.trace_iters = w.trace_iters;
    A.bar = bar;
    A.status = status;
    A.rotate = (p.rotate ? 1 : 0) | (p.l2pf ? 2 : 0);
    void* args[] = {&A};
    cudaError_t e = cudaMemsetAsync(bar, 0, sizeof(unsigned), s);  // grid-barrier arrival counter
    if (e != cudaSuccess) return e;
    return cudaLaunchCooperativeKernel((const void*)k_nmf_persist<K, LP, NB, NG>, dim3(p.nblk_f), dim3(NG * TG),
                                       args, p.smem_f, s);
}

// (K, LP, NBG, NGRP) dispatch to a callable templated on the four
template <int K, int LP, class F>
inline cudaError_t disp_nb(const NmfPlan& p, F&& f) {
    constexpr int NG4 = fits4(K, LP) ? 4 : 3;
    if (p.ngrp == 4 && NG4 != 4) return cudaErrorInvalidValue;
    switch (p.nbuf * 10 + p.ngrp) {
        case 22:
            if constexpr (K > 8) return f.template operator()<K, LP, 2, 2>();
            return cudaErrorInvalidValue;
        case 32:
            if constexpr (K > 8) return f.template operator()<K, LP, 3, 2>();
            return cudaErrorInvalidValue;
        case 23: return f.template operator()<K, LP, 2, 3>();
        case 33: return f.template operator()<K, LP, 3, 3>();
        case 24: return f.template operator()<K, LP, 2, NG4>();
        case 34: return f.template operator()<K, LP, 3, NG4>();
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
cudaError_t fused_launch_k(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D, int it,
                           unsigned* status, cudaStream_t s) {
    return disp_lp<K>(p, [&]<int KK, int LP, int NB, int NG>() {
        return fused_klb<KK, LP, NB, NG>(g, p, w, V, D, it, status, s);
    });
}
template <int K>
cudaError_t persist_launch_k(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D, int n_iter,
                             double* obj, unsigned* bar, unsigned* status, cudaStream_t s) {
    return disp_lp<K>(p, [&]<int KK, int LP, int NB, int NG>() {
        return persist_klb<KK, LP, NB, NG>(g, p, w, V, D, n_iter, obj, bar, status, s);
    });
}
#define HSNCT_FUSED_EXTERN(KV)                                                                                  \
    extern template cudaError_t fused_launch_k<KV>(const Geometry&, const NmfPlan&, const NmfWs&, float*,       \
                                                   const float*, int, unsigned*, cudaStream_t);                 \
    extern template cudaError_t persist_launch_k<KV>(const Geometry&, const NmfPlan&, const NmfWs&, float*,     \
                                                     float*, int, double*, unsigned*, unsigned*, cudaStream_t);
HSNCT_FUSED_EXTERN(1) HSNCT_FUSED_EXTERN(2) HSNCT_FUSED_EXTERN(3) HSNCT_FUSED_EXTERN(4)
HSNCT_FUSED_EXTERN(5) HSNCT_FUSED_EXTERN(6) HSNCT_FUSED_EXTERN(7) HSNCT_FUSED_EXTERN(8)
HSNCT_FUSED_EXTERN(9) HSNCT_FUSED_EXTERN(10) HSNCT_FUSED_EXTERN(11) HSNCT_FUSED_EXTERN(12)
HSNCT_FUSED_EXTERN(13) HSNCT_FUSED_EXTERN(14) HSNCT_FUSED_EXTERN(15) HSNCT_FUSED_EXTERN(16)

}  // namespace hsnct
