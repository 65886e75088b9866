// Host side of the fused NMF path: plan, Y+ preparation launch, per-K dispatch.
#include "nmf_fused.cuh"

#include <cstdlib>

namespace hsnct {

// Static shared memory of k_nmf_persist<K, ., nb, ngrp> (FusedShared + the D-update arrays),
// with slack for alignment.
static size_t persist_static_bytes(int K, int nb, int ngrp) {
    const size_t KK = (size_t)K * K, GK = (size_t)RG * K, KP = (size_t)((K + 3) & ~3), nth = (size_t)ngrp * TG;
    const size_t fs = 8 * ngrp * nb + 16 * ngrp + 4 * ngrp * nb + 4 * ngrp * 2 * GW * GK + 4 * ngrp * GW * RG * KP +
                      4 * KK + 8 * ngrp * KK + 8 * ngrp + 4;
    return fs + 24 * KK + 8 * nth + 8 * (nth / 32) + 8 * (size_t)K * 64 + 256;
}

// Ring slots per compute group: 3 when they fit the shared-memory budget, else 2.  K <= 8: the
// measured 208 KB dynamic budget; K > 8 (larger static arrays): 227 KB less the static part
// and the 1 KB the driver reserves per CTA.
static int nbuf_for(int Nkp, int LP, int K, int ngrp) {
    for (int nb = 3; nb >= 2; --nb) {
        const size_t dyn = fused_smem_bytes(Nkp, K, LP, nb, ngrp);
        const bool fits = K <= 8 ? dyn <= 208 * 1024 : dyn + persist_static_bytes(K, nb, ngrp) <= 226 * 1024;
        if (fits) return nb;
    }
    return 0;
}

bool nmf_fused_plan(const Geometry& g, int num_sms, NmfPlan* p) {
    // K = 9..16: the V update takes NE = ceil(RG K / 32) (tile row, component) elements per lane
    if (g.K > 16) return false;
    const int Nkp = (g.Nk + 3) & ~3;
    const int pairs = (g.Nk + 1) / 2;
    const int LP = (pairs + TG - 1) / TG;
    if (LP > lp_cap(g.K)) return false;
    // four groups (more tiles in flight) when the registers and two slots per group fit
    int ngrp = fits4(g.K, LP) && nbuf_for(Nkp, LP, g.K, 4) >= 2 ? 4 : 3;
    // K > 8: two groups (8 warps, up to 255 registers): three spill 100-300 B of accumulators
    // (C6, K = 9, LP = 5: 16.5 -> 15.5 ms per iteration)
    if (g.K > 8) ngrp = 2;
    const char* ng = getenv("HSNCT_NGRP");
    if (ng && ng[0] == '3') ngrp = 3;
    const int nbuf = nbuf_for(Nkp, LP, g.K, ngrp);
    if (nbuf < 2) return false;
    p->LP = LP;
    p->nbuf = nbuf;
    p->ngrp = ngrp;
    // rotating the ragged lambda slots over the SM sub-partitions: +1% with four groups (C2);
    // with three groups it pays once the warps without a last lambda pair skip that slot
    // (Pass::SKIP): C4 6.61 -> 6.24 ms per iteration (rotation alone: -1%)
    const char* rt = getenv("HSNCT_ROTATE");
    p->rotate = rt ? rt[0] == '1' : true;
    const char* pf = getenv("HSNCT_L2PF");
    p->l2pf = pf ? pf[0] == '1' : false;  // measured -1.6% at C4: the pass is issue-bound
    p->fthreads = ngrp * TG;
    p->smem_f = fused_smem_bytes(Nkp, g.K, LP, nbuf, ngrp);
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    const int64_t ntiles = (Np + RG - 1) / RG;
    p->nblk_f = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)num_sms));
    const char* nbk = getenv("HSNCT_NBLK");  // A/B: fewer persistent CTAs (grid barrier / partial count)
    if (nbk && atoi(nbk) > 0) p->nblk_f = std::min(p->nblk_f, atoi(nbk));
    p->PB = p->nblk_f;
    // the persistent kernel's D update gives every CTA a lambda slice of SL = ceil(Nk / nCTA)
    // bins: dnew holds 64 per component, the fp64 B slice SCR/2 values, and threads
    // [0, K*K + K*SL) produce its outputs.  Shapes beyond that (few rows, long spectra) run
    // the per-iteration launches (k_nmf_fused + k_dred) instead.
    const int SL = (g.Nk + p->nblk_f - 1) / p->nblk_f;
    p->persist_fits = SL <= 64 && g.K * SL <= SCR / 2 && g.K * g.K + g.K * SL <= p->fthreads;
    p->nby = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms * 8, (Np + 7) / 8));
    return true;
}

cudaError_t nmf_yplus_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y, int64_t ld_y,
                             unsigned* status, cudaStream_t s) {
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    k_yplus<<<p.nby, 256, 0, s>>>(Y, ld_y, Np, g.Nk, p.Nkp, w.Yp, w.ypart, status, w.nclamp);
    return cudaGetLastError();
}

#define HSNCT_K8(M) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15) M(16)

cudaError_t nmf_fused_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D,
                             int it, unsigned* status, cudaStream_t s) {
    switch (g.K) {
#define M(KV) \
    case KV: return fused_launch_k<KV>(g, p, w, V, D, it, status, s);
        HSNCT_K8(M)
#undef M
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t nmf_persist_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D, int n_iter,
                               double* obj, unsigned* bar, unsigned* status, cudaStream_t s) {
    if (p.mma) return nmf_mma_persist_launch(g, p, w, V, D, n_iter, obj, bar, status, s);
    switch (g.K) {
#define M(KV) \
    case KV: return persist_launch_k<KV>(g, p, w, V, D, n_iter, obj, bar, status, s);
        HSNCT_K8(M)
#undef M
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace hsnct
