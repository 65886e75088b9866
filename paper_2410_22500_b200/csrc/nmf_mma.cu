// Host side of the tensor-core NMF path (nmf_mma.cuh): plan, Y+ split launch, per-K dispatch.
#include "nmf_mma.cuh"

#include <cstdlib>

namespace hsnct {

bool nmf_mma_plan(const Geometry& g, int num_sms, NmfPlan* p) {
    // Opt-in (HSNCT_MMA=1): measured slower than the FFMA kernel on B200 (DESIGN.md §5.1:
    // per-8-row-tile overheads of the 12-way bin split dominate its tensor work).
    const char* on = getenv("HSNCT_MMA");
    if (!(on && on[0] == '1')) return false;
    if (g.K > 8) return false;
    const int N16 = (g.Nk + 15) & ~15;
    const int spw = mma_spw(N16);
    if (spw < 1 || spw > MSPW_MAX) return false;
    const int nslot = mma_nslot(N16, g.K);
    if (nslot < 2) return false;
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    const int64_t ntiles = (Np + MR - 1) / MR;
    p->N16 = N16;
    p->spw = spw;
    p->nslot = nslot;
    p->smem_m = (size_t)nslot * mma_slot_bytes(N16, g.K);
    p->nblk_f = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)num_sms));
    if ((g.Nk + p->nblk_f - 1) / p->nblk_f > 16) return false;  // D-update slice <= 16 bins
    p->nby = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms * 8, (Np + 7) / 8));
    return true;
}

cudaError_t nmf_ysplit_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y, int64_t ld_y,
                              unsigned* status, cudaStream_t s) {
    const int64_t Np = (int64_t)g.Nv * g.Nr * g.Nc;
    k_ysplit<<<p.nby, 256, 0, s>>>(Y, ld_y, Np, g.Nk, p.N16, reinterpret_cast<__half*>(w.Yp), w.ypart, status);
    return cudaGetLastError();
}

cudaError_t nmf_mma_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D, int n_iter,
                           double* obj, unsigned* bar, unsigned* status, cudaStream_t s) {
    switch (g.K) {
#define M(KV) \
    case KV: return mma_launch_k<KV>(g, p, w, V, D, n_iter, obj, bar, status, s);
        M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8)
#undef M
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace hsnct
