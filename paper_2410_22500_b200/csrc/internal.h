// Internal declarations shared by the C ABI (api.cpp) and the CUDA kernels.
// Nothing here is exported; the public surface is include/hsnct.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

namespace hsnct {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: a kernel's attribute is
// raised on the calling thread's current device the first time a launch there needs more
// than 48 KB, and remembered per device (atomic; a race only repeats the call).
constexpr int MAX_DEVICES = 64;
struct SmemAttr {
    std::atomic<int> bytes[MAX_DEVICES] = {};
};
inline cudaError_t ensure_smem(const void* func, int bytes, SmemAttr& a) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < MAX_DEVICES && a.bytes[dev].load(std::memory_order_acquire) >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < MAX_DEVICES) {
        int cur = a.bytes[dev].load(std::memory_order_relaxed);
        while (cur < bytes && !a.bytes[dev].compare_exchange_weak(cur, bytes, std::memory_order_release)) {
        }
    }
    return cudaSuccess;
}

// Device status word bits (deferred errors, read back by hsnct_sync).
enum : unsigned {
    ST_Y_NONFINITE = 1u,     // E_DATA
    ST_Y_ALLZERO = 2u,       // E_DATA
    ST_INIT_BAD = 4u,        // E_DATA: V0/D0 non-finite or negative
    ST_NUMERIC = 8u,         // E_NUMERIC: V or D became non-finite
    ST_LABEL_BAD = 16u,      // E_DATA: an FMD label outside [-1, n_mat)
    ST_REGION_EMPTY = 32u,   // E_DATA: an FMD user region has no voxel
};

struct Geometry {
    int Nv, Nr, Nc, Nk, K;
    int P;       // FFT length = next_pow2(2 Nc)
    int logP;
    int num_sms; // SMs of the handle's device
};

// Per-handle device constants (small, owned by the handle).
struct DeviceTables {
    float* cos_t = nullptr;     // [Nv]
    float* sin_t = nullptr;     // [Nv]
    float* Hhat = nullptr;      // [P] real, even DFT of the zero-padded ramp kernel, / P folded in
    float2* twiddle = nullptr;  // [P/2] exp(-2 pi i t / P)
    unsigned* status = nullptr; // device status word
    unsigned* counter = nullptr;// grid "last block" tickets (zero between launches)
    unsigned long long* nclamp = nullptr;  // negative Y entries clamped to 0 by the last decompose
    int* mbir_groups = nullptr; // [mbir_ng][mbir_vb + 1] projector view groups (mbir.cu)
    double* logtab = nullptr;   // [256] ln(max(n, 1/2)), fp64 (counts.cu, R7)
    int mbir_ng = 0, mbir_vb = 0;
};

// ---------------------------------------------------------------- NMF (nmf.cu)
constexpr int DG2 = 8;  // chunk groups of the D-update reduction
constexpr int TC_CLUSTER = 4;  // CTAs per cluster of the tcgen05 row pass (bin ranges)
struct TcRanges {
    int l0[TC_CLUSTER];   // first bin of cluster rank j's range (multiple of 16)
    int L[TC_CLUSTER];    // bins in the range (multiple of 16)
    int nch[TC_CLUSTER];  // chunks of W bins in the range (the last one may be shorter)
    int W;                // chunk width in bins (multiple of 16, <= 128)
};
struct NmfPlan {
    int Nkp;         // Nk rounded up to 4
    int nbx;         // D-update column blocks = ceil(Nk / 32)
    int P;           // number of per-CTA B partials
    int PH;          // number of per-CTA H partials
    int nvp;         // number of per-CTA objective partials
    // fused single-pass path (nmf_fused.cu), K <= 8
    bool fused;
    bool persist;    // run all iterations in one cooperative launch (fused or mma path)
    bool persist_fits;  // the persistent kernel's lambda slice fits its D-update buffers
    int LP;          // lambda pairs per thread
    int nbuf;        // ring slots per compute group
    int ngrp;        // compute groups of 4 warps (3 or 4)
    bool rotate;     // rotate the lambda slots per group over the SM sub-partitions
    bool l2pf;       // L2 prefetch one tile beyond the ring (per group)
    int PB;          // B partials of the fused kernel (2 per CTA)
    int nby;         // blocks of the Y+ preparation kernel
    int fthreads;    // threads per CTA
    int nblk_f;      // CTAs (persistent, static tile schedule)
    size_t smem_f;   // dynamic smem (tile ring)
    // tcgen05 row pass (nmf_tc.cu), K <= 8: one launch per iteration + k_dred
    bool tc;
    int tc_ncl;      // clusters (TC_CLUSTER CTAs each)
    int tc_R;        // ring slots per CTA
    int tc_R2;       // phase-2 ring slots (0: phase 2 reads the phase-1 ring)
    int tc_maxch;    // chunks of the longest bin range
    size_t tc_smem;  // dynamic smem
    TcRanges tc_rg;
    int tc_Nk16;     // Nk rounded up to 16
    int64_t tc_Npad; // Np rounded up to the 64-row tile
    // mma.sync row pass (nmf_mma.cu), K <= 8: one launch per iteration + k_dred
    bool mma;
    int mma_NB;      // 16-bin blocks per row = ceil(Nk / 16)
    int mma_NBW;     // blocks per warp (template instance >= ceil(NB / mma_MW))
    int mma_MW;      // warps per CTA: 8, or 16 (K = 9..16 with HSNCT_MMA_MW=16)
    int64_t mma_Npad;// Np rounded up to the 16-row tile
    // two-pass fallback (nmf.cu)
    int nblk_v, nchunk, bthreads, nlam_blk;
    int64_t rows_per_chunk;
    size_t smem_v;
};
struct NmfWs {
    double* Gd;      // [K*K]   G = D D^T used by the current V half-step
    double* vpart;   // [nvp*2] per-CTA <V_new, A>, ||Y+||^2
    double* dpart;   // [nbx]   per-column <B, D_new>
    double* Gpart;   // [nbx*K*K] per-column partials of D_new D_new^T
    double* ysq;     // [1]
    double* Hpart;   // [P*K*K]
    float* Bpart;    // [P*K*Nkp]
    double* L2B;     // [nbx*DG2*K*32]
    double* L2H;     // [nbx*DG2*K*K]
    float* Yp;       // [Np*Nkp] Y+ (fused path only)
    double* ypart;   // [nby] ||Y+||^2 partials (fused and tc paths)
    unsigned long long* nclamp = nullptr;  // clamped-entry counter (handle-owned, zeroed per call)
    void* Yc;        // [Npad*Nk16] Y+ as fp16 hi/lo pairs in the tcgen05 layout (tc path)
    unsigned* ymax;  // bits of max(Y+) (tc path)
    int* texp;       // [ntiles] per-tile Y+ scale exponents (mma path)
    // diagnostics (hsnct_debug_trace): per-iteration, per-CTA %globaltimer stamps
    uint64_t* trace = nullptr;  // [trace_iters][nCTA][TRACE_SLOTS] or null
    int trace_iters = 0;
};
constexpr int TRACE_SLOTS = 16;  // persist: [iteration][CTA] iteration start, pass end, barrier 1, D update
                                 // done, iteration end, partials reduced, D slice updated, G reduced +
                                 // D restaged; tc: [tile][CTA] (nmf_tc.cu, TcStamp)
NmfPlan nmf_plan(const Geometry& g, int num_sms);
bool nmf_fused_plan(const Geometry& g, int num_sms, NmfPlan* p);
size_t nmf_ws_bytes(const Geometry& g, const NmfPlan& p);
NmfWs nmf_ws_carve(const Geometry& g, const NmfPlan& p, void* ws);
// Enqueues the per-call preparation: G = D D^T for the initial D, and Y+ for the
// fused path (nmf_init_launches launches).
// counts-domain input (NEXT-1): uint8 y [Np][Nk], y0 [Nr Nc][Nk], offset b [Nv][Nk] (nullable)
struct CountsIn {
    const uint8_t* y;
    const uint8_t* y0;
    const float* b;
};
// mode 0: raw Y into out [Np][ld_out]; mode 1: Y+ into out [Np][Nkp] with the k_yplus partials
// (nblk blocks: ypart[nblk], nclamp)
cudaError_t counts_decode(const Geometry& g, const DeviceTables& t, const CountsIn& cin, float* out, int64_t ld_out,
                          int mode, int nblk, double* ypart, unsigned long long* nclamp, cudaStream_t s);
cudaError_t nmf_launch_init(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y, int64_t ld_y,
                            const float* D, unsigned* status, cudaStream_t s, const DeviceTables* t = nullptr,
                            const CountsIn* cin = nullptr);
int nmf_init_launches(const NmfPlan& p);
// Enqueues one Lee-Seung iteration (nmf_launches_per_iter launches).
cudaError_t nmf_launch_iter(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y,
                            int64_t ld_y, float* V, float* D, int it, double* obj2,
                            unsigned* status, unsigned* counter, cudaStream_t s);
cudaError_t nmf_fused_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D,
                             int it, unsigned* status, cudaStream_t s);
// All n_iter iterations in one cooperative launch (fused path); bar = 2 zeroed words.
cudaError_t nmf_persist_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D, int n_iter,
                               double* obj, unsigned* bar, unsigned* status, cudaStream_t s);
cudaError_t nmf_yplus_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y, int64_t ld_y,
                             unsigned* status, cudaStream_t s);
// tcgen05 path: plan (fills the tc_* fields), input preparation (max / ||Y+||^2 / non-finite
// check, then the fp16 hi/lo conversion), one row pass
bool nmf_tc_plan(const Geometry& g, int num_sms, NmfPlan* p);
cudaError_t nmf_tc_prepare(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y, int64_t ld_y,
                           unsigned* status, cudaStream_t s);
cudaError_t nmf_tc_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D, int it,
                          unsigned* status, cudaStream_t s);
// mma.sync path: plan (mma_* fields, nblk_f, nby), input preparation, one row pass
bool nmf_mma_plan(const Geometry& g, int num_sms, NmfPlan* p);
cudaError_t nmf_mma_prepare(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y, int64_t ld_y,
                            unsigned* status, cudaStream_t s);
cudaError_t nmf_mma_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, const float* D, int it,
                           unsigned* status, cudaStream_t s);
// the mma input preparation from counts (NEXT-1): Eq. 2 decoded into the block layout
cudaError_t nmf_mma_prepare_counts(const Geometry& g, const NmfPlan& p, const NmfWs& w, const DeviceTables& t,
                                   const CountsIn& cin, unsigned* status, cudaStream_t s);
// all n_iter iterations in one cooperative launch (mma path, persist_fits); bar = 1 zeroed word
cudaError_t nmf_mma_persist_launch(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* V, float* D,
                                   int n_iter, double* obj, unsigned* bar, unsigned* status, cudaStream_t s);
int nmf_launches_per_iter(const NmfPlan& p);
// sharded decomposition (NEXT-4): one row pass -> the rank's sums in red (fp64 [K*N_k + K*K + 2]);
// the D update from the all-reduced sums (identical on every rank)
size_t nmf_red_size(const Geometry& g);
cudaError_t nmf_shard_rowpass(const Geometry& g, const NmfPlan& p, const NmfWs& w, const float* Y, int64_t ld_y,
                              float* V, const float* D, int it, double* red, unsigned* status, cudaStream_t s);
cudaError_t nmf_shard_dupdate(const Geometry& g, const NmfPlan& p, const NmfWs& w, float* D, const double* red,
                              int it, double* obj2, unsigned* status, unsigned* counter, cudaStream_t s);
std::string nmf_plan_desc(const Geometry& g, const NmfPlan& p);
// counter words needed by the handle: 1 + ceil(Nk / 32)

// ------------------------------------------------------------- FBP (fbp.cu)
// Ramp filter of Nch channels of every (v, r) sinogram row of the slice window
// [s0, s0+ns):  element (v, r, c, ch) is in[((v*Nr + r)*Nc + c)*ld_in + ch].
// Output Q[(r-s0)][v][c][Kc] (Kc >= Nch; channels >= Nch are written as 0).
cudaError_t ramp_filter(const Geometry& g, const DeviceTables& t, const float* in, int64_t ld_in,
                        int Nch, int s0, int ns, float* Q, int Kc, cudaStream_t s);
// Backprojection of Q[(r-s0)][v][c][Kc] for slices [s0, s0+ns).
// mode 0 (FHR): X[ch][r][i][j] for ch < Nch (channel-planar, plane stride Nx).
// mode 1 (DHR): Xh[((r-s0)*Nc + i)*Nc + j][ld_out] columns col0 + ch, ch < Nch.
cudaError_t backproject(const Geometry& g, const DeviceTables& t, const float* Q, int Kc, int Nch,
                        int s0, int ns, int mode, float* out, int64_t ld_out, int64_t col0,
                        cudaStream_t s);
int ramp_launches();
int backproject_launches();

// ---------------------------------------------- FMD back half (fmd.cu, NEXT-2)
int fmd_tblocks(const Geometry& g);
size_t fmd_ws_bytes(const Geometry& g);
cudaError_t fmd_transform(const Geometry& g, const float* X, const int32_t* labels, int Nm, float* T, void* ws,
                          unsigned* status, cudaStream_t s);
cudaError_t fmd_materials(const Geometry& g, const float* X, const float* T, int Nm, float* Xm, void* ws,
                          unsigned* status, cudaStream_t s);
cudaError_t fmd_spectra(const Geometry& g, const float* D, const float* T, int Nm, float* Dm, cudaStream_t s);

// ----------------------------------------------------------- MBIR (mbir.cu, NEXT-3)
struct MbirPrm {
    double sigma_v, sigma_x, p, q, T;
};
// Projector view groups: views split by orientation class (|cos| >= |sin|: 1, else 0), VB per
// group; table[g*(vb+1)] = class, then VB views (-1 = empty slot).
struct MbirGroups {
    std::vector<int> table;
    int ng = 0, vb = 0;
};
MbirGroups mbir_groups(const Geometry& g, const float* cs, const float* sn);
int mbir_kp(int K);  // K rounded up to even: channels per voxel of the internal iterate Xi
// X[k][n] -> Xi[n][KP]
cudaError_t mbir_to_inner(const float* X, int K, int64_t Nx, float* Xi, cudaStream_t s);
// Xi1[n][2] = (1, 0), n < Nc^2
cudaError_t mbir_ones(float* Xi1, int Nc, cudaStream_t s);
// A x of Nr slices of Xi (K channels, KP = mbir_kp(K) per voxel).  mode 0: E[r][v][c][Kc] = Y - A x
// (Y [Np][K] nullable), osc * (sum of squares) added to *obj (nullable); mode 1: P[Np][K] = A x.
cudaError_t mbir_project(const Geometry& g, const DeviceTables& t, const float* Xi, int Nr, int K, const float* Y,
                         int mode, float* out, int Kc, double* obj, double osc, cudaStream_t s);
// one SQS step Xc -> Xn (update = 1; Xout nullable: also channel-planar), or only the prior term
// of the objective at Xc (update = 0); G = (pi/Nv) A^T e [K][Nx], G1 = (pi/Nv) A^T (-A 1) [Nc^2]
cudaError_t mbir_sqs(const Geometry& g, const MbirPrm& prm, const float* Xc, const float* G, const float* G1,
                     float* Xn, float* Xout, double* obj, int update, unsigned* status, cudaStream_t s);

// ------------------------------------------------------- synthesis (synth.cu)
cudaError_t synthesize(const Geometry& g, const float* X, const float* D, int s0, int ns, int b0,
                       int nb, float* Xh, int64_t ld_xh, cudaStream_t s);

}  // namespace hsnct
