// C ABI of libhsnct.so (include/hsnct.h): argument validation, workspace
// carving, constant tables and launch sequencing.  Every numerical step runs
// in the CUDA kernels of nmf.cu / fbp.cu / synth.cu; this file does no
// arithmetic on the data.
#include "hsnct.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "internal.h"

using namespace hsnct;

struct hsnct_s {
    int device = 0;
    Geometry g{};
    DeviceTables t{};
    NmfPlan nmf{};
    unsigned* status_host = nullptr;  // pinned mirror of t.status
    uint64_t launches = 0;
    uint64_t* trace = nullptr;        // diagnostics buffer (HSNCT_TRACE=1 at create)
    int trace_iters = 0;
    cudaEvent_t fbp_ev[3] = {nullptr, nullptr, nullptr};  // stage timing of hsnct_fbp (diagnostics)
    bool fbp_timed = false;                               // events of the last call are recorded
    cudaEvent_t nmf_ev[3] = {nullptr, nullptr, nullptr};  // stage timing of decompose (diagnostics)
    bool nmf_timed = false;
    // hsnct_fhr_stream: D2H copy stream and per-window-buffer events (created on first use)
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_syn[2] = {nullptr, nullptr}, ev_cpy[2] = {nullptr, nullptr};
};

namespace {

thread_local std::string g_last_error;

hsnct_status fail(hsnct_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

hsnct_status cuda_fail(cudaError_t e, const char* where) {
    return fail(HSNCT_E_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CK(expr, where)                                   \
    do {                                                  \
        cudaError_t e_ = (expr);                          \
        if (e_ != cudaSuccess) return cuda_fail(e_, where); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

size_t a256(size_t b) { return (b + 255) & ~size_t(255); }

// NVTX range around every ABI call (visible to nsys / ncu --nvtx; no cost without a tool)
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
};

int trace_ctas(const NmfPlan& p) { return p.tc ? TC_CLUSTER * p.tc_ncl : p.nblk_f; }

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

struct Range {
    uintptr_t lo, hi;
};
Range rng(const void* p, size_t bytes) {
    uintptr_t a = reinterpret_cast<uintptr_t>(p);
    return Range{a, a + bytes};
}
bool overlap(Range a, Range b) { return a.lo < b.hi && b.lo < a.hi && a.hi > a.lo && b.hi > b.lo; }

int64_t Np_of(const Geometry& g) { return (int64_t)g.Nv * g.Nr * g.Nc; }
int64_t Nx_of(const Geometry& g) { return (int64_t)g.Nr * g.Nc * g.Nc; }
// FHR channels per filtered-sinogram sample: K exactly up to 8 (no padding in Q), else 16
int kc_of(int K) { return K <= 8 ? K : 16; }
int dhr_kc(const Geometry& g) { return g.P <= 1024 ? 16 : 8; }

// hsnct_subspace_decompose_counts: the decompose workspace, plus (plans that read Y itself: tc,
// two-pass) the decoded Y [Np][Nkp]
size_t counts_ws(const Geometry& g, const NmfPlan& p) {
    return a256(nmf_ws_bytes(g, p)) + ((p.fused || p.mma) ? 0 : a256((size_t)Np_of(g) * ((g.Nk + 3) & ~3) * sizeof(float)));
}

// hsnct_mbir workspace: two iterates Xi [Nx][KP], residual E [Np][Kc] (the backprojector's Q
// layout), G = (pi/Nv) A^T E [K][Nx], and for A^T A 1: G1 [Nc^2], the ones image [Nc^2][2], E1 [Nv Nc]
struct MbirLayout {
    size_t xa, e, gk, g1, ones, e1, total;
};
MbirLayout mbir_layout(const Geometry& g) {
    MbirLayout L{};
    L.xa = a256((size_t)g.Nr * g.Nc * g.Nc * mbir_kp(g.K) * sizeof(float));
    L.e = a256((size_t)g.Nv * g.Nr * g.Nc * (g.K <= 8 ? g.K : 16) * sizeof(float));
    L.gk = a256((size_t)g.K * g.Nr * g.Nc * g.Nc * sizeof(float));
    L.g1 = a256((size_t)g.Nc * g.Nc * sizeof(float));
    L.ones = a256((size_t)g.Nc * g.Nc * 2 * sizeof(float));
    L.e1 = a256((size_t)g.Nv * g.Nc * sizeof(float));
    L.total = 2 * L.xa + L.e + L.gk + L.g1 + L.ones + L.e1;
    return L;
}

size_t fbp_ws(const Geometry& g) { return a256((size_t)Np_of(g) * kc_of(g.K) * sizeof(float)); }
// Filtered sinograms of one slice for one chunk of dhr_kc bins.
size_t dhr_ws_chunk_slice(const Geometry& g) { return (size_t)g.Nv * g.Nc * dhr_kc(g) * sizeof(float); }
// Workspace for one slice and all N_k bins (hsnct_workspace_bytes(DHR)); a workspace of
// a single chunk-slice is the minimum.
size_t dhr_ws_per_slice(const Geometry& g) {
    return dhr_ws_chunk_slice(g) * (size_t)((g.Nk + dhr_kc(g) - 1) / dhr_kc(g));
}
int64_t fhr_window_slices(const Geometry& g) {
    const size_t per = (size_t)g.Nc * g.Nc * g.Nk * sizeof(float);
    const size_t budget = size_t(2) << 30;
    return std::max<int64_t>(1, std::min<int64_t>(g.Nr, (int64_t)(budget / std::max<size_t>(per, 1))));
}
struct FhrHostLayout {
    size_t y, v, d, x, xh, nmf, fbp, total;
    int Nkp;
};
FhrHostLayout fhr_layout(const Geometry& g, const NmfPlan& p) {
    FhrHostLayout L{};
    L.Nkp = (g.Nk + 3) & ~3;
    L.y = a256((size_t)Np_of(g) * L.Nkp * sizeof(float));
    L.v = a256((size_t)Np_of(g) * g.K * sizeof(float));
    L.d = a256((size_t)g.K * g.Nk * sizeof(float));
    L.x = a256((size_t)g.K * Nx_of(g) * sizeof(float));
    L.xh = a256((size_t)fhr_window_slices(g) * g.Nc * g.Nc * g.Nk * sizeof(float));
    L.nmf = a256(nmf_ws_bytes(g, p));
    L.fbp = fbp_ws(g);
    L.total = L.y + L.v + L.d + L.x + L.xh + L.nmf + L.fbp;
    return L;
}

// hsnct_fhr_stream: as fhr_layout, with two device windows of window_slices slices
FhrHostLayout stream_layout(const Geometry& g, const NmfPlan& p, int window_slices) {
    FhrHostLayout L = fhr_layout(g, p);
    L.total -= L.xh;
    L.xh = a256((size_t)window_slices * g.Nc * g.Nc * g.Nk * sizeof(float));
    L.total += 2 * L.xh;
    return L;
}

// hsnct_fhr_stream_counts: stream_layout; the counts y, y0, b live in the Y region when the plan
// decodes them in its input preparation (fused, mma), else behind it
size_t stream_counts_bytes(const Geometry& g, const NmfPlan& p, int window_slices) {
    const FhrHostLayout L = stream_layout(g, p, window_slices);
    const size_t cb = a256((size_t)Np_of(g) * g.Nk) + a256((size_t)g.Nr * g.Nc * g.Nk) + a256((size_t)g.Nv * g.Nk * 4);
    return (p.fused || p.mma) ? L.total + (cb > L.y ? cb - L.y : 0) : L.total + cb;
}

hsnct_status check_ws(void* ws, size_t have, size_t need, const char* op) {
    if (need == 0) return HSNCT_OK;
    if (!ws) return fail(HSNCT_E_ARG, "%s: workspace is NULL (need %zu bytes)", op, need);
    if (!aligned(ws, 256)) return fail(HSNCT_E_ARG, "%s: workspace must be 256-byte aligned", op);
    if (have < need) return fail(HSNCT_E_ARG, "%s: workspace %zu bytes < required %zu", op, have, need);
    return HSNCT_OK;
}

hsnct_status check_window(const Geometry& g, int s0, int ns, int b0, int nb, int64_t ld, const char* op) {
    if (s0 < 0 || ns < 0 || (int64_t)s0 + ns > g.Nr)
        return fail(HSNCT_E_ARG, "%s: slice window [%d, %d+%d) outside [0, %d)", op, s0, s0, ns, g.Nr);
    if (b0 < 0 || nb < 0 || (int64_t)b0 + nb > g.Nk)
        return fail(HSNCT_E_ARG, "%s: bin window [%d, %d+%d) outside [0, %d)", op, b0, b0, nb, g.Nk);
    if (ld < nb) return fail(HSNCT_E_ARG, "%s: ld_xh=%lld < n_bins=%d", op, (long long)ld, nb);
    return HSNCT_OK;
}

hsnct_status check_y(const Geometry& g, const float* Y, int64_t ld, const char* op) {
    if (!Y) return fail(HSNCT_E_ARG, "%s: Y is NULL", op);
    if (!aligned(Y, 16)) return fail(HSNCT_E_ARG, "%s: Y must be 16-byte aligned", op);
    if (ld < g.Nk || ld % 4 != 0)
        return fail(HSNCT_E_ARG, "%s: ld_y=%lld must be >= N_k=%d and a multiple of 4", op, (long long)ld, g.Nk);
    return HSNCT_OK;
}

// Enqueue decompose on device buffers (shared by the ABI call and fhr_host).
hsnct_status run_decompose(hsnct_t h, const float* Y, int64_t ld, float* V, float* D, int n_iter,
                           double* obj, void* ws, cudaStream_t s, const CountsIn* cin = nullptr) {
    if (n_iter == 0) return HSNCT_OK;
    NmfWs w = nmf_ws_carve(h->g, h->nmf, ws);
    w.nclamp = h->t.nclamp;
    CK(cudaMemsetAsync(h->t.nclamp, 0, sizeof(unsigned long long), s), "decompose stats");
    w.trace = h->trace;
    w.trace_iters = h->trace_iters;
    const bool timed = h->nmf_ev[0] != nullptr;
    if (timed) CK(cudaEventRecord(h->nmf_ev[0], s), "decompose timing");
    CK(nmf_launch_init(h->g, h->nmf, w, Y, ld, D, h->t.status, s, &h->t, cin), "decompose init");
    h->launches += nmf_init_launches(h->nmf);
    if (timed) CK(cudaEventRecord(h->nmf_ev[1], s), "decompose timing");
    h->nmf_timed = timed;
    if (h->nmf.persist) {
        const int nbx = (h->g.Nk + 31) / 32;
        cudaError_t e = nmf_persist_launch(h->g, h->nmf, w, V, D, n_iter, obj, h->t.counter + 1 + nbx + 1,
                                           h->t.status, s);
        if (e == cudaSuccess) {
            h->launches += 1;
            if (timed) CK(cudaEventRecord(h->nmf_ev[2], s), "decompose timing");
            return HSNCT_OK;
        }
        // cooperative launch refused (e.g. SMs shared with other work): per-iteration launches
        (void)cudaGetLastError();
    }
    for (int it = 0; it < n_iter; ++it) {
        CK(nmf_launch_iter(h->g, h->nmf, w, Y, ld, V, D, it, obj ? obj + 2 * it : nullptr,
                           h->t.status, h->t.counter, s),
           "decompose iteration");
        h->launches += nmf_launches_per_iter(h->nmf);
    }
    if (timed) CK(cudaEventRecord(h->nmf_ev[2], s), "decompose timing");
    return HSNCT_OK;
}

hsnct_status run_fbp(hsnct_t h, const float* V, float* X, void* ws, cudaStream_t s) {
    const Geometry& g = h->g;
    float* Q = static_cast<float*>(ws);
    const int kc = kc_of(g.K);
    const bool timed = h->fbp_ev[0] != nullptr;
    if (timed) CK(cudaEventRecord(h->fbp_ev[0], s), "fbp timing");
    CK(ramp_filter(g, h->t, V, g.K, g.K, 0, g.Nr, Q, kc, s), "fbp ramp filter");
    if (timed) CK(cudaEventRecord(h->fbp_ev[1], s), "fbp timing");
    CK(backproject(g, h->t, Q, kc, g.K, 0, g.Nr, 0, X, 0, 0, s), "fbp backprojection");
    if (timed) CK(cudaEventRecord(h->fbp_ev[2], s), "fbp timing");
    h->fbp_timed = timed;
    h->launches += 2;
    return HSNCT_OK;
}

hsnct_status read_status(hsnct_t h, cudaStream_t s) {
    CK(cudaMemcpyAsync(h->status_host, h->t.status, sizeof(unsigned), cudaMemcpyDeviceToHost, s), "sync");
    CK(cudaStreamSynchronize(s), "sync");
    const unsigned st = *h->status_host;
    if (st) {
        CK(cudaMemsetAsync(h->t.status, 0, sizeof(unsigned), s), "sync");
        CK(cudaStreamSynchronize(s), "sync");
    }
    if (st & (ST_Y_NONFINITE | ST_Y_ALLZERO | ST_INIT_BAD | ST_LABEL_BAD | ST_REGION_EMPTY))
        return fail(HSNCT_E_DATA, "data error (status 0x%x):%s%s%s%s%s", st,
                    (st & ST_Y_NONFINITE) ? " non-finite Y;" : "",
                    (st & ST_Y_ALLZERO) ? " Y+ is identically zero;" : "",
                    (st & ST_INIT_BAD) ? " V0/D0 non-finite or negative;" : "",
                    (st & ST_LABEL_BAD) ? " FMD label outside [-1, n_mat);" : "",
                    (st & ST_REGION_EMPTY) ? " an FMD user region is empty;" : "");
    if (st & ST_NUMERIC) return fail(HSNCT_E_NUMERIC, "numerical error: NaN/Inf produced in V or D");
    return HSNCT_OK;
}

}  // namespace

extern "C" {

int hsnct_abi_version(void) { return HSNCT_ABI_VERSION; }

const char* hsnct_last_error(void) { return g_last_error.c_str(); }

const char* hsnct_status_string(hsnct_status st) {
    switch (st) {
        case HSNCT_OK: return "ok";
        case HSNCT_E_ARG: return "invalid argument";
        case HSNCT_E_DATA: return "data error";
        case HSNCT_E_NUMERIC: return "numerical error";
        case HSNCT_E_CUDA: return "CUDA error";
        case HSNCT_E_NOMEM: return "out of memory";
    }
    return "unknown status";
}

hsnct_status hsnct_create(const hsnct_geom* gp, int device, hsnct_t* out) {
    Nvtx nvtx_("hsnct_create");
    g_last_error.clear();
    if (!out) return fail(HSNCT_E_ARG, "create: out is NULL");
    *out = nullptr;
    if (!gp) return fail(HSNCT_E_ARG, "create: geometry is NULL");
    const hsnct_geom& G = *gp;
    if (G.n_views < 2) return fail(HSNCT_E_ARG, "create: n_views=%d < 2", G.n_views);
    if (G.n_rows < 1) return fail(HSNCT_E_ARG, "create: n_rows=%d < 1", G.n_rows);
    if (G.n_cols < 2 || G.n_cols > 1024) return fail(HSNCT_E_ARG, "create: n_cols=%d outside [2, 1024]", G.n_cols);
    if (G.n_bins < 1) return fail(HSNCT_E_ARG, "create: n_bins=%d < 1", G.n_bins);
    if (G.n_sub < 1 || G.n_sub > HSNCT_MAX_SUB || G.n_sub > G.n_bins)
        return fail(HSNCT_E_ARG, "create: n_sub=%d outside [1, min(16, n_bins)]", G.n_sub);
    if ((int64_t)G.n_sub * ((G.n_bins + 3) & ~3) > 51200)
        return fail(HSNCT_E_ARG, "create: n_sub * n_bins = %lld exceeds 51200 (row-pass D tile)",
                    (long long)G.n_sub * G.n_bins);
    const int64_t Np = (int64_t)G.n_views * G.n_rows * G.n_cols;
    if (Np > (int64_t)1 << 40) return fail(HSNCT_E_ARG, "create: N_p too large");
    if (G.angles)
        for (int v = 0; v < G.n_views; ++v)
            if (!std::isfinite(G.angles[v])) return fail(HSNCT_E_ARG, "create: angle %d is not finite", v);

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(HSNCT_E_CUDA, "create: no CUDA device");
    if (device < 0 || device >= ndev) return fail(HSNCT_E_ARG, "create: device %d outside [0, %d)", device, ndev);
    DeviceGuard guard(device);

    hsnct_t h = new (std::nothrow) hsnct_s();
    if (!h) return fail(HSNCT_E_NOMEM, "create: host allocation failed");
    h->device = device;
    Geometry& g = h->g;
    g.Nv = G.n_views;
    g.Nr = G.n_rows;
    g.Nc = G.n_cols;
    g.Nk = G.n_bins;
    g.K = G.n_sub;
    g.P = 1;
    g.logP = 0;
    while (g.P < 2 * g.Nc) {
        g.P <<= 1;
        ++g.logP;
    }
    cudaDeviceGetAttribute(&g.num_sms, cudaDevAttrMultiProcessorCount, device);
    h->nmf = nmf_plan(g, g.num_sms);

    // Constant tables, built in fp64 on the host.
    std::vector<float> cs(g.Nv), sn(g.Nv);
    for (int v = 0; v < g.Nv; ++v) {
        const double th = G.angles ? G.angles[v] : (double)v * M_PI / (double)g.Nv;
        cs[v] = (float)std::cos(th);
        sn[v] = (float)std::sin(th);
    }
    // Circularly arranged Kak-Slaney kernel (tau = 1): hc[n] = h[n], hc[P-n] = h[n], |n| <= Nc-1.
    std::vector<double> hc(g.P, 0.0);
    auto hk = [](long d) -> double {
        if (d == 0) return 0.25;
        if (d % 2 == 0) return 0.0;
        return -1.0 / (M_PI * M_PI * (double)d * (double)d);
    };
    for (int n = 0; n < g.Nc; ++n) {
        hc[n] = hk(n);
        if (n > 0) hc[g.P - n] = hk(n);
    }
    std::vector<float> Hhat(g.P);
    for (int f = 0; f < g.P; ++f) {
        double s = 0.0;
        for (int n = 0; n < g.P; ++n) {
            if (hc[n] == 0.0) continue;
            const long fn = ((long)f * n) % g.P;
            s += hc[n] * std::cos(2.0 * M_PI * (double)fn / (double)g.P);
        }
        Hhat[f] = (float)(s / (double)g.P);  // inverse-FFT 1/P folded in
    }
    std::vector<float2> tw(g.P / 2);
    for (int t = 0; t < g.P / 2; ++t) {
        const double a = -2.0 * M_PI * (double)t / (double)g.P;
        tw[t] = make_float2((float)std::cos(a), (float)std::sin(a));
    }
    cudaError_t e = cudaSuccess;
    auto al = [&](void** p, size_t b) {
        if (e == cudaSuccess) e = cudaMalloc(p, b);
    };
    al((void**)&h->t.cos_t, g.Nv * sizeof(float));
    al((void**)&h->t.sin_t, g.Nv * sizeof(float));
    al((void**)&h->t.Hhat, g.P * sizeof(float));
    al((void**)&h->t.twiddle, (g.P / 2) * sizeof(float2));
    al((void**)&h->t.status, sizeof(unsigned));
    al((void**)&h->t.nclamp, sizeof(unsigned long long));
    al((void**)&h->t.counter, (size_t)(4 + (g.Nk + 31) / 32) * sizeof(unsigned));
    std::vector<double> lt(256);
    for (int n = 0; n < 256; ++n) lt[n] = std::log(n > 0 ? (double)n : 0.5);  // R7: ln(max(n, 1/2))
    al((void**)&h->t.logtab, 256 * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpy(h->t.logtab, lt.data(), 256 * sizeof(double), cudaMemcpyHostToDevice);
    const MbirGroups mg = mbir_groups(g, cs.data(), sn.data());
    h->t.mbir_ng = mg.ng;
    h->t.mbir_vb = mg.vb;
    al((void**)&h->t.mbir_groups, mg.table.size() * sizeof(int));
    if (e == cudaSuccess)
        e = cudaMemcpy(h->t.mbir_groups, mg.table.data(), mg.table.size() * sizeof(int), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaHostAlloc((void**)&h->status_host, sizeof(unsigned), cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaMemcpy(h->t.cos_t, cs.data(), g.Nv * sizeof(float), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(h->t.sin_t, sn.data(), g.Nv * sizeof(float), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(h->t.Hhat, Hhat.data(), g.P * sizeof(float), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(h->t.twiddle, tw.data(), (g.P / 2) * sizeof(float2), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(h->t.status, 0, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(h->t.nclamp, 0, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(h->t.counter, 0, (size_t)(4 + (g.Nk + 31) / 32) * sizeof(unsigned));
    const char* tr = getenv("HSNCT_TRACE");
    if (e == cudaSuccess && tr && tr[0] == '1' && (h->nmf.persist || h->nmf.tc)) {
        h->trace_iters = 256;
        const size_t tb = (size_t)h->trace_iters * trace_ctas(h->nmf) * TRACE_SLOTS * sizeof(uint64_t);
        e = cudaMalloc((void**)&h->trace, tb);
        if (e == cudaSuccess) e = cudaMemset(h->trace, 0, tb);
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        hsnct_destroy(h);
        return cuda_fail(e, "create");
    }
    *out = h;
    return HSNCT_OK;
}

void hsnct_destroy(hsnct_t h) {
    if (!h) return;
    DeviceGuard guard(h->device);
    cudaDeviceSynchronize();
    cudaFree(h->t.cos_t);
    cudaFree(h->t.sin_t);
    cudaFree(h->t.Hhat);
    cudaFree(h->t.twiddle);
    cudaFree(h->t.status);
    cudaFree(h->t.nclamp);
    cudaFree(h->t.counter);
    cudaFree(h->t.mbir_groups);
    cudaFree(h->t.logtab);
    cudaFree(h->trace);
    for (cudaEvent_t e : h->fbp_ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : h->nmf_ev)
        if (e) cudaEventDestroy(e);
    for (int i = 0; i < 2; ++i) {
        if (h->ev_syn[i]) cudaEventDestroy(h->ev_syn[i]);
        if (h->ev_cpy[i]) cudaEventDestroy(h->ev_cpy[i]);
    }
    if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
    if (h->status_host) cudaFreeHost(h->status_host);
    delete h;
}

size_t hsnct_workspace_bytes(hsnct_t h, int op) {
    if (!h) return 0;
    switch (op) {
        case HSNCT_OP_DECOMPOSE: return a256(nmf_ws_bytes(h->g, h->nmf));
        case HSNCT_OP_FBP: return fbp_ws(h->g);
        case HSNCT_OP_DHR: return a256(dhr_ws_per_slice(h->g));
        case HSNCT_OP_FHR_HOST: return fhr_layout(h->g, h->nmf).total;
        case HSNCT_OP_FMD: return fmd_ws_bytes(h->g);
        case HSNCT_OP_MBIR: return mbir_layout(h->g).total;
        case HSNCT_OP_PROJECT: return mbir_layout(h->g).xa;
        case HSNCT_OP_DECOMPOSE_COUNTS: return counts_ws(h->g, h->nmf);
        default: return 0;
    }
}

hsnct_status hsnct_subspace_decompose(hsnct_t h, const float* Y, int64_t ld_y, float* V, float* D,
                                      int n_iter, double* obj_trace, void* ws, size_t ws_bytes,
                                      void* stream) {
    Nvtx nvtx_("hsnct_subspace_decompose");
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "decompose: handle is NULL");
    const Geometry& g = h->g;
    hsnct_status st = check_y(g, Y, ld_y, "decompose");
    if (st) return st;
    if (!V || !D) return fail(HSNCT_E_ARG, "decompose: V or D is NULL");
    // V rows are bulk-copied (cp.async.bulk) by the row-pass kernels: 16-byte aligned base
    if (!aligned(V, 16) || !aligned(D, 4))
        return fail(HSNCT_E_ARG, "decompose: V must be 16-byte aligned and D 4-byte aligned");
    if (n_iter < 0) return fail(HSNCT_E_ARG, "decompose: n_iter=%d < 0", n_iter);
    if (obj_trace && !aligned(obj_trace, 8)) return fail(HSNCT_E_ARG, "decompose: obj_trace misaligned");
    const size_t need = a256(nmf_ws_bytes(g, h->nmf));
    if ((st = check_ws(ws, ws_bytes, need, "decompose"))) return st;
    const Range rY = rng(Y, (size_t)Np_of(g) * ld_y * sizeof(float));
    const Range rV = rng(V, (size_t)Np_of(g) * g.K * sizeof(float));
    const Range rD = rng(D, (size_t)g.K * g.Nk * sizeof(float));
    const Range rW = rng(ws, need);
    const Range rO = rng(obj_trace, obj_trace ? (size_t)2 * n_iter * sizeof(double) : 0);
    if (overlap(rV, rD) || overlap(rV, rY) || overlap(rD, rY) || overlap(rW, rV) || overlap(rW, rD) ||
        overlap(rW, rY) || overlap(rO, rV) || overlap(rO, rD) || overlap(rO, rW) || overlap(rO, rY))
        return fail(HSNCT_E_ARG, "decompose: Y, V, D, obj_trace and workspace must not overlap");
    DeviceGuard guard(h->device);
    return run_decompose(h, Y, ld_y, V, D, n_iter, obj_trace, ws, (cudaStream_t)stream);
}

hsnct_status check_counts(const Geometry& g, const uint8_t* y, const uint8_t* y0, const float* b, const char* op) {
    if (!y || !y0) return fail(HSNCT_E_ARG, "%s: y or y0 is NULL", op);
    if (b && !aligned(b, 4)) return fail(HSNCT_E_ARG, "%s: b must be 4-byte aligned", op);
    (void)g;
    return HSNCT_OK;
}

hsnct_status hsnct_subspace_decompose_counts(hsnct_t h, const uint8_t* y, const uint8_t* y0, const float* b, float* V,
                                             float* D, int n_iter, double* obj_trace, void* ws, size_t ws_bytes,
                                             void* stream) {
    Nvtx nvtx_("hsnct_subspace_decompose_counts");
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "decompose_counts: handle is NULL");
    const Geometry& g = h->g;
    hsnct_status st = check_counts(g, y, y0, b, "decompose_counts");
    if (st) return st;
    if (!V || !D) return fail(HSNCT_E_ARG, "decompose_counts: V or D is NULL");
    if (!aligned(V, 16) || !aligned(D, 4))
        return fail(HSNCT_E_ARG, "decompose_counts: V must be 16-byte aligned and D 4-byte aligned");
    if (n_iter < 0) return fail(HSNCT_E_ARG, "decompose_counts: n_iter=%d < 0", n_iter);
    if (obj_trace && !aligned(obj_trace, 8)) return fail(HSNCT_E_ARG, "decompose_counts: obj_trace misaligned");
    const size_t need = counts_ws(g, h->nmf);
    if ((st = check_ws(ws, ws_bytes, need, "decompose_counts"))) return st;
    const Range ry = rng(y, (size_t)Np_of(g) * g.Nk), ry0 = rng(y0, (size_t)g.Nr * g.Nc * g.Nk);
    const Range rb = rng(b, b ? (size_t)g.Nv * g.Nk * sizeof(float) : 0);
    const Range rV = rng(V, (size_t)Np_of(g) * g.K * sizeof(float));
    const Range rD = rng(D, (size_t)g.K * g.Nk * sizeof(float));
    const Range rW = rng(ws, need);
    const Range rO = rng(obj_trace, obj_trace ? (size_t)2 * n_iter * sizeof(double) : 0);
    const Range outs[4] = {rV, rD, rW, rO}, ins[3] = {ry, ry0, rb};
    for (int i = 0; i < 4; ++i) {
        for (int j = i + 1; j < 4; ++j)
            if (overlap(outs[i], outs[j])) return fail(HSNCT_E_ARG, "decompose_counts: V, D, obj_trace, ws overlap");
        for (int j = 0; j < 3; ++j)
            if (overlap(outs[i], ins[j]))
                return fail(HSNCT_E_ARG, "decompose_counts: outputs and workspace must not overlap y, y0, b");
    }
    if (n_iter == 0) return HSNCT_OK;
    DeviceGuard guard(h->device);
    const cudaStream_t s = (cudaStream_t)stream;
    const CountsIn cin{y, y0, b};
    if (h->nmf.fused || h->nmf.mma) return run_decompose(h, nullptr, 0, V, D, n_iter, obj_trace, ws, s, &cin);
    // tc / two-pass plans read Y itself: decode it into the workspace tail first
    float* Yd = reinterpret_cast<float*>(static_cast<char*>(ws) + a256(nmf_ws_bytes(g, h->nmf)));
    const int Nkp = (g.Nk + 3) & ~3;
    CK(counts_decode(g, h->t, cin, Yd, Nkp, 0, h->nmf.nby > 0 ? h->nmf.nby : g.num_sms * 8, nullptr, nullptr, s),
       "decompose_counts decode");
    h->launches += 1;
    return run_decompose(h, Yd, Nkp, V, D, n_iter, obj_trace, ws, s);
}

hsnct_status hsnct_counts_to_projections(hsnct_t h, const uint8_t* y, const uint8_t* y0, const float* b, float* Y,
                                         int64_t ld_y, void* stream) {
    Nvtx nvtx_("hsnct_counts_to_projections");
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "counts_to_projections: handle is NULL");
    const Geometry& g = h->g;
    hsnct_status st = check_counts(g, y, y0, b, "counts_to_projections");
    if (st) return st;
    if (!Y || !aligned(Y, 4)) return fail(HSNCT_E_ARG, "counts_to_projections: Y is NULL or misaligned");
    if (ld_y < g.Nk) return fail(HSNCT_E_ARG, "counts_to_projections: ld_y=%lld < N_k", (long long)ld_y);
    const Range rY = rng(Y, ((size_t)Np_of(g) - 1) * ld_y * sizeof(float) + g.Nk * sizeof(float));
    if (overlap(rY, rng(y, (size_t)Np_of(g) * g.Nk)) || overlap(rY, rng(y0, (size_t)g.Nr * g.Nc * g.Nk)) ||
        overlap(rY, rng(b, b ? (size_t)g.Nv * g.Nk * sizeof(float) : 0)))
        return fail(HSNCT_E_ARG, "counts_to_projections: Y must not overlap y, y0, b");
    DeviceGuard guard(h->device);
    CK(counts_decode(g, h->t, CountsIn{y, y0, b}, Y, ld_y, 0, g.num_sms * 8, nullptr, nullptr, (cudaStream_t)stream),
       "counts_to_projections");
    h->launches += 1;
    return HSNCT_OK;
}

size_t hsnct_nmf_red_size(hsnct_t h) { return h ? nmf_red_size(h->g) : 0; }

hsnct_status hsnct_nmf_begin(hsnct_t h, const float* Y, int64_t ld_y, const float* D, void* ws, size_t ws_bytes,
                             void* stream) {
    Nvtx nvtx_("hsnct_nmf_begin");
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "nmf_begin: handle is NULL");
    const Geometry& g = h->g;
    hsnct_status st = check_y(g, Y, ld_y, "nmf_begin");
    if (st) return st;
    if (!D || !aligned(D, 4)) return fail(HSNCT_E_ARG, "nmf_begin: D is NULL or misaligned");
    const size_t need = a256(nmf_ws_bytes(g, h->nmf));
    if ((st = check_ws(ws, ws_bytes, need, "nmf_begin"))) return st;
    DeviceGuard guard(h->device);
    cudaStream_t s = (cudaStream_t)stream;
    NmfWs w = nmf_ws_carve(g, h->nmf, ws);
    w.nclamp = h->t.nclamp;
    CK(cudaMemsetAsync(h->t.nclamp, 0, sizeof(unsigned long long), s), "nmf_begin");
    CK(nmf_launch_init(g, h->nmf, w, Y, ld_y, D, h->t.status, s), "nmf_begin");
    h->launches += nmf_init_launches(h->nmf);
    return HSNCT_OK;
}

hsnct_status hsnct_nmf_rowpass(hsnct_t h, const float* Y, int64_t ld_y, float* V, const float* D, int it, void* ws,
                               size_t ws_bytes, double* red, void* stream) {
    Nvtx nvtx_("hsnct_nmf_rowpass");
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "nmf_rowpass: handle is NULL");
    const Geometry& g = h->g;
    hsnct_status st = check_y(g, Y, ld_y, "nmf_rowpass");
    if (st) return st;
    if (!V || !D || !red) return fail(HSNCT_E_ARG, "nmf_rowpass: V, D or red is NULL");
    if (!aligned(V, 16) || !aligned(D, 4) || !aligned(red, 8))
        return fail(HSNCT_E_ARG, "nmf_rowpass: V must be 16-byte, D 4-byte and red 8-byte aligned");
    if (it < 0) return fail(HSNCT_E_ARG, "nmf_rowpass: it=%d < 0", it);
    const size_t need = a256(nmf_ws_bytes(g, h->nmf));
    if ((st = check_ws(ws, ws_bytes, need, "nmf_rowpass"))) return st;
    const Range rV = rng(V, (size_t)Np_of(g) * g.K * sizeof(float));
    const Range rR = rng(red, nmf_red_size(g) * sizeof(double));
    if (overlap(rV, rR) || overlap(rR, rng(ws, need)) || overlap(rV, rng(ws, need)) ||
        overlap(rV, rng(D, (size_t)g.K * g.Nk * sizeof(float))))
        return fail(HSNCT_E_ARG, "nmf_rowpass: V, D, red and the workspace must not overlap");
    DeviceGuard guard(h->device);
    NmfWs w = nmf_ws_carve(g, h->nmf, ws);
    w.nclamp = h->t.nclamp;
    CK(nmf_shard_rowpass(g, h->nmf, w, Y, ld_y, V, D, it, red, h->t.status, (cudaStream_t)stream), "nmf_rowpass");
    h->launches += nmf_launches_per_iter(h->nmf);  // row pass (+ column pass) + the local reduction
    return HSNCT_OK;
}

hsnct_status hsnct_nmf_dupdate(hsnct_t h, float* D, const double* red, int it, double* obj2, void* ws,
                               size_t ws_bytes, void* stream) {
    Nvtx nvtx_("hsnct_nmf_dupdate");
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "nmf_dupdate: handle is NULL");
    const Geometry& g = h->g;
    if (!D || !red) return fail(HSNCT_E_ARG, "nmf_dupdate: D or red is NULL");
    if (!aligned(D, 4) || !aligned(red, 8) || (obj2 && !aligned(obj2, 8)))
        return fail(HSNCT_E_ARG, "nmf_dupdate: D, red or obj2 misaligned");
    if (it < 0) return fail(HSNCT_E_ARG, "nmf_dupdate: it=%d < 0", it);
    const size_t need = a256(nmf_ws_bytes(g, h->nmf));
    hsnct_status st;
    if ((st = check_ws(ws, ws_bytes, need, "nmf_dupdate"))) return st;
    DeviceGuard guard(h->device);
    NmfWs w = nmf_ws_carve(g, h->nmf, ws);
    CK(nmf_shard_dupdate(g, h->nmf, w, D, red, it, obj2, h->t.status, h->t.counter, (cudaStream_t)stream),
       "nmf_dupdate");
    h->launches += 1;
    return HSNCT_OK;
}

hsnct_status hsnct_fbp(hsnct_t h, const float* V, float* X, void* ws, size_t ws_bytes, void* stream) {
    Nvtx nvtx_("hsnct_fbp");
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "fbp: handle is NULL");
    const Geometry& g = h->g;
    if (!V || !X) return fail(HSNCT_E_ARG, "fbp: V or X is NULL");
    if (!aligned(V, 4) || !aligned(X, 4)) return fail(HSNCT_E_ARG, "fbp: V, X must be 4-byte aligned");
    hsnct_status st;
    const size_t need = fbp_ws(g);
    if ((st = check_ws(ws, ws_bytes, need, "fbp"))) return st;
    const Range rV = rng(V, (size_t)Np_of(g) * g.K * sizeof(float));
    const Range rX = rng(X, (size_t)Nx_of(g) * g.K * sizeof(float));
    const Range rW = rng(ws, need);
    if (overlap(rV, rX) || overlap(rW, rX) || overlap(rW, rV))
        return fail(HSNCT_E_ARG, "fbp: V, X and workspace must not overlap");
    DeviceGuard guard(h->device);
    return run_fbp(h, V, X, ws, (cudaStream_t)stream);
}

hsnct_status hsnct_synthesize(hsnct_t h, const float* X, const float* D, int slice0, int n_slices,
                              int bin0, int n_bins, float* Xh, int64_t ld_xh, void* stream) {
    Nvtx nvtx_("hsnct_synthesize");
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "synthesize: handle is NULL");
    const Geometry& g = h->g;
    hsnct_status st = check_window(g, slice0, n_slices, bin0, n_bins, ld_xh, "synthesize");
    if (st) return st;
    if (n_slices == 0 || n_bins == 0) return HSNCT_OK;
    if (!X || !D || !Xh) return fail(HSNCT_E_ARG, "synthesize: X, D or Xh is NULL");
    if (!aligned(X, 4) || !aligned(D, 4) || !aligned(Xh, 4))
        return fail(HSNCT_E_ARG, "synthesize: X, D, Xh must be 4-byte aligned");
    const Range rXh = rng(Xh, ((size_t)(n_slices) * g.Nc * g.Nc - 1) * ld_xh * sizeof(float) + n_bins * sizeof(float));
    if (overlap(rXh, rng(X, (size_t)Nx_of(g) * g.K * sizeof(float))) ||
        overlap(rXh, rng(D, (size_t)g.K * g.Nk * sizeof(float))))
        return fail(HSNCT_E_ARG, "synthesize: Xh must not overlap X or D");
    DeviceGuard guard(h->device);
    CK(synthesize(g, X, D, slice0, n_slices, bin0, n_bins, Xh, ld_xh, (cudaStream_t)stream), "synthesize");
    h->launches += 1;
    return HSNCT_OK;
}

hsnct_status hsnct_dhr(hsnct_t h, const float* Y, int64_t ld_y, int slice0, int n_slices, int bin0,
                       int n_bins, float* Xh, int64_t ld_xh, void* ws, size_t ws_bytes, void* stream) {
    Nvtx nvtx_("hsnct_dhr");
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "dhr: handle is NULL");
    const Geometry& g = h->g;
    hsnct_status st = check_window(g, slice0, n_slices, bin0, n_bins, ld_xh, "dhr");
    if (st) return st;
    if ((st = check_y(g, Y, ld_y, "dhr"))) return st;
    if (n_slices == 0 || n_bins == 0) return HSNCT_OK;
    if (!Xh || !aligned(Xh, 4)) return fail(HSNCT_E_ARG, "dhr: Xh is NULL or misaligned");
    const size_t per = dhr_ws_chunk_slice(g);
    if ((st = check_ws(ws, ws_bytes, a256(per), "dhr"))) return st;
    const Range rXh = rng(Xh, ((size_t)(n_slices) * g.Nc * g.Nc - 1) * ld_xh * sizeof(float) + n_bins * sizeof(float));
    if (overlap(rXh, rng(Y, (size_t)Np_of(g) * ld_y * sizeof(float))) || overlap(rXh, rng(ws, ws_bytes)))
        return fail(HSNCT_E_ARG, "dhr: Xh must not overlap Y or the workspace");
    DeviceGuard guard(h->device);
    cudaStream_t s = (cudaStream_t)stream;
    const int kc = dhr_kc(g);
    // one ramp + one backprojection launch per pass over (slices x bin chunks) that fits the
    // workspace: as many bin chunks as possible (the whole window when it fits), then slices
    const int nchunk_all = (n_bins + kc - 1) / kc;
    const size_t cap = ws_bytes / per;  // chunk-slices per pass (>= 1)
    const int chunks_pass = (int)std::min<size_t>((size_t)nchunk_all, cap);
    const int ns_pass = (int)std::max<size_t>(1, std::min<size_t>((size_t)n_slices, cap / chunks_pass));
    float* Q = static_cast<float*>(ws);
    for (int c0 = 0; c0 < nchunk_all; c0 += chunks_pass) {
        const int b = bin0 + c0 * kc;
        const int nch = std::min(chunks_pass * kc, bin0 + n_bins - b);
        for (int r = slice0; r < slice0 + n_slices; r += ns_pass) {
            const int ns = std::min(ns_pass, slice0 + n_slices - r);
            CK(ramp_filter(g, h->t, Y + b, ld_y, nch, r, ns, Q, kc, s), "dhr ramp filter");
            float* out = Xh + (int64_t)(r - slice0) * g.Nc * g.Nc * ld_xh;
            CK(backproject(g, h->t, Q, kc, nch, r, ns, 1, out, ld_xh, b - bin0, s), "dhr backprojection");
            h->launches += 2;
        }
    }
    return HSNCT_OK;
}

hsnct_status hsnct_fhr_host(hsnct_t h, const float* Y_host, int64_t ld_y, const float* V0_host,
                            const float* D0_host, int n_iter, float* Xh_host, float* V_host,
                            float* D_host, void* ws, size_t ws_bytes, void* stream) {
    Nvtx nvtx_("hsnct_fhr_host");
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "fhr_host: handle is NULL");
    const Geometry& g = h->g;
    if (!Y_host || !V0_host || !D0_host || !Xh_host)
        return fail(HSNCT_E_ARG, "fhr_host: Y, V0, D0 and Xh host buffers are required");
    if (ld_y < g.Nk) return fail(HSNCT_E_ARG, "fhr_host: ld_y=%lld < N_k=%d", (long long)ld_y, g.Nk);
    if (n_iter < 0) return fail(HSNCT_E_ARG, "fhr_host: n_iter=%d < 0", n_iter);
    const FhrHostLayout L = fhr_layout(g, h->nmf);
    hsnct_status st = check_ws(ws, ws_bytes, L.total, "fhr_host");
    if (st) return st;
    DeviceGuard guard(h->device);
    cudaStream_t s = (cudaStream_t)stream;
    char* c = static_cast<char*>(ws);
    float* Yd = (float*)c;
    c += L.y;
    float* Vd = (float*)c;
    c += L.v;
    float* Dd = (float*)c;
    c += L.d;
    float* Xd = (float*)c;
    c += L.x;
    float* Xhd = (float*)c;
    c += L.xh;
    void* wn = c;
    c += L.nmf;
    void* wf = c;
    const int64_t Np = Np_of(g);
    CK(cudaMemcpy2DAsync(Yd, (size_t)L.Nkp * sizeof(float), Y_host, (size_t)ld_y * sizeof(float),
                         (size_t)g.Nk * sizeof(float), (size_t)Np, cudaMemcpyHostToDevice, s),
       "fhr_host H2D Y");
    CK(cudaMemcpyAsync(Vd, V0_host, (size_t)Np * g.K * sizeof(float), cudaMemcpyHostToDevice, s), "fhr_host H2D V0");
    CK(cudaMemcpyAsync(Dd, D0_host, (size_t)g.K * g.Nk * sizeof(float), cudaMemcpyHostToDevice, s), "fhr_host H2D D0");
    if ((st = run_decompose(h, Yd, L.Nkp, Vd, Dd, n_iter, nullptr, wn, s))) return st;
    if ((st = run_fbp(h, Vd, Xd, wf, s))) return st;
    const int64_t wsl = fhr_window_slices(g);
    const size_t slice_elems = (size_t)g.Nc * g.Nc * g.Nk;
    for (int64_t r = 0; r < g.Nr; r += wsl) {
        const int ns = (int)std::min<int64_t>(wsl, g.Nr - r);
        CK(synthesize(g, Xd, Dd, (int)r, ns, 0, g.Nk, Xhd, g.Nk, s), "fhr_host synthesize");
        h->launches += 1;
        CK(cudaMemcpyAsync(Xh_host + (size_t)r * slice_elems, Xhd, (size_t)ns * slice_elems * sizeof(float),
                           cudaMemcpyDeviceToHost, s),
           "fhr_host D2H Xh");
    }
    if (V_host)
        CK(cudaMemcpyAsync(V_host, Vd, (size_t)Np * g.K * sizeof(float), cudaMemcpyDeviceToHost, s), "fhr_host D2H V");
    if (D_host)
        CK(cudaMemcpyAsync(D_host, Dd, (size_t)g.K * g.Nk * sizeof(float), cudaMemcpyDeviceToHost, s), "fhr_host D2H D");
    return read_status(h, s);
}

size_t hsnct_fhr_stream_bytes(hsnct_t h, int window_slices) {
    if (!h || window_slices < 1) return 0;
    return stream_layout(h->g, h->nmf, std::min(window_slices, h->g.Nr)).total;
}

}  // extern "C"

// hsnct_fhr_stream (Y_host, ld_y) and hsnct_fhr_stream_counts (ch: host counts, Eq. 2 on the device)
static hsnct_status fhr_stream_impl(hsnct_t h, const float* Y_host, int64_t ld_y, const CountsIn* ch,
                                    const float* V0_host, const float* D0_host, int n_iter, int window_slices,
                                    float* ring_host, hsnct_window_fn on_window, void* user, float* V_host,
                                    float* D_host, void* ws, size_t ws_bytes, void* stream) {
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "fhr_stream: handle is NULL");
    const Geometry& g = h->g;
    if ((!Y_host && !ch) || !V0_host || !D0_host || !ring_host)
        return fail(HSNCT_E_ARG, "fhr_stream: Y (or y, y0), V0, D0 and the ring are required");
    if (ch) {
        hsnct_status sc = check_counts(g, ch->y, ch->y0, ch->b, "fhr_stream_counts");
        if (sc) return sc;
    } else if (ld_y < g.Nk) {
        return fail(HSNCT_E_ARG, "fhr_stream: ld_y=%lld < N_k=%d", (long long)ld_y, g.Nk);
    }
    if (n_iter < 0) return fail(HSNCT_E_ARG, "fhr_stream: n_iter=%d < 0", n_iter);
    if (window_slices < 1) return fail(HSNCT_E_ARG, "fhr_stream: window_slices=%d < 1", window_slices);
    const int wsl = std::min(window_slices, g.Nr);
    const FhrHostLayout L = stream_layout(g, h->nmf, wsl);
    hsnct_status st = check_ws(ws, ws_bytes, ch ? stream_counts_bytes(g, h->nmf, wsl) : L.total, "fhr_stream");
    if (st) return st;
    DeviceGuard guard(h->device);
    cudaStream_t s = (cudaStream_t)stream;
    if (!h->copy_stream) {
        CK(cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking), "fhr_stream stream");
        for (int i = 0; i < 2; ++i) {
            CK(cudaEventCreateWithFlags(&h->ev_syn[i], cudaEventDisableTiming), "fhr_stream events");
            CK(cudaEventCreateWithFlags(&h->ev_cpy[i], cudaEventDisableTiming), "fhr_stream events");
        }
    }
    char* c = static_cast<char*>(ws);
    float* Yd = (float*)c;
    c += L.y;
    float* Vd = (float*)c;
    c += L.v;
    float* Dd = (float*)c;
    c += L.d;
    float* Xd = (float*)c;
    c += L.x;
    float* Xw[2] = {(float*)c, (float*)(c + L.xh)};
    c += 2 * L.xh;
    void* wn = c;
    c += L.nmf;
    void* wf = c;
    const int64_t Np = Np_of(g);
    if (!ch) {
        CK(cudaMemcpy2DAsync(Yd, (size_t)L.Nkp * sizeof(float), Y_host, (size_t)ld_y * sizeof(float),
                             (size_t)g.Nk * sizeof(float), (size_t)Np, cudaMemcpyHostToDevice, s),
           "fhr_stream H2D Y");
    }
    CK(cudaMemcpyAsync(Vd, V0_host, (size_t)Np * g.K * sizeof(float), cudaMemcpyHostToDevice, s), "fhr_stream H2D V0");
    CK(cudaMemcpyAsync(Dd, D0_host, (size_t)g.K * g.Nk * sizeof(float), cudaMemcpyHostToDevice, s), "fhr_stream H2D D0");
    if (ch) {
        // the counts (1 + 1/N_v bytes per element) in the Y region when the plan decodes them in its
        // input preparation, else behind the workspace (and decoded into the Y region first)
        const bool inprep = h->nmf.fused || h->nmf.mma;
        const size_t ny = (size_t)Np * g.Nk, ny0 = (size_t)g.Nr * g.Nc * g.Nk;
        char* cb = inprep ? reinterpret_cast<char*>(Yd) : static_cast<char*>(ws) + L.total;
        uint8_t* yd = reinterpret_cast<uint8_t*>(cb);
        uint8_t* y0d = yd + a256(ny);
        float* bd = ch->b ? reinterpret_cast<float*>(y0d + a256(ny0)) : nullptr;
        CK(cudaMemcpyAsync(yd, ch->y, ny, cudaMemcpyHostToDevice, s), "fhr_stream_counts H2D y");
        CK(cudaMemcpyAsync(y0d, ch->y0, ny0, cudaMemcpyHostToDevice, s), "fhr_stream_counts H2D y0");
        if (bd)
            CK(cudaMemcpyAsync(bd, ch->b, (size_t)g.Nv * g.Nk * sizeof(float), cudaMemcpyHostToDevice, s),
               "fhr_stream_counts H2D b");
        const CountsIn cin{yd, y0d, bd};
        if (inprep) {
            if ((st = run_decompose(h, nullptr, 0, Vd, Dd, n_iter, nullptr, wn, s, &cin))) return st;
        } else {
            CK(counts_decode(g, h->t, cin, Yd, L.Nkp, 0, h->nmf.nby > 0 ? h->nmf.nby : g.num_sms * 8, nullptr,
                             nullptr, s),
               "fhr_stream_counts decode");
            h->launches += 1;
            if ((st = run_decompose(h, Yd, L.Nkp, Vd, Dd, n_iter, nullptr, wn, s))) return st;
        }
    } else if ((st = run_decompose(h, Yd, L.Nkp, Vd, Dd, n_iter, nullptr, wn, s))) {
        return st;
    }
    if ((st = run_fbp(h, Vd, Xd, wf, s))) return st;
    if (V_host)
        CK(cudaMemcpyAsync(V_host, Vd, (size_t)Np * g.K * sizeof(float), cudaMemcpyDeviceToHost, s), "fhr_stream D2H V");
    if (D_host)
        CK(cudaMemcpyAsync(D_host, Dd, (size_t)g.K * g.Nk * sizeof(float), cudaMemcpyDeviceToHost, s), "fhr_stream D2H D");
    const size_t slice_elems = (size_t)g.Nc * g.Nc * g.Nk;
    const int nwin = (g.Nr + wsl - 1) / wsl;
    auto deliver = [&](int w) -> hsnct_status {
        CK(cudaEventSynchronize(h->ev_cpy[w & 1]), "fhr_stream D2H");
        const int s0 = w * wsl, ns = std::min(wsl, g.Nr - s0);
        if (on_window) on_window(user, s0, ns, ring_host + (size_t)(w & 1) * wsl * slice_elems);
        return HSNCT_OK;
    };
    for (int w = 0; w < nwin; ++w) {
        const int b = w & 1;
        const int s0 = w * wsl, ns = std::min(wsl, g.Nr - s0);
        if (w >= 2) {  // window w-2 used this device buffer and host slot: wait for its copy
            if ((st = deliver(w - 2))) return st;
            CK(cudaStreamWaitEvent(s, h->ev_cpy[b], 0), "fhr_stream order");
        }
        CK(synthesize(g, Xd, Dd, s0, ns, 0, g.Nk, Xw[b], g.Nk, s), "fhr_stream synthesize");
        h->launches += 1;
        CK(cudaEventRecord(h->ev_syn[b], s), "fhr_stream order");
        CK(cudaStreamWaitEvent(h->copy_stream, h->ev_syn[b], 0), "fhr_stream order");
        CK(cudaMemcpyAsync(ring_host + (size_t)b * wsl * slice_elems, Xw[b], (size_t)ns * slice_elems * sizeof(float),
                           cudaMemcpyDeviceToHost, h->copy_stream),
           "fhr_stream D2H Xh");
        CK(cudaEventRecord(h->ev_cpy[b], h->copy_stream), "fhr_stream order");
    }
    for (int w = std::max(0, nwin - 2); w < nwin; ++w)
        if ((st = deliver(w))) return st;
    // the caller's stream must not run ahead of the last copies (the device windows are its workspace)
    CK(cudaStreamWaitEvent(s, h->ev_cpy[(nwin - 1) & 1], 0), "fhr_stream order");
    if (nwin >= 2) CK(cudaStreamWaitEvent(s, h->ev_cpy[(nwin - 2) & 1], 0), "fhr_stream order");
    return read_status(h, s);
}

extern "C" {

hsnct_status hsnct_fhr_stream(hsnct_t h, const float* Y_host, int64_t ld_y, const float* V0_host,
                              const float* D0_host, int n_iter, int window_slices, float* ring_host,
                              hsnct_window_fn on_window, void* user, float* V_host, float* D_host,
                              void* ws, size_t ws_bytes, void* stream) {
    Nvtx nvtx_("hsnct_fhr_stream");
    return fhr_stream_impl(h, Y_host, ld_y, nullptr, V0_host, D0_host, n_iter, window_slices, ring_host, on_window,
                           user, V_host, D_host, ws, ws_bytes, stream);
}

size_t hsnct_fhr_stream_counts_bytes(hsnct_t h, int window_slices) {
    if (!h || window_slices < 1) return 0;
    return stream_counts_bytes(h->g, h->nmf, std::min(window_slices, h->g.Nr));
}

hsnct_status hsnct_fhr_stream_counts(hsnct_t h, const uint8_t* y_host, const uint8_t* y0_host, const float* b_host,
                                     const float* V0_host, const float* D0_host, int n_iter, int window_slices,
                                     float* ring_host, hsnct_window_fn on_window, void* user, float* V_host,
                                     float* D_host, void* ws, size_t ws_bytes, void* stream) {
    Nvtx nvtx_("hsnct_fhr_stream_counts");
    const CountsIn ch{y_host, y0_host, b_host};
    return fhr_stream_impl(h, nullptr, 0, &ch, V0_host, D0_host, n_iter, window_slices, ring_host, on_window, user,
                           V_host, D_host, ws, ws_bytes, stream);
}

static hsnct_status check_nmat(const Geometry& g, int n_mat, const char* op) {
    if (n_mat < 1 || n_mat > std::min(g.K, 8))
        return fail(HSNCT_E_ARG, "%s: n_mat=%d outside [1, min(K=%d, 8)]", op, n_mat, g.K);
    return HSNCT_OK;
}

hsnct_status hsnct_fmd_transform(hsnct_t h, const float* X, const int32_t* labels, int n_mat, float* T,
                                 void* ws, size_t ws_bytes, void* stream) {
    Nvtx nvtx_("hsnct_fmd_transform");
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "fmd_transform: handle is NULL");
    const Geometry& g = h->g;
    hsnct_status st = check_nmat(g, n_mat, "fmd_transform");
    if (st) return st;
    if (!X || !labels || !T) return fail(HSNCT_E_ARG, "fmd_transform: X, labels or T is NULL");
    if (!aligned(X, 4) || !aligned(labels, 4) || !aligned(T, 4))
        return fail(HSNCT_E_ARG, "fmd_transform: X, labels, T must be 4-byte aligned");
    if ((st = check_ws(ws, ws_bytes, fmd_ws_bytes(g), "fmd_transform"))) return st;
    const Range rT = rng(T, (size_t)n_mat * g.K * sizeof(float));
    if (overlap(rT, rng(X, (size_t)Nx_of(g) * g.K * sizeof(float))) ||
        overlap(rT, rng(labels, (size_t)Nx_of(g) * sizeof(int32_t))) || overlap(rT, rng(ws, ws_bytes)))
        return fail(HSNCT_E_ARG, "fmd_transform: T must not overlap X, labels or the workspace");
    DeviceGuard guard(h->device);
    CK(fmd_transform(g, X, labels, n_mat, T, ws, h->t.status, (cudaStream_t)stream), "fmd_transform");
    h->launches += 1 + (n_mat + std::max(1, std::min(8, 48 / g.K)) - 1) / std::max(1, std::min(8, 48 / g.K));
    return HSNCT_OK;
}

hsnct_status hsnct_fmd_materials(hsnct_t h, const float* X, const float* T, int n_mat, float* Xm,
                                 void* ws, size_t ws_bytes, void* stream) {
    Nvtx nvtx_("hsnct_fmd_materials");
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "fmd_materials: handle is NULL");
    const Geometry& g = h->g;
    hsnct_status st = check_nmat(g, n_mat, "fmd_materials");
    if (st) return st;
    if (!X || !T || !Xm) return fail(HSNCT_E_ARG, "fmd_materials: X, T or Xm is NULL");
    if (!aligned(X, 4) || !aligned(T, 4) || !aligned(Xm, 4))
        return fail(HSNCT_E_ARG, "fmd_materials: X, T, Xm must be 4-byte aligned");
    if ((st = check_ws(ws, ws_bytes, fmd_ws_bytes(g), "fmd_materials"))) return st;
    const Range rXm = rng(Xm, (size_t)n_mat * Nx_of(g) * sizeof(float));
    if (overlap(rXm, rng(X, (size_t)Nx_of(g) * g.K * sizeof(float))) ||
        overlap(rXm, rng(T, (size_t)n_mat * g.K * sizeof(float))) || overlap(rXm, rng(ws, ws_bytes)))
        return fail(HSNCT_E_ARG, "fmd_materials: Xm must not overlap X, T or the workspace");
    DeviceGuard guard(h->device);
    CK(fmd_materials(g, X, T, n_mat, Xm, ws, h->t.status, (cudaStream_t)stream), "fmd_materials");
    h->launches += 2;
    return HSNCT_OK;
}

hsnct_status hsnct_fmd_spectra(hsnct_t h, const float* D, const float* T, int n_mat, float* Dm, void* stream) {
    Nvtx nvtx_("hsnct_fmd_spectra");
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "fmd_spectra: handle is NULL");
    const Geometry& g = h->g;
    hsnct_status st = check_nmat(g, n_mat, "fmd_spectra");
    if (st) return st;
    if (!D || !T || !Dm) return fail(HSNCT_E_ARG, "fmd_spectra: D, T or Dm is NULL");
    if (!aligned(D, 4) || !aligned(T, 4) || !aligned(Dm, 4))
        return fail(HSNCT_E_ARG, "fmd_spectra: D, T, Dm must be 4-byte aligned");
    const Range rDm = rng(Dm, (size_t)n_mat * g.Nk * sizeof(float));
    if (overlap(rDm, rng(D, (size_t)g.K * g.Nk * sizeof(float))) || overlap(rDm, rng(T, (size_t)n_mat * g.K * sizeof(float))))
        return fail(HSNCT_E_ARG, "fmd_spectra: Dm must not overlap D or T");
    DeviceGuard guard(h->device);
    CK(fmd_spectra(g, D, T, n_mat, Dm, (cudaStream_t)stream), "fmd_spectra");
    h->launches += 1;
    return HSNCT_OK;
}

hsnct_status hsnct_mbir(hsnct_t h, const float* V, float* X, int n_iter, const hsnct_mbir_params* prm,
                        double* obj_trace, void* ws, size_t ws_bytes, void* stream) {
    Nvtx nvtx_("hsnct_mbir");
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "mbir: handle is NULL");
    const Geometry& g = h->g;
    if (!V || !X || !prm) return fail(HSNCT_E_ARG, "mbir: V, X or params is NULL");
    if (!aligned(V, 4) || !aligned(X, 4)) return fail(HSNCT_E_ARG, "mbir: V, X must be 4-byte aligned");
    if (obj_trace && !aligned(obj_trace, 8)) return fail(HSNCT_E_ARG, "mbir: obj_trace misaligned");
    if (n_iter < 0) return fail(HSNCT_E_ARG, "mbir: n_iter=%d < 0", n_iter);
    const MbirPrm P{prm->sigma_v, prm->sigma_x, prm->p, prm->q, prm->T};
    if (!(std::isfinite(P.sigma_v) && P.sigma_v > 0) || !(std::isfinite(P.sigma_x) && P.sigma_x > 0) ||
        !(P.p >= 1.0 && P.p <= 2.0) || P.q != 2.0 || !(std::isfinite(P.T) && P.T > 0))
        return fail(HSNCT_E_ARG, "mbir: need sigma_v > 0, sigma_x > 0, 1 <= p <= 2, q == 2, T > 0");
    const MbirLayout L = mbir_layout(g);
    hsnct_status st;
    if ((st = check_ws(ws, ws_bytes, L.total, "mbir"))) return st;
    const Range rV = rng(V, (size_t)Np_of(g) * g.K * sizeof(float));
    const Range rX = rng(X, (size_t)Nx_of(g) * g.K * sizeof(float));
    const Range rW = rng(ws, L.total);
    const Range rO = rng(obj_trace, obj_trace ? (size_t)(n_iter + 1) * sizeof(double) : 0);
    if (overlap(rV, rX) || overlap(rW, rX) || overlap(rW, rV) || overlap(rO, rX) || overlap(rO, rV) || overlap(rO, rW))
        return fail(HSNCT_E_ARG, "mbir: V, X, obj_trace and workspace must not overlap");
    DeviceGuard guard(h->device);
    const cudaStream_t s = (cudaStream_t)stream;
    char* w = static_cast<char*>(ws);
    float* Xa = reinterpret_cast<float*>(w);
    float* Xb = reinterpret_cast<float*>(w + L.xa);
    float* E = reinterpret_cast<float*>(w + 2 * L.xa);
    float* Gk = reinterpret_cast<float*>(w + 2 * L.xa + L.e);
    float* G1 = reinterpret_cast<float*>(w + 2 * L.xa + L.e + L.gk);
    float* ones = reinterpret_cast<float*>(w + 2 * L.xa + L.e + L.gk + L.g1);
    float* E1 = reinterpret_cast<float*>(w + 2 * L.xa + L.e + L.gk + L.g1 + L.ones);
    const int kc = kc_of(g.K);
    const double osc = 0.5 / (P.sigma_v * P.sigma_v);  // data term 1/(2 sv^2) ||y - A x||^2
    if (obj_trace) CK(cudaMemsetAsync(obj_trace, 0, (size_t)(n_iter + 1) * sizeof(double), s), "mbir");
    uint64_t nl = 0;
    if (n_iter > 0) {  // data curvature A^T A 1 of one slice (the same for every slice and channel)
        Geometry g1 = g;
        g1.Nr = 1;
        g1.K = 1;
        CK(mbir_ones(ones, g.Nc, s), "mbir ones");
        CK(mbir_project(g, h->t, ones, 1, 1, nullptr, 0, E1, 1, nullptr, 0.0, s), "mbir project");
        CK(backproject(g1, h->t, E1, 1, 1, 0, 1, 0, G1, 0, 0, s), "mbir backprojection");
        nl += 3;
    }
    CK(mbir_to_inner(X, g.K, Nx_of(g), Xa, s), "mbir");
    nl += 1;
    for (int it = 0; it < n_iter; ++it) {
        double* o = obj_trace ? obj_trace + it : nullptr;
        CK(mbir_project(g, h->t, Xa, g.Nr, g.K, V, 0, E, kc, o, osc, s), "mbir project");
        CK(backproject(g, h->t, E, kc, g.K, 0, g.Nr, 0, Gk, 0, 0, s), "mbir backprojection");
        CK(mbir_sqs(g, P, Xa, Gk, G1, Xb, it == n_iter - 1 ? X : nullptr, o, 1, h->t.status, s), "mbir update");
        std::swap(Xa, Xb);
        nl += 3;
    }
    if (obj_trace) {  // objective of the final iterate
        CK(mbir_project(g, h->t, Xa, g.Nr, g.K, V, 0, E, kc, obj_trace + n_iter, osc, s), "mbir project");
        CK(mbir_sqs(g, P, Xa, nullptr, nullptr, nullptr, nullptr, obj_trace + n_iter, 0, h->t.status, s), "mbir");
        nl += 2;
    }
    h->launches += nl;
    return HSNCT_OK;
}

hsnct_status hsnct_project(hsnct_t h, const float* X, float* P, void* ws, size_t ws_bytes, void* stream) {
    Nvtx nvtx_("hsnct_project");
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "project: handle is NULL");
    const Geometry& g = h->g;
    if (!X || !P) return fail(HSNCT_E_ARG, "project: X or P is NULL");
    if (!aligned(X, 4) || !aligned(P, 4)) return fail(HSNCT_E_ARG, "project: X, P must be 4-byte aligned");
    const size_t need = mbir_layout(g).xa;
    hsnct_status st;
    if ((st = check_ws(ws, ws_bytes, need, "project"))) return st;
    const Range rP = rng(P, (size_t)Np_of(g) * g.K * sizeof(float));
    const Range rX = rng(X, (size_t)Nx_of(g) * g.K * sizeof(float));
    const Range rW = rng(ws, need);
    if (overlap(rP, rX) || overlap(rW, rX) || overlap(rW, rP))
        return fail(HSNCT_E_ARG, "project: X, P and workspace must not overlap");
    DeviceGuard guard(h->device);
    const cudaStream_t s = (cudaStream_t)stream;
    float* Xi = static_cast<float*>(ws);
    CK(mbir_to_inner(X, g.K, Nx_of(g), Xi, s), "project");
    CK(mbir_project(g, h->t, Xi, g.Nr, g.K, nullptr, 1, P, g.K, nullptr, 0.0, s), "project");
    h->launches += 2;
    return HSNCT_OK;
}

hsnct_status hsnct_sync(hsnct_t h, void* stream) {
    Nvtx nvtx_("hsnct_sync");
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "sync: handle is NULL");
    DeviceGuard guard(h->device);
    return read_status(h, (cudaStream_t)stream);
}

uint64_t hsnct_kernel_launches(hsnct_t h) { return h ? h->launches : 0; }

hsnct_status hsnct_debug_trace(hsnct_t h, uint64_t* host, size_t n, size_t* n_out, int* n_cta) {
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "debug_trace: handle is NULL");
    const size_t avail = h->trace ? (size_t)h->trace_iters * trace_ctas(h->nmf) * TRACE_SLOTS : 0;
    const size_t m = std::min(n, avail);
    if (n_out) *n_out = avail;
    if (n_cta) *n_cta = trace_ctas(h->nmf);
    if (m == 0) return HSNCT_OK;
    if (!host) return fail(HSNCT_E_ARG, "debug_trace: host buffer is NULL");
    DeviceGuard guard(h->device);
    CK(cudaMemcpy(host, h->trace, m * sizeof(uint64_t), cudaMemcpyDeviceToHost), "debug_trace");
    return HSNCT_OK;
}

hsnct_status hsnct_decompose_stats(hsnct_t h, int64_t* n_clamped, void* stream) {
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "decompose_stats: handle is NULL");
    if (!n_clamped) return fail(HSNCT_E_ARG, "decompose_stats: n_clamped is NULL");
    DeviceGuard guard(h->device);
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(&v, h->t.nclamp, sizeof v, cudaMemcpyDeviceToHost, (cudaStream_t)stream), "decompose_stats");
    CK(cudaStreamSynchronize((cudaStream_t)stream), "decompose_stats");
    *n_clamped = (int64_t)v;
    return HSNCT_OK;
}

hsnct_status hsnct_debug_plan(hsnct_t h, char* buf, size_t n) {
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "debug_plan: handle is NULL");
    if (!buf || n == 0) return fail(HSNCT_E_ARG, "debug_plan: buffer is NULL or empty");
    const std::string d = nmf_plan_desc(h->g, h->nmf);
    const size_t m = std::min(n - 1, d.size());
    memcpy(buf, d.data(), m);
    buf[m] = 0;
    return HSNCT_OK;
}

hsnct_status hsnct_debug_fbp_timing(hsnct_t h, int on) {
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "debug_fbp_timing: handle is NULL");
    DeviceGuard guard(h->device);
    if (on && !h->fbp_ev[0]) {
        for (cudaEvent_t& e : h->fbp_ev) CK(cudaEventCreate(&e), "debug_fbp_timing");
    } else if (!on && h->fbp_ev[0]) {
        CK(cudaDeviceSynchronize(), "debug_fbp_timing");
        for (cudaEvent_t& e : h->fbp_ev) {
            cudaEventDestroy(e);
            e = nullptr;
        }
    }
    h->fbp_timed = false;
    return HSNCT_OK;
}

hsnct_status hsnct_debug_fbp_times(hsnct_t h, float* ms) {
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "debug_fbp_times: handle is NULL");
    if (!ms) return fail(HSNCT_E_ARG, "debug_fbp_times: ms is NULL");
    if (!h->fbp_timed) return fail(HSNCT_E_ARG, "debug_fbp_times: no timed hsnct_fbp call");
    DeviceGuard guard(h->device);
    CK(cudaEventSynchronize(h->fbp_ev[2]), "debug_fbp_times");
    CK(cudaEventElapsedTime(&ms[0], h->fbp_ev[0], h->fbp_ev[1]), "debug_fbp_times");
    CK(cudaEventElapsedTime(&ms[1], h->fbp_ev[1], h->fbp_ev[2]), "debug_fbp_times");
    return HSNCT_OK;
}

hsnct_status hsnct_debug_nmf_timing(hsnct_t h, int on) {
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "debug_nmf_timing: handle is NULL");
    DeviceGuard guard(h->device);
    if (on && !h->nmf_ev[0]) {
        for (cudaEvent_t& e : h->nmf_ev) CK(cudaEventCreate(&e), "debug_nmf_timing");
    } else if (!on && h->nmf_ev[0]) {
        CK(cudaDeviceSynchronize(), "debug_nmf_timing");
        for (cudaEvent_t& e : h->nmf_ev) {
            cudaEventDestroy(e);
            e = nullptr;
        }
    }
    h->nmf_timed = false;
    return HSNCT_OK;
}

hsnct_status hsnct_debug_nmf_times(hsnct_t h, float* ms) {
    g_last_error.clear();
    if (!h) return fail(HSNCT_E_ARG, "debug_nmf_times: handle is NULL");
    if (!ms) return fail(HSNCT_E_ARG, "debug_nmf_times: ms is NULL");
    if (!h->nmf_timed) return fail(HSNCT_E_ARG, "debug_nmf_times: no timed decompose call");
    DeviceGuard guard(h->device);
    CK(cudaEventSynchronize(h->nmf_ev[2]), "debug_nmf_times");
    CK(cudaEventElapsedTime(&ms[0], h->nmf_ev[0], h->nmf_ev[1]), "debug_nmf_times");
    CK(cudaEventElapsedTime(&ms[1], h->nmf_ev[1], h->nmf_ev[2]), "debug_nmf_times");
    return HSNCT_OK;
}

}  // extern "C"
