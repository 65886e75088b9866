/*
 * hsnct.h -- C ABI of libhsnct.so, the B200 (sm_100a) hot path of fast
 * hyperspectral neutron tomography (FHR), arXiv 2410.22500.
 *
 * The calls follow the paper's statement of the problem:
 *   Algorithm 1, "Input p, N_s -> Output x^h":
 *     hsnct_subspace_decompose   subspace extraction, Eq. 4
 *     hsnct_fbp                  tomographic reconstruction of the N_s subspace
 *                                sinograms (FBP per DESIGN.md R10)
 *     hsnct_synthesize           subspace expansion, Eq. 6
 *   and the paper's baseline:
 *     hsnct_dhr                  direct hyperspectral reconstruction, one FBP per
 *                                wavelength bin
 *   and, in place of FBP, the paper's model-based reconstruction (NEXT-3):
 *     hsnct_mbir                 Eq. 5, QGGMRF prior, SQS iterations
 *     hsnct_project              the forward projector A of Eq. 5
 *   plus hsnct_fhr_host, the whole of Algorithm 1 on HOST buffers (the
 *   end-to-end entry point: host->device copy, the three stages, device->host).
 *
 * Notation: N_v views, N_r detector rows (= slices),
 * N_c detector columns (= image width), N_k wavelength bins,
 * N_p = N_v N_r N_c projections, N_x = N_r N_c N_c voxels, K = N_s subspace
 * dimension.
 *
 * Layouts (all fp32, row-major, caller-owned DEVICE memory unless stated):
 *   Y   [N_p][ld_y]   projection data p, row p = (v*N_r + r)*N_c + c,
 *                     bin index fastest.  ld_y >= N_k, ld_y % 4 == 0,
 *                     16-byte aligned; all N_p*ld_y floats must be readable (the
 *                     padding columns are read and ignored).
 *   V   [N_p][K]      subspace views V^s, row p as for Y; 16-byte
 *                     aligned in hsnct_subspace_decompose (rows are bulk-copied).
 *   D   [K][N_k]      subspace basis, stored as (D^s)^T.
 *   X   [K][N_r][N_c][N_c]  subspace reconstructions x^s,
 *                     channel-planar; voxel (r, i, j) at x = j-(N_c-1)/2,
 *                     y = i-(N_c-1)/2 (R14).
 *   Xh  [n_slices*N_c*N_c][ld_xh]  a window of x^h: voxels of
 *                     slices [slice0, slice0+n_slices), bins [bin0, bin0+n_bins),
 *                     bin fastest; ld_xh >= n_bins.
 * Geometry (R11-R16): theta_v = v*pi/N_v unless angles are given;
 * Kak-Slaney Ram-Lak filter (tau = 1); linear interpolation; scale pi/N_v;
 * detector samples outside [0, N_c-1] are zero; no FOV mask.
 *
 * Ownership: every array is allocated and freed by the caller (PyTorch).
 * The library allocates only small per-handle constant tables (angles,
 * filter spectrum, FFT twiddles, a status word) in hsnct_create and frees
 * them in hsnct_destroy.  Scratch space is the caller's workspace buffer
 * (device, 256-byte aligned, size from hsnct_workspace_bytes).
 *
 * Streams: every call only ENQUEUES work on the caller's CUDA stream
 * (a cudaStream_t passed as void*; NULL = legacy default stream) and
 * returns; a handle must be used by one stream at a time.
 *
 * Errors: argument errors (null / misaligned pointers, shapes, windows,
 * workspace too small, overlapping outputs) are detected on the host before
 * any launch and returned synchronously as HSNCT_E_ARG (SPEC "config" class).
 * Data-dependent errors are recorded in a device status word and returned
 * by hsnct_sync: HSNCT_E_DATA for non-finite Y / V0 / D0 or an all-zero Y+
 * (SPEC "data" class), HSNCT_E_NUMERIC for a non-finite V or D produced by
 * the iteration (SPEC "numerical" class).  HSNCT_E_CUDA reports a CUDA
 * runtime failure (launch or copy), details in hsnct_last_error.
 */
#ifndef HSNCT_H_
#define HSNCT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HSNCT_ABI_VERSION 1
#define HSNCT_MAX_SUB 16 /* K = N_s <= 16 */

typedef struct hsnct_s* hsnct_t;

typedef enum {
    HSNCT_OK = 0,
    HSNCT_E_ARG = 1,     /* bad shape / range / null / misaligned / aliasing / window / workspace */
    HSNCT_E_DATA = 2,    /* non-finite input, negative init, Y+ identically zero (deferred)      */
    HSNCT_E_NUMERIC = 3, /* NaN/Inf produced during the iteration (deferred)                     */
    HSNCT_E_CUDA = 4,    /* CUDA runtime error                                                   */
    HSNCT_E_NOMEM = 5    /* host or handle-table allocation failed                               */
} hsnct_status;

typedef enum {
    HSNCT_OP_DECOMPOSE = 0, /* hsnct_subspace_decompose                    */
    HSNCT_OP_FBP = 1,       /* hsnct_fbp                                   */
    HSNCT_OP_DHR = 2,       /* hsnct_dhr, any window (the minimum is used) */
    HSNCT_OP_FHR_HOST = 3,  /* hsnct_fhr_host                              */
    HSNCT_OP_FMD = 4,       /* hsnct_fmd_transform / hsnct_fmd_materials   */
    HSNCT_OP_MBIR = 5,      /* hsnct_mbir                                  */
    HSNCT_OP_PROJECT = 6,   /* hsnct_project                               */
    HSNCT_OP_DECOMPOSE_COUNTS = 7 /* hsnct_subspace_decompose_counts       */
} hsnct_op;

typedef struct {
    int32_t n_views; /* N_v >= 2                 */
    int32_t n_rows;  /* N_r >= 1                 */
    int32_t n_cols;  /* 2 <= N_c <= 1024 (FFT length P = next_pow2(2 N_c) <= 2048) */
    int32_t n_bins;  /* N_k >= 1, and K * round_up(N_k, 4) <= 51200 (the row pass
                        keeps D [K][N_k] in shared memory)                       */
    int32_t n_sub;   /* 1 <= K <= min(16, N_k)   */
    const double* angles; /* HOST array of N_v view angles in radians, copied at create;
                             NULL => theta_v = v*pi/N_v (R13)            */
} hsnct_geom;

/* Validates the geometry, selects device `device` and builds the constant
 * tables (cos/sin per view; the DFT of the zero-padded Kak-Slaney kernel,
 * P = next_pow2(2 N_c); FFT twiddles) in fp64 on the host.  *out receives the
 * handle.  E_ARG on a bad geometry, E_CUDA / E_NOMEM on allocation failure. */
hsnct_status hsnct_create(const hsnct_geom* g, int device, hsnct_t* out);

/* Frees the handle's tables.  Safe on NULL.  Synchronizes the device. */
void hsnct_destroy(hsnct_t h);

/* Workspace bytes the caller must provide for `op` (hsnct_op).  0 on a bad
 * handle / op.  HSNCT_OP_DHR returns the size for one slice and all N_k bins
 * (filtered sinograms); hsnct_dhr accepts any workspace of at least one slice x 16
 * bins and processes as many (bin chunks x slices) per launch as fit. */
size_t hsnct_workspace_bytes(hsnct_t h, int op);

/* Subspace extraction, Eq. 4: n_iter Lee-Seung
 * multiplicative-update iterations (R1-R3, V half first) on
 * Y+ = max(Y, 0) (R6), starting from the caller's V (= V0, strictly > 0) and
 * D (= D0, strictly > 0), both overwritten in place with V_n, D_n (raw,
 * unnormalised iterates, R9).  One iteration:
 *   V <- V .* (Y+ D^T) ./ max(V (D D^T), 1e-30);  D <- D .* (V^T Y+) ./ max((V^T V) D, 1e-30).
 * obj_trace (device fp64, 2*n_iter entries, nullable) receives ||Y+ - V D||_F^2
 * after each half-step, evaluated in fp64 from the Gram identity.
 * n_iter == 0 is a no-op.  Deterministic: static schedule, fixed reduction
 * order, no floating-point atomics.  Resume = call again with the same V, D. */
hsnct_status hsnct_subspace_decompose(hsnct_t h, const float* Y, int64_t ld_y, float* V, float* D,
                                      int n_iter, double* obj_trace, void* ws, size_t ws_bytes,
                                      void* stream);

/* Counts-domain input (NEXT-1): Eq. 2 with the Appendix-A offset
 * and the 1/2-count floor (R7),
 *   Y[p][k] = fp32( (L[y0[rc][k]] - L[y[p][k]]) - b[v][k] ),  L[n] = ln(max(n, 1/2)) in fp64,
 *   p = (v N_r + r) N_c + c, rc = r N_c + c:
 * y uint8 [N_p][N_k] (transmitted counts, row p as for Y), y0 uint8 [N_r N_c][N_k] (the open
 * beam, shared by every view), b fp32 [N_v][N_k] or NULL (= 0), all DEVICE memory, b 4-byte
 * aligned.  The single fp64 -> fp32 rounding makes Y bit-identical to fp32 of the fp64 formula.
 * hsnct_counts_to_projections writes Y [N_p][ld_y] (ld_y >= N_k; padding untouched; a
 * non-finite b is a deferred E_DATA).
 * hsnct_subspace_decompose_counts is hsnct_subspace_decompose on that Y, decoded inside the
 * input preparation (1 byte of y per element instead of 4 of Y; y0 is read once per view and
 * served from L2): V, D, the objective trace and the clamped count are bit-identical to
 * hsnct_subspace_decompose on the materialised Y.  Workspace:
 * hsnct_workspace_bytes(h, HSNCT_OP_DECOMPOSE_COUNTS) (device, 256-byte aligned); outputs
 * and workspace must not overlap y, y0, b. */
hsnct_status hsnct_counts_to_projections(hsnct_t h, const uint8_t* y, const uint8_t* y0, const float* b, float* Y,
                                         int64_t ld_y, void* stream);
hsnct_status hsnct_subspace_decompose_counts(hsnct_t h, const uint8_t* y, const uint8_t* y0, const float* b, float* V,
                                             float* D, int n_iter, double* obj_trace, void* ws, size_t ws_bytes,
                                             void* stream);

/* Sharded subspace extraction (NEXT-4): Eq. 4 on Y distributed over ranks by
 * rows (e.g. slice ranges: parallel-beam slices decouple, so a rank's rows are all views of its
 * slices).  The iteration of hsnct_subspace_decompose, split at its one exchange step:
 *
 *   hsnct_nmf_begin(Y, D)                     once: Y+ preparation, G = D D^T
 *   for it in 0..n_iter-1:
 *     hsnct_nmf_rowpass(Y, V, D, it, red)     this rank's rows: V half-step (row-local) and its
 *                                             sums red = [B = V^T Y+ (K x N_k) | H = V^T V (K x K)
 *                                             | <V_new, A> | ||Y+||^2], fp64
 *     (caller) all-reduce SUM of red over the ranks, e.g. NCCL via torch.distributed
 *     hsnct_nmf_dupdate(D, red, it, obj2)     D <- D .* B ./ max(H D, 1e-30) from the global
 *                                             sums, G for the next row pass, the two objective
 *                                             values (obj2, device fp64[2], nullable)
 *
 * Every rank holds the full D (K x N_k, identical on all ranks) and its own rows of Y and V;
 * the handle is created with the rank's local geometry (its N_r slices).  On one rank the
 * sequence computes what hsnct_subspace_decompose computes (up to the order of the fp64 sums).
 * ws: HSNCT_OP_DECOMPOSE workspace of the handle, reused across the calls of one decomposition.
 * red: device fp64 array of hsnct_nmf_red_size(h) values.  Errors as hsnct_subspace_decompose. */
size_t hsnct_nmf_red_size(hsnct_t h);
hsnct_status hsnct_nmf_begin(hsnct_t h, const float* Y, int64_t ld_y, const float* D, void* ws, size_t ws_bytes,
                             void* stream);
hsnct_status hsnct_nmf_rowpass(hsnct_t h, const float* Y, int64_t ld_y, float* V, const float* D, int it, void* ws,
                               size_t ws_bytes, double* red, void* stream);
hsnct_status hsnct_nmf_dupdate(hsnct_t h, float* D, const double* red, int it, double* obj2, void* ws,
                               size_t ws_bytes, void* stream);

/* FBP of the K subspace sinograms (Algorithm 1 lines "Tomographic
 * Reconstruction", FBP per R10): column k of V, reshaped
 * (N_v, N_r, N_c), is ramp-filtered along c and backprojected into X[k].
 * X must not overlap V or ws. */
hsnct_status hsnct_fbp(hsnct_t h, const float* V, float* X, void* ws, size_t ws_bytes, void* stream);

/* Model-based reconstruction of the K subspace sinograms (NEXT-3; Eq. 5, PAPER.md:224-228,
 * DESIGN.md R24-R26), every channel k and slice r independently:
 *   x = argmin_{x >= 0} 1/(2 sigma_v^2) ||y - A x||^2 + h(x),   y = column k of V on slice r,
 * A the linear-interpolation projector (the exact adjoint of hsnct_fbp's backprojector without
 * its pi/N_v factor: (A x)[v][c] = sum_ij x[i][j] max(0, 1 - |u_ij(v) - c|)), h the QGGMRF prior
 * on the 8-neighbourhood of the slice: h(x) = sum_{pairs} b_ij rho(x_i - x_j),
 *   rho(d) = |d|^p / (p sigma_x^p) * u / (1 + u),  u = |d / (T sigma_x)|^(q - p),
 *   b = 1/(4 + 4/sqrt 2) for edge neighbours, b / sqrt 2 for diagonal ones.
 * Solver: n_iter Jacobi separable-quadratic-surrogate steps (monotone in the objective)
 *   x <- max(0, x - grad / ((1/sigma_v^2) A^T A 1 + sum_j 2 b_ij w(x_i - x_j))),  w = rho'(d)/d.
 * X [K][N_r][N_c][N_c]: in x0 (e.g. the FBP), out the n_iter-th iterate (unchanged if n_iter
 * == 0).  obj_trace (device fp64, n_iter + 1 entries, nullable): the objective summed over
 * channels and slices at iterates 0..n_iter.  Parameters: sigma_v > 0, sigma_x > 0,
 * 1 <= p <= 2, q == 2, T > 0, else E_ARG.  Workspace: hsnct_workspace_bytes(h, HSNCT_OP_MBIR).
 * X, V, obj_trace and ws must not overlap.  A non-finite iterate sets E_NUMERIC (hsnct_sync).
 * fp32 arithmetic; the objective sums use fp64 atomics (order not fixed). */
typedef struct {
    double sigma_v, sigma_x, p, q, T;
} hsnct_mbir_params;
hsnct_status hsnct_mbir(hsnct_t h, const float* V, float* X, int n_iter, const hsnct_mbir_params* prm,
                        double* obj_trace, void* ws, size_t ws_bytes, void* stream);

/* Forward projection of Eq. 5: P = A X, P [N_p][K] in the layout of V (row (v N_r + r) N_c + c),
 * X [K][N_r][N_c][N_c].  Workspace: hsnct_workspace_bytes(h, HSNCT_OP_PROJECT). */
hsnct_status hsnct_project(hsnct_t h, const float* X, float* P, void* ws, size_t ws_bytes, void* stream);

/* Subspace expansion, Eq. 6, x^h = x^s (D^s)^T, on a
 * window: Xh[n][b] = sum_k X[k][slice0*N_c*N_c + n] * D[k][bin0 + b].
 * Empty windows (n_slices == 0 or n_bins == 0) are a no-op. */
hsnct_status hsnct_synthesize(hsnct_t h, const float* X, const float* D, int slice0, int n_slices,
                              int bin0, int n_bins, float* Xh, int64_t ld_xh, void* stream);

/* Direct hyperspectral reconstruction, the baseline: every
 * bin b of the window is reconstructed separately by FBP of the raw
 * (unclamped, R6) sinogram Y[., bin0 + b]; output layout as hsnct_synthesize. */
hsnct_status hsnct_dhr(hsnct_t h, const float* Y, int64_t ld_y, int slice0, int n_slices, int bin0,
                       int n_bins, float* Xh, int64_t ld_xh, void* ws, size_t ws_bytes, void* stream);

/* The whole of Algorithm 1 on HOST buffers (end to end): copies Y_host
 * [N_p][ld_y], V0_host [N_p][K], D0_host [K][N_k] to the device workspace,
 * runs decompose(n_iter) -> fbp -> synthesize over all slices and bins in
 * windows, and copies x^h back to Xh_host [N_x][N_k] (ld = N_k), V and D back
 * to V_host / D_host (nullable).  Host buffers should be page-locked for
 * full copy bandwidth.  Blocks until the result is on the host; returns the
 * deferred data/numeric status like hsnct_sync. */
hsnct_status hsnct_fhr_host(hsnct_t h, const float* Y_host, int64_t ld_y, const float* V0_host,
                            const float* D0_host, int n_iter, float* Xh_host, float* V_host,
                            float* D_host, void* ws, size_t ws_bytes, void* stream);

/* Algorithm 1 end to end on HOST buffers for volumes whose x^h does not fit in host or
 * device memory (C4: 215 GB, C5: 430 GB): like hsnct_fhr_host, but x^h leaves the device in
 * windows of window_slices slices (all N_k bins) through a caller-owned page-locked HOST
 * ring of two windows, ring_host [2][window_slices*N_c*N_c][N_k].  Window w is synthesized
 * on `stream` into one of two device window buffers while window w-1 is copied D2H on a
 * second stream of the handle; when window w's copy has completed, on_window(user, slice0,
 * n_slices, xh) is called on the calling thread with xh pointing into the ring (valid until
 * the call returns; the slot is then reused for window w+2).  on_window may be NULL.
 * Workspace: hsnct_fhr_stream_bytes(h, window_slices).  V_host / D_host nullable as in
 * hsnct_fhr_host.  Blocks until the last window has been delivered; returns the deferred
 * data/numeric status like hsnct_sync. */
typedef void (*hsnct_window_fn)(void* user, int slice0, int n_slices, const float* xh);
size_t hsnct_fhr_stream_bytes(hsnct_t h, int window_slices);
hsnct_status hsnct_fhr_stream(hsnct_t h, const float* Y_host, int64_t ld_y, const float* V0_host,
                              const float* D0_host, int n_iter, int window_slices, float* ring_host,
                              hsnct_window_fn on_window, void* user, float* V_host, float* D_host,
                              void* ws, size_t ws_bytes, void* stream);

/* hsnct_fhr_stream from the detector counts (NEXT-1 end to end; Eq. 2, with the
 * Appendix-A offset): the HOST arrays y_host uint8 [N_p][N_k], y0_host uint8
 * [N_r N_c][N_k] and b_host fp32 [N_v][N_k] (nullable: b = 0) go to the device (1 + 1/N_v bytes
 * per element instead of 4) and the decomposition decodes Y = fp32((L[y0] - L[y]) - b) as
 * hsnct_subspace_decompose_counts does -- the results equal hsnct_fhr_stream's on the decoded Y
 * bit for bit.  Everything else as hsnct_fhr_stream; workspace hsnct_fhr_stream_counts_bytes. */
size_t hsnct_fhr_stream_counts_bytes(hsnct_t h, int window_slices);
hsnct_status hsnct_fhr_stream_counts(hsnct_t h, const uint8_t* y_host, const uint8_t* y0_host, const float* b_host,
                                     const float* V0_host, const float* D0_host, int n_iter, int window_slices,
                                     float* ring_host, hsnct_window_fn on_window, void* user, float* V_host,
                                     float* D_host, void* ws, size_t ws_bytes, void* stream);

/* ---- Fast material decomposition, semi-supervised back half (NEXT-2):
 * Algorithm 2 after the subspace reconstruction, on X
 * [K][N_x] (hsnct_fbp's output).  1 <= n_mat <= min(K, 8).  Workspace:
 * hsnct_workspace_bytes(h, HSNCT_OP_FMD) (device, 256-byte aligned).
 *
 * Transformation matrix, Eq. 7: T[i][j] = mean of X[j][n]
 * over the voxels n with labels[n] == i (labels: DEVICE int32 [N_x], values
 * -1 (no region) or 0..n_mat-1, the user-provided homogeneous regions M_i).
 * T: DEVICE fp32 [n_mat][K].  Deferred errors (hsnct_sync): a label >= n_mat or
 * an empty region -> HSNCT_E_DATA. */
hsnct_status hsnct_fmd_transform(hsnct_t h, const float* X, const int32_t* labels, int n_mat, float* T,
                                 void* ws, size_t ws_bytes, void* stream);

/* Material estimation, Eq. 8: for every voxel n,
 * Xm[:, n] = argmin_{x >= 0} || X[:, n] - T^T x ||_2 (non-negative least
 * squares, exact KKT solution).  Xm: DEVICE fp32 [n_mat][N_x] (material-planar).
 * A singular T T^T -> HSNCT_E_NUMERIC (deferred). */
hsnct_status hsnct_fmd_materials(hsnct_t h, const float* X, const float* T, int n_mat, float* Xm,
                                 void* ws, size_t ws_bytes, void* stream);

/* mu-spectra estimation, Eq. 9: D^m = D^s T^T, i.e. with D
 * stored as (D^s)^T [K][N_k]:  Dm[i][l] = sum_k T[i][k] D[k][l],  Dm: DEVICE fp32
 * [n_mat][N_k]. */
hsnct_status hsnct_fmd_spectra(hsnct_t h, const float* D, const float* T, int n_mat, float* Dm, void* stream);

/* Waits for the stream, then returns and clears the deferred status
 * (HSNCT_OK, HSNCT_E_DATA or HSNCT_E_NUMERIC), or HSNCT_E_CUDA. */
hsnct_status hsnct_sync(hsnct_t h, void* stream);

/* Number of kernels this handle has launched since create (for launch-count
 * accounting in bench.py). */
uint64_t hsnct_kernel_launches(hsnct_t h);

/* Diagnostics.  When the environment variable HSNCT_TRACE=1 is set at
 * hsnct_create, the persistent decompose kernel records %globaltimer stamps (ns)
 * per iteration and CTA: [iter][cta][8] = iteration start, row pass end, first
 * grid barrier passed, D update done, iteration end, partials reduced, D slice
 * updated, G reduced and D restaged (first 256 iterations of the last call).  Copies min(n, available) values to the HOST buffer; *n_out
 * receives the number available (0 when tracing is off), *n_cta the CTA count
 * (both nullable).  Synchronous. */
hsnct_status hsnct_debug_trace(hsnct_t h, uint64_t* host, size_t n, size_t* n_out, int* n_cta);

/* Statistic of the last hsnct_subspace_decompose on this handle (SPEC's clamped-count
 * statistic, reading R6): *n_clamped receives the number of entries of Y (bins < N_k of the
 * N_p rows) that were negative and entered the NMF as 0.  Waits for `stream` (the call's
 * stream).  Counted with integer atomics, so exact and deterministic. */
hsnct_status hsnct_decompose_stats(hsnct_t h, int64_t* n_clamped, void* stream);

/* Diagnostics: the subspace-extraction plan chosen at create (which row-pass kernel, its
 * template parameters and grid), as a NUL-terminated string copied to the HOST buffer
 * buf (at most n bytes, truncated).  Shapes that differ only in N_r beyond a few row
 * tiles select the same plan; the GPU tests use this to show that the slice-reduced
 * full-iteration parity configs run the bench configs' kernels. */
hsnct_status hsnct_debug_plan(hsnct_t h, char* buf, size_t n);

/* Diagnostics: stage timing of hsnct_fbp (bench.py's per-stage rooflines).
 * hsnct_debug_fbp_timing(h, 1) makes every later hsnct_fbp call record CUDA events
 * around its ramp-filter and backprojection launches (on the call's stream);
 * hsnct_debug_fbp_timing(h, 0) stops it (synchronises the device).
 * hsnct_debug_fbp_times waits for the last timed call and writes its two durations in
 * milliseconds to the HOST array ms[2] = {ramp filter, backprojection};
 * HSNCT_E_ARG when no timed call was made since timing was switched on. */
hsnct_status hsnct_debug_fbp_timing(hsnct_t h, int on);
hsnct_status hsnct_debug_fbp_times(hsnct_t h, float* ms);

/* Diagnostics: stage timing of hsnct_subspace_decompose / _counts (bench.py's NMF roofline, measured
 * on the dominant kernel's own launches).  hsnct_debug_nmf_timing(h, 1) makes every later
 * decompose record CUDA events (on the call's stream) around its input preparation (Y+ or counts
 * into the row pass's layout, G = D0 D0^T) and around its iterations (the one persistent launch,
 * or the per-iteration launches); hsnct_debug_nmf_timing(h, 0) stops it (synchronises the
 * device).  hsnct_debug_nmf_times waits for the last timed call and writes ms[2] = {preparation,
 * iterations} (HOST array, milliseconds); HSNCT_E_ARG when no timed call was made since timing
 * was switched on. */
hsnct_status hsnct_debug_nmf_timing(hsnct_t h, int on);
hsnct_status hsnct_debug_nmf_times(hsnct_t h, float* ms);

/* Static description of a status code; never NULL. */
const char* hsnct_status_string(hsnct_status st);

/* Thread-local description of the last error raised by any call on this
 * thread (argument that failed, CUDA error string); "" if none. */
const char* hsnct_last_error(void);

/* HSNCT_ABI_VERSION of the loaded library. */
int hsnct_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HSNCT_H_ */
