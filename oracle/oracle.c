/*
 * oracle/oracle.c -- plain, slow, fp64 CPU oracle for the FHR hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2410_22500_b200/csrc); neither side includes or links the other.
 *
 * Every function follows a passage of /root/reference/PAPER.md (cited as
 * PAPER.md:<line>, with the equation/algorithm it falls in) or, where the
 * paper is silent, a reading listed in DESIGN.md §3 ("Readings").  All
 * arithmetic is IEEE fp64 in the order the formula states; OpenMP is used
 * only across independent outputs, each of which is accumulated in a fixed
 * sequential order, so results do not depend on the thread count.
 *
 * Notation (§II): N_v views, N_r detector rows (slices),
 * N_c detector columns (image width), N_k wavelength bins, N_p = N_v N_r N_c,
 * N_x = N_r N_c N_c.  The projection matrix p in R^{N_p x N_k}
 * is stored row-major with row index p = (v*N_r + r)*N_c + c and the bin
 * index fastest ("y_{v,r,c,k}").  The subspace dimension N_s
 * is called K here; D is stored as (D^s)^T, K x N_k.
 *
 * Parity pins: see tests/test_oracle_*.py.  Nothing in this file is
 * "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_PI 3.14159265358979323846264338327950288

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* Subspace extraction: Eq. 4                            */
/*   (V^s, D^s) = argmin_{V>=0, D>=0} || p - V D^T ||_F^2                    */
/* solved (reading R1, R2, R3 in DESIGN.md) by the textbook Lee-Seung        */
/* Frobenius multiplicative updates, V half-step first, denominators         */
/* floored at 1e-30, on Y+ = max(Y, 0) (reading R6).                         */
/* ------------------------------------------------------------------------ */

static inline double yplus(const float* Y, int64_t ld, int64_t p, int64_t l) {
    double y = (double)Y[p * ld + l];
    return y > 0.0 ? y : 0.0;
}

/* || Y+ - V D ||_F^2, straight from the definition. */
double oracle_nmf_objective(const float* Y, int64_t Np, int64_t Nk, int64_t ld_y, int K,
                            const double* V, const double* D, int nthreads) {
    set_threads(nthreads);
    double* rows = (double*)malloc(sizeof(double) * (size_t)(Np > 0 ? Np : 1));
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < Np; ++p) {
        double s = 0.0;
        for (int64_t l = 0; l < Nk; ++l) {
            double vd = 0.0;
            for (int k = 0; k < K; ++k) vd += V[p * K + k] * D[(int64_t)k * Nk + l];
            double e = yplus(Y, ld_y, p, l) - vd;
            s += e * e;
        }
        rows[p] = s;
    }
    double f = 0.0;
    for (int64_t p = 0; p < Np; ++p) f += rows[p];
    free(rows);
    return f;
}

/*
 * n_iter Lee-Seung iterations from the caller's (V, D) (in/out, fp64).
 * One iteration (reading R2, V first):
 *   A = Y+ D^T;  G = D D^T;  V <- V .* A ./ max(V G, 1e-30)
 *   B = V^T Y+;  H = V^T V;  D <- D .* B ./ max(H D, 1e-30)
 * obj (nullable, 2*n_iter): ||Y+ - V D||^2 after the V half and after the D
 * half of every iteration, by oracle_nmf_objective.
 */
int oracle_nmf(const float* Y, int64_t Np, int64_t Nk, int64_t ld_y, int K,
               double* V, double* D, int n_iter, double* obj, int nthreads) {
    if (Np < 0 || Nk < 0 || K < 1 || K > 16 || ld_y < Nk || n_iter < 0) return 1;
    set_threads(nthreads);
    double* G = (double*)malloc(sizeof(double) * K * K);
    double* H = (double*)malloc(sizeof(double) * K * K);
    double* B = (double*)malloc(sizeof(double) * (size_t)K * (size_t)(Nk > 0 ? Nk : 1));
    for (int it = 0; it < n_iter; ++it) {
        /* G = D D^T */
        for (int a = 0; a < K; ++a)
            for (int b = 0; b < K; ++b) {
                double s = 0.0;
                for (int64_t l = 0; l < Nk; ++l) s += D[(int64_t)a * Nk + l] * D[(int64_t)b * Nk + l];
                G[a * K + b] = s;
            }
        /* V half-step: rows are independent. */
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < Np; ++p) {
            double A[64], VG[64];
            for (int k = 0; k < K; ++k) {
                double s = 0.0;
                for (int64_t l = 0; l < Nk; ++l) s += yplus(Y, ld_y, p, l) * D[(int64_t)k * Nk + l];
                A[k] = s;
            }
            for (int k = 0; k < K; ++k) {
                double s = 0.0;
                for (int j = 0; j < K; ++j) s += V[p * K + j] * G[j * K + k];
                VG[k] = s;
            }
            for (int k = 0; k < K; ++k) {
                double den = VG[k] > 1e-30 ? VG[k] : 1e-30;
                V[p * K + k] = V[p * K + k] * A[k] / den;
            }
        }
        if (obj) obj[2 * it] = oracle_nmf_objective(Y, Np, Nk, ld_y, K, V, D, nthreads);
        /* H = V^T V (fixed row order). */
        for (int a = 0; a < K; ++a)
            for (int b = 0; b < K; ++b) {
                double s = 0.0;
                for (int64_t p = 0; p < Np; ++p) s += V[p * K + a] * V[p * K + b];
                H[a * K + b] = s;
            }
        /* B = V^T Y+: every (k, l) output sums rows in order p = 0..Np-1. */
#pragma omp parallel for schedule(static)
        for (int64_t l0 = 0; l0 < Nk; l0 += 64) {
            int64_t l1 = l0 + 64 < Nk ? l0 + 64 : Nk;
            double acc[16 * 64];
            for (int k = 0; k < K; ++k)
                for (int64_t l = l0; l < l1; ++l) acc[k * 64 + (l - l0)] = 0.0;
            for (int64_t p = 0; p < Np; ++p)
                for (int64_t l = l0; l < l1; ++l) {
                    double y = yplus(Y, ld_y, p, l);
                    for (int k = 0; k < K; ++k) acc[k * 64 + (l - l0)] += V[p * K + k] * y;
                }
            for (int k = 0; k < K; ++k)
                for (int64_t l = l0; l < l1; ++l) B[(int64_t)k * Nk + l] = acc[k * 64 + (l - l0)];
        }
        /* D half-step: columns are independent. */
        for (int64_t l = 0; l < Nk; ++l) {
            double HD[64];
            for (int k = 0; k < K; ++k) {
                double s = 0.0;
                for (int j = 0; j < K; ++j) s += H[k * K + j] * D[(int64_t)j * Nk + l];
                HD[k] = s;
            }
            for (int k = 0; k < K; ++k) {
                double den = HD[k] > 1e-30 ? HD[k] : 1e-30;
                D[(int64_t)k * Nk + l] = D[(int64_t)k * Nk + l] * B[(int64_t)k * Nk + l] / den;
            }
        }
        if (obj) obj[2 * it + 1] = oracle_nmf_objective(Y, Np, Nk, ld_y, K, V, D, nthreads);
    }
    free(G);
    free(H);
    free(B);
    return 0;
}

/*
 * Sampled single-iteration checks at sizes the full oracle cannot reach
 * (tests at BASELINE.json full size): from the GPU's (V_n, D_n) the oracle
 * recomputes, for the listed rows, the V half-step of iteration n+1
 * (row-local, PAPER.md:191 via reading R2), and for the listed bins, the
 * D half-step given the full V_{n+1} (column-local).  Same formulas as
 * oracle_nmf, restricted to the requested outputs.
 */
int oracle_nmf_vstep_rows(const float* Y, int64_t Np, int64_t Nk, int64_t ld_y, int K,
                          const double* V, const double* D, const int64_t* rows, int64_t nrows,
                          double* Vout /* nrows x K */, int nthreads) {
    set_threads(nthreads);
    double G[256];
    for (int a = 0; a < K; ++a)
        for (int b = 0; b < K; ++b) {
            double s = 0.0;
            for (int64_t l = 0; l < Nk; ++l) s += D[(int64_t)a * Nk + l] * D[(int64_t)b * Nk + l];
            G[a * K + b] = s;
        }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nrows; ++i) {
        int64_t p = rows[i];
        for (int k = 0; k < K; ++k) {
            double A = 0.0, VG = 0.0;
            for (int64_t l = 0; l < Nk; ++l) A += yplus(Y, ld_y, p, l) * D[(int64_t)k * Nk + l];
            for (int j = 0; j < K; ++j) VG += V[p * K + j] * G[j * K + k];
            double den = VG > 1e-30 ? VG : 1e-30;
            Vout[i * K + k] = V[p * K + k] * A / den;
        }
    }
    (void)Np;
    return 0;
}

int oracle_nmf_dstep_cols(const float* Y, int64_t Np, int64_t Nk, int64_t ld_y, int K,
                          const double* V /* V_{n+1}, Np x K */, const double* D /* D_n */,
                          const int64_t* cols, int64_t ncols, double* Dout /* K x ncols */,
                          int nthreads) {
    set_threads(nthreads);
    double H[256];
    for (int a = 0; a < K; ++a)
        for (int b = 0; b < K; ++b) {
            double s = 0.0;
            for (int64_t p = 0; p < Np; ++p) s += V[p * K + a] * V[p * K + b];
            H[a * K + b] = s;
        }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < ncols; ++i) {
        int64_t l = cols[i];
        for (int k = 0; k < K; ++k) {
            double B = 0.0, HD = 0.0;
            for (int64_t p = 0; p < Np; ++p) B += V[p * K + k] * yplus(Y, ld_y, p, l);
            for (int j = 0; j < K; ++j) HD += H[k * K + j] * D[(int64_t)j * Nk + l];
            double den = HD > 1e-30 ? HD : 1e-30;
            Dout[(int64_t)k * ncols + i] = D[(int64_t)k * Nk + l] * B / den;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Tomographic reconstruction by FBP (reading R10-R16).    */
/* ------------------------------------------------------------------------ */

/* Kak-Slaney discrete Ram-Lak kernel with detector pitch tau = 1 (R11):
 * h[0] = 1/4, h[even != 0] = 0, h[odd d] = -1/(pi^2 d^2). */
double oracle_ramp_kernel(int64_t d) {
    if (d == 0) return 0.25;
    if (d % 2 == 0) return 0.0;
    return -1.0 / (OR_PI * OR_PI * (double)d * (double)d);
}

/* Direct linear convolution q[c] = sum_{m=0}^{Nc-1} h[c-m] s[m] of each of
 * nrows contiguous rows of length Nc (R11: no FFT in the oracle). */
static void ramp_filter_row(const double* sr, double* qr, int64_t Nc) {
    for (int64_t c = 0; c < Nc; ++c) {
        double acc = 0.0;
        for (int64_t m = 0; m < Nc; ++m) acc += oracle_ramp_kernel(c - m) * sr[m];
        qr[c] = acc;
    }
}

void oracle_ramp_filter_rows(const double* s, double* q, int64_t nrows, int64_t Nc, int nthreads) {
    set_threads(nthreads);
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < nrows; ++row) ramp_filter_row(s + row * Nc, q + row * Nc, Nc);
}

/* theta_v = v*pi/Nv (R13) unless the caller passes angles. */
static double view_angle(const double* angles, int64_t v, int64_t Nv) {
    return angles ? angles[v] : (double)v * OR_PI / (double)Nv;
}

/* Voxel-driven linear-interpolation backprojection of one slice (R12, R14,
 * R16): X[i][j] = (pi/Nv) sum_v [(1-w) q_v[i0] + w q_v[i0+1]],
 * u = x_j cos(theta_v) + y_i sin(theta_v) + (Nc-1)/2, i0 = floor(u),
 * w = u - i0, q outside [0, Nc-1] = 0, x_j = j-(Nc-1)/2, y_i = i-(Nc-1)/2.
 * q is [Nv][Nc] (filtered sinogram of the slice). */
void oracle_backproject_slice(const double* q, int64_t Nv, int64_t Nc, const double* angles,
                              double* X) {
    double half = 0.5 * (double)(Nc - 1);
    for (int64_t i = 0; i < Nc; ++i)
        for (int64_t j = 0; j < Nc; ++j) {
            double x = (double)j - half, y = (double)i - half, acc = 0.0;
            for (int64_t v = 0; v < Nv; ++v) {
                double th = view_angle(angles, v, Nv);
                double u = x * cos(th) + y * sin(th) + half;
                double fl = floor(u);
                int64_t i0 = (int64_t)fl;
                double w = u - fl;
                double a = (i0 >= 0 && i0 < Nc) ? q[v * Nc + i0] : 0.0;
                double b = (i0 + 1 >= 0 && i0 + 1 < Nc) ? q[v * Nc + i0 + 1] : 0.0;
                acc += (1.0 - w) * a + w * b;
            }
            X[i * Nc + j] = OR_PI / (double)Nv * acc;
        }
}

/* Exact matrix adjoint of oracle_backproject_slice (without the pi/Nv
 * factor's transpose being special: it is a scalar): a voxel-driven
 * "splat" forward projector.  Check-only tool for the adjoint pin. */
void oracle_splat_project_slice(const double* X, int64_t Nv, int64_t Nc, const double* angles,
                                double* P) {
    double half = 0.5 * (double)(Nc - 1);
    for (int64_t t = 0; t < Nv * Nc; ++t) P[t] = 0.0;
    for (int64_t v = 0; v < Nv; ++v) {
        double th = view_angle(angles, v, Nv);
        for (int64_t i = 0; i < Nc; ++i)
            for (int64_t j = 0; j < Nc; ++j) {
                double x = (double)j - half, y = (double)i - half;
                double u = x * cos(th) + y * sin(th) + half;
                double fl = floor(u);
                int64_t i0 = (int64_t)fl;
                double w = u - fl, val = OR_PI / (double)Nv * X[i * Nc + j];
                if (i0 >= 0 && i0 < Nc) P[v * Nc + i0] += (1.0 - w) * val;
                if (i0 + 1 >= 0 && i0 + 1 < Nc) P[v * Nc + i0 + 1] += w * val;
            }
    }
}

/* Naive ray-sampled Radon transform of an Nc x Nc image (check-only tool):
 * P[v][c] = sum_s f(t e_theta + s e_perp) * ds, bilinear sampling of the
 * pixel grid (pixel (i,j) at (x_j, y_i)), ds = step, s in [-Nc, Nc]. */
void oracle_radon_naive(const double* img, int64_t Nc, int64_t Nv, const double* angles,
                        double step, double* P, int nthreads) {
    set_threads(nthreads);
    double half = 0.5 * (double)(Nc - 1);
#pragma omp parallel for schedule(static)
    for (int64_t vc = 0; vc < Nv * Nc; ++vc) {
        int64_t v = vc / Nc, c = vc % Nc;
        double th = view_angle(angles, v, Nv);
        double ct = cos(th), st = sin(th), t = (double)c - half, acc = 0.0;
        int64_t ns = (int64_t)ceil((double)Nc / step);
        for (int64_t n = -ns; n <= ns; ++n) {
            double s = (double)n * step;
            double x = t * ct - s * st, y = t * st + s * ct;
            double fj = x + half, fi = y + half;
            double j0 = floor(fj), i0 = floor(fi);
            double wj = fj - j0, wi = fi - i0;
            int64_t J = (int64_t)j0, I = (int64_t)i0;
            double val = 0.0;
            for (int di = 0; di < 2; ++di)
                for (int dj = 0; dj < 2; ++dj) {
                    int64_t ii = I + di, jj = J + dj;
                    if (ii < 0 || ii >= Nc || jj < 0 || jj >= Nc) continue;
                    double wgt = (di ? wi : 1.0 - wi) * (dj ? wj : 1.0 - wj);
                    val += wgt * img[ii * Nc + jj];
                }
            acc += val * step;
        }
        P[vc] = acc;
    }
}

/* FBP of K subspace sinograms (Algorithm 1, "Tomographic Reconstruction",
 * PAPER.md:240-243, with FBP per reading R10).  V is the N_p x K subspace
 * view matrix V^s; column k reshaped to (N_v, N_r, N_c) is
 * sinogram k.  X out: [K][N_r][N_c][N_c] (x^s in R^{N_x x N_s}, PAPER.md:223,
 * stored channel-planar). */
int oracle_fbp(const double* V, int64_t Nv, int64_t Nr, int64_t Nc, int K, const double* angles,
               double* X, int nthreads) {
    if (Nv < 1 || Nr < 1 || Nc < 1 || K < 1) return 1;
    set_threads(nthreads);
#pragma omp parallel for schedule(dynamic) collapse(2)
    for (int k = 0; k < K; ++k)
        for (int64_t r = 0; r < Nr; ++r) {
            double* s = (double*)malloc(sizeof(double) * Nv * Nc);
            double* q = (double*)malloc(sizeof(double) * Nv * Nc);
            for (int64_t v = 0; v < Nv; ++v)
                for (int64_t c = 0; c < Nc; ++c) s[v * Nc + c] = V[((v * Nr + r) * Nc + c) * K + k];
            for (int64_t v = 0; v < Nv; ++v) ramp_filter_row(s + v * Nc, q + v * Nc, Nc);
            oracle_backproject_slice(q, Nv, Nc, angles, X + ((int64_t)k * Nr + r) * Nc * Nc);
            free(s);
            free(q);
        }
    return 0;
}

/* Subspace expansion, Eq. 6: x^h = x^s (D^s)^T, as the
 * triple loop xh[n][l] = sum_k X[k][n] D[k][l] over the window of slices
 * [s0, s0+ns) and bins [b0, b0+nb).  Xh out: [ns*Nc*Nc][nb]. */
int oracle_synthesize(const double* X, const double* D, int64_t Nr, int64_t Nc, int64_t Nk, int K,
                      int64_t s0, int64_t ns, int64_t b0, int64_t nb, double* Xh, int nthreads) {
    if (s0 < 0 || ns < 0 || s0 + ns > Nr || b0 < 0 || nb < 0 || b0 + nb > Nk) return 1;
    set_threads(nthreads);
    int64_t Nx = Nr * Nc * Nc, n0 = s0 * Nc * Nc, nn = ns * Nc * Nc;
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < nn; ++n)
        for (int64_t l = 0; l < nb; ++l) {
            double acc = 0.0;
            for (int k = 0; k < K; ++k) acc += X[(int64_t)k * Nx + n0 + n] * D[(int64_t)k * Nk + b0 + l];
            Xh[n * nb + l] = acc;
        }
    return 0;
}

/* Direct hyperspectral reconstruction, the paper's baseline (PAPER.md:441-442:
 * "DHR performs N_k individual 3D reconstructions, one for each wavelength
 * bin in p ... using FBP"): for each bin l in the window the sinogram
 * Y[(v,r,c), l] (raw, unclamped: R6) is ramp-filtered and backprojected.
 * Xh out: [ns*Nc*Nc][nb]. */
int oracle_dhr(const float* Y, int64_t ld_y, int64_t Nv, int64_t Nr, int64_t Nc, int64_t Nk,
               const double* angles, int64_t s0, int64_t ns, int64_t b0, int64_t nb, double* Xh,
               int nthreads) {
    if (s0 < 0 || ns < 0 || s0 + ns > Nr || b0 < 0 || nb < 0 || b0 + nb > Nk) return 1;
    set_threads(nthreads);
    int64_t NN = Nc * Nc;
#pragma omp parallel for schedule(dynamic) collapse(2)
    for (int64_t r = s0; r < s0 + ns; ++r)
        for (int64_t l = b0; l < b0 + nb; ++l) {
            double* s = (double*)malloc(sizeof(double) * Nv * Nc);
            double* q = (double*)malloc(sizeof(double) * Nv * Nc);
            double* x = (double*)malloc(sizeof(double) * NN);
            for (int64_t v = 0; v < Nv; ++v)
                for (int64_t c = 0; c < Nc; ++c) s[v * Nc + c] = (double)Y[((v * Nr + r) * Nc + c) * ld_y + l];
            for (int64_t v = 0; v < Nv; ++v) ramp_filter_row(s + v * Nc, q + v * Nc, Nc);
            oracle_backproject_slice(q, Nv, Nc, angles, x);
            for (int64_t n = 0; n < NN; ++n) Xh[((r - s0) * NN + n) * nb + (l - b0)] = x[n];
            free(s);
            free(q);
            free(x);
        }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Fast material decomposition, semi-supervised back half (*/
/* Section "Fast Material Decomposition", Algorithm 2), on the subspace      */
/* reconstructions x^s (stored channel-planar X[K][Nx], reading R10).        */
/* ------------------------------------------------------------------------ */

/* Transformation matrix, Eq. 7:
 *   T[i][j] = (1/|M_i|) sum_{n in M_i} x^s[n][j],
 * with the regions M_i given as labels[n] = i (labels < 0: no region).
 * counts[i] = |M_i|.  Returns 1 on a bad label, 2 if some region is empty. */
int oracle_fmd_transform(const double* X, int64_t Nx, int K, const int32_t* labels, int Nm, double* T,
                         int64_t* counts) {
    for (int i = 0; i < Nm; ++i) {
        counts[i] = 0;
        for (int j = 0; j < K; ++j) T[i * K + j] = 0.0;
    }
    for (int64_t n = 0; n < Nx; ++n) {
        const int32_t i = labels[n];
        if (i < 0) continue;
        if (i >= Nm) return 1;
        counts[i] += 1;
        for (int j = 0; j < K; ++j) T[i * K + j] += X[(int64_t)j * Nx + n];
    }
    for (int i = 0; i < Nm; ++i) {
        if (counts[i] == 0) return 2;
        for (int j = 0; j < K; ++j) T[i * K + j] /= (double)counts[i];
    }
    return 0;
}

/* Solve the m x m system A z = r (A row-major, copied) by Gaussian elimination with
 * partial pivoting.  Returns 1 if singular. */
static int solve_small(const double* A, const double* r, int m, double* z) {
    double M[64 * 65];
    for (int i = 0; i < m; ++i) {
        for (int j = 0; j < m; ++j) M[i * (m + 1) + j] = A[i * m + j];
        M[i * (m + 1) + m] = r[i];
    }
    for (int c = 0; c < m; ++c) {
        int p = c;
        for (int i = c + 1; i < m; ++i)
            if (fabs(M[i * (m + 1) + c]) > fabs(M[p * (m + 1) + c])) p = i;
        if (M[p * (m + 1) + c] == 0.0) return 1;
        if (p != c)
            for (int j = 0; j <= m; ++j) {
                double t = M[c * (m + 1) + j];
                M[c * (m + 1) + j] = M[p * (m + 1) + j];
                M[p * (m + 1) + j] = t;
            }
        for (int i = c + 1; i < m; ++i) {
            double f = M[i * (m + 1) + c] / M[c * (m + 1) + c];
            for (int j = c; j <= m; ++j) M[i * (m + 1) + j] -= f * M[c * (m + 1) + j];
        }
    }
    for (int i = m - 1; i >= 0; --i) {
        double s = M[i * (m + 1) + m];
        for (int j = i + 1; j < m; ++j) s -= M[i * (m + 1) + j] * z[j];
        z[i] = s / M[i * (m + 1) + i];
    }
    return 0;
}

/* Non-negative least squares min_{x >= 0} ||A x - y||_2 for A (rows x m, row-major),
 * following Lawson & Hanson, "Solving Least Squares Problems" (1974), Ch. 23,
 * Algorithm NNLS (the algorithm named by Eq. 8: argmin_{x>=0}).
 * Working on the normal equations (A^T A) x = A^T y restricted to the passive set.
 * m <= 64.  x (m) out.  Returns the number of outer iterations, or -1 on failure. */
int oracle_nnls(const double* A, int rows, int m, const double* y, double* x) {
    double AtA[64 * 64], Aty[64], z[64], sub[64 * 64], rhs[64];
    int P[64];
    if (m < 1 || m > 64) return -1;
    for (int i = 0; i < m; ++i) {
        x[i] = 0.0;
        P[i] = 0;
        double s = 0.0;
        for (int r = 0; r < rows; ++r) s += A[r * m + i] * y[r];
        Aty[i] = s;
        for (int j = 0; j < m; ++j) {
            double t = 0.0;
            for (int r = 0; r < rows; ++r) t += A[r * m + i] * A[r * m + j];
            AtA[i * m + j] = t;
        }
    }
    double amax = 0.0;
    for (int i = 0; i < m; ++i) amax = fabs(Aty[i]) > amax ? fabs(Aty[i]) : amax;
    const double tol = 1e-13 * amax + 1e-300; /* w_i > tol: a real improvement direction */
    int outer = 0;
    for (; outer < 3 * m + 3; ++outer) {
        /* step 2: w = A^T (y - A x) */
        int t = -1;
        double wmax = 0.0;
        for (int i = 0; i < m; ++i) {
            double s = Aty[i];
            for (int j = 0; j < m; ++j) s -= AtA[i * m + j] * x[j];
            if (!P[i] && s > tol && s > wmax) {
                wmax = s;
                t = i;
            }
        }
        if (t < 0) return outer; /* step 3: KKT satisfied */
        P[t] = 1;                /* step 5 */
        for (;;) {
            /* step 6: z = LS solution on the passive set, 0 elsewhere */
            int idx[64], np = 0;
            for (int i = 0; i < m; ++i)
                if (P[i]) idx[np++] = i;
            for (int a = 0; a < np; ++a) {
                rhs[a] = Aty[idx[a]];
                for (int b = 0; b < np; ++b) sub[a * np + b] = AtA[idx[a] * m + idx[b]];
            }
            double zp[64];
            if (solve_small(sub, rhs, np, zp)) return -1;
            for (int i = 0; i < m; ++i) z[i] = 0.0;
            for (int a = 0; a < np; ++a) z[idx[a]] = zp[a];
            /* step 7: all passive z > 0 -> accept */
            int ok = 1;
            for (int a = 0; a < np; ++a)
                if (z[idx[a]] <= 0.0) ok = 0;
            if (ok) {
                for (int i = 0; i < m; ++i) x[i] = z[i];
                break;
            }
            /* steps 8-11: move towards z until a passive variable hits 0 */
            double alpha = 1e300;
            for (int a = 0; a < np; ++a) {
                const int i = idx[a];
                if (z[i] <= 0.0) {
                    const double al = x[i] / (x[i] - z[i]);
                    if (al < alpha) alpha = al;
                }
            }
            for (int i = 0; i < m; ++i) x[i] += alpha * (z[i] - x[i]);
            for (int a = 0; a < np; ++a) {
                const int i = idx[a];
                if (fabs(x[i]) <= 1e-15) {
                    x[i] = 0.0;
                    P[i] = 0;
                }
            }
        }
    }
    return outer;
}

/* Material estimation, Eq. 8: for every voxel n,
 *   x^m[n] = argmin_{x >= 0} || x^s[n] - x T ||^2,
 * i.e. NNLS with A = T^T (K x Nm) and y = x^s[n] (K).  Xm out: [Nm][Nx] material-planar.
 * Returns the number of voxels where NNLS failed. */
int64_t oracle_fmd_materials(const double* X, int64_t Nx, int K, const double* T, int Nm, double* Xm,
                             int nthreads) {
    set_threads(nthreads);
    double At[64 * 8];
    for (int j = 0; j < K; ++j)
        for (int i = 0; i < Nm; ++i) At[j * Nm + i] = T[i * K + j];
    int64_t fails = 0;
#pragma omp parallel for schedule(static) reduction(+ : fails)
    for (int64_t n = 0; n < Nx; ++n) {
        double y[64], x[8];
        for (int j = 0; j < K; ++j) y[j] = X[(int64_t)j * Nx + n];
        if (oracle_nnls(At, K, Nm, y, x) < 0) fails += 1;
        for (int i = 0; i < Nm; ++i) Xm[(int64_t)i * Nx + n] = x[i];
    }
    return fails;
}

/* mu-spectra estimation, Eq. 9: D^m = D^s T^T.  With D stored as
 * (D^s)^T [K][Nk], the output is (D^m)^T [Nm][Nk]:  Dm[i][l] = sum_k T[i][k] D[k][l]. */
void oracle_fmd_spectra(const double* D, int64_t Nk, int K, const double* T, int Nm, double* Dm) {
    for (int i = 0; i < Nm; ++i)
        for (int64_t l = 0; l < Nk; ++l) {
            double s = 0.0;
            for (int k = 0; k < K; ++k) s += T[i * K + k] * D[(int64_t)k * Nk + l];
            Dm[(int64_t)i * Nk + l] = s;
        }
}

/* ------------------------------------------------------------------ MBIR (NEXT-3)
 * Eq. 5 for one subspace channel of one slice:
 *   x = argmin_{x >= 0} 1/(2 sv^2) ||y - A x||^2 + h(x),
 * A the linear projection operator: (A x)[v][c] = sum_{i,j} x[i][j] max(0, 1 - |u_ij(v) - c|),
 * u_ij(v) = x_j cos(theta_v) + y_i sin(theta_v) + (Nc-1)/2 (readings R13, R14, R16; the exact
 * adjoint of the backprojector without its pi/Nv factor), h the QGGMRF prior (
 * the pairwise form of SPEC.md:199 with q = 2, reading R24):
 *   h(x) = sum over unordered 8-neighbour pairs {i, j} of b_ij rho(x_i - x_j),
 *   rho(d) = |d|^p / (p sx^p) * u / (1 + u),  u = |d / (T sx)|^(q - p),
 *   b = b1 for edge neighbours, b1 / sqrt(2) for diagonal ones, 4 b1 + 4 b1/sqrt(2) = 1 (R25).
 * Solver (reading R26): separable-quadratic-surrogate majorize-minimize iterations.  With
 * w(d) = rho'(d) / d (the half-quadratic curvature, non-increasing in |d| for p <= q = 2):
 *   dd[i] = (1/sv^2) (A^T A 1)[i]                                   (data curvature, A >= 0)
 *   e = y - A x;  g[i] = -(1/sv^2) (A^T e)[i] + sum_{j in N(i)} b_ij rho'(x_i - x_j)
 *   dp[i] = sum_{j in N(i)} 2 b_ij w(x_i - x_j)
 *   x[i] <- max(0, x[i] - g[i] / (dd[i] + dp[i]))          (every voxel from the same x: Jacobi)
 * so the objective is non-increasing at every iteration (majorization).  y: [Nv][Nc];
 * x: [Nc][Nc], in: x0, out: the n_iter-th iterate; obj (nullable): [n_iter + 1] objective
 * values of the iterates 0..n_iter.  prm = {sv, sx, p, q, T}; q must be 2 (w(0) finite). */
static double qg_rho(double d, const double* prm) {
    const double sx = prm[1], p = prm[2], q = prm[3], T = prm[4];
    const double a = fabs(d);
    if (a == 0.0) return 0.0;
    const double u = pow(a / (T * sx), q - p);
    return pow(a, p) / (p * pow(sx, p)) * u / (1.0 + u);
}
/* w(d) = rho'(d)/d = |d|^(p-2)/sx^p * u/(1+u) * (1 + (q-p)/(p (1+u))); with q = 2,
 * |d|^(p-2) u = 1/(T sx)^(2-p), so w(d) = 1/(sx^p (T sx)^(2-p)) / (1+u) * (1 + (2-p)/(p(1+u))). */
static double qg_omega(double d, const double* prm) {
    const double sx = prm[1], p = prm[2], T = prm[4];
    const double u = pow(fabs(d) / (T * sx), 2.0 - p);
    return 1.0 / (pow(sx, p) * pow(T * sx, 2.0 - p)) / (1.0 + u) * (1.0 + (2.0 - p) / (p * (1.0 + u)));
}
double oracle_qggmrf_rho(double d, const double* prm) { return qg_rho(d, prm); }
double oracle_qggmrf_omega(double d, const double* prm) { return qg_omega(d, prm); }

void oracle_mbir_project_slice(const double* X, int64_t Nv, int64_t Nc, const double* angles, double* P) {
    double half = 0.5 * (double)(Nc - 1);
    for (int64_t t = 0; t < Nv * Nc; ++t) P[t] = 0.0;
    for (int64_t v = 0; v < Nv; ++v) {
        double th = view_angle(angles, v, Nv);
        for (int64_t i = 0; i < Nc; ++i)
            for (int64_t j = 0; j < Nc; ++j) {
                double u = ((double)j - half) * cos(th) + ((double)i - half) * sin(th) + half;
                double fl = floor(u), w = u - fl;
                int64_t i0 = (int64_t)fl;
                if (i0 >= 0 && i0 < Nc) P[v * Nc + i0] += (1.0 - w) * X[i * Nc + j];
                if (i0 + 1 >= 0 && i0 + 1 < Nc) P[v * Nc + i0 + 1] += w * X[i * Nc + j];
            }
    }
}
void oracle_mbir_backproject_slice(const double* R, int64_t Nv, int64_t Nc, const double* angles, double* X) {
    double half = 0.5 * (double)(Nc - 1);
    for (int64_t i = 0; i < Nc; ++i)
        for (int64_t j = 0; j < Nc; ++j) {
            double acc = 0.0;
            for (int64_t v = 0; v < Nv; ++v) {
                double th = view_angle(angles, v, Nv);
                double u = ((double)j - half) * cos(th) + ((double)i - half) * sin(th) + half;
                double fl = floor(u), w = u - fl;
                int64_t i0 = (int64_t)fl;
                double a = (i0 >= 0 && i0 < Nc) ? R[v * Nc + i0] : 0.0;
                double b = (i0 + 1 >= 0 && i0 + 1 < Nc) ? R[v * Nc + i0 + 1] : 0.0;
                acc += (1.0 - w) * a + w * b;
            }
            X[i * Nc + j] = acc;
        }
}

static const int NB_DI[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
static const int NB_DJ[8] = {-1, 0, 1, -1, 1, -1, 0, 1};

static double mbir_objective(const double* y, const double* ax, int64_t Nv, int64_t Nc, const double* x,
                             const double* prm, double b1) {
    double data = 0.0, prior = 0.0;
    for (int64_t t = 0; t < Nv * Nc; ++t) data += (y[t] - ax[t]) * (y[t] - ax[t]);
    for (int64_t i = 0; i < Nc; ++i)
        for (int64_t j = 0; j < Nc; ++j)
            for (int n = 0; n < 8; ++n) {  /* each unordered pair once: neighbours after (i, j) */
                int64_t i2 = i + NB_DI[n], j2 = j + NB_DJ[n];
                if (i2 < 0 || i2 >= Nc || j2 < 0 || j2 >= Nc) continue;
                if (i2 * Nc + j2 <= i * Nc + j) continue;
                double b = (NB_DI[n] != 0 && NB_DJ[n] != 0) ? b1 / sqrt(2.0) : b1;
                prior += b * qg_rho(x[i * Nc + j] - x[i2 * Nc + j2], prm);
            }
    return data / (2.0 * prm[0] * prm[0]) + prior;
}

int oracle_mbir_slice(const double* y, int64_t Nv, int64_t Nc, const double* angles, const double* prm,
                      int n_iter, double* x, double* obj) {
    if (prm[3] != 2.0 || prm[0] <= 0.0 || prm[1] <= 0.0 || prm[2] < 1.0 || prm[2] > 2.0 || prm[4] <= 0.0) return 1;
    const double iv = 1.0 / (prm[0] * prm[0]);
    const double b1 = 1.0 / (4.0 + 4.0 / sqrt(2.0));
    int64_t n = Nc * Nc, m = Nv * Nc;
    double* one = calloc((size_t)n, sizeof(double));
    double* dd = malloc(sizeof(double) * n);
    double* ax = malloc(sizeof(double) * m);
    double* e = malloc(sizeof(double) * m);
    double* g = malloc(sizeof(double) * n);
    double* xn = malloc(sizeof(double) * n);
    for (int64_t t = 0; t < n; ++t) one[t] = 1.0;
    oracle_mbir_project_slice(one, Nv, Nc, angles, ax);
    oracle_mbir_backproject_slice(ax, Nv, Nc, angles, dd);
    for (int64_t t = 0; t < n; ++t) dd[t] *= iv;
    for (int it = 0; it <= n_iter; ++it) {
        oracle_mbir_project_slice(x, Nv, Nc, angles, ax);
        if (obj) obj[it] = mbir_objective(y, ax, Nv, Nc, x, prm, b1);
        if (it == n_iter) break;
        for (int64_t t = 0; t < m; ++t) e[t] = y[t] - ax[t];
        oracle_mbir_backproject_slice(e, Nv, Nc, angles, g);
        for (int64_t i = 0; i < Nc; ++i)
            for (int64_t j = 0; j < Nc; ++j) {
                double gi = -iv * g[i * Nc + j], di = dd[i * Nc + j];
                for (int k = 0; k < 8; ++k) {
                    int64_t i2 = i + NB_DI[k], j2 = j + NB_DJ[k];
                    if (i2 < 0 || i2 >= Nc || j2 < 0 || j2 >= Nc) continue;
                    double b = (NB_DI[k] != 0 && NB_DJ[k] != 0) ? b1 / sqrt(2.0) : b1;
                    double d = x[i * Nc + j] - x[i2 * Nc + j2], w = qg_omega(d, prm);
                    gi += b * w * d;      /* rho'(d) = w(d) d */
                    di += 2.0 * b * w;
                }
                double v = x[i * Nc + j] - gi / di;
                xn[i * Nc + j] = v > 0.0 ? v : 0.0;
            }
        memcpy(x, xn, sizeof(double) * n);
    }
    free(one);
    free(dd);
    free(ax);
    free(e);
    free(g);
    free(xn);
    return 0;
}

/* MBIR of the K subspace sinograms (Algorithm 1 with Eq. 5 in place of FBP):
 * V [Np][K] (row p = (v Nr + r) Nc + c), X [K][Nr][Nc][Nc] in: x0, out: x_n; every (channel,
 * slice) independently (2-D prior, R25). */
int oracle_mbir(const double* V, int64_t Nv, int64_t Nr, int64_t Nc, int K, const double* angles,
                const double* prm, int n_iter, double* X, int nthreads) {
    set_threads(nthreads);
    int bad = 0;
#pragma omp parallel for schedule(dynamic) reduction(| : bad)
    for (int64_t kr = 0; kr < (int64_t)K * Nr; ++kr) {
        int64_t k = kr / Nr, r = kr % Nr;
        double* y = malloc(sizeof(double) * Nv * Nc);
        for (int64_t v = 0; v < Nv; ++v)
            for (int64_t c = 0; c < Nc; ++c) y[v * Nc + c] = V[((v * Nr + r) * Nc + c) * K + k];
        bad |= oracle_mbir_slice(y, Nv, Nc, angles, prm, n_iter, X + (k * Nr + r) * Nc * Nc, NULL);
        free(y);
    }
    return bad;
}

/* ------------------------------------------------------------------ counts -> projections (NEXT-1)
 * Eq. 2 with the Appendix-A offset and the 1/2-count floor
 * of reading R7:  p[v][r][c][k] = -log(max(y, 1/2) / max(y0, 1/2)) - b[v][k]
 *                                = ln(max(y0, 1/2)) - ln(max(y, 1/2)) - b[v][k],  fp64.
 * y: uint8 [Np][Nk], row p = (v Nr + r) Nc + c; y0: uint8 [Nr Nc][Nk] (open beam, one per (r, c));
 * b: [Nv][Nk] (NULL = 0); P: [Np][Nk]. */
void oracle_counts_to_projections(const uint8_t* y, const uint8_t* y0, const double* b, int64_t Nv, int64_t NrNc,
                                  int64_t Nk, double* P) {
    for (int64_t v = 0; v < Nv; ++v)
        for (int64_t rc = 0; rc < NrNc; ++rc) {
            const int64_t p = v * NrNc + rc;
            for (int64_t k = 0; k < Nk; ++k) {
                const double a = y0[rc * Nk + k] > 0 ? (double)y0[rc * Nk + k] : 0.5;
                const double t = y[p * Nk + k] > 0 ? (double)y[p * Nk + k] : 0.5;
                P[p * Nk + k] = log(a) - log(t) - (b ? b[v * Nk + k] : 0.0);
            }
        }
}
