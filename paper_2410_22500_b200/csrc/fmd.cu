// Fast material decomposition, semi-supervised back half (NEXT-2; PAPER.md:268-373,
// Algorithm 2 after the subspace reconstruction), on the subspace reconstructions
// X [K][N_x] (hsnct_fbp's output):
//
//   k_fmd_tpart / k_fmd_tfinal  Eq. 7: T[i][j] = mean of X[j][n] over the
//                               voxels labelled i; per-block fp64 partial sums over a static
//                               voxel partition, reduced in a fixed block order.
//   k_fmd_prep                  G = T T^T (fp64) and the inverse of every principal
//                               submatrix G_PP, P a subset of the N_m materials.
//   k_fmd_nnls                  Eq. 8: per voxel, the non-negative least
//                               squares solution of min_{x >= 0} ||X[:, n] - T^T x|| as the
//                               passive set that satisfies the KKT conditions, searched in
//                               order of increasing size (fp64; the solution is unique when G
//                               is positive definite, so any KKT set gives the same x).
//   k_fmd_spectra               Eq. 9: (D^m)^T = T D, fp64 accumulation.
#include <algorithm>

#include "internal.h"

namespace hsnct {
namespace {

constexpr int FT = 256;          // threads per block
constexpr int FMD_MAXM = 8;      // materials
constexpr int FMD_RACC = 48;     // fp64 accumulators per thread in the transform pass
#ifndef FMD_NNLS_MINB
#define FMD_NNLS_MINB 2  // two blocks per SM (128 registers): 3.68 -> 2.61 ms at C4; three spill
#endif

__device__ __forceinline__ double warp_sum_dd(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Partial sums of X over the voxels of regions [i0, i0 + nr) for block b's voxel range;
// thread t takes voxels t, t + FT, ... of the range (fixed order), then a fixed-order
// block reduction.  part[b][i - i0][k] (fp64), cnt[b][i - i0] (int64).
template <int K, int RMAX>
__global__ void __launch_bounds__(FT, 2) k_fmd_tpart(const float* __restrict__ X, int64_t Nx,
                                                  const int32_t* __restrict__ labels, int Nm, int i0, int nr,
                                                  int64_t per_blk, double* __restrict__ part,
                                                  long long* __restrict__ cnt, unsigned* __restrict__ status) {
    __shared__ double red[FT / 32][RMAX * K];
    __shared__ long long redc[FT / 32][RMAX];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int64_t n0 = (int64_t)blockIdx.x * per_blk, n1 = min(Nx, n0 + per_blk);
    double s[RMAX][K];
    long long c[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
        c[r] = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) s[r][k] = 0.0;
    }
    unsigned bad = 0;
    for (int64_t n = n0 + tid; n < n1; n += FT) {
        const int lab = labels[n];
        if (lab >= Nm || lab < -1) bad = ST_LABEL_BAD;
        const int rr = lab - i0;
        if (rr < 0 || rr >= nr) continue;
        float x[K];
#pragma unroll
        for (int k = 0; k < K; ++k) x[k] = __ldg(X + (int64_t)k * Nx + n);
#pragma unroll
        for (int r = 0; r < RMAX; ++r)
            if (r == rr) {
                c[r] += 1;
#pragma unroll
                for (int k = 0; k < K; ++k) s[r][k] += (double)x[k];
            }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    if (lane == 0 && bad) atomicOr(status, bad);
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
        long long cc = c[r];
#pragma unroll
        for (int o = 16; o; o >>= 1) cc += __shfl_xor_sync(0xffffffffu, cc, o);
        if (lane == 0) redc[w][r] = cc;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const double v = warp_sum_dd(s[r][k]);
            if (lane == 0) red[w][r * K + k] = v;
        }
    }
    __syncthreads();
    for (int o = tid; o < nr * K; o += FT) {
        double v = 0.0;
        for (int ww = 0; ww < FT / 32; ++ww) v += red[ww][o];
        part[((int64_t)blockIdx.x * FMD_MAXM + i0) * K + o] = v;
    }
    for (int o = tid; o < nr; o += FT) {
        long long v = 0;
        for (int ww = 0; ww < FT / 32; ++ww) v += redc[ww][o];
        cnt[(int64_t)blockIdx.x * FMD_MAXM + i0 + o] = v;
    }
}

// T = (sum over blocks, fixed order) / count; an empty region flags ST_REGION_EMPTY (E_DATA).
__global__ void __launch_bounds__(FT) k_fmd_tfinal(const double* __restrict__ part, const long long* __restrict__ cnt,
                                                   int nblk, int Nm, int K, float* __restrict__ T,
                                                   unsigned* __restrict__ status) {
    for (int o = threadIdx.x; o < Nm * K; o += FT) {
        const int i = o / K;
        double s = 0.0;
        long long c = 0;
        for (int b = 0; b < nblk; ++b) {
            s += part[(int64_t)b * FMD_MAXM * K + o];
            c += cnt[(int64_t)b * FMD_MAXM + i];
        }
        if (c == 0) {
            atomicOr(status, (unsigned)ST_REGION_EMPTY);
            T[o] = 0.f;
        } else {
            T[o] = (float)(s / (double)c);
        }
    }
}

// Offset of subset P's inverse in the packed table: sum over masks Q < P of popcount(Q)^2.
__host__ __device__ inline int inv_off(int P) {
    int o = 0;
    for (int Q = 0; Q < P; ++Q) {
        int c = 0;
        for (int v = Q; v; v &= v - 1) ++c;
        o += c * c;
    }
    return o;
}

// G = T T^T and, for every non-empty subset P (bit mask), the inverse of G_PP (Gauss-Jordan
// with partial pivoting, fp64), packed: |P| x |P| row-major at tab + inv_off(P).
__global__ void __launch_bounds__(FT) k_fmd_prep(const float* __restrict__ T, int Nm, int K,
                                                 double* __restrict__ G, double* __restrict__ tab,
                                                 unsigned* __restrict__ status) {
    __shared__ double Gs[FMD_MAXM * FMD_MAXM];
    for (int o = threadIdx.x; o < Nm * Nm; o += FT) {
        const int a = o / Nm, b = o - (o / Nm) * Nm;
        double s = 0.0;
        for (int k = 0; k < K; ++k) s += (double)T[a * K + k] * (double)T[b * K + k];
        Gs[o] = s;
        G[o] = s;
    }
    __syncthreads();
    for (int P = 1 + threadIdx.x; P < (1 << Nm); P += FT) {
        int idx[FMD_MAXM], m = 0;
        for (int i = 0; i < Nm; ++i)
            if (P & (1 << i)) idx[m++] = i;
        double M[FMD_MAXM][2 * FMD_MAXM];
        for (int a = 0; a < m; ++a)
            for (int b = 0; b < 2 * m; ++b) M[a][b] = b < m ? Gs[idx[a] * Nm + idx[b]] : (b - m == a ? 1.0 : 0.0);
        bool sing = false;
        for (int col = 0; col < m; ++col) {
            int p = col;
            for (int r = col + 1; r < m; ++r)
                if (fabs(M[r][col]) > fabs(M[p][col])) p = r;
            if (!(fabs(M[p][col]) > 0.0)) {
                sing = true;
                break;
            }
            if (p != col)
                for (int b = 0; b < 2 * m; ++b) {
                    const double t = M[col][b];
                    M[col][b] = M[p][b];
                    M[p][b] = t;
                }
            const double inv = 1.0 / M[col][col];
            for (int b = 0; b < 2 * m; ++b) M[col][b] *= inv;
            for (int r = 0; r < m; ++r)
                if (r != col) {
                    const double f = M[r][col];
                    for (int b = 0; b < 2 * m; ++b) M[r][b] -= f * M[col][b];
                }
        }
        double* out = tab + inv_off(P);
        for (int a = 0; a < m; ++a)
            for (int b = 0; b < m; ++b) out[a * m + b] = sing ? 0.0 : M[a][m + b];
        if (sing) atomicOr(status, (unsigned)ST_NUMERIC);
    }
}

// Per voxel NNLS by passive-set search in order of increasing size (subset order table in
// smem), KKT test in fp64.  Xm [Nm][Nx].
template <int K, int NM>
__global__ void __launch_bounds__(FT, FMD_NNLS_MINB) k_fmd_nnls(const float* __restrict__ X, int64_t Nx, const float* __restrict__ T,
                                                 const double* __restrict__ G, const double* __restrict__ tab,
                                                 float* __restrict__ Xm, unsigned* __restrict__ status) {
    constexpr int NS = 1 << NM;
    constexpr int NINV = NM * (NM + 1) * (NS / 4 > 0 ? NS / 4 : 1);  // sum_P |P|^2 = n (n+1) 2^(n-2)
    __shared__ double Ts[NM * K], Gs[NM * NM];
    __shared__ double inv[NINV + 1];
    __shared__ unsigned char order[NS];
    __shared__ short offs[NS];
    for (int o = threadIdx.x; o < NM * K; o += FT) Ts[o] = (double)T[o];
    for (int o = threadIdx.x; o < NM * NM; o += FT) Gs[o] = G[o];
    for (int o = threadIdx.x; o < inv_off(NS); o += FT) inv[o] = tab[o];
    if (threadIdx.x == 0) {  // subsets by increasing size, then by mask (fixed order)
        int q = 0;
        for (int sz = 0; sz <= NM; ++sz)
            for (int P = 0; P < NS; ++P)
                if (__popc(P) == sz) order[q++] = (unsigned char)P;
        int o = 0;
        for (int P = 0; P < NS; ++P) {
            offs[P] = (short)o;
            o += __popc(P) * __popc(P);
        }
    }
    __syncthreads();
    unsigned bad = 0;
    for (int64_t n = (int64_t)blockIdx.x * FT + threadIdx.x; n < Nx; n += (int64_t)gridDim.x * FT) {
        double y[K];
#pragma unroll
        for (int k = 0; k < K; ++k) y[k] = (double)__ldg(X + (int64_t)k * Nx + n);
        double b[NM], bmax = 0.0;
#pragma unroll
        for (int i = 0; i < NM; ++i) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < K; ++k) s = fma(Ts[i * K + k], y[k], s);
            b[i] = s;
            bmax = fmax(bmax, fabs(s));
        }
        const double tol = 1e-12 * bmax;
        double x[NM], best[NM], fbest = 1e300;
        bool found = false;
        // x_P = inv(G_PP) b_P (zero off P); true when every x_P > 0
        auto solve = [&](int P, double* z) {
            const int mP = __popc(P);
            const double* Ip = inv + offs[P];
            bool pos = true;
            int a = 0;
#pragma unroll
            for (int i = 0; i < NM; ++i) {
                z[i] = 0.0;
                if (P & (1 << i)) {
                    double s = 0.0;
                    int c2 = 0;
#pragma unroll
                    for (int j = 0; j < NM; ++j)
                        if (P & (1 << j)) s = fma(Ip[a * mP + c2++], b[j], s);
                    z[i] = s;
                    pos = pos && (s > 0.0);
                    ++a;
                }
            }
            return pos;
        };
        // Lawson-Hanson active set first: a few passive-set solves per voxel instead of up to
        // 2^NM. It accepts only a solve with x_P > 0 whose off-set gradient is <= tol -- the
        // enumeration's KKT test, so both return the unique solution; any stall (an added index
        // that cannot stay, the iteration cap) hands the voxel to the enumeration below.
        {
            int P = 0, banned = 0;
            bool sol = true, stall = false;
            double xl[NM];
#pragma unroll
            for (int i = 0; i < NM; ++i) xl[i] = 0.0;
            for (int it = 0; it < 2 * NM && !found && !stall; ++it) {
                int jb = -1;
                double wb = tol;
#pragma unroll
                for (int j = 0; j < NM; ++j) {
                    double g = b[j];
#pragma unroll
                    for (int i = 0; i < NM; ++i) g = fma(-Gs[j * NM + i], xl[i], g);
                    if (!((P | banned) & (1 << j)) && g > wb) {
                        wb = g;
                        jb = j;
                    }
                }
                if (jb < 0) {
                    if (sol && !banned) {
#pragma unroll
                        for (int i = 0; i < NM; ++i) x[i] = xl[i];
                        found = true;
                    } else {
                        stall = true;
                    }
                    break;
                }
                P |= 1 << jb;
                sol = false;
                for (int inner = 0; inner < NM && P && !stall; ++inner) {
                    double z[NM];
                    if (solve(P, z)) {
#pragma unroll
                        for (int i = 0; i < NM; ++i) xl[i] = z[i];
                        sol = true;
                        break;
                    }
                    if (z[jb] <= 0.0 && inner == 0) {  // the new index cannot enter: give up
                        stall = true;
                        banned |= 1 << jb;
                        break;
                    }
                    double alpha = 1.0;
                    int imin = -1;
#pragma unroll
                    for (int i = 0; i < NM; ++i)
                        if ((P & (1 << i)) && z[i] <= 0.0) {
                            const double ai = xl[i] / (xl[i] - z[i]);
                            if (ai < alpha || imin < 0) {
                                alpha = ai;
                                imin = i;
                            }
                        }
#pragma unroll
                    for (int i = 0; i < NM; ++i) xl[i] = fma(alpha, z[i] - xl[i], xl[i]);
                    xl[imin] = 0.0;  // the blocking index leaves the set
#pragma unroll
                    for (int i = 0; i < NM; ++i)
                        if ((P & (1 << i)) && (i == imin || xl[i] <= 0.0)) {
                            P &= ~(1 << i);
                            xl[i] = 0.0;
                        }
                }
                if (!sol && !P) sol = true;  // back to the empty set: x = 0 is its solve
                if (!sol) stall = true;
            }
        }
        for (int q = 0; q < NS && !found; ++q) {
            const int P = order[q];
            const int mP = __popc(P);
            const double* Ip = inv + offs[P];
            // x_P = inv(G_PP) b_P, packed in the order of P's members
            bool pos = true;
            int a = 0;
#pragma unroll
            for (int i = 0; i < NM; ++i) {
                x[i] = 0.0;
                if (P & (1 << i)) {
                    double s = 0.0;
                    int c2 = 0;
#pragma unroll
                    for (int j = 0; j < NM; ++j)
                        if (P & (1 << j)) s = fma(Ip[a * mP + c2++], b[j], s);
                    x[i] = s;
                    pos = pos && (s > 0.0);
                    ++a;
                }
            }
            if (!pos) continue;
            // KKT: gradient G x - b >= 0 off the passive set; track the best feasible point
            bool kkt = true;
            double f = 0.0;
#pragma unroll
            for (int i = 0; i < NM; ++i) {
                double gi = -b[i];
#pragma unroll
                for (int j = 0; j < NM; ++j) gi = fma(Gs[i * NM + j], x[j], gi);
                if (!(P & (1 << i)) && gi < -tol) kkt = false;
                f += x[i] * (0.5 * (gi + b[i]) - b[i]);
            }
            if (kkt) {
                found = true;
            } else if (f < fbest) {
                fbest = f;
#pragma unroll
                for (int i = 0; i < NM; ++i) best[i] = x[i];
            }
        }
        if (!found) {
            if (fbest < 1e300) {
#pragma unroll
                for (int i = 0; i < NM; ++i) x[i] = best[i];
            } else {
#pragma unroll
                for (int i = 0; i < NM; ++i) x[i] = 0.0;
            }
            bad |= ST_NUMERIC;
        }
#pragma unroll
        for (int i = 0; i < NM; ++i) Xm[(int64_t)i * Nx + n] = (float)x[i];
    }
    if (bad) atomicOr(status, bad);
}

__global__ void __launch_bounds__(FT) k_fmd_spectra(const float* __restrict__ D, int Nk, int K,
                                                    const float* __restrict__ T, int Nm, float* __restrict__ Dm) {
    for (int64_t o = (int64_t)blockIdx.x * FT + threadIdx.x; o < (int64_t)Nm * Nk; o += (int64_t)gridDim.x * FT) {
        const int i = (int)(o / Nk), l = (int)(o - (int64_t)i * Nk);
        double s = 0.0;
        for (int k = 0; k < K; ++k) s = fma((double)T[i * K + k], (double)D[(int64_t)k * Nk + l], s);
        Dm[o] = (float)s;
    }
}

template <int K>
cudaError_t tpart_k(const float* X, int64_t Nx, const int32_t* labels, int Nm, int nblk, int64_t per_blk,
                    double* part, long long* cnt, unsigned* status, cudaStream_t s) {
    constexpr int RMAX = std::max(1, std::min(FMD_MAXM, FMD_RACC / K));
    for (int i0 = 0; i0 < Nm; i0 += RMAX) {
        const int nr = std::min(RMAX, Nm - i0);
        k_fmd_tpart<K, RMAX><<<nblk, FT, 0, s>>>(X, Nx, labels, Nm, i0, nr, per_blk, part, cnt, status);
    }
    return cudaGetLastError();
}

template <int K, int NM>
cudaError_t nnls_km(const float* X, int64_t Nx, const float* T, const double* G, const double* tab, float* Xm,
                    unsigned* status, int num_sms, cudaStream_t s) {
    const int64_t want = (int64_t)num_sms * 8;
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(want, (Nx + FT - 1) / FT));
    k_fmd_nnls<K, NM><<<nb, FT, 0, s>>>(X, Nx, T, G, tab, Xm, status);
    return cudaGetLastError();
}

template <int K>
cudaError_t nnls_k(int Nm, const float* X, int64_t Nx, const float* T, const double* G, const double* tab, float* Xm,
                   unsigned* status, int num_sms, cudaStream_t s) {
    switch (Nm) {
#define M(NMV) \
    case NMV: return NMV <= K ? nnls_km<K, (NMV <= K ? NMV : 1)>(X, Nx, T, G, tab, Xm, status, num_sms, s) : cudaErrorInvalidValue;
        M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8)
#undef M
        default: return cudaErrorInvalidValue;
    }
}

#define HSNCT_K_CASES(M) \
    M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15) M(16)

}  // namespace

int fmd_tblocks(const Geometry& g) {
    const int64_t Nx = (int64_t)g.Nr * g.Nc * g.Nc;
    return (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)g.num_sms * 4, (Nx + FT - 1) / FT));
}

size_t fmd_ws_bytes(const Geometry& g) {
    const size_t nblk = (size_t)fmd_tblocks(g);
    size_t b = nblk * FMD_MAXM * g.K * sizeof(double);                    // partial sums
    b = (b + 255) & ~size_t(255);
    b += ((nblk * FMD_MAXM * sizeof(long long)) + 255) & ~size_t(255);    // counts
    b += (FMD_MAXM * FMD_MAXM * sizeof(double) + 255) & ~size_t(255);     // G
    b += (size_t)FMD_MAXM * (FMD_MAXM + 1) * (1 << (FMD_MAXM - 2)) * sizeof(double);  // packed inverses
    return (b + 255) & ~size_t(255);
}

cudaError_t fmd_transform(const Geometry& g, const float* X, const int32_t* labels, int Nm, float* T, void* ws,
                          unsigned* status, cudaStream_t s) {
    const int64_t Nx = (int64_t)g.Nr * g.Nc * g.Nc;
    const int nblk = fmd_tblocks(g);
    const int64_t per_blk = (Nx + nblk - 1) / nblk;
    char* c = static_cast<char*>(ws);
    double* part = reinterpret_cast<double*>(c);
    c += ((size_t)nblk * FMD_MAXM * g.K * sizeof(double) + 255) & ~size_t(255);
    long long* cnt = reinterpret_cast<long long*>(c);
    cudaError_t e = cudaSuccess;
    switch (g.K) {
#define M(KV) \
    case KV: e = tpart_k<KV>(X, Nx, labels, Nm, nblk, per_blk, part, cnt, status, s); break;
        HSNCT_K_CASES(M)
#undef M
        default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    k_fmd_tfinal<<<1, FT, 0, s>>>(part, cnt, nblk, Nm, g.K, T, status);
    return cudaGetLastError();
}

cudaError_t fmd_materials(const Geometry& g, const float* X, const float* T, int Nm, float* Xm, void* ws,
                          unsigned* status, cudaStream_t s) {
    const int64_t Nx = (int64_t)g.Nr * g.Nc * g.Nc;
    const int nblk = fmd_tblocks(g);
    char* c = static_cast<char*>(ws);
    c += ((size_t)nblk * FMD_MAXM * g.K * sizeof(double) + 255) & ~size_t(255);
    c += ((size_t)nblk * FMD_MAXM * sizeof(long long) + 255) & ~size_t(255);
    double* G = reinterpret_cast<double*>(c);
    c += (FMD_MAXM * FMD_MAXM * sizeof(double) + 255) & ~size_t(255);
    double* tab = reinterpret_cast<double*>(c);
    k_fmd_prep<<<1, FT, 0, s>>>(T, Nm, g.K, G, tab, status);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    switch (g.K) {
#define M(KV) \
    case KV: return nnls_k<KV>(Nm, X, Nx, T, G, tab, Xm, status, g.num_sms, s);
        HSNCT_K_CASES(M)
#undef M
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t fmd_spectra(const Geometry& g, const float* D, const float* T, int Nm, float* Dm, cudaStream_t s) {
    const int64_t tot = (int64_t)Nm * g.Nk;
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)g.num_sms * 4, (tot + FT - 1) / FT));
    k_fmd_spectra<<<nb, FT, 0, s>>>(D, g.Nk, g.K, T, Nm, Dm);
    return cudaGetLastError();
}

}  // namespace hsnct
