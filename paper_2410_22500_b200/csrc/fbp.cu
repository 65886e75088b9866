// FBP of parallel-beam sinograms (R10-R16):
//
//   k_ramp         Kak-Slaney ramp filter (tau = 1) as an FFT convolution:
//                  zero-pad each detector row to P = next_pow2(2 N_c), radix-2 FFT in
//                  shared memory, multiply by the real, even spectrum H^ of the
//                  circularly arranged kernel, inverse FFT, keep c < N_c.  P >= 2 N_c - 1,
//                  so the circular convolution equals the linear one exactly.  Two
//                  real channels ride in one complex transform (H^ is real and even).
//   k_backproject  voxel-driven linear-interpolation backprojection, scale pi/N_v.
//                  A 16x16 voxel tile stages, per view, only the detector window its
//                  voxels project into (<= 16 (|cos|+|sin|) + 4 bins) with zero fill
//                  outside [0, N_c-1]; channels are innermost (float4 LDS).
//
// The same two kernels serve FHR (channels = the K subspace sinograms, output
// X[k][r][i][j]) and the DHR baseline (channels = a chunk of wavelength bins,
// output Xh[voxel][bin]).
#include <algorithm>

#include "internal.h"

namespace hsnct {
namespace {

constexpr int RT = 256;      // ramp-filter threads
constexpr int TILE = 16;     // backprojection voxel tile edge
constexpr int WMAX = 28;     // detector window per view per tile (>= 16*sqrt(2) + 4)

__device__ __forceinline__ unsigned bitrev(unsigned x, int logP) { return __brev(x) >> (32 - logP); }

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// One (v, r) detector row-set per block: Nch channels -> npair complex rows of length P.
__global__ void __launch_bounds__(RT) k_ramp(const float* __restrict__ in, int64_t ld_in, int Nch,
                                             int Nv, int Nr, int Nc, int P, int logP, int s0,
                                             const float* __restrict__ Hhat,
                                             const float2* __restrict__ tw,
                                             float* __restrict__ Q, int Kc) {
    extern __shared__ float2 z[];  // [npair][P]
    const int v = blockIdx.x, rl = blockIdx.y, r = s0 + rl;
    const int npair = (Nch + 1) >> 1;
    const int tid = threadIdx.x;
    const int64_t row0 = ((int64_t)v * Nr + r) * Nc;
    // load, zero-padded, into bit-reversed positions (DIT input order)
    for (int i = tid; i < npair * P; i += RT) {
        const int pr = i / P, c = i - pr * P;
        float2 val = make_float2(0.f, 0.f);
        if (c < Nc) {
            const float* src = in + (row0 + c) * ld_in;
            const int ch = 2 * pr;
            val.x = src[ch];
            if (ch + 1 < Nch) val.y = src[ch + 1];
        }
        z[pr * P + bitrev(c, logP)] = val;
    }
    __syncthreads();
    const int half = P >> 1;
    // forward DIT FFT (natural order out)
    for (int m = 1; m < P; m <<= 1) {
        const int tstride = half / m;
        for (int i = tid; i < npair * half; i += RT) {
            const int pr = i / half, b = i - pr * half;
            const int j = b & (m - 1);
            const int i0 = ((b - j) << 1) + j, i1 = i0 + m;
            float2* zp = z + pr * P;
            const float2 t = cmul(tw[j * tstride], zp[i1]);
            const float2 a = zp[i0];
            zp[i0] = make_float2(a.x + t.x, a.y + t.y);
            zp[i1] = make_float2(a.x - t.x, a.y - t.y);
        }
        __syncthreads();
    }
    // multiply by the (real, even, 1/P-scaled) filter spectrum
    for (int i = tid; i < npair * P; i += RT) {
        const int f = i % P;
        const float hf = Hhat[f];
        z[i].x *= hf;
        z[i].y *= hf;
    }
    __syncthreads();
    // inverse DIF FFT with conjugate twiddles (bit-reversed order out)
    for (int m = half; m >= 1; m >>= 1) {
        const int tstride = half / m;
        for (int i = tid; i < npair * half; i += RT) {
            const int pr = i / half, b = i - pr * half;
            const int j = b & (m - 1);
            const int i0 = ((b - j) << 1) + j, i1 = i0 + m;
            float2* zp = z + pr * P;
            const float2 a = zp[i0], c = zp[i1];
            float2 w = tw[j * tstride];
            w.y = -w.y;
            zp[i0] = make_float2(a.x + c.x, a.y + c.y);
            zp[i1] = cmul(make_float2(a.x - c.x, a.y - c.y), w);
        }
        __syncthreads();
    }
    // store q[c], c < Nc: Q[rl][v][c][Kc]
    float* dst = Q + (((int64_t)rl * Nv + v) * Nc) * Kc;
    for (int i = tid; i < Nc * Kc; i += RT) {
        const int c = i / Kc, ch = i - c * Kc;
        float val = 0.f;
        if (ch < Nch) {
            const float2 zz = z[(ch >> 1) * P + bitrev(c, logP)];
            val = (ch & 1) ? zz.y : zz.x;
        }
        dst[i] = val;
    }
}

template <int KC>
__global__ void __launch_bounds__(TILE * TILE) k_backproject(
    const float* __restrict__ Q, int Nch, int Nv, int Nc, int s0, const float* __restrict__ cos_t,
    const float* __restrict__ sin_t, int mode, float* __restrict__ out, int64_t ld_out, int64_t col0,
    int64_t Nx, int vchunk) {
    extern __shared__ __align__(16) float Qs[];  // [vchunk][WMAX][KC]
    __shared__ int clo[64];
    const int tx = threadIdx.x % TILE, ty = threadIdx.x / TILE;
    const int j = blockIdx.x * TILE + tx, i = blockIdx.y * TILE + ty;
    const int rl = blockIdx.z, r = s0 + rl;
    const float half = 0.5f * (float)(Nc - 1);
    const float x = (float)j - half, y = (float)i - half;
    const float xa = (float)(blockIdx.x * TILE) - half, ya = (float)(blockIdx.y * TILE) - half;
    const float xb = xa + (TILE - 1), yb = ya + (TILE - 1);
    float acc[KC];
#pragma unroll
    for (int c = 0; c < KC; ++c) acc[c] = 0.f;
    const float* Qr = Q + (int64_t)rl * Nv * Nc * KC;
    for (int v0 = 0; v0 < Nv; v0 += vchunk) {
        const int nv = min(vchunk, Nv - v0);
        __syncthreads();
        if ((int)threadIdx.x < nv) {
            const int v = v0 + threadIdx.x;
            const float cs = cos_t[v], sn = sin_t[v];
            const float u1 = fmaf(xa, cs, fmaf(ya, sn, half));
            const float u2 = fmaf(xb, cs, fmaf(ya, sn, half));
            const float u3 = fmaf(xa, cs, fmaf(yb, sn, half));
            const float u4 = fmaf(xb, cs, fmaf(yb, sn, half));
            const float umin = fminf(fminf(u1, u2), fminf(u3, u4));
            clo[threadIdx.x] = (int)floorf(umin) - 1;
        }
        __syncthreads();
        // cooperative load of the per-view windows (zero outside the detector)
        for (int t = threadIdx.x; t < nv * WMAX * (KC / 4); t += TILE * TILE) {
            const int vv = t / (WMAX * (KC / 4));
            const int rem = t - vv * (WMAX * (KC / 4));
            const int w = rem / (KC / 4), c4 = rem - w * (KC / 4);
            const int c = clo[vv] + w;
            float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
            if (c >= 0 && c < Nc)
                val = __ldg(reinterpret_cast<const float4*>(Qr + ((int64_t)(v0 + vv) * Nc + c) * KC) + c4);
            reinterpret_cast<float4*>(Qs + (vv * WMAX + w) * KC)[c4] = val;
        }
        __syncthreads();
        for (int vv = 0; vv < nv; ++vv) {
            const int v = v0 + vv;
            const float u = fmaf(x, cos_t[v], fmaf(y, sin_t[v], half));
            const float fl = floorf(u);
            const float wt = u - fl;
            const int li = (int)fl - clo[vv];
            const float4* q0 = reinterpret_cast<const float4*>(Qs + (vv * WMAX + li) * KC);
            const float4* q1 = q0 + KC / 4;
#pragma unroll
            for (int c4 = 0; c4 < KC / 4; ++c4) {
                const float4 a = q0[c4], b = q1[c4];
                acc[4 * c4 + 0] += fmaf(wt, b.x - a.x, a.x);
                acc[4 * c4 + 1] += fmaf(wt, b.y - a.y, a.y);
                acc[4 * c4 + 2] += fmaf(wt, b.z - a.z, a.z);
                acc[4 * c4 + 3] += fmaf(wt, b.w - a.w, a.w);
            }
        }
    }
    if (i >= Nc || j >= Nc) return;
    const float scale = 3.14159265358979323846f / (float)Nv;
    const int64_t vox = ((int64_t)rl * Nc + i) * Nc + j;
    if (mode == 0) {
        const int64_t n = (int64_t)r * Nc * Nc + (int64_t)i * Nc + j;
#pragma unroll
        for (int c = 0; c < KC; ++c)
            if (c < Nch) out[(int64_t)c * Nx + n] = acc[c] * scale;
    } else {
        float* o = out + vox * ld_out + col0;
#pragma unroll
        for (int c = 0; c < KC; ++c)
            if (c < Nch) o[c] = acc[c] * scale;
    }
}

}  // namespace

cudaError_t ramp_filter(const Geometry& g, const DeviceTables& t, const float* in, int64_t ld_in,
                        int Nch, int s0, int ns, float* Q, int Kc, cudaStream_t s) {
    if (ns <= 0) return cudaSuccess;
    const int npair = (Nch + 1) / 2;
    const size_t smem = (size_t)npair * g.P * sizeof(float2);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_ramp, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    dim3 grid(g.Nv, ns);
    k_ramp<<<grid, RT, smem, s>>>(in, ld_in, Nch, g.Nv, g.Nr, g.Nc, g.P, g.logP, s0, t.Hhat, t.twiddle,
                                  Q, Kc);
    return cudaGetLastError();
}

template <int KC>
static cudaError_t bp_k(const Geometry& g, const DeviceTables& t, const float* Q, int Nch, int s0,
                        int ns, int mode, float* out, int64_t ld_out, int64_t col0, cudaStream_t s) {
    const int per_view = WMAX * KC * (int)sizeof(float);
    int vchunk = std::min(std::min(g.Nv, 64), std::max(1, (96 * 1024) / per_view));
    const size_t smem = (size_t)vchunk * per_view;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_backproject<KC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    dim3 grid((g.Nc + TILE - 1) / TILE, (g.Nc + TILE - 1) / TILE, ns);
    k_backproject<KC><<<grid, TILE * TILE, smem, s>>>(Q, Nch, g.Nv, g.Nc, s0, t.cos_t, t.sin_t, mode,
                                                     out, ld_out, col0,
                                                     (int64_t)g.Nr * g.Nc * g.Nc, vchunk);
    return cudaGetLastError();
}

cudaError_t backproject(const Geometry& g, const DeviceTables& t, const float* Q, int Kc, int Nch,
                        int s0, int ns, int mode, float* out, int64_t ld_out, int64_t col0,
                        cudaStream_t s) {
    if (ns <= 0) return cudaSuccess;
    switch (Kc) {
        case 4: return bp_k<4>(g, t, Q, Nch, s0, ns, mode, out, ld_out, col0, s);
        case 8: return bp_k<8>(g, t, Q, Nch, s0, ns, mode, out, ld_out, col0, s);
        case 12: return bp_k<12>(g, t, Q, Nch, s0, ns, mode, out, ld_out, col0, s);
        case 16: return bp_k<16>(g, t, Q, Nch, s0, ns, mode, out, ld_out, col0, s);
        default: return cudaErrorInvalidValue;
    }
}

int ramp_launches() { return 1; }
int backproject_launches() { return 1; }

}  // namespace hsnct
