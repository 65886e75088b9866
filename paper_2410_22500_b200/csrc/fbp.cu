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
// floats per staged detector sample: KC, plus 4 when KC/4 is even (an odd number of
// 16-byte chunks per sample spreads consecutive samples over all bank groups)
__host__ __device__ constexpr int bp_pitch(int KC) { return KC + (((KC / 4) % 2 == 0) ? 4 : 0); }

__device__ __forceinline__ unsigned bitrev(unsigned x, int logP) { return __brev(x) >> (32 - logP); }

// (x, x) * b + c on both halves: one packed FFMA2 with a broadcast scalar
__device__ __forceinline__ float2 ffma2s(float x, float2 b, float2 c) {
    float2 r;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %2};\n\t"
        "mov.b64 rb, {%3, %4};\n\t"
        "mov.b64 rc, {%5, %6};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
        "mov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(x), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// One (v, r) detector row-set per block: Nch channels -> npair complex rows of length P.
__global__ void __launch_bounds__(RT) k_ramp(const float* __restrict__ in, int64_t ld_in, int NchAll,
                                             int Nv, int Nr, int Nc, int P, int logP, int s0, int ns,
                                             const float* __restrict__ Hhat,
                                             const float2* __restrict__ tw,
                                             float* __restrict__ Q, int Kc) {
    extern __shared__ float2 z[];  // [npair][P]
    // blockIdx.y = chunk * ns + slice: channel chunk of Kc channels, slice of the window
    const int v = blockIdx.x, rl = blockIdx.y % ns, chunk = blockIdx.y / ns, r = s0 + rl;
    in += (int64_t)chunk * Kc;
    const int Nch = min(Kc, NchAll - chunk * Kc);
    const int npair = (Nch + 1) >> 1;
    const int tid = threadIdx.x;
    const int64_t row0 = ((int64_t)v * Nr + r) * Nc;
    // load, zero-padded, into bit-reversed positions (DIT input order)
    // channel pairs fastest: consecutive threads read consecutive channels of one detector bin
    for (int i = tid; i < npair * P; i += RT) {
        const int c = i / npair, pr = i - c * npair;
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
    float* dst = Q + ((((int64_t)chunk * ns + rl) * Nv + v) * Nc) * Kc;
    for (int i = tid; i < Nc * Kc; i += RT) {  // channels fastest: coalesced stores
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
    const float* __restrict__ Q, int NchAll, int Nv, int Nc, int s0, int ns, const float* __restrict__ cos_t,
    const float* __restrict__ sin_t, int mode, float* __restrict__ out, int64_t ld_out, int64_t col0,
    int64_t Nx, int vchunk) {
    // [vchunk][WMAX][SP]: one detector sample's KC channels, padded so that the samples
    // read by a quarter-warp's LDS.128 fall in distinct 16-byte bank groups
    constexpr int SP = bp_pitch(KC);
    extern __shared__ __align__(16) float Qs[];
    __shared__ int clo[64];
    const int tx = threadIdx.x % TILE, ty = threadIdx.x / TILE;
    const int j = blockIdx.x * TILE + tx, i = blockIdx.y * TILE + ty;
    // blockIdx.z = chunk * ns + slice (channel chunk of KC, slice of the window)
    const int rl = blockIdx.z % ns, chunk = blockIdx.z / ns, r = s0 + rl;
    const int Nch = min(KC, NchAll - chunk * KC);
    col0 += (int64_t)chunk * KC;
    const float half = 0.5f * (float)(Nc - 1);
    const float x = (float)j - half, y = (float)i - half;
    const float xa = (float)(blockIdx.x * TILE) - half, ya = (float)(blockIdx.y * TILE) - half;
    const float xb = xa + (TILE - 1), yb = ya + (TILE - 1);
    float2 acc[KC / 2];  // channel pairs; (1 - w) a + w b as two packed FMAs per pair
#pragma unroll
    for (int c = 0; c < KC / 2; ++c) acc[c] = make_float2(0.f, 0.f);
    const float* Qr = Q + ((int64_t)chunk * ns + rl) * Nv * Nc * KC;
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
            reinterpret_cast<float4*>(Qs + (vv * WMAX + w) * SP)[c4] = val;
        }
        __syncthreads();
        for (int vv = 0; vv < nv; ++vv) {
            const int v = v0 + vv;
            const float u = fmaf(x, cos_t[v], fmaf(y, sin_t[v], half));
            const float fl = floorf(u);
            const float wt = u - fl, w1 = 1.f - wt;
            const int li = (int)fl - clo[vv];
            const float4* q0 = reinterpret_cast<const float4*>(Qs + (vv * WMAX + li) * SP);
            const float4* q1 = q0 + SP / 4;
#pragma unroll
            for (int c4 = 0; c4 < KC / 4; ++c4) {
                const float4 a = q0[c4], b = q1[c4];
                acc[2 * c4 + 0] = ffma2s(wt, make_float2(b.x, b.y), ffma2s(w1, make_float2(a.x, a.y), acc[2 * c4 + 0]));
                acc[2 * c4 + 1] = ffma2s(wt, make_float2(b.z, b.w), ffma2s(w1, make_float2(a.z, a.w), acc[2 * c4 + 1]));
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
            if (c < Nch) out[(int64_t)c * Nx + n] = ((c & 1) ? acc[c >> 1].y : acc[c >> 1].x) * scale;
    } else {
        float* o = out + vox * ld_out + col0;
#pragma unroll
        for (int c = 0; c < KC; ++c)
            if (c < Nch) o[c] = ((c & 1) ? acc[c >> 1].y : acc[c >> 1].x) * scale;
    }
}

}  // namespace

cudaError_t ramp_filter(const Geometry& g, const DeviceTables& t, const float* in, int64_t ld_in,
                        int Nch, int s0, int ns, float* Q, int Kc, cudaStream_t s) {
    if (ns <= 0) return cudaSuccess;
    const int npair = (std::min(Nch, Kc) + 1) / 2;
    const size_t smem = (size_t)npair * g.P * sizeof(float2);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_ramp, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    const int nchunk = (Nch + Kc - 1) / Kc;
    dim3 grid(g.Nv, ns * nchunk);
    k_ramp<<<grid, RT, smem, s>>>(in, ld_in, Nch, g.Nv, g.Nr, g.Nc, g.P, g.logP, s0, ns, t.Hhat, t.twiddle,
                                  Q, Kc);
    return cudaGetLastError();
}

template <int KC>
static cudaError_t bp_k(const Geometry& g, const DeviceTables& t, const float* Q, int Nch, int s0,
                        int ns, int mode, float* out, int64_t ld_out, int64_t col0, cudaStream_t s) {
    const int per_view = WMAX * bp_pitch(KC) * (int)sizeof(float);
    int vchunk = std::min(std::min(g.Nv, 64), std::max(1, (96 * 1024) / per_view));
    const size_t smem = (size_t)vchunk * per_view;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_backproject<KC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    const int nchunk = (Nch + KC - 1) / KC;
    dim3 grid((g.Nc + TILE - 1) / TILE, (g.Nc + TILE - 1) / TILE, ns * nchunk);
    k_backproject<KC><<<grid, TILE * TILE, smem, s>>>(Q, Nch, g.Nv, g.Nc, s0, ns, t.cos_t, t.sin_t, mode,
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
