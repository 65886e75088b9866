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
#include <cstdlib>

#include "internal.h"

namespace hsnct {
namespace {

constexpr int RT = 256;      // ramp-filter threads
// k_ramp_reg: three blocks per SM (80 registers) for P <= 512 (C3 0.062 -> 0.055 ms), two
// for P = 1024, whose 32-point transforms need the registers (three: C4 0.122 -> 0.131 ms)
constexpr int BTX = 16;            // backprojection voxel tile: 16 columns x 16 VPT rows
// detector window per view per tile: the tile's voxels span <= 15|cos| + 31|sin| <= 34.4 bins,
// plus the interpolation neighbour and a one-bin margin on each side of floor()
// (16 x 16 tiles: <= 15(|cos| + |sin|) + 3 <= 24.3 -> 28)
__host__ __device__ constexpr int bp_wmax(int VPT) { return VPT == 2 ? 40 : 28; }
constexpr int BVMAX = 64;          // views per staged chunk (upper bound)
// floats per staged detector sample: KC, plus 4 when KC is a multiple of 8 (an odd number
// of 16-byte chunks per sample spreads a quarter-warp's LDS.128 over all bank groups; the
// other widths are conflict-free as they are for neighbouring samples)
// K = 3 and 5 are padded to 4 and 6 (one LDS.128 / three LDS.64 per sample instead of 3 / 5
// scalar loads; the pad channel is never stored)
__host__ __device__ constexpr int bp_pitch(int KC) {
    return KC % 8 == 0 ? KC + 4 : (KC == 3 || KC == 5 ? KC + 1 : KC);
}

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

// complex a + b and a - b as one packed f32x2 instruction each (FADD2): the butterflies' adds
// are ~60% of the FFT's floating-point instructions
__device__ __forceinline__ float2 cadd2(float2 a, float2 b) {
    float2 r;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ float2 csub2(float2 a, float2 b) {
    float2 r;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
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

// cp.async of VEC floats with zero fill (src_bytes = 0 -> zeros); 4/8/16-byte forms
// ---------------------------------------------------------------------------------------
// Ramp filter for P = 32 B <= 1024 (B in {4, 8, 16, 32}): the same FFT convolution as k_ramp,
// computed as a four-step FFT whose short DFTs run in registers.  With n = 32 j + l and
// k = k1 + B k2:
//   pass 1  thread (pair, l):  B-point DFT over j of x[32 j + l] (j >= B/2 is the zero
//           padding, P >= 2 N_c), times W_P^(l k1)                      -> T[k1][l]
//   pass 2  thread (pair, k1): 32-point DFT over l -> X[k1 + B k2]; times H^[k1 + B k2];
//           32-point inverse DFT over k2; times W_P^(-l k1)              -> T[k1][l]
//   pass 3  thread (pair, l):  B-point inverse DFT over k1 -> q[l + 32 j], kept for < N_c.
// Shared memory only between the passes (rows of 33 complex values: conflict-free).

// cos(k pi / 16) for any integer k (exact table of the first octant)
__host__ __device__ constexpr double cos16(int k) {
    constexpr double C[9] = {1.0,
                             0.98078528040323044913,
                             0.92387953251128675613,
                             0.83146961230254523708,
                             0.70710678118654752440,
                             0.55557023301960222474,
                             0.38268343236508977173,
                             0.19509032201612826785,
                             0.0};
    k = ((k % 32) + 32) % 32;
    return k <= 8 ? C[k] : (k <= 16 ? -C[16 - k] : (k <= 24 ? -C[k - 16] : C[32 - k]));
}
// W_N^k = exp(-2 pi i k / N) (INV: conjugate), N | 32
template <int N, bool INV>
__device__ __forceinline__ float2 wn(int k) {
    const int q = k * (32 / N);  // in units of pi / 16: 2 pi k / N = q pi / 16
    const float c = (float)cos16(q), sn = (float)cos16(q - 8);  // sin x = cos(x - pi/2)
    return make_float2(c, INV ? sn : -sn);
}
__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n / 2); }
__host__ __device__ constexpr int brevc(int i, int bits) {
    int r = 0;
    for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
    return r;
}
// In-register radix-2 DIT DFT of length N (natural order in and out), unnormalised.
template <int N, bool INV>
__device__ __forceinline__ void dft_reg(float2 (&x)[N]) {
    constexpr int L = ilog2c(N);
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const int j = brevc(i, L);
        if (j > i) {
            const float2 t = x[i];
            x[i] = x[j];
            x[j] = t;
        }
    }
#pragma unroll
    for (int m = 1; m < N; m <<= 1) {
#pragma unroll
        for (int i0 = 0; i0 < N; i0 += 2 * m) {
#pragma unroll
            for (int j = 0; j < m; ++j) {
                const int q = j * (N / (2 * m));  // twiddle W_N^q (compile-time)
                const float2 tw = wn<N, INV>(q);
                const float2 a = x[i0 + j], b0 = x[i0 + j + m];
                // W = 1 and W = -i (+i inverse) are exact swaps / negations
                const float2 b = (q == 0)       ? b0
                                 : (4 * q == N) ? (INV ? make_float2(-b0.y, b0.x) : make_float2(b0.y, -b0.x))
                                                : cmul(tw, b0);
                x[i0 + j] = cadd2(a, b);
                x[i0 + j + m] = csub2(a, b);
            }
        }
    }
}
// Forward DFT of length N whose inputs x[N/2..N) are zero (the zero padding of pass 1): the
// first decimation-in-frequency split leaves two N/2-point DFTs, of x and of x W_N^j.
template <int N>
__device__ __forceinline__ void dft_reg_halfzero(float2 (&x)[N]) {
    float2 e[N / 2], o[N / 2];
#pragma unroll
    for (int j = 0; j < N / 2; ++j) {
        e[j] = x[j];
        o[j] = j == 0 ? x[0] : (4 * j == N ? make_float2(x[j].y, -x[j].x) : cmul(wn<N, false>(j), x[j]));
    }
    dft_reg<N / 2, false>(e);
    dft_reg<N / 2, false>(o);
#pragma unroll
    for (int k = 0; k < N / 2; ++k) {
        x[2 * k] = e[k];
        x[2 * k + 1] = o[k];
    }
}
// W_P^m from the [P/2] table (m in [0, P))
__device__ __forceinline__ float2 twp(const float2* __restrict__ tw, int m, int half) {
    const float2 w = __ldg(tw + (m < half ? m : m - half));
    return m < half ? w : make_float2(-w.x, -w.y);
}

template <int B>
__global__ void __launch_bounds__(256, B <= 16 ? 3 : 2) k_ramp_reg(const float* __restrict__ in, int64_t ld_in, int NchAll,
                                                    int Nv, int Nr, int Nc, int s0, int ns,
                                                    const float* __restrict__ Hhat,
                                                    const float2* __restrict__ tw, float* __restrict__ Q,
                                                    int Kc) {
    constexpr int P = 32 * B, RS = 33;  // row stride of T (complex)
    extern __shared__ float2 T[];       // [npair][B][RS]
    const int v = blockIdx.x, rl = blockIdx.y % ns, chunk = blockIdx.y / ns, r = s0 + rl;
    in += (int64_t)chunk * Kc;
    const int Nch = min(Kc, NchAll - chunk * Kc);
    const int npair = (Nch + 1) >> 1;
    const int tid = threadIdx.x;
    const int64_t row0 = ((int64_t)v * Nr + r) * Nc;
    // ---- pass 1
    if (tid < 32 * npair) {
        const int pr = tid >> 5, l = tid & 31, ch = 2 * pr;
        float2 x[B];
#pragma unroll
        for (int j = 0; j < B; ++j) {
            x[j] = make_float2(0.f, 0.f);
            const int c = 32 * j + l;
            if (j < B / 2 && c < Nc) {
                const float* src = in + (row0 + c) * ld_in + ch;
                x[j].x = __ldg(src);
                if (ch + 1 < Nch) x[j].y = __ldg(src + 1);
            }
        }
        dft_reg_halfzero<B>(x);
        float2* t = T + (pr * B) * RS + l;
#pragma unroll
        for (int k1 = 0; k1 < B; ++k1) t[k1 * RS] = k1 == 0 ? x[0] : cmul(twp(tw, l * k1, P / 2), x[k1]);
    }
    __syncthreads();
    // ---- pass 2
    if (tid < B * npair) {
        const int pr = tid / B, k1 = tid - (tid / B) * B;
        float2* t = T + (pr * B + k1) * RS;
        float2 z[32];
#pragma unroll
        for (int l = 0; l < 32; ++l) z[l] = t[l];
        dft_reg<32, false>(z);
#pragma unroll
        for (int k2 = 0; k2 < 32; ++k2) {
            const float h = __ldg(Hhat + k1 + B * k2);
            z[k2].x *= h;
            z[k2].y *= h;
        }
        dft_reg<32, true>(z);
#pragma unroll
        for (int l = 0; l < 32; ++l) {
            const float2 w = twp(tw, l * k1, P / 2);
            t[l] = k1 == 0 ? z[l] : cmul(make_float2(w.x, -w.y), z[l]);
        }
    }
    __syncthreads();
    // ---- pass 3, store q[c], c < Nc: Q[chunk][rl][v][c][Kc]
    if (tid < 32 * npair) {
        const int pr = tid >> 5, l = tid & 31, ch = 2 * pr;
        const float2* t = T + (pr * B) * RS + l;
        float2 x[B];
#pragma unroll
        for (int k1 = 0; k1 < B; ++k1) x[k1] = t[k1 * RS];
        dft_reg<B, true>(x);
        float* dst = Q + ((((int64_t)chunk * ns + rl) * Nv + v) * Nc) * Kc;
#pragma unroll
        for (int j = 0; j < B / 2; ++j) {
            const int c = 32 * j + l;
            if (c < Nc) {
                dst[(int64_t)c * Kc + ch] = x[j].x;
                if (ch + 1 < Kc) dst[(int64_t)c * Kc + ch + 1] = ch + 1 < Nch ? x[j].y : 0.f;
            }
        }
    }
}

template <int VEC>
__device__ __forceinline__ void cp_async_zfill(float* dst, const float* src, bool ok) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    const int n = ok ? 4 * VEC : 0;
    if constexpr (VEC == 4)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
    else if constexpr (VEC == 2)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Voxel-driven backprojection.  Block = a BTX x BTY voxel tile of one slice (and one channel
// chunk), 256 threads, two voxels per thread (rows ty and ty + 16).  Views are processed in
// chunks of vch: per view the tile's detector window (BWMAX samples from clo, KC channels
// each, stored exactly as in Q so a window is one contiguous run of floats) is staged by
// cp.async into one of two buffers while the other chunk is being used.  Per voxel and view:
// u = x cos + y sin + (N_c - 1)/2, l = floor(u), w = u - l, acc += (1 - w) q[l] + w q[l + 1].
template <int KC, int VPT>
__global__ void __launch_bounds__(BTX * 16, KC <= 8 ? 4 : 2) k_backproject(
    const float* __restrict__ Q, int NchAll, int Nv, int Nc, int s0, int ns, const float* __restrict__ cos_t,
    const float* __restrict__ sin_t, int mode, float* __restrict__ out, int64_t ld_out, int64_t col0,
    int64_t Nx, int vch) {
    constexpr int NT = BTX * 16;
    constexpr int BTY = 16 * VPT;      // tile rows; VPT voxels per thread (rows ty, ty + 16)
    constexpr int BWMAX = bp_wmax(VPT);
    constexpr int VEC = KC % 4 == 0 ? 4 : (KC % 2 == 0 ? 2 : 1);  // floats per copy (global alignment)
    constexpr int SP = bp_pitch(KC);                               // floats per staged sample
    constexpr int LV = SP % 4 == 0 ? 4 : (SP % 2 == 0 ? 2 : 1);    // floats per shared-memory load
    constexpr int WQ = BWMAX * KC;                                 // floats per view window in Q
    constexpr int WIN = BWMAX * SP;                                // ... and in shared memory
    extern __shared__ __align__(16) float Ws[];                    // [2][vch][WIN]
    __shared__ float2 csn[2][BVMAX];
    __shared__ int clo[2][BVMAX];
    const int tid = threadIdx.x;
    const int tx = tid % BTX, ty = tid / BTX;
    const int j = blockIdx.x * BTX + tx, i0 = blockIdx.y * BTY + ty;
    // blockIdx.z = chunk * ns + slice (channel chunk of KC, slice of the window)
    const int rl = blockIdx.z % ns, chunk = blockIdx.z / ns, r = s0 + rl;
    const int Nch = min(KC, NchAll - chunk * KC);
    col0 += (int64_t)chunk * KC;
    const float half = 0.5f * (float)(Nc - 1);
    const float x = (float)j - half, y0 = (float)i0 - half, y1 = y0 + (float)(BTY / 2);
    const float xa = (float)(blockIdx.x * BTX) - half, ya = (float)(blockIdx.y * BTY) - half;
    const float xb = xa + (BTX - 1), yb = ya + (BTY - 1);
    const float* Qr = Q + ((int64_t)chunk * ns + rl) * Nv * Nc * KC;
    const int nchk = (Nv + vch - 1) / vch;

    // view metadata of chunk ck into buffer b: (cos, sin) and the window start
    auto meta = [&](int ck, int b) {
        const int v = ck * vch + tid;
        if (tid < vch && v < Nv) {
            const float cs = cos_t[v], sn = sin_t[v];
            const float u1 = fmaf(xa, cs, fmaf(ya, sn, half));
            const float u2 = fmaf(xb, cs, fmaf(ya, sn, half));
            const float u3 = fmaf(xa, cs, fmaf(yb, sn, half));
            const float u4 = fmaf(xb, cs, fmaf(yb, sn, half));
            clo[b][tid] = (int)floorf(fminf(fminf(u1, u2), fminf(u3, u4))) - 1;
            csn[b][tid] = make_float2(cs, sn);
        }
    };
    // windows of chunk ck into buffer b (zero outside the detector), one cp.async group
    auto stage = [&](int ck, int b) {
        const int v0 = ck * vch, nv = min(vch, Nv - v0);
        float* dst = Ws + (size_t)b * vch * WIN;
        for (int t = tid; t < nv * (WQ / VEC); t += NT) {
            const int vv = t / (WQ / VEC), e = (t - vv * (WQ / VEC)) * VEC;
            const int w = e / KC, c = clo[b][vv] + w;
            const bool ok = c >= 0 && c < Nc;
            const float* src = ok ? Qr + ((int64_t)(v0 + vv) * Nc + clo[b][vv]) * KC + e : Qr;
            cp_async_zfill<VEC>(dst + vv * WIN + w * SP + (e - w * KC), src, ok);
        }
        cp_async_commit();
    };

    float2 acc0[(KC + 1) / 2], acc1[(KC + 1) / 2];
#pragma unroll
    for (int c = 0; c < (KC + 1) / 2; ++c) acc0[c] = acc1[c] = make_float2(0.f, 0.f);
    // (1 - w) q[l] + w q[l + 1] into acc, KC channels from the window at p
    auto interp = [&](float2* acc, const float* p, float wt) {
        const float w1 = 1.f - wt;
        float a[SP + 1], bq[SP + 1];
#pragma unroll
        for (int c = 0; c < KC; c += LV) {
            if constexpr (LV == 4) {
                const float4 qa = *reinterpret_cast<const float4*>(p + c);
                const float4 qb = *reinterpret_cast<const float4*>(p + SP + c);
                a[c] = qa.x; a[c + 1] = qa.y; a[c + 2] = qa.z; a[c + 3] = qa.w;
                bq[c] = qb.x; bq[c + 1] = qb.y; bq[c + 2] = qb.z; bq[c + 3] = qb.w;
            } else if constexpr (LV == 2) {
                const float2 qa = *reinterpret_cast<const float2*>(p + c);
                const float2 qb = *reinterpret_cast<const float2*>(p + SP + c);
                a[c] = qa.x; a[c + 1] = qa.y;
                bq[c] = qb.x; bq[c + 1] = qb.y;
            } else {
                a[c] = p[c];
                bq[c] = p[SP + c];
            }
        }
        a[KC] = bq[KC] = 0.f;
#pragma unroll
        for (int c = 0; c < (KC + 1) / 2; ++c)
            acc[c] = ffma2s(wt, make_float2(bq[2 * c], bq[2 * c + 1]),
                            ffma2s(w1, make_float2(a[2 * c], a[2 * c + 1]), acc[c]));
    };

    meta(0, 0);
    __syncthreads();
    stage(0, 0);
    for (int ck = 0; ck < nchk; ++ck) {
        const int b = ck & 1;
        if (ck + 1 < nchk) {  // prefetch the next chunk into the other buffer
            meta(ck + 1, b ^ 1);
            __syncthreads();
            stage(ck + 1, b ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int nv = min(vch, Nv - ck * vch);
        const float* win = Ws + (size_t)b * vch * WIN;
        for (int vv = 0; vv < nv; ++vv) {
            const float2 t = csn[b][vv];
            const int cl = clo[b][vv];
            const float u0 = fmaf(x, t.x, fmaf(y0, t.y, half));
            const float u1 = fmaf(x, t.x, fmaf(y1, t.y, half));
            const float f0 = floorf(u0), f1 = floorf(u1);
            interp(acc0, win + vv * WIN + ((int)f0 - cl) * SP, u0 - f0);
            if constexpr (VPT == 2) interp(acc1, win + vv * WIN + ((int)f1 - cl) * SP, u1 - f1);
        }
        __syncthreads();  // buffer b is refilled by the next iteration's prefetch
    }
    if (j >= Nc) return;
    const float scale = 3.14159265358979323846f / (float)Nv;
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
        const int i = i0 + q * 16;
        if (i >= Nc) break;
        const float2* acc = q ? acc1 : acc0;
        if (mode == 0) {
            const int64_t n = (int64_t)r * Nc * Nc + (int64_t)i * Nc + j;
#pragma unroll
            for (int c = 0; c < KC; ++c)
                if (c < Nch) out[(int64_t)c * Nx + n] = ((c & 1) ? acc[c >> 1].y : acc[c >> 1].x) * scale;
        } else {
            const int64_t vox = ((int64_t)rl * Nc + i) * Nc + j;
            float* o = out + vox * ld_out + col0;
#pragma unroll
            for (int c = 0; c < KC; ++c)
                if (c < Nch) o[c] = ((c & 1) ? acc[c >> 1].y : acc[c >> 1].x) * scale;
        }
    }
}

}  // namespace

template <int B>
static cudaError_t ramp_reg(const Geometry& g, const DeviceTables& t, const float* in, int64_t ld_in, int Nch,
                            int s0, int ns, float* Q, int Kc, cudaStream_t s) {
    const int npair = (std::min(Nch, Kc) + 1) / 2;
    const size_t smem = (size_t)npair * B * 33 * sizeof(float2);
    static SmemAttr attr;
    cudaError_t e = ensure_smem((const void*)k_ramp_reg<B>, (int)smem, attr);
    if (e != cudaSuccess) return e;
    const int nchunk = (Nch + Kc - 1) / Kc;
    dim3 grid(g.Nv, ns * nchunk);
    k_ramp_reg<B><<<grid, 32 * npair, smem, s>>>(in, ld_in, Nch, g.Nv, g.Nr, g.Nc, s0, ns, t.Hhat, t.twiddle, Q,
                                                Kc);
    return cudaGetLastError();
}

cudaError_t ramp_filter(const Geometry& g, const DeviceTables& t, const float* in, int64_t ld_in,
                        int Nch, int s0, int ns, float* Q, int Kc, cudaStream_t s) {
    if (ns <= 0) return cudaSuccess;
    if (Kc <= 16 && getenv("HSNCT_RAMP_SMEM") == nullptr) {  // register four-step FFT for P <= 1024
        switch (g.P) {
            case 128: return ramp_reg<4>(g, t, in, ld_in, Nch, s0, ns, Q, Kc, s);
            case 256: return ramp_reg<8>(g, t, in, ld_in, Nch, s0, ns, Q, Kc, s);
            case 512: return ramp_reg<16>(g, t, in, ld_in, Nch, s0, ns, Q, Kc, s);
            case 1024: return ramp_reg<32>(g, t, in, ld_in, Nch, s0, ns, Q, Kc, s);
            default: break;
        }
    }
    const int npair = (std::min(Nch, Kc) + 1) / 2;
    const size_t smem = (size_t)npair * g.P * sizeof(float2);
    static SmemAttr attr;
    cudaError_t e = ensure_smem((const void*)k_ramp, (int)smem, attr);
    if (e != cudaSuccess) return e;
    const int nchunk = (Nch + Kc - 1) / Kc;
    dim3 grid(g.Nv, ns * nchunk);
    k_ramp<<<grid, RT, smem, s>>>(in, ld_in, Nch, g.Nv, g.Nr, g.Nc, g.P, g.logP, s0, ns, t.Hhat, t.twiddle,
                                  Q, Kc);
    return cudaGetLastError();
}

template <int KC, int VPT>
static cudaError_t bp_kv(const Geometry& g, const DeviceTables& t, const float* Q, int Nch, int s0, int ns, int mode,
                         float* out, int64_t ld_out, int64_t col0, cudaStream_t s) {
    // views per chunk: two buffers of about 20 KB (KC <= 8: four blocks per SM) or 40 KB
    // (KC = 16: two blocks per SM, 128 registers) each
    const int per_view = bp_wmax(VPT) * bp_pitch(KC) * (int)sizeof(float);
    const int vch = std::max(1, std::min(std::min(g.Nv, BVMAX), ((KC <= 8 ? 20 : 40) * 1024) / per_view));
    const size_t smem = (size_t)2 * vch * per_view;
    static SmemAttr attr;
    cudaError_t e = ensure_smem((const void*)k_backproject<KC, VPT>, (int)smem, attr);
    if (e != cudaSuccess) return e;
    const int nchunk = (Nch + KC - 1) / KC;
    dim3 grid((g.Nc + BTX - 1) / BTX, (g.Nc + 16 * VPT - 1) / (16 * VPT), ns * nchunk);
    k_backproject<KC, VPT><<<grid, BTX * 16, smem, s>>>(Q, Nch, g.Nv, g.Nc, s0, ns, t.cos_t, t.sin_t, mode, out,
                                                        ld_out, col0, (int64_t)g.Nr * g.Nc * g.Nc, vch);
    return cudaGetLastError();
}

// Two voxels per thread (16 x 32 tiles) unless that leaves fewer than two blocks per SM
// (C1, C2: one slice), then 16 x 16 tiles with one voxel per thread.
template <int KC>
static cudaError_t bp_k(const Geometry& g, const DeviceTables& t, const float* Q, int Nch, int s0, int ns, int mode,
                        float* out, int64_t ld_out, int64_t col0, cudaStream_t s) {
    const int64_t blocks2 = (int64_t)((g.Nc + BTX - 1) / BTX) * ((g.Nc + 31) / 32) * ns * ((Nch + KC - 1) / KC);
    if (blocks2 < 2 * (int64_t)g.num_sms) return bp_kv<KC, 1>(g, t, Q, Nch, s0, ns, mode, out, ld_out, col0, s);
    return bp_kv<KC, 2>(g, t, Q, Nch, s0, ns, mode, out, ld_out, col0, s);
}

cudaError_t backproject(const Geometry& g, const DeviceTables& t, const float* Q, int Kc, int Nch,
                        int s0, int ns, int mode, float* out, int64_t ld_out, int64_t col0,
                        cudaStream_t s) {
    if (ns <= 0) return cudaSuccess;
    switch (Kc) {
        case 1: return bp_k<1>(g, t, Q, Nch, s0, ns, mode, out, ld_out, col0, s);
        case 2: return bp_k<2>(g, t, Q, Nch, s0, ns, mode, out, ld_out, col0, s);
        case 3: return bp_k<3>(g, t, Q, Nch, s0, ns, mode, out, ld_out, col0, s);
        case 4: return bp_k<4>(g, t, Q, Nch, s0, ns, mode, out, ld_out, col0, s);
        case 5: return bp_k<5>(g, t, Q, Nch, s0, ns, mode, out, ld_out, col0, s);
        case 6: return bp_k<6>(g, t, Q, Nch, s0, ns, mode, out, ld_out, col0, s);
        case 7: return bp_k<7>(g, t, Q, Nch, s0, ns, mode, out, ld_out, col0, s);
        case 8: return bp_k<8>(g, t, Q, Nch, s0, ns, mode, out, ld_out, col0, s);
        case 16: return bp_k<16>(g, t, Q, Nch, s0, ns, mode, out, ld_out, col0, s);
        default: return cudaErrorInvalidValue;
    }
}

int ramp_launches() { return 1; }
int backproject_launches() { return 1; }

}  // namespace hsnct
