// Throughput of legacy mma.sync (HMMA) and packed FFMA2 on this GPU: each warp runs
// independent chains; reports TFLOP/s over the whole grid.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

template <int NACC>
__global__ void k_hmma(float* out, int iters) {
    unsigned a0 = 0x3c003c00u ^ threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 0x3c003c00u, b1 = b0 + 7;
    float c[NACC][4];
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void k_hmma_tf32(float* out, int iters) {
    unsigned a0 = 0x3f800000u ^ threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 0x3f800000u, b1 = b0 + 7;
    float c[NACC][4];
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, int iters) {
    float2 c[8];
    float2 a = make_float2(1.0001f + threadIdx.x * 1e-7f, 0.9999f), b = make_float2(1e-7f, 2e-7f);
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = make_float2(i, i + 1);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            asm volatile("{.reg .b64 ra, rb, rc; mov.b64 ra, {%2,%3}; mov.b64 rb, {%4,%5}; mov.b64 rc, {%0,%1}; fma.rn.f32x2 rc, ra, rb, rc; mov.b64 {%0,%1}, rc;}"
                         : "+f"(c[i].x), "+f"(c[i].y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i].x + c[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma(float* out, int iters) {
    float c[8];
    float a = 1.0001f + threadIdx.x * 1e-7f, b = 1e-7f;
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(c[i]) : "f"(a), "f"(b));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, 1 << 24);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int warps : {4, 8, 16}) {
        dim3 grid(sms), block(32 * warps);
        auto run = [&](const char* name, void (*k)(float*, int), double flop_per_iter_warp) {
            k<<<grid, block>>>(out, 100);
            cudaEventRecord(e0);
            k<<<grid, block>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double fl = flop_per_iter_warp * iters * warps * sms;
            printf("%-22s warps/SM=%2d  %8.1f TFLOP/s  (%.3f ms)\n", name, warps, fl / ms * 1e-9, ms);
        };
        run("hmma f16 m16n8k16 x4", k_hmma<4>, 4.0 * 2 * 16 * 8 * 16);
        run("hmma f16 m16n8k16 x8", k_hmma<8>, 8.0 * 2 * 16 * 8 * 16);
        run("hmma tf32 m16n8k8 x8", k_hmma_tf32<8>, 8.0 * 2 * 16 * 8 * 8);
        run("ffma2 (f32x2) x8", k_ffma2, 8.0 * 2 * 2 * 32);
        run("ffma x8", k_ffma, 8.0 * 2 * 32);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
