// Microbenchmark: FP32 FFMA vs packed fma.rn.f32x2 (sm_100a) throughput per SM, and MUFU.RSQ rate.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ub scripts/ubench_fp32x2.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ffma(float *out, int iters) {
    float a[8], b = 1.0001f, c = 0.9999f;
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

__global__ void k_ffma2(float *out, int iters) {
    unsigned long long a[4];
    float2 bb = make_float2(1.0001f, 1.0001f), cc = make_float2(0.9999f, 0.9999f);
    unsigned long long b = *(unsigned long long *)&bb, c = *(unsigned long long *)&cc;
    for (int i = 0; i < 4; ++i) {
        float2 t = make_float2(threadIdx.x * 0.001f + 2 * i, threadIdx.x * 0.001f + 2 * i + 1);
        a[i] = *(unsigned long long *)&t;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = fma2(a[i], b, c);
    }
    float s = 0;
    for (int i = 0; i < 4; ++i) {
        float2 t = *(float2 *)&a[i];
        s += t.x + t.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// mixed: 4 packed FFMA2 chains + 4 scalar FFMA chains per iteration (12 lane-ops per lane per iteration)
__global__ void k_mixed(float *out, int iters) {
    unsigned long long a[4];
    float f[4], b1 = 1.0001f, c1 = 0.9999f;
    float2 bb = make_float2(1.0001f, 1.0001f), cc = make_float2(0.9999f, 0.9999f);
    unsigned long long b = *(unsigned long long *)&bb, c = *(unsigned long long *)&cc;
    for (int i = 0; i < 4; ++i) {
        float2 t = make_float2(threadIdx.x * 0.001f + 2 * i, threadIdx.x * 0.001f + 2 * i + 1);
        a[i] = *(unsigned long long *)&t;
        f[i] = threadIdx.x * 0.002f + i;
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            a[i] = fma2(a[i], b, c);
            f[i] = fmaf(f[i], b1, c1);
        }
    }
    float s = 0;
    for (int i = 0; i < 4; ++i) {
        float2 t = *(float2 *)&a[i];
        s += t.x + t.y + f[i];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_rsqrt(float *out, int iters) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = 1.0f + threadIdx.x * 0.001f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float y;
            asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i]));
            a[i] = y + 1.0f;
        }
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float *out;
    cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
    const int iters = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        for (int kind = 0; kind < 4; ++kind) {
            cudaEventRecord(a);
            if (kind == 0) k_ffma<<<sms * 8, 256>>>(out, iters);
            if (kind == 1) k_ffma2<<<sms * 8, 256>>>(out, iters);
            if (kind == 2) k_rsqrt<<<sms * 8, 256>>>(out, iters);
            if (kind == 3) k_mixed<<<sms * 8, 256>>>(out, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double lane_ops = (double)sms * 8 * 256 * iters * (kind == 3 ? 12 : 8);  // ffma2 counts 2 per lane
            double per_sm_clk = lane_ops / (ms * 1e-3) / sms / (clk * 1e3);
            printf("%s: %.3f ms, %.1f lane-ops/clk/SM at nominal %d MHz (%.2f Tops/s)\n",
                   kind == 0 ? "FFMA     " : kind == 1 ? "FFMA2x2  " : kind == 2 ? "MUFU.RSQ " : "MIXED    ", ms, per_sm_clk, clk / 1000,
                   lane_ops / (ms * 1e-3) / 1e12);
        }
    }
    return 0;
}
