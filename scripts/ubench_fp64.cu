// Microbenchmark: FP64 DFMA throughput per SM per clock on sm_100a (the fp64 eval's roofline denominator:
// k_eval_gravity<double> issues 13 FP64-pipe instructions per pair -- 8 DFMA + 3 DMUL + 2 DADD, from SASS --
// plus MUFU.RSQ64H / MUFU.RCP64H seeds).
// usage: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubd scripts/ubench_fp64.cu && /tmp/ubd
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double *out, long long *cyc, int iters, double b, double c) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    long long *cyc, *h = new long long[sms * 8];
    cudaMalloc(&out, sizeof(double) * sms * 8 * 256);
    cudaMalloc(&cyc, sizeof(long long) * sms * 8);
    const int iters = 4000;
    for (int ctas : {2, 4, 8}) {
        const int grid = sms * ctas;
        k_dfma<<<grid, 256>>>(out, cyc, iters, 1.0000001, 1e-9);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        k_dfma<<<grid, 256>>>(out, cyc, iters, 1.0000001, 1e-9);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        cudaMemcpy(h, cyc, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        const double ops = (double)grid * 256 * iters * 8;  // DFMA lane-ops
        printf("DFMA ctas/SM %d: %.3f ms, %.3e DFMA/s = %.2f TFLOP/s, %.1f DFMA lane-ops/clk/SM (clock64), f_eff %.0f MHz\n",
               ctas, ms, ops / (ms * 1e-3), 2 * ops / (ms * 1e-3) / 1e12, ops / sms / mx, mx / (ms * 1e-3) / 1e6);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
    return 0;
}
