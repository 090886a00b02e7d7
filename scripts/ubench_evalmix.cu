// Microbenchmark of the gravity eval hot loop's instruction mix on sm_100a (k_eval_gravity.cu hot_loop +
// Tgt<float,4>::interact): 4 shared-memory sources per iteration x 4 register targets (2 packed pairs).
// Reports FP32 lane-ops per SM per SM-clock (clock64) = the fraction of the 128 lane-ops/clk/SM FP32 peak the
// loop reaches, for instruction-mix variants that give the SAME bits:
//   mode 0  current: FADD2 / FFMA2 / FMUL2 + 2 MUFU.RSQ per pair
//   mode 1  every FADD2 as FFMA2(x, 1, y) and every FMUL2 as FFMA2(a, b, -0) (bit-identical: one rounding)
//   mode 2  FADD2 -> FFMA2 only
//   mode 3  FMUL2 -> FFMA2 only
//   mode 4  (perf probe, not bit-identical) mode 0 with MUFU replaced by a dependent FMUL
// usage: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubm scripts/ubench_evalmix.cu && /tmp/ubm
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 bc(float v) { return make_float2(v, v); }
__device__ __forceinline__ float rsq(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int MODE>
struct Mix {
    float2 one, nz;
    __device__ __forceinline__ float2 add(float2 a, float2 b) const {
        if (MODE == 1 || MODE == 2) return __ffma2_rn(a, one, b);
        return __fadd2_rn(a, b);
    }
    __device__ __forceinline__ float2 mul(float2 a, float2 b) const {
        if (MODE == 1 || MODE == 3) return __ffma2_rn(a, b, nz);
        return __fmul2_rn(a, b);
    }
};

template <int MODE, int K = 4, int MINB = 1>
__global__ void __launch_bounds__(128, MINB) k_mix(const float4 *gsrc, float *out, long long *cyc, int iters, float one,
                                                    float nzero) {
    constexpr int NP = K / 2;
    __shared__ float4 src[1024 + 64];  // 64 records of slack: a 4-source step at the wrap point reads past 1024
    for (int i = threadIdx.x; i < 1024 + 64; i += blockDim.x) src[i] = gsrc[i & 1023];
    __syncthreads();
    Mix<MODE> M;
    M.one = bc(one);
    M.nz = bc(nzero);
    float2 tx[NP], ty[NP], tz[NP], ap[NP], ax[NP], ay[NP], az[NP];
    for (int p = 0; p < NP; ++p) {
        // every target coordinate distinct and runtime-dependent (constant or repeated targets let ptxas share
        // the d = s - t of equal targets across pairs -- the first version of this benchmark did, and over-reported)
        const float u = (float)(threadIdx.x + 1) * one;
        tx[p] = make_float2(-0.011f * u - 0.13f * p, -0.017f * u - 0.29f * p - 0.07f);
        ty[p] = make_float2(-0.023f * u - 0.31f * p - 0.05f, -0.019f * u - 0.37f * p - 0.11f);
        tz[p] = make_float2(-0.029f * u - 0.41f * p - 0.03f, -0.013f * u - 0.43f * p - 0.17f);
        ap[p] = ax[p] = ay[p] = az[p] = make_float2(0.f, 0.f);
    }
    const float2 E = bc(1e-6f);
    __syncthreads();
    long long t0 = clock64();
    uint32_t sa = (uint32_t)__cvta_generic_to_shared(src) + (threadIdx.x & 31) * 16;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(src);
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        float4 s[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(s[q].x), "=f"(s[q].y), "=f"(s[q].z), "=f"(s[q].w)
                         : "r"(sa + q * 64) : "memory");
        sa = base + ((sa + 256 - base) & 16383u);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const float2 dx = M.add(bc(s[q].x), tx[p]);
                const float2 dy = M.add(bc(s[q].y), ty[p]);
                const float2 dz = M.add(bc(s[q].z), tz[p]);
                float2 r2 = __ffma2_rn(dx, dx, E);
                r2 = __ffma2_rn(dy, dy, r2);
                r2 = __ffma2_rn(dz, dz, r2);
                float2 ri;
                if (MODE == 4) ri = __fmul2_rn(r2, bc(0.5f));
                else ri = make_float2(rsq(r2.x), rsq(r2.y));
                const float2 mri = M.mul(bc(s[q].w), ri);
                ap[p] = M.add(ap[p], mri);
                const float2 m3 = M.mul(mri, M.mul(ri, ri));
                ax[p] = __ffma2_rn(m3, dx, ax[p]);
                ay[p] = __ffma2_rn(m3, dy, ay[p]);
                az[p] = __ffma2_rn(m3, dz, az[p]);
            }
        }
    }
    long long t1 = clock64();
    float acc = 0.f;
    for (int p = 0; p < NP; ++p) acc += ap[p].x + ap[p].y + ax[p].x + ax[p].y + ay[p].x + ay[p].y + az[p].x + az[p].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE, int K = 4, int MINB = 1>
void run(int ctas_per_sm, int sms, const float4 *src, float *out, long long *cyc, long long *hcyc) {
    const int iters = 4000 * 4 / K;
    const int grid = sms * ctas_per_sm;
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_mix<MODE, K, MINB>);
    k_mix<MODE, K, MINB><<<grid, 128>>>(src, out, cyc, iters, 1.0f, -0.0f);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_mix<MODE, K, MINB><<<grid, 128>>>(src, out, cyc, iters, 1.0f, -0.0f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaMemcpy(hcyc, cyc, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
        printf("mode %d: %s\n", MODE, cudaGetErrorString(e));
        return;
    }
    long long mx = 0;
    for (int i = 0; i < grid; ++i) mx = hcyc[i] > mx ? hcyc[i] : mx;
    // lane-ops per SM: ctas * 128 threads * iters * 4 sources * 4 targets * 13
    const double ops_sm = (double)ctas_per_sm * 128 * iters * 4 * K * 13;
    const double pairs = (double)grid * 128 * iters * 4 * K;
    printf("mode %d K %d regs %3d ctas/SM %d: %.3f ms, %.3e pairs/s, %.1f lane-ops/clk/SM (frac of 128: %.3f), "
           "f_eff %.0f MHz\n", MODE, K, fa.numRegs, ctas_per_sm, ms, pairs / (ms * 1e-3), ops_sm / mx, ops_sm / mx / 128.0,
           mx / (ms * 1e-3) / 1e6);
}

#define CK(x)                                                                                      \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess) {                                                                   \
            printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));               \
            fflush(stdout);                                                                        \
            return 1;                                                                              \
        }                                                                                          \
    } while (0)

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    printf("SMs %d\n", sms);
    static float4 h[1024];
    for (int i = 0; i < 1024; ++i) h[i] = make_float4(0.001f * i, 0.002f * (i % 37), 0.003f * (i % 11), 1.0f + i);
    float4 *src;
    float *out;
    long long *cyc, *hcyc = new long long[sms * 16];
    CK(cudaMalloc(&src, sizeof(h)));
    CK(cudaMemcpy(src, h, sizeof(h), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&out, sizeof(float) * sms * 16 * 128));
    CK(cudaMalloc(&cyc, sizeof(long long) * sms * 16));
    for (int c : {3, 4, 5, 6, 8}) {
        run<0, 4>(c, sms, src, out, cyc, hcyc);
        run<2, 4>(c, sms, src, out, cyc, hcyc);
        run<0, 8>(c, sms, src, out, cyc, hcyc);
        run<2, 8>(c, sms, src, out, cyc, hcyc);
        run<0, 6>(c, sms, src, out, cyc, hcyc);
        run<2, 6>(c, sms, src, out, cyc, hcyc);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(e));
    return 0;
}
