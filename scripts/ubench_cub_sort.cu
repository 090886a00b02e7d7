// Reference measurement (not on the product path): CUB's DeviceRadixSort::SortPairs on the a2 workload --
// 12.5M (u32 key, u32 value) pairs, 24-bit Morton keys of the c5w Plummer tile's box distribution approximated by
// uniformly random 24-bit keys -- against which the hand-written Onesweep sort (k_sort.cu) is compared.
// usage: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cubs scripts/ubench_cub_sort.cu && /tmp/cubs
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cub/cub.cuh>

int main() {
    const int n = 12500000;
    std::vector<uint32_t> hk(n), hv(n);
    std::mt19937 rng(1);
    for (int i = 0; i < n; ++i) { hk[i] = rng() & 0xFFFFFFu; hv[i] = i; }
    uint32_t *k0, *k1, *v0, *v1;
    cudaMalloc(&k0, 4 * n); cudaMalloc(&k1, 4 * n); cudaMalloc(&v0, 4 * n); cudaMalloc(&v1, 4 * n);
    cudaMemcpy(k0, hk.data(), 4 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(v0, hv.data(), 4 * n, cudaMemcpyHostToDevice);
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, v0, v1, n, 0, 24);
    void *dtmp; cudaMalloc(&dtmp, tmp);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) cub::DeviceRadixSort::SortPairs(dtmp, tmp, k0, k1, v0, v1, n, 0, 24);
    float best = 1e9;
    for (int rep = 0; rep < 10; ++rep) {
        cudaEventRecord(a);
        cub::DeviceRadixSort::SortPairs(dtmp, tmp, k0, k1, v0, v1, n, 0, 24);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
    }
    printf("CUB SortPairs 12.5M u32/u32, 24 bits: best %.1f us\n", best * 1e3);
    return 0;
}
