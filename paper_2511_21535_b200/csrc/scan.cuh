// scan.cuh -- device-wide exclusive scan (reduce -> scan partials -> downsweep), generic over the value
// type and over "get"/"put" functors so inputs need not be materialised (a4 run heads, a5 offsets).
// The element count may live on the device (`nptr`, e.g. the box count B); launches are sized by the
// host-side capacity `ncap` and early-exit beyond *nptr.
#pragma once
#include "common.cuh"

namespace p2p {

constexpr int SC_THREADS = 256;
constexpr int SC_ITEMS = 8;
constexpr int SC_TILE = SC_THREADS * SC_ITEMS;

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T x) {
    const unsigned lane = threadIdx.x & 31u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (unsigned)o) x += y;
    }
    return x;
}

// exclusive block scan (SC_THREADS threads); returns exclusive prefix, *total = block sum
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T *total) {
    __shared__ T wt[SC_THREADS / 32];
    const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    T x = warp_incl_scan(v);
    if (lane == 31) wt[w] = x;
    __syncthreads();
    T add = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < SC_THREADS / 32; ++i) {
        T t = wt[i];
        add += (i < (int)w) ? t : T(0);
        tot += t;
    }
    __syncthreads();
    *total = tot;
    return x - v + add;
}

template <typename T, typename Get>
__global__ void __launch_bounds__(SC_THREADS) k_scan_reduce(Get get, const uint32_t *nptr, uint64_t ncap,
                                                            T *partials) {
    const uint64_t n = nptr ? min((uint64_t)*nptr, ncap) : ncap;  // a device count never exceeds the capacity
    const uint64_t base = (uint64_t)blockIdx.x * SC_TILE;
    T s = 0;
    if (base < n) {
#pragma unroll
        for (int i = 0; i < SC_ITEMS; ++i) {
            uint64_t idx = base + (uint64_t)i * SC_THREADS + threadIdx.x;
            if (idx < n) s += get(idx);
        }
    }
    T tot;
    block_excl_scan<T>(s, &tot);
    if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

// single block: exclusive scan of the partials in place, writes the grand total
template <typename T>
__global__ void __launch_bounds__(SC_THREADS) k_scan_partials(T *partials, uint32_t nparts, T *total_out) {
    T carry = 0;
    for (uint32_t b0 = 0; b0 < nparts; b0 += SC_THREADS) {
        uint32_t i = b0 + threadIdx.x;
        T v = i < nparts ? partials[i] : T(0);
        T tot;
        T e = block_excl_scan<T>(v, &tot);
        if (i < nparts) partials[i] = carry + e;
        carry += tot;
    }
    if (threadIdx.x == 0 && total_out) *total_out = carry;
}

template <typename T, typename Get, typename Put>
__global__ void __launch_bounds__(SC_THREADS) k_scan_down(Get get, Put put, const uint32_t *nptr, uint64_t ncap,
                                                          const T *partials) {
    const uint64_t n = nptr ? min((uint64_t)*nptr, ncap) : ncap;  // a device count never exceeds the capacity
    const uint64_t base = (uint64_t)blockIdx.x * SC_TILE;
    if (base >= n) return;  // whole block beyond n: uniform exit (no barrier below is skipped partially)
    // thread-contiguous items: thread t owns [base + t*ITEMS, base + (t+1)*ITEMS)
    T vals[SC_ITEMS];
    T s = 0;
#pragma unroll
    for (int i = 0; i < SC_ITEMS; ++i) {
        uint64_t idx = base + (uint64_t)threadIdx.x * SC_ITEMS + i;
        vals[i] = idx < n ? get(idx) : T(0);
        s += vals[i];
    }
    T tot;
    T e = block_excl_scan<T>(s, &tot) + partials[blockIdx.x];
#pragma unroll
    for (int i = 0; i < SC_ITEMS; ++i) {
        uint64_t idx = base + (uint64_t)threadIdx.x * SC_ITEMS + i;
        if (idx < n) put(idx, e, vals[i]);
        e += vals[i];
    }
}

// run the three phases; `ncap` = capacity (launch size), `nptr` = optional device count
// scratch: >= scan_partials_bytes(ncap) bytes (plan-owned, reused by consecutive scans on one stream)
static inline size_t scan_partials_bytes(uint64_t ncap) { return 8 * (size_t)div_up(ncap, SC_TILE) + 8; }

template <typename T, typename Get, typename Put>
cudaError_t device_scan(Get get, Put put, const uint32_t *nptr, uint64_t ncap, T *total_out, void *scratch,
                        cudaStream_t st) {
    if (ncap == 0) {
        if (total_out) cudaMemsetAsync(total_out, 0, sizeof(T), st);
        return cudaGetLastError();
    }
    const unsigned nblk = div_up(ncap, SC_TILE);
    T *partials = (T *)scratch;
    P2P_LAUNCH((k_scan_reduce<T, Get>), nblk, SC_THREADS, 0, st, get, nptr, ncap, partials);
    P2P_LAUNCH((k_scan_partials<T>), 1, SC_THREADS, 0, st, partials, nblk, total_out);
    P2P_LAUNCH((k_scan_down<T, Get, Put>), nblk, SC_THREADS, 0, st, get, put, nptr, ncap, partials);
    return cudaGetLastError();
}

}  // namespace p2p
