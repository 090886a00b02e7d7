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
    constexpr uint32_t PER = 32;  // up to 8192 partials: thread t owns a contiguous range, all loads in flight, one
                                  // block scan (the looped form below paid a block scan per 256: 12 us on c5w)
    if (nparts <= PER * SC_THREADS) {
        const uint32_t per = (nparts + SC_THREADS - 1) / SC_THREADS, t0 = threadIdx.x * per;
        T v[PER];
        T sum = 0;
#pragma unroll
        for (uint32_t i = 0; i < PER; ++i) {
            v[i] = (i < per && t0 + i < nparts) ? partials[t0 + i] : T(0);
            sum += v[i];
        }
        T tot;
        T e = block_excl_scan<T>(sum, &tot);
#pragma unroll
        for (uint32_t i = 0; i < PER; ++i) {
            if (i < per && t0 + i < nparts) partials[t0 + i] = e;
            e += v[i];
        }
        if (threadIdx.x == 0 && total_out) *total_out = tot;
        return;
    }
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

// ---- single-pass scan (u32 values < 2^30) with decoupled look-back: reads the input ONCE (the 3-phase scan
// above reads it twice and launches three kernels).  Tiles are claimed in launch order through `tile_ctr`, so every
// predecessor of a tile is already running; a tile publishes its aggregate, then a warp walks back 32 predecessors
// per step to the nearest inclusive prefix.  `status` holds >= ceil(ncap / SCL_TILE) words, zeroed before the
// launch together with *tile_ctr.
constexpr int SCL_ITEMS = 16;
constexpr int SCL_TILE = SC_THREADS * SCL_ITEMS;
constexpr uint32_t SCL_AGG = 1u << 30, SCL_INC = 2u << 30, SCL_VAL = (1u << 30) - 1u;

template <typename Get, typename Put>
__global__ void __launch_bounds__(SC_THREADS) k_scan_lb(Get get, Put put, const uint32_t *nptr, uint64_t ncap,
                                                        uint32_t *status, uint32_t *tile_ctr, uint32_t *total_out) {
    __shared__ uint32_t s_tile, s_excl;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t n = nptr ? min((uint64_t)*nptr, ncap) : ncap;
    const uint64_t base = (uint64_t)tile * SCL_TILE;
    if (base >= n) return;  // no successor of this tile holds elements either
    uint32_t vals[SCL_ITEMS];
    uint32_t sum = 0;
#pragma unroll
    for (int i = 0; i < SCL_ITEMS; ++i) {
        const uint64_t idx = base + (uint64_t)threadIdx.x * SCL_ITEMS + i;
        vals[i] = idx < n ? get(idx) : 0u;
        sum += vals[i];
    }
    uint32_t tot;
    const uint32_t bex = block_excl_scan<uint32_t>(sum, &tot);
    if (threadIdx.x < 32) {
        const unsigned lane = threadIdx.x;
        volatile uint32_t *vs = status;
        uint32_t excl = 0;
        if (tile == 0) {
            if (lane == 0) vs[0] = SCL_INC | tot;
        } else {
            if (lane == 0) vs[tile] = SCL_AGG | tot;
            for (int64_t t = (int64_t)tile - 1;; t -= 32) {
                const int64_t q = t - (int64_t)lane;
                uint32_t v = SCL_INC;  // before tile 0: an inclusive zero
                if (q >= 0)
                    do {
                        v = vs[q];
                    } while ((v & ~SCL_VAL) == 0u);
                const uint32_t inc = __ballot_sync(0xffffffffu, (v & ~SCL_VAL) == SCL_INC);
                const int first = inc ? __ffs(inc) - 1 : 32;  // nearest predecessor with an inclusive prefix
                uint32_t part = (int)lane <= first ? (v & SCL_VAL) : 0u;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                excl += part;
                if (inc) break;
            }
            __threadfence();
            if (lane == 0) vs[tile] = SCL_INC | (excl + tot);
        }
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    uint32_t e = s_excl + bex;
#pragma unroll
    for (int i = 0; i < SCL_ITEMS; ++i) {
        const uint64_t idx = base + (uint64_t)threadIdx.x * SCL_ITEMS + i;
        if (idx < n) put(idx, e, vals[i]);
        e += vals[i];
    }
    if (total_out && base + SCL_TILE >= n && threadIdx.x == 0) *total_out = s_excl + tot;  // the last tile
}

static inline size_t scan_lb_status_words(uint64_t ncap) { return div_up(ncap, SCL_TILE) + 1; }

template <typename Get, typename Put>
cudaError_t device_scan_lb(Get get, Put put, const uint32_t *nptr, uint64_t ncap, uint32_t *total_out,
                           uint32_t *status, uint32_t *tile_ctr, cudaStream_t st) {
    if (ncap == 0) {
        if (total_out) cudaMemsetAsync(total_out, 0, sizeof(uint32_t), st);
        return cudaGetLastError();
    }
    const unsigned ntiles = div_up(ncap, SCL_TILE);
    cudaMemsetAsync(status, 0, sizeof(uint32_t) * ntiles, st);
    cudaMemsetAsync(tile_ctr, 0, sizeof(uint32_t), st);
    if (total_out) cudaMemsetAsync(total_out, 0, sizeof(uint32_t), st);
    P2P_LAUNCH((k_scan_lb<Get, Put>), ntiles, SC_THREADS, 0, st, get, put, nptr, ncap, status, tile_ctr, total_out);
    return cudaGetLastError();
}

}  // namespace p2p
