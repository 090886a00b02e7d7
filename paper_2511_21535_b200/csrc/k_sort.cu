// k_sort.cu -- hand-written stable LSD radix sort of (u32 key, u32 value) pairs for sm_100a
// (SURVEY §8a-a2 "Morton-key radix sort"; BASELINE north_star forbids a library sort on the path).
//
// Design (Onesweep-style, one read + one write of the pairs per 8-bit digit):
//   k_radix_hist      one pass over the keys builds the 256-bin histogram of EVERY digit at once
//   k_radix_hist_scan exclusive scan of each digit histogram -> global digit offsets
//   k_radix_pass      per digit: each CTA takes the next 4096-key tile (tile ids handed out by an atomic
//                     counter in launch order, so look-back never waits on an unscheduled tile), counts its
//                     digits, publishes them and resolves its exclusive prefix by decoupled look-back over
//                     earlier tiles (before the ranking: the inclusive prefixes propagate at look-back speed),
//                     ranks its keys stably in input order (8 bit-sliced ballots per key: digit_peers),
//                     stages the tile in shared memory in digit order and writes each digit run
//                     contiguously (coalesced) to its global position.
// Stability: within a tile keys are ranked in (warp, item, lane) order, which is input order; tiles are
// ordered by id = input order.  HBM traffic per pass: 8 B read + 8 B write per pair (+ look-back words).
#include "plan.hpp"

namespace p2p {

namespace {
#ifndef P2P_RS_THREADS
#define P2P_RS_THREADS 256
#endif
#ifndef P2P_RS_ITEMS
#define P2P_RS_ITEMS 16
#endif
#ifndef P2P_RS_MINB
#define P2P_RS_MINB 3
#endif
#ifndef P2P_RS_LB
#define P2P_RS_LB 8
#endif
constexpr int RS_THREADS = P2P_RS_THREADS;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = P2P_RS_ITEMS;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // 4096 keys per tile
constexpr uint32_t FLAG_AGG = 1u << 30;
constexpr uint32_t FLAG_INC = 2u << 30;
constexpr uint32_t VAL_MASK = (1u << 30) - 1u;

__global__ void __launch_bounds__(256) k_radix_hist(const uint32_t *__restrict__ keys, uint32_t n, int passes,
                                                    uint32_t *__restrict__ hist) {
    __shared__ uint32_t sh[4][256];
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t k = keys[i];
        for (int p = 0; p < passes; ++p) atomicAdd(&sh[p][(k >> (8 * p)) & 255u], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) {
        uint32_t v = (&sh[0][0])[i];
        if (v) atomicAdd(&hist[i], v);
    }
}

// block-wide exclusive scan of one value per thread (256 threads)
__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t v, uint32_t *warp_tot /*[8]*/, uint32_t *total) {
    const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (unsigned)o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    uint32_t add = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < RS_WARPS; ++i) {
        uint32_t t = warp_tot[i];
        add += (i < (int)w) ? t : 0u;
        tot += t;
    }
    __syncthreads();
    if (total) *total = tot;
    return x - v + add;
}

__global__ void __launch_bounds__(256) k_radix_hist_scan(uint32_t *hist) {
    __shared__ uint32_t wt[RS_WARPS];
    uint32_t *h = hist + blockIdx.x * 256;
    uint32_t v = h[threadIdx.x];
    uint32_t e = block_excl_scan256(v, wt, nullptr);
    h[threadIdx.x] = e;
}

// lanes of `mask` whose 8-bit digit equals this lane's: bit-sliced, 8 ballots (default).  __match_any_sync
// (P2P_SORT_MATCH=1) costs one pass per DISTINCT value in the warp on sm_100a: ~28 on uniform digits, so the
// histogram kernel ran at 0.55 TB/s on passes 0-1 and 1.0 TB/s on the skewed top digit (ncu, gpurun_out/sort)
#ifndef P2P_SORT_XORPEERS
#define P2P_SORT_XORPEERS 1
#endif
__device__ __forceinline__ uint32_t digit_peers(uint32_t mask, uint32_t d) {
#if defined(P2P_SORT_MATCH) && P2P_SORT_MATCH
    return __match_any_sync(mask, d);
#else
#if P2P_SORT_XORPEERS
    // lanes whose digit differs from this lane's in any bit: OR over the bits of (ballot XOR my-bit-broadcast);
    // the bit sits in the sign of (d << (31 - b)), which gives both the ballot predicate and the broadcast mask
    uint32_t diff = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const int32_t sb = (int32_t)(d << (31 - b));
        const uint32_t bb = __ballot_sync(mask, sb < 0);
        diff |= bb ^ (uint32_t)(sb >> 31);
    }
    return mask & ~diff;
#else
    uint32_t peers = mask;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const bool one = (d >> b) & 1u;
        const uint32_t bb = __ballot_sync(mask, one);
        peers &= one ? bb : ~bb;
    }
    return peers;
#endif
#endif
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile(uint32_t *p, uint32_t v) {
    asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 3 resident CTAs per SM (<= 85 registers): measured 377 us per c5w sort vs 438 at 2 CTAs and 390 at 4 (spills)
__global__ void __launch_bounds__(RS_THREADS, P2P_RS_MINB) k_radix_pass(const uint32_t *__restrict__ kin,
                                                           const uint32_t *__restrict__ vin, uint32_t *__restrict__ kout,
                                                           uint32_t *__restrict__ vout, uint32_t n, int shift,
                                                           const uint32_t *__restrict__ digit_off,
                                                           uint32_t *status, uint32_t *tile_ctr, bool iota) {
    __shared__ uint32_t s_whist[RS_WARPS][256];
    __shared__ uint32_t s_tdig[256];
    __shared__ uint32_t s_goff[256];
    extern __shared__ uint32_t s_dyn[];  // the tile staged in digit order: keys, then values (dynamic: > 48 KB tiles)
    uint32_t *s_keys = s_dyn, *s_vals = s_dyn + RS_TILE;
    __shared__ uint32_t s_wt[RS_WARPS];
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_thist[256];

    const unsigned tid = threadIdx.x, lane = tid & 31u, w = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
    for (int i = tid; i < RS_WARPS * 256; i += RS_THREADS) (&s_whist[0][0])[i] = 0;
    s_thist[tid] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint32_t base = tile * RS_TILE;
    const uint32_t seg = base + w * 32 * RS_ITEMS;
    const uint32_t lt_mask = (1u << lane) - 1u;

    uint32_t k[RS_ITEMS], v[RS_ITEMS], r[RS_ITEMS];
#pragma unroll
    for (int i = 0; i < RS_ITEMS; ++i) {
        uint32_t idx = seg + i * 32 + lane;
        bool ok = idx < n;
        k[i] = ok ? kin[idx] : 0u;
        v[i] = iota ? idx : (ok ? vin[idx] : 0u);  // iota: the first pass's values are the input positions
    }
    // the tile's digit counts first (shared-memory atomics), published as the tile aggregate BEFORE the
    // ranking: successors looking back find it early, and this tile's own look-back (after the ranking) mostly
    // finds its predecessors already resolved
#pragma unroll
    for (int i = 0; i < RS_ITEMS; ++i)
        if (seg + i * 32 + lane < n) atomicAdd(&s_thist[(k[i] >> shift) & 255u], 1u);
    __syncthreads();
    // per digit: publish the aggregate, look back for the exclusive prefix, publish the inclusive prefix --
    // all BEFORE the ranking, so the chain of inclusive prefixes across tiles advances at look-back speed and the
    // ranking work stays off it
    {
        const uint32_t d = tid, cnt = s_thist[d];
        uint32_t *my = status + (size_t)tile * 256 + d;
        uint32_t excl = 0;
        if (tile == 0) {
            st_volatile(my, FLAG_INC | cnt);
        } else {
            st_volatile(my, FLAG_AGG | cnt);
            // walk back LB predecessors per step (independent loads in flight; tile 0 is always inclusive, so
            // the walk never passes it): a chain of one dependent load per predecessor made the look-back the
            // pass's critical path
            constexpr int LB = P2P_RS_LB;
            for (int64_t t = (int64_t)tile - 1;;) {
                uint32_t sv[LB];
#pragma unroll
                for (int i = 0; i < LB; ++i) sv[i] = t - i >= 0 ? ld_volatile(status + (size_t)(t - i) * 256 + d) : FLAG_INC;
                bool done = false;
                int adv = LB;
#pragma unroll
                for (int i = 0; i < LB; ++i) {
                    if (done || adv < LB) continue;
                    const uint32_t f = sv[i] & ~VAL_MASK;
                    if (f == 0) {  // predecessor not published yet: resume from it after a back-off
                        adv = i;
                        continue;
                    }
                    excl += sv[i] & VAL_MASK;
                    if (f == FLAG_INC) done = true;
                }
                if (done) break;
                t -= adv;
                if (adv < LB) __nanosleep(50);
            }
            st_volatile(my, FLAG_INC | (excl + cnt));
        }
        s_goff[d] = digit_off[d] + excl;
    }
#pragma unroll
    for (int i = 0; i < RS_ITEMS; ++i) {
        uint32_t idx = seg + i * 32 + lane;
        bool ok = idx < n;
        uint32_t mask = __ballot_sync(0xffffffffu, ok);
        if (ok) {
            uint32_t d = (k[i] >> shift) & 255u;
            const uint32_t peers = digit_peers(mask, d);
            uint32_t cnt = s_whist[w][d];
            r[i] = cnt + __popc(peers & lt_mask);
            __syncwarp(mask);
            if (lane == (uint32_t)(__ffs(peers) - 1)) s_whist[w][d] = cnt + __popc(peers);
        }
        __syncwarp();
    }
    __syncthreads();

    // per digit: exclusive prefix across warps, tile-local digit start
    {
        const uint32_t d = tid;
        uint32_t sum = 0;
#pragma unroll
        for (int ww = 0; ww < RS_WARPS; ++ww) {
            uint32_t c = s_whist[ww][d];
            s_whist[ww][d] = sum;
            sum += c;
        }
        s_tdig[d] = block_excl_scan256(sum, s_wt, nullptr);
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < RS_ITEMS; ++i) {
        uint32_t idx = seg + i * 32 + lane;
        if (idx < n) {
            uint32_t d = (k[i] >> shift) & 255u;
            uint32_t pos = s_tdig[d] + s_whist[w][d] + r[i];
            s_keys[pos] = k[i];
            s_vals[pos] = v[i];
        }
    }
    __syncthreads();
    const uint32_t tile_n = min((uint32_t)RS_TILE, n - base);
    for (uint32_t j = tid; j < tile_n; j += RS_THREADS) {
        uint32_t key = s_keys[j];
        uint32_t d = (key >> shift) & 255u;
        uint32_t dst = s_goff[d] + (j - s_tdig[d]);
        kout[dst] = key;
        vout[dst] = s_vals[j];
    }
}

__global__ void k_iota_u32(uint32_t *__restrict__ v, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = i;
}

__global__ void k_copy_u32(const uint32_t *__restrict__ a, uint32_t *__restrict__ b, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) b[i] = a[i];
}
}  // namespace

size_t radix_status_words(uint64_t n, int passes) { return (size_t)passes * div_up(n, RS_TILE) * 256; }

cudaError_t radix_sort_pairs(uint32_t *kin, uint32_t *vin, uint32_t *kalt, uint32_t *valt, uint32_t n, int passes,
                             DevCounters *ctr, uint32_t *hist, uint32_t *status, cudaStream_t st, uint32_t **kout,
                             uint32_t **vout, bool iota_values, bool hist_ready) {
    *kout = kin;
    *vout = vin;
    if (n == 0) return cudaSuccess;
    if (passes == 0) {  // one box: the order is the input order
        if (iota_values) P2P_LAUNCH(k_iota_u32, std::min<unsigned>(div_up(n, 256), 148 * 8), 256, 0, st, vin, n);
        return cudaGetLastError();
    }
    const uint32_t ntiles = div_up(n, RS_TILE);
    cudaMemsetAsync(status, 0, radix_status_words(n, passes) * sizeof(uint32_t), st);
    cudaMemsetAsync(ctr->sort_tile_ctr, 0, sizeof(ctr->sort_tile_ctr), st);
    if (!hist_ready) {  // else the caller's key kernel built the digit histograms (k_bin_gravity)
        cudaMemsetAsync(hist, 0, (size_t)passes * 256 * sizeof(uint32_t), st);
        unsigned hg = std::min<unsigned>(div_up(n, 256 * 8), 148 * 8);
        P2P_LAUNCH(k_radix_hist, hg, 256, 0, st, kin, n, passes, hist);
    }
    P2P_LAUNCH(k_radix_hist_scan, passes, 256, 0, st, hist);
    static bool smem_set = false;
    if (!smem_set) {  // static (12 KB) + dynamic staging may exceed the 48 KB default
        cudaFuncSetAttribute(k_radix_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * RS_TILE);
        smem_set = true;
    }
    uint32_t *a_k = kin, *a_v = vin, *b_k = kalt, *b_v = valt;
    for (int p = 0; p < passes; ++p) {
        P2P_LAUNCH(k_radix_pass, ntiles, RS_THREADS, 8 * RS_TILE, st, a_k, a_v, b_k, b_v, n, 8 * p, hist + 256 * p,
                   status + (size_t)p * ntiles * 256, &ctr->sort_tile_ctr[p], iota_values && p == 0);
        std::swap(a_k, b_k);
        std::swap(a_v, b_v);
    }
    *kout = a_k;
    *vout = a_v;
    return cudaGetLastError();
}

}  // namespace p2p
