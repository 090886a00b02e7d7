// k_dist.cu -- the multi-GPU path: Morton-range sharding with a halo exchange.
//
// Collective plan build on every rank (all steps stream-ordered; ONE host synchronisation for the exchange sizes):
//   1. bin + key the rank's input particles (the binning arithmetic of k_bin_gravity, DESIGN C6);
//   2. coarse histogram over 2^sc_bits Morton "supercells" (key >> shift), all-reduced (sum) on the device;
//   3. k_splitters: identical count-balanced splitters on every rank, computed on the device from the reduced
//      histogram (= p2p_partition_splitters, C20): rank r owns keys [spl[r], spl[r+1]), contiguous Morton ranges
//      aligned to supercells;
//   4. route: every input particle goes to its owner (as a target + source) and to every OTHER rank that owns a
//      box of its 26-neighbourhood (as a halo source).  A particle whose 3x3x3 neighbourhood fits in one
//      Morton-aligned cube lying inside one rank range needs no halo test (the common case: O(1) per particle);
//      the rest test the 26 neighbour owners;
//   5. the per-tile route counts are scanned per destination group (rank r, owned | halo) and all-gathered;
//      ONE device->host read-back gives the splitters, every rank's send counts and the out-of-domain flag;
//   6. a stable multi-split scatters {x,y,z,m} records straight from the caller's arrays into one send buffer
//      laid out [to rank 0: owned ; halo][to rank 1: owned ; halo]...; ONE all-to-all-v delivers them;
//   7. the local plan = the ordinary a1..a5 over the received records with target boxes restricted to the owned
//      range (halo boxes are sources only).
// Within every box the particles keep increasing GLOBAL input order (received runs are rank-major, each in its
// sender's input order, and the local radix sort is stable), so every target's redundant run -- records, order and
// rebased bits -- is identical to the 1-GPU plan on the concatenated input: results are bitwise independent of the
// GPU count.
// Eval: the local eval, then the reverse all-to-all-v returns the owned part of every received run to the rank and
// input slot it came from.
#include <algorithm>
#include <vector>

#include <cstdlib>

#include "plan.hpp"
#include "scan.cuh"

namespace p2p {

namespace {
template <typename T> struct V4T;
template <> struct V4T<float> { using type = float4; };
template <> struct V4T<double> { using type = double4; };

constexpr int MAX_RANKS = 64;  // halo masks are u64
constexpr int RT_THREADS = 256, RT_WARPS = RT_THREADS / 32, RT_ITEMS = 16, RT_TILE = RT_THREADS * RT_ITEMS;

// positions at pos[i*3 + d] (same binning arithmetic as k_structs.cu k_bin_gravity, DESIGN C6); an out-of-domain
// particle records its index in *err and gets box coordinate 0 in the offending dimension (a valid key)
template <typename T>
__global__ void k_keys(const T *__restrict__ pos, uint32_t n, Geom g, uint32_t *__restrict__ key,
                       unsigned long long *err) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t c[3];
        bool bad = false;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            double f = floor(__ddiv_rn(__dsub_rn((double)pos[(size_t)3 * i + d], g.lo[d]), g.h));
            if (!(f >= 0.0 && f < (double)g.nbox[d])) {
                bad = true;
                f = 0.0;
            }
            c[d] = (uint32_t)f;
        }
        if (bad) atomicMin(err, (unsigned long long)i);
        key[i] = spread3(c[0]) | (spread3(c[1]) << 1) | (spread3(c[2]) << 2);
    }
}

// supercell histogram: SC_COPIES striped copies (copy = block % SC_COPIES) spread the atomics on the dense
// centre supercells of clustered inputs (one copy: 277 us on the c5w tile), then k_sc_fold sums the copies
constexpr int SC_COPIES = 32;
__global__ void k_sc_hist(const uint32_t *__restrict__ key, uint32_t n, int shift, size_t nbins,
                          unsigned int *__restrict__ hist) {
    unsigned int *h = hist + (size_t)(blockIdx.x % SC_COPIES) * nbins;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        atomicAdd(&h[key[i] >> shift], 1u);
}
__global__ void k_sc_fold(const unsigned int *__restrict__ hist, size_t nbins, unsigned long long *__restrict__ out) {
    for (size_t b = (size_t)blockIdx.x * blockDim.x + threadIdx.x; b < nbins; b += (size_t)gridDim.x * blockDim.x) {
        unsigned long long s = 0;
#pragma unroll
        for (int c = 0; c < SC_COPIES; ++c) s += hist[(size_t)c * nbins + b];
        out[b] = s;
    }
}

__global__ void k_err_flag(const unsigned long long *err, unsigned long long *flag) {
    *flag = *err != ~0ull ? 1ull : 0ull;
}

// The splitters of compute_splitters (below) from the all-reduced device histogram, one block of 1024 threads:
// spl[r] = (first supercell b with excl(b) * G >= r * total) << shift, where excl(b) = particles in supercells < b;
// no such b < nbins -> nbins << shift.  Warp w owns the bins [w 32 C, (w + 1) 32 C), read in rows of 32 consecutive
// bins (coalesced); pass 1 sums them, a block scan gives every warp its base, pass 2 scans each row and lane j of a
// row resolves the ranks whose threshold falls in (excl(b) G, excl(b + 1) G] of its bin b (each crossing is found
// by exactly one lane: excl is non-decreasing).  Also copies the out-of-domain count hist[nbins] and the
// splitters into the read-back words.
constexpr int SPL_THREADS = 1024;
__global__ void __launch_bounds__(SPL_THREADS) k_splitters(const unsigned long long *__restrict__ hist, uint32_t nbins,
                                                           int shift, int key_bits, int G, uint32_t *__restrict__ spl,
                                                           unsigned long long *__restrict__ xfer_spl,
                                                           unsigned long long *__restrict__ xfer_err) {
    constexpr unsigned FULL = 0xffffffffu;
    __shared__ unsigned long long s_w[SPL_THREADS / 32];
    __shared__ uint32_t s_spl[MAX_RANKS + 1];
    const unsigned t = threadIdx.x, lane = t & 31u, w = t >> 5;
    const uint32_t C = (nbins + SPL_THREADS - 1) / SPL_THREADS;  // rows per warp
    const uint32_t wb = w * 32u * C;                              // the warp's first bin
    constexpr uint32_t U = 8;                                     // rows loaded per batch (loads in flight)
    auto ld = [&](uint32_t j) -> unsigned long long {
        const uint32_t b = wb + 32u * j + lane;
        return (j < C && b < nbins) ? hist[b] : 0ull;
    };
    unsigned long long s = 0;
    for (uint32_t j0 = 0; j0 < C; j0 += U) {
        unsigned long long v[U];
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) v[u] = ld(j0 + u);
#pragma unroll
        for (uint32_t u = 0; u < U; ++u) s += v[u];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (lane == 0) s_w[w] = s;
    const uint32_t dflt = (uint32_t)min((unsigned long long)nbins << shift, 0xffffffffull);
    if (t <= (unsigned)G) s_spl[t] = t == 0 ? 0u : (t == (unsigned)G ? (uint32_t)min(1ull << key_bits, 0xffffffffull) : dflt);
    __syncthreads();
    unsigned long long base = 0, total = 0;
    for (int i = 0; i < SPL_THREADS / 32; ++i) {
        base += i < (int)w ? s_w[i] : 0ull;
        total += s_w[i];
    }
    if (total == 0) {
        if (t > 0 && t < (unsigned)G) s_spl[t] = 0u;  // host loop: every r crosses at b = 0
    } else {
        // the thresholds r total (r = 1 .. G-1) that fall in this warp's range (base G, (base + s) G]: the warp
        // walks its rows only if there is one, and compares each bin with the next pending threshold only
        const unsigned long long GG = (unsigned long long)G;
        uint32_t r = 1;
        while (r < (uint32_t)G && (unsigned long long)r * total <= base * GG) ++r;
        if (r < (uint32_t)G && (unsigned long long)r * total <= (base + s) * GG) {
            for (uint32_t j0 = 0; j0 < C && r < (uint32_t)G; j0 += U) {
                unsigned long long v[U];
#pragma unroll
                for (uint32_t u = 0; u < U; ++u) v[u] = ld(j0 + u);
                for (uint32_t u = 0; u < U && r < (uint32_t)G; ++u) {
                    unsigned long long x = v[u];
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const unsigned long long y = __shfl_up_sync(FULL, x, o);
                        if (lane >= (unsigned)o) x += y;
                    }
                    const unsigned long long e1 = base + x;  // excl(b + 1) of lane's bin b
                    const uint32_t b = wb + 32u * (j0 + u) + lane;
                    // every pending threshold reached inside this row: first lane with e1 G >= r total
                    while (r < (uint32_t)G) {
                        const unsigned m = __ballot_sync(FULL, e1 * GG >= (unsigned long long)r * total);
                        if (!m) break;
                        const uint32_t bl = __shfl_sync(FULL, b, __ffs(m) - 1);
                        if (lane == 0) s_spl[r] = bl + 1 < nbins ? (uint32_t)((bl + 1) << shift) : dflt;
                        ++r;
                    }
                    base += __shfl_sync(FULL, x, 31);
                }
            }
        }
    }
    __syncthreads();
    if (t <= (unsigned)G) {
        spl[t] = s_spl[t];
        xfer_spl[t] = s_spl[t];
    }
    if (t == 0) *xfer_err = hist[nbins];
}

__device__ __forceinline__ int owner_of(uint32_t key, const uint32_t *spl, int G) {
    int lo = 0, hi = G - 1;  // largest r with spl[r] <= key
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (spl[mid] <= key) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// ranks other than `r0` that own a key of the box's 26-neighbourhood: they need the box's particles as halo
__device__ unsigned long long halo_mask(const Geom &g, uint32_t key, const uint32_t *spl, int G, int r0) {
    const uint32_t c[3] = {compact3(key), compact3(key >> 1), compact3(key >> 2)};
    unsigned long long m = 0ull;
    for (int slot = 0; slot < 27; ++slot) {
        if (slot == 13) continue;
        const int dd[3] = {slot % 3 - 1, (slot / 3) % 3 - 1, slot / 9 - 1};
        uint32_t nc[3];
        bool ok = true;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            int v = (int)c[d] + dd[d];
            if (v < 0 || v >= g.nbox[d]) {
                if (!((g.periodic >> d) & 1u)) ok = false;
                v = v < 0 ? v + g.nbox[d] : v - g.nbox[d];
            }
            nc[d] = (uint32_t)v;
        }
        if (!ok) continue;
        const int r = owner_of(spread3(nc[0]) | (spread3(nc[1]) << 1) | (spread3(nc[2]) << 2), spl, G);
        if (r != r0) m |= 1ull << r;
    }
    return m;
}

// halo_mask with an O(1) exit: if the box's 3x3x3 neighbourhood lies inside the Morton-aligned cube of side 2^l
// (l = smallest level at which no coordinate sits on the cube's faces, i.e. its low l bits are neither all 0 nor
// all 1) with no domain wrap, and both ends of that cube's key range belong to r0, every neighbour key is r0's
// (rank ranges are contiguous in key order): no halo.
__device__ __forceinline__ unsigned long long halo_of(const Geom &g, uint32_t key, const uint32_t *spl, int G,
                                                      int r0) {
    if (G == 1) return 0ull;
    const uint32_t c[3] = {compact3(key), compact3(key >> 1), compact3(key >> 2)};
    int l = 0;
    bool fast = true;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        if (c[d] == 0u || c[d] + 1u >= (uint32_t)g.nbox[d]) fast = false;
        const int tz = __ffs(c[d]) - 1, to = __ffs(~c[d]) - 1;  // trailing zeros / ones (c[d] != 0 if fast)
        l = max(l, max(tz, to) + 1);
    }
    if (fast && 3 * l < 32) {
        const uint32_t span = (1u << (3 * l)) - 1u;
        if (owner_of(key & ~span, spl, G) == r0 && owner_of(key | span, spl, G) == r0) return 0ull;
    }
    return halo_mask(g, key, spl, G, r0);
}

// route, pass 1 (tile = 4096 input particles): owner + halo mask of every particle, and the tile's count per
// destination group (group 2r = owned by rank r, 2r+1 = halo for rank r), column-major tcnt[group][tile]
__global__ void __launch_bounds__(RT_THREADS) k_route_count(Geom g, const uint32_t *__restrict__ key, uint32_t n,
                                                            const uint32_t *__restrict__ spl, int G,
                                                            uint8_t *__restrict__ r0_out,
                                                            unsigned long long *__restrict__ mask_out,
                                                            uint32_t *__restrict__ tcnt, uint32_t ntiles) {
    __shared__ uint32_t s_spl[MAX_RANKS + 1];
    __shared__ uint32_t s_cnt[2 * MAX_RANKS];
    const unsigned t = threadIdx.x;
    if (t <= (unsigned)G) s_spl[t] = spl[t];
    if (t < 2u * G) s_cnt[t] = 0u;
    __syncthreads();
    const uint32_t base = blockIdx.x * RT_TILE;
#pragma unroll 4
    for (int i = 0; i < RT_ITEMS; ++i) {
        const uint32_t p = base + i * RT_THREADS + t;
        if (p >= n) break;
        const uint32_t k = key[p];
        const int r0 = owner_of(k, s_spl, G);
        const unsigned long long m = halo_of(g, k, s_spl, G, r0);
        r0_out[p] = (uint8_t)r0;
        mask_out[p] = m;
        atomicAdd(&s_cnt[2 * r0], 1u);
        for (unsigned long long mm = m; mm; mm &= mm - 1) atomicAdd(&s_cnt[2 * (__ffsll((long long)mm) - 1) + 1], 1u);
    }
    __syncthreads();
    if (t < 2u * G) tcnt[(size_t)t * ntiles + blockIdx.x] = s_cnt[t];
}

// route, pass 2: block g scans column g of tcnt in place (exclusive tile offsets inside the group) and writes the
// group total gtot[g]
__global__ void __launch_bounds__(1024) k_route_scan(uint32_t *__restrict__ tcnt, uint32_t ntiles,
                                                     unsigned long long *__restrict__ gtot) {
    __shared__ uint32_t s_w[32];
    const unsigned t = threadIdx.x, lane = t & 31u, w = t >> 5;
    uint32_t *col = tcnt + (size_t)blockIdx.x * ntiles;
    uint32_t carry = 0;
    for (uint32_t b0 = 0; b0 < ntiles; b0 += 1024) {
        const uint32_t i = b0 + t;
        const uint32_t v = i < ntiles ? col[i] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (unsigned)o) x += y;
        }
        if (lane == 31) s_w[w] = x;
        __syncthreads();
        uint32_t add = 0, tot = 0;
        for (int j = 0; j < 32; ++j) {
            add += j < (int)w ? s_w[j] : 0u;
            tot += s_w[j];
        }
        if (i < ntiles) col[i] = carry + x - v + add;
        carry += tot;
        __syncthreads();
    }
    if (t == 0) gtot[blockIdx.x] = carry;
}

// route, pass 3: stable multi-split.  The send buffer is laid out by group (to rank 0: owned, halo; to rank 1: ...),
// each group in input order: tile offsets (pass 2) + per-warp offsets (pass A below) + the in-warp rank (match /
// ballot, in input order).  Records {x,y,z,m} are read straight from the caller's arrays (coalesced) and written
// to their send slot; perm_send[j] = input index of the j-th OWNED entry (rank-major), used by the result return.
template <typename T, typename V4>
__global__ void __launch_bounds__(RT_THREADS) k_route_scatter(const T *__restrict__ pos, const T *__restrict__ q,
                                                              const uint8_t *__restrict__ r0_in,
                                                              const unsigned long long *__restrict__ mask_in,
                                                              uint32_t n, int G, const uint32_t *__restrict__ toff,
                                                              uint32_t ntiles,
                                                              const unsigned long long *__restrict__ gtot,
                                                              V4 *__restrict__ send, uint32_t *__restrict__ perm_send) {
    __shared__ unsigned long long s_gbase[2 * MAX_RANKS];
    __shared__ uint32_t s_obase[MAX_RANKS];
    __shared__ uint32_t s_w[RT_WARPS][2 * MAX_RANKS];
    const unsigned t = threadIdx.x, lane = t & 31u, w = t >> 5;
    const int NG = 2 * G;
    if (t == 0) {
        unsigned long long a = 0, o = 0;
        for (int gi = 0; gi < NG; ++gi) {
            s_gbase[gi] = a;
            a += gtot[gi];
            if (!(gi & 1)) {
                s_obase[gi >> 1] = (uint32_t)o;
                o += gtot[gi];
            }
        }
    }
    for (int i = t; i < RT_WARPS * NG; i += RT_THREADS) s_w[i / NG][i % NG] = 0u;
    __syncthreads();
    const uint32_t seg = blockIdx.x * RT_TILE + w * 32 * RT_ITEMS;
    // pass A: per-warp counts per group
    for (int i = 0; i < RT_ITEMS; ++i) {
        const uint32_t p = seg + i * 32 + lane;
        if (p >= n) break;
        atomicAdd(&s_w[w][2 * r0_in[p]], 1u);
        for (unsigned long long mm = mask_in[p]; mm; mm &= mm - 1)
            atomicAdd(&s_w[w][2 * (__ffsll((long long)mm) - 1) + 1], 1u);
    }
    __syncthreads();
    if (t < (unsigned)NG) {  // exclusive prefix over the warps + the tile's offset inside the group
        uint32_t a = toff[(size_t)t * ntiles + blockIdx.x];
        for (int ww = 0; ww < RT_WARPS; ++ww) {
            const uint32_t c = s_w[ww][t];
            s_w[ww][t] = a;
            a += c;
        }
    }
    __syncthreads();
    // pass B: in input order, stable ranks inside the warp
    const uint32_t lt = (1u << lane) - 1u;
    for (int i = 0; i < RT_ITEMS; ++i) {
        const uint32_t p = seg + i * 32 + lane;
        const bool ok = p < n;
        const uint32_t act = __ballot_sync(0xffffffffu, ok);
        if (!act) break;  // warp-uniform
        const int r0 = ok ? (int)r0_in[p] : -1;
        const unsigned long long m = ok ? mask_in[p] : 0ull;
        V4 rec;
        if (ok) {
            rec.x = pos[(size_t)3 * p + 0];
            rec.y = pos[(size_t)3 * p + 1];
            rec.z = pos[(size_t)3 * p + 2];
            rec.w = q[p];
        }
        const uint32_t peers = __match_any_sync(0xffffffffu, r0);
        uint32_t slot = 0;
        if (ok) slot = s_w[w][2 * r0] + __popc(peers & lt);
        __syncwarp();
        if (ok) {
            if (lane == (unsigned)(__ffs(peers) - 1)) s_w[w][2 * r0] += __popc(peers);
            send[s_gbase[2 * r0] + slot] = rec;
            perm_send[s_obase[r0] + slot] = p;
        }
        __syncwarp();
        if (__ballot_sync(0xffffffffu, m != 0ull)) {
            for (int r = 0; r < G; ++r) {
                const uint32_t bm = __ballot_sync(0xffffffffu, (m >> r) & 1ull);
                if (!bm) continue;
                if ((m >> r) & 1ull) send[s_gbase[2 * r + 1] + s_w[w][2 * r + 1] + __popc(bm & lt)] = rec;
                __syncwarp();
                if (lane == 0) s_w[w][2 * r + 1] += __popc(bm);
                __syncwarp();
            }
        }
    }
}

// packs the results of local positions [i0, i0 + n): the owned head of one received run (halo positions are
// source-only, never written by the eval and never sent back)
template <typename T, typename V4>
__global__ void k_pack_results(const T *__restrict__ phi, const T *__restrict__ field, uint32_t i0, uint32_t n,
                               V4 *__restrict__ res) {
    for (uint32_t i = i0 + blockIdx.x * blockDim.x + threadIdx.x; i < i0 + n; i += gridDim.x * blockDim.x) {
        V4 r;
        r.x = phi[i];
        r.y = field[3 * (size_t)i + 0];
        r.z = field[3 * (size_t)i + 1];
        r.w = field[3 * (size_t)i + 2];
        res[i] = r;
    }
}

template <typename T, typename V4>
__global__ void k_unpack_results(const V4 *__restrict__ res, const uint32_t *__restrict__ perm_send, uint32_t n,
                                 T *__restrict__ phi, T *__restrict__ field) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const uint32_t i = perm_send[j];
        const V4 r = res[j];
        phi[i] = r.x;
        if (field) {
            field[3 * (size_t)i + 0] = r.y;
            field[3 * (size_t)i + 1] = r.z;
            field[3 * (size_t)i + 2] = r.w;
        }
    }
}

// rank r owns keys [spl[r], spl[r+1]): spl[r] = (first supercell whose exclusive prefix count >= r*total/G)
// << shift -- a pure function of the all-reduced histogram, so every rank derives the same splitters
void compute_splitters(const unsigned long long *h, int64_t nbins, int shift, int key_bits, int G, uint32_t *spl) {
    unsigned long long total = 0;
    for (int64_t b = 0; b < nbins; ++b) total += h[b];
    spl[0] = 0u;
    int r = 1;
    unsigned long long cum = 0;
    for (int64_t b = 0; b < nbins && r < G; ++b) {
        while (r < G && (unsigned __int128)cum * G >= (unsigned __int128)r * total) spl[r++] = (uint32_t)(b << shift);
        cum += h[b];
    }
    for (; r < G; ++r) spl[r] = (uint32_t)std::min<uint64_t>((uint64_t)nbins << shift, 0xffffffffull);
    spl[G] = (uint32_t)std::min<uint64_t>((uint64_t)1 << key_bits, 0xffffffffull);
}

unsigned grid1(uint64_t n, int num_sms) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(div_up(n, 256), (uint64_t)num_sms * 16));
}

struct Tmp {  // stream-ordered temporaries of the build
    cudaStream_t st;
    std::vector<void *> bufs;
    template <typename X>
    cudaError_t get(X **p, size_t bytes) {
        cudaError_t e = dalloc((void **)p, bytes, st);
        if (e == cudaSuccess) bufs.push_back(*p);
        return e;
    }
    ~Tmp() {
        for (void *b : bufs) dfree(b, st);
    }
};

template <typename T>
p2p_status build_dist_t(p2p_plan *P, const void *pos_v, const void *q_v) {
    using V4 = typename V4T<T>::type;
    free_distributed(P);  // a previous build's exchange buffers (p2p_plan_update on a collective plan)
    CommBase *C = P->comm;
    const int G = C->nranks, me = C->rank, NG = 2 * G;
    if (G > MAX_RANKS) {
        set_error("multi-GPU plans support at most 64 ranks (u64 halo masks)");
        return P2P_ERR_UNSUPPORTED;
    }
    cudaStream_t st = P->stream;
    const uint32_t n_in = (uint32_t)P->n_in;
    const T *pos = (const T *)pos_v, *q = (const T *)q_v;
    Tmp tmp{st, {}};
    const unsigned gb = grid1(std::max<uint32_t>(n_in, 1), P->num_sms);
    const size_t nn = std::max<uint32_t>(n_in, 1);
    const uint32_t ntiles = div_up(n_in, RT_TILE);
    // read-back words: [G][NG] all-gathered group totals | [NG] this rank's totals | [G+1] splitters |
    // out-of-domain count (all ranks) | this rank's first out-of-domain index
    const size_t x_gall = 0, x_gtot = (size_t)G * NG, x_spl = x_gtot + NG, x_erra = x_spl + G + 1, x_erri = x_erra + 1;
    const size_t xwords = x_erri + 1;
    uint32_t *key = nullptr, *spl = nullptr, *tcnt = nullptr;
    uint8_t *r0 = nullptr;
    unsigned long long *err = nullptr, *hmask = nullptr, *xfer = nullptr;
    P2P_CUDA_TRY(tmp.get(&key, 4 * nn));
    P2P_CUDA_TRY(tmp.get(&err, 8));
    P2P_CUDA_TRY(tmp.get(&xfer, 8 * xwords));
    P2P_CUDA_TRY(tmp.get(&spl, 4 * (G + 1)));
    P2P_CUDA_TRY(tmp.get(&r0, nn));
    P2P_CUDA_TRY(tmp.get(&hmask, 8 * nn));
    P2P_CUDA_TRY(tmp.get(&tcnt, 4 * (size_t)NG * std::max<uint32_t>(ntiles, 1)));
    P2P_CUDA_TRY(cudaMemsetAsync(err, 0xff, 8, st));
    // ---- 1. keys of the input particles ----
    if (n_in) P2P_LAUNCH(k_keys<T>, gb, 256, 0, st, pos, n_in, P->geom, key, err);
    // ---- 2. supercell histogram (+ one extra bin: ranks with an out-of-domain input), all-reduced ----
    // supercells span >= 4 keys (shift >= 2): the splitters are multiples of 4 keys, so an aligned key block -- a
    // multi-box quad of the REDUNDANT eval (k_structs.cu mb_role) -- never straddles two ranks
    const int sc_bits = std::max(0, std::min(P->key_bits - 2, 18)), shift = P->key_bits - sc_bits;
    const size_t nbins = (size_t)1 << sc_bits;
    unsigned long long *hist = nullptr;
    unsigned int *hist32 = nullptr;
    P2P_CUDA_TRY(tmp.get(&hist, 8 * (nbins + 1)));
    P2P_CUDA_TRY(tmp.get(&hist32, 4 * SC_COPIES * nbins));
    P2P_CUDA_TRY(cudaMemsetAsync(hist32, 0, 4 * SC_COPIES * nbins, st));
    if (n_in) P2P_LAUNCH(k_sc_hist, gb, 256, 0, st, key, n_in, shift, nbins, hist32);
    P2P_LAUNCH(k_sc_fold, grid1(nbins, P->num_sms), 256, 0, st, hist32, nbins, hist);
    P2P_LAUNCH(k_err_flag, 1, 1, 0, st, err, hist + nbins);
    p2p_status s = C->allreduce_sum_u64(hist, nbins + 1, st);
    if (s != P2P_OK) return s;
    // ---- 3. count-balanced splitters on the device, identical on every rank (C20) ----
    P2P_LAUNCH(k_splitters, 1, SPL_THREADS, 0, st, hist, (uint32_t)nbins, shift, P->key_bits, G, spl, xfer + x_spl,
               xfer + x_erra);
    // ---- 4./5. route counts per destination group, scanned and all-gathered ----
    if (ntiles)
        P2P_LAUNCH(k_route_count, ntiles, RT_THREADS, 0, st, P->geom, key, n_in, spl, G, r0, hmask, tcnt, ntiles);
    P2P_LAUNCH(k_route_scan, NG, 1024, 0, st, tcnt, ntiles, xfer + x_gtot);
    s = C->allgather_u64(xfer + x_gtot, xfer + x_gall, NG, st);
    if (s != P2P_OK) return s;
    P2P_CUDA_TRY(cudaMemcpyAsync(xfer + x_erri, err, 8, cudaMemcpyDeviceToDevice, st));
    std::vector<unsigned long long> hx(xwords);
    P2P_CUDA_TRY(cudaMemcpyAsync(hx.data(), xfer, 8 * xwords, cudaMemcpyDeviceToHost, st));
    P2P_CUDA_TRY(cudaStreamSynchronize(st));  // the ONE host synchronisation of the collective build
    if (hx[x_erra]) {  // every rank bails out consistently
        if (hx[x_erri] != ~0ull) {
            char buf[160];
            snprintf(buf, sizeof buf, "position of input particle %llu is outside the domain (C6)", hx[x_erri]);
            set_error(buf);
        } else {
            set_error("another rank has a position outside the domain (C6)");
        }
        return P2P_ERR_OUT_OF_DOMAIN;
    }
    P->splitters.assign(G + 1, 0u);
    for (int r = 0; r <= G; ++r) P->splitters[r] = (uint32_t)hx[x_spl + r];
    const uint32_t lo = P->splitters[me], hi = P->splitters[me + 1];
    P->geom.tkey_lo = lo;
    P->geom.tkey_hi = hi > lo ? hi - 1 : 0u;
    if (hi <= lo) P->geom.tkey_lo = 1;  // empty range: no target box
    // send: to rank r the run [owned by r ; halo for r]; receive from rank s: [owned from s ; halo from s]
    // rp_scnt[r] / rp_soff[r]: owned entries sent to r and their offset among this rank's owned entries (result
    // return); rp_rcnt[s] / rp_roff[s]: owned entries received from s and the offset of s's run in the local input
    const unsigned long long *gme = &hx[x_gall + (size_t)me * NG];
    P->rp_scnt.assign(G, 0);
    P->rp_soff.assign(G, 0);
    P->rp_rcnt.assign(G, 0);
    P->rp_roff.assign(G, 0);
    std::vector<int64_t> so(G), sc(G), ro(G), rc(G);
    int64_t e_send = 0, n_loc = 0, n_own = 0, o_sent = 0;
    for (int r = 0; r < G; ++r) {
        const unsigned long long *gr = &hx[x_gall + (size_t)r * NG];
        P->rp_scnt[r] = (int64_t)gme[2 * r];
        P->rp_soff[r] = o_sent;
        o_sent += P->rp_scnt[r];
        so[r] = e_send * (int64_t)sizeof(V4);
        sc[r] = (int64_t)(gme[2 * r] + gme[2 * r + 1]) * (int64_t)sizeof(V4);
        e_send += (int64_t)(gme[2 * r] + gme[2 * r + 1]);
        P->rp_rcnt[r] = (int64_t)gr[2 * me];
        P->rp_roff[r] = n_loc;
        ro[r] = n_loc * (int64_t)sizeof(V4);
        rc[r] = (int64_t)(gr[2 * me] + gr[2 * me + 1]) * (int64_t)sizeof(V4);
        n_loc += (int64_t)(gr[2 * me] + gr[2 * me + 1]);
        n_own += (int64_t)gr[2 * me];
    }
    if (o_sent != (int64_t)n_in || n_loc >= ((int64_t)1 << 30)) {
        set_error(o_sent != (int64_t)n_in ? "route: owned entries != input particles (internal)"
                                          : "local plan over owned + halo particles would reach 2^30 (radix look-back 30-bit digit prefixes)");
        return o_sent != (int64_t)n_in ? P2P_ERR_CUDA : P2P_ERR_UNSUPPORTED;
    }
    P->n_own = n_own;
    // ---- 6. stable multi-split of the records into the send buffer, ONE all-to-all-v ----
    V4 *send = nullptr, *local = nullptr;
    P2P_CUDA_TRY(tmp.get(&send, sizeof(V4) * std::max<int64_t>(e_send, 1)));
    P2P_CUDA_TRY(tmp.get(&local, sizeof(V4) * std::max<int64_t>(n_loc, 1)));
    P2P_CUDA_TRY(dalloc((void **)&P->perm_send, 4 * nn, st));
    if (ntiles)
        P2P_LAUNCH((k_route_scatter<T, V4>), ntiles, RT_THREADS, 0, st, pos, q, r0, hmask, n_in, G, tcnt, ntiles,
                   xfer + x_gtot, send, P->perm_send);
    s = C->alltoallv(send, so.data(), sc.data(), local, ro.data(), rc.data(), st);
    if (s != P2P_OK) return s;
    // ---- 7. the local plan over the received records, targets = this rank's Morton range ----
    // capacity buffers persist across p2p_plan_update calls (grow only); the temporaries above are released
    // stream-ordered (cudaFreeAsync), after every collective that reads them has completed on this stream
    P->n = n_loc;
    // result-return buffers first: a rank whose Morton range is empty (several splitters inside one supercell
    // holding > 1/G of the particles) keeps no particle but still receives its inputs' results
    const size_t nl = (size_t)std::max<int64_t>(n_loc, 1);
    P2P_CUDA_TRY(dalloc(&P->phi_loc, sizeof(T) * nl, st));
    P2P_CUDA_TRY(dalloc(&P->field_loc, 3 * sizeof(T) * nl, st));
    P2P_CUDA_TRY(dalloc(&P->res_own, sizeof(V4) * nl, st));
    P2P_CUDA_TRY(dalloc(&P->res_back, sizeof(V4) * nn, st));
    if (P->n == 0) {
        // no local particle, but the build's collectives (the item cost cap's all-reduce, k_structs.cu) still
        // need this rank's (zero) contribution
        P2P_CUDA_TRY(cudaMemsetAsync(&P->ctr->sum_nb2, 0, sizeof(unsigned long long), st));
        return P->comm->allreduce_sum_u64(&P->ctr->sum_nb2, 1, st);
    }
    if (P->n > P->cap) {
        free_capacity(P);
        s = alloc_capacity(P, P->n);
        if (s != P2P_OK) return s;
    }
    return build_gravity_structs(P, nullptr, nullptr, local);
}

template <typename T>
p2p_status eval_dist_t(p2p_plan *P, p2p_layout layout, void *phi, void *field) {
    using V4 = typename V4T<T>::type;
    cudaStream_t st = P->stream;
    const int G = P->comm->nranks;
    const uint32_t nl = (uint32_t)P->n, ni = (uint32_t)P->n_in;
    static const bool peer_ok = [] {
        const char *e = getenv("P2P_PEER_RESULTS");  // 0: the pack + all-to-all-v + unpack path on any communicator
        return !(e && e[0] == '0');
    }();
    if (peer_ok && P->comm->has_peer_results() && G <= PEER_MAX) {
        // a7 + a9 fused with the reverse all-to-all-v over peer memory: the eval epilogue stores every owned target's
        // {phi, fx, fy, fz} straight into its origin rank's receive buffer (comm_ipc.cu), laid out like res_back
        std::vector<char *> dst(G);
        std::vector<int64_t> dst_off(G), my_off(G);
        for (int r = 0; r < G; ++r) my_off[r] = P->rp_soff[r];
        char *recv = nullptr;
        p2p_status s = P->comm->peer_results_begin((uint64_t)std::max<uint32_t>(ni, 1) * sizeof(V4), my_off.data(),
                                                   dst.data(), dst_off.data(), &recv, st);
        if (s != P2P_OK) return s;
        if (nl > 0) {
            PeerRes h{};
            h.G = G;
            for (int r = 0; r < G; ++r) {
                h.lo[r] = (uint32_t)P->rp_roff[r];
                h.dst[r] = dst[r];
                h.off[r] = dst_off[r];
            }
            if (!P->peer_tab) P2P_CUDA_TRY(cudaMalloc(&P->peer_tab, sizeof(PeerRes)));
            P2P_CUDA_TRY(cudaMemcpy(P->peer_tab, &h, sizeof(PeerRes), cudaMemcpyHostToDevice));
            s = eval_gravity(P, layout, nullptr, nullptr, (const PeerRes *)P->peer_tab);
            if (s != P2P_OK) return s;
        }
        s = P->comm->peer_results_end(st);
        if (s != P2P_OK) return s;
        if (ni) P2P_LAUNCH((k_unpack_results<T, V4>), grid1(ni, P->num_sms), 256, 0, st, (const V4 *)recv,
                           P->perm_send, ni, (T *)phi, (T *)field);
        P2P_CUDA_TRY(cudaGetLastError());
        return P2P_OK;
    }
    if (nl > 0) {
        // results land at the local (received) positions; halo positions are not written and never sent back
        p2p_status s = eval_gravity(P, layout, P->phi_loc, P->field_loc);
        if (s != P2P_OK) return s;
        for (int r = 0; r < G; ++r)
            if (P->rp_rcnt[r] > 0)
                P2P_LAUNCH((k_pack_results<T, V4>), grid1((uint64_t)P->rp_rcnt[r], P->num_sms), 256, 0, st,
                           (const T *)P->phi_loc, (const T *)P->field_loc, (uint32_t)P->rp_roff[r],
                           (uint32_t)P->rp_rcnt[r], (V4 *)P->res_own);
    }
    std::vector<int64_t> so(G), sc(G), ro(G), rc(G);
    for (int r = 0; r < G; ++r) {  // the owned head of every received run goes back to its sender
        so[r] = P->rp_roff[r] * (int64_t)sizeof(V4);
        sc[r] = P->rp_rcnt[r] * (int64_t)sizeof(V4);
        ro[r] = P->rp_soff[r] * (int64_t)sizeof(V4);
        rc[r] = P->rp_scnt[r] * (int64_t)sizeof(V4);
    }
    p2p_status s = P->comm->alltoallv(P->res_own, so.data(), sc.data(), P->res_back, ro.data(), rc.data(), st);
    if (s != P2P_OK) return s;
    if (ni) P2P_LAUNCH((k_unpack_results<T, V4>), grid1(ni, P->num_sms), 256, 0, st, (const V4 *)P->res_back,
                       P->perm_send, ni, (T *)phi, (T *)field);
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}
}  // namespace

p2p_status build_distributed(p2p_plan *P, const void *pos, const void *q) {
    return P->cfg.precision == P2P_FP64 ? build_dist_t<double>(P, pos, q) : build_dist_t<float>(P, pos, q);
}

p2p_status eval_distributed(p2p_plan *P, p2p_layout layout, void *phi, void *field) {
    return P->cfg.precision == P2P_FP64 ? eval_dist_t<double>(P, layout, phi, field)
                                        : eval_dist_t<float>(P, layout, phi, field);
}

}  // namespace p2p

extern "C" p2p_status p2p_partition_splitters(const uint64_t *hist, int64_t nbins, int shift, int key_bits,
                                              int nranks, uint32_t *splitters_out) {
    if (!hist || !splitters_out || nbins < 1 || nranks < 1 || shift < 0 || key_bits < 0 || key_bits > 32 ||
        (nbins << shift) > ((int64_t)1 << 32)) {
        p2p::set_error("invalid splitter arguments");
        return P2P_ERR_INVALID_ARGUMENT;
    }
    p2p::compute_splitters((const unsigned long long *)hist, nbins, shift, key_bits, nranks, splitters_out);
    return P2P_OK;
}

namespace p2p {

void free_distributed(p2p_plan *P) {
    void *bufs[] = {P->perm_send, P->phi_loc, P->field_loc, P->res_own, P->res_back};
    for (void *b : bufs) dfree(b, P->stream);
    P->perm_send = nullptr;
    P->phi_loc = P->field_loc = P->res_own = P->res_back = nullptr;
    if (P->peer_tab) cudaFree(P->peer_tab);
    P->peer_tab = nullptr;
}

}  // namespace p2p
