// k_structs.cu -- method steps a1..a5 on the device:
//   a1 bin + Morton key (fp64 IEEE binning, DESIGN C6/C7), a2 stable radix sort (k_sort.cu),
//   a3 permute into Morton-ordered AoS records, a4 box-offset scan (run heads -> compact box table),
//   a5 neighbour CSR (ascending stencil slot, C10) + redundant offsets red_off + eval work items.
// Bit-exactness with the oracle: every fp64 operation that decides an integer (box index, sub-cell) is an
// explicit IEEE intrinsic (__dsub_rn, __ddiv_rn, __fma_rn) so no contraction or reassociation can change
// a rounding.
#include <algorithm>

#include <cstdlib>

#include "items.cuh"
#include "plan.hpp"
#include "scan.cuh"

namespace p2p {

// ------------------------------------------------------------------------------------------------ a1
// floor(fl(a / h)) (C6: the IEEE fp64 division, then floor) without the division in the common case: q = fl(a *
// fl(1/h)) is within 2^-52 |q| (1 + 2^-52) of a/h and fl(a/h) within 2^-53 of it, so floor(q) == floor(fl(a/h))
// whenever q is farther than 2^-50 |q| from an integer (q - f and f + 1 - q are exact: Sterbenz); otherwise -- a
// point within a few ulp of a box face -- the division decides, exactly as the oracle (face tests pin both paths)
__device__ __forceinline__ double floor_div_exact(double a, double h, double inv_h) {
    const double q = a * inv_h;
    const double f = floor(q);
    const double margin = fabs(q) * 0x1p-50;
    if (q - f > margin && (f + 1.0) - q > margin) return f;
    return floor(__ddiv_rn(a, h));
}

// positions at pos[i * ps + d] (ps = 3: the caller's [N][3] array; ps = 4: {x,y,z,m} records).  With `aos` the
// caller's SoA input is also packed into {x,y,z,m} records in input order (read sequentially here), so that the a3
// gather touches ONE 16-byte record per particle instead of a position and a mass in two arrays (two DRAM bursts)
// The a2 sort's digit histograms are built here too (the keys are in registers; the sort's own histogram pass
// re-read 50 MB at c5w), and its first pass takes the input positions as values (no iota array written / read).
#ifndef P2P_BIN_MINB
#define P2P_BIN_MINB 0  // 0: no register cap
#endif
template <typename T, typename V4>
__global__ void __launch_bounds__(256, P2P_BIN_MINB) k_bin_gravity(const T *__restrict__ pos, int ps, uint32_t n, Geom g,
                                                     uint32_t *__restrict__ key, DevCounters *ctr,
                                                     const T *__restrict__ q, V4 *__restrict__ aos, int passes,
                                                     uint32_t *__restrict__ hist) {
    __shared__ uint32_t sh[4][256];
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();
    const double inv_h = 1.0 / g.h;
    // BIN_U particles per thread per iteration, every load issued before the first use (memory-level parallelism:
    // one particle per iteration left the kernel at 0.55 of HBM with 67% warps active)
#ifndef P2P_BIN_U
#define P2P_BIN_U 4
#endif
    constexpr int BIN_U = P2P_BIN_U;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i0 = blockIdx.x * blockDim.x * BIN_U + threadIdx.x; i0 < n; i0 += stride * BIN_U) {
        T xd[BIN_U][3], qm[BIN_U];
#pragma unroll
        for (int u = 0; u < BIN_U; ++u) {
            const uint32_t i = i0 + u * blockDim.x;
            const bool ok = i < n;
#pragma unroll
            for (int d = 0; d < 3; ++d) xd[u][d] = ok ? pos[(size_t)ps * i + d] : (T)g.lo[d];
            qm[u] = (ok && aos) ? q[i] : (T)0;
        }
#pragma unroll
        for (int u = 0; u < BIN_U; ++u) {
            const uint32_t i = i0 + u * blockDim.x;
            if (i >= n) break;
            uint32_t c[3];
            bool bad = false;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                double f = floor_div_exact(__dsub_rn((double)xd[u][d], g.lo[d]), g.h, inv_h);
                if (!(f >= 0.0 && f < (double)g.nbox[d])) {
                    bad = true;
                    f = 0.0;
                }
                c[d] = (uint32_t)f;
            }
            if (bad) atomicMin(&ctr->err_index, (unsigned long long)i);
            const uint32_t k = spread3(c[0]) | (spread3(c[1]) << 1) | (spread3(c[2]) << 2);
            key[i] = k;
            for (int p = 0; p < passes; ++p) atomicAdd(&sh[p][(k >> (8 * p)) & 255u], 1u);
            if (aos) {
                V4 r;
                r.x = xd[u][0];
                r.y = xd[u][1];
                r.z = xd[u][2];
                r.w = qm[u];
                aos[i] = r;
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) {
        const uint32_t v = (&sh[0][0])[i];
        if (v) atomicAdd(&hist[i], v);
    }
}

// Helmholtz: key = morton2(box) * t + subcell, subcell = sy*st + sx, s_d = floor((x_d - o_d)/Delta),
// o_d = fma(ib_d, h, lo_d), Delta = h / st (DESIGN C8)
template <typename T>
__global__ void k_bin_helmholtz(const T *__restrict__ pos, uint32_t n, Geom g, int st, double delta, uint32_t t,
                                uint32_t *__restrict__ key, uint32_t *__restrict__ idx, DevCounters *ctr) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t c[2], s[2];
        bool bad = false, irr = false;
#pragma unroll
        for (int d = 0; d < 2; ++d) {
            double x = (double)pos[2 * (size_t)i + d];
            double f = floor(__ddiv_rn(__dsub_rn(x, g.lo[d]), g.h));
            if (!(f >= 0.0 && f < (double)g.nbox[d])) {
                bad = true;
                f = 0.0;
            }
            c[d] = (uint32_t)f;
            double o = __fma_rn((double)c[d], g.h, g.lo[d]);
            double sf = floor(__ddiv_rn(__dsub_rn(x, o), delta));
            if (!(sf >= 0.0 && sf < (double)st)) {
                irr = true;
                sf = 0.0;
            }
            s[d] = (uint32_t)sf;
        }
        if (bad) atomicMin(&ctr->err_index, (unsigned long long)i);
        if (irr && !bad) atomicOr(&ctr->irregular, 1u);
        key[i] = (spread2(c[0]) | (spread2(c[1]) << 1)) * t + (s[1] * (uint32_t)st + s[0]);
        idx[i] = i;
    }
}

// ------------------------------------------------------------------------------------------------ a3
// random gather (input order is arbitrary) of {x,y,z,m} records: one 16 B (fp64: 32 B) load per particle,
// 4 particles per thread iteration, all loads issued before the stores (memory-level parallelism)
#ifndef P2P_PERMUTE_CS
#define P2P_PERMUTE_CS 1
#endif
#if P2P_PERMUTE_CS  // streaming perm reads / record stores leave L2 to the gathered lines (8 records each): 231 -> 227 us
#define P2P_PERM_LD(p) __ldcs(p)
#define P2P_REC_ST(p, v) st_stream(p, v)
#else
#define P2P_PERM_LD(p) (*(p))
#define P2P_REC_ST(p, v) (*(p) = (v))
#endif
__device__ __forceinline__ void st_stream(float4 *p, const float4 &v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double4 *p, const double4 &v) {
    __stcs(reinterpret_cast<double2 *>(p), make_double2(v.x, v.y));
    __stcs(reinterpret_cast<double2 *>(p) + 1, make_double2(v.z, v.w));
}
#ifndef P2P_PERM_U
#define P2P_PERM_U 4
#endif
template <typename V4>
__global__ void k_permute_gravity(const V4 *__restrict__ src, const uint32_t *__restrict__ perm, uint32_t n,
                                  V4 *__restrict__ rec) {
    constexpr int U = P2P_PERM_U;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t p0 = blockIdx.x * blockDim.x + threadIdx.x; p0 < n; p0 += U * stride) {
        uint32_t i[U];
#pragma unroll
        for (int u = 0; u < U; ++u) i[u] = p0 + u * stride < n ? P2P_PERM_LD(perm + p0 + u * stride) : 0u;
        V4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (p0 + u * stride < n) r[u] = src[i[u]];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (p0 + u * stride < n) P2P_REC_ST(rec + p0 + u * stride, r[u]);
    }
}

template <typename C2>
__global__ void k_permute_complex(const C2 *__restrict__ x, const uint32_t *__restrict__ perm, uint32_t n,
                                  C2 *__restrict__ xs) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) xs[p] = x[perm[p]];
}

// ------------------------------------------------------------------------------------------------ a4
struct HeadGet {
    const uint32_t *skey;
    uint32_t div;
    __device__ uint32_t operator()(uint64_t p) const {
        return (p == 0 || skey[p] / div != skey[p - 1] / div) ? 1u : 0u;
    }
};
struct HeadGet1 {  // gravity: the box key is the sorted key itself (no division)
    const uint32_t *skey;
    __device__ uint32_t operator()(uint64_t p) const { return (p == 0 || skey[p] != skey[p - 1]) ? 1u : 0u; }
};
struct HeadPut {
    const uint32_t *skey;
    uint32_t div;
    uint32_t *bkey, *bstart, *box_of;
    uint32_t n;
    uint32_t *occ = nullptr;  // optional occupancy bitmap of the key space (gravity)
    __device__ void operator()(uint64_t p, uint32_t e, uint32_t v) const {
        if (v) {
            uint32_t bk = skey[p] / div;
            bkey[e] = bk;
            bstart[e] = (uint32_t)p;
            if (box_of) box_of[bk] = e;
            if (occ) atomicOr(&occ[bk >> 5], 1u << (bk & 31u));
        }
        if (p == n - 1) bstart[e + v] = n;
    }
};

// gravity run heads with vectorised key loads: thread t holds keys i0 .. i0 + 7 (i0 = tile + 8 t) in registers from two
// 16-byte loads plus its predecessor, instead of the generic scan's two scalar loads per element (HeadGet1)
__device__ __forceinline__ uint32_t head_bits(const uint32_t *__restrict__ skey, uint32_t n, uint64_t i0,
                                              uint32_t (&k)[8]) {
    if (i0 + 8 <= n) {
        const uint4 a = *reinterpret_cast<const uint4 *>(skey + i0), b = *reinterpret_cast<const uint4 *>(skey + i0 + 4);
        k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w; k[4] = b.x; k[5] = b.y; k[6] = b.z; k[7] = b.w;
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) k[i] = i0 + i < n ? skey[i0 + i] : 0u;
    }
    uint32_t prev = i0 > 0 && i0 < n ? skey[i0 - 1] : ~k[0];
    uint32_t h = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (i0 + i < n && k[i] != prev) h |= 1u << i;
        prev = k[i];
    }
    return h;
}
__global__ void __launch_bounds__(SC_THREADS) k_head_reduce(const uint32_t *__restrict__ skey, uint32_t n,
                                                           uint32_t *__restrict__ partials) {
    const uint64_t i0 = (uint64_t)blockIdx.x * SC_TILE + (uint64_t)threadIdx.x * SC_ITEMS;
    uint32_t k[8];
    const uint32_t h = i0 < n ? head_bits(skey, n, i0, k) : 0u;
    uint32_t tot;
    block_excl_scan<uint32_t>((uint32_t)__popc(h), &tot);
    if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(SC_THREADS) k_head_down(const uint32_t *__restrict__ skey, uint32_t n,
                                                         const uint32_t *__restrict__ partials,
                                                         uint32_t *__restrict__ bkey, uint32_t *__restrict__ bstart) {
    const uint64_t base = (uint64_t)blockIdx.x * SC_TILE;
    if (base >= n) return;  // whole block beyond n: uniform exit
    const uint64_t i0 = base + (uint64_t)threadIdx.x * SC_ITEMS;
    uint32_t k[8];
    const uint32_t h = i0 < n ? head_bits(skey, n, i0, k) : 0u;
    uint32_t tot;
    uint32_t e = block_excl_scan<uint32_t>((uint32_t)__popc(h), &tot) + partials[blockIdx.x];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if ((h >> i) & 1u) {
            bkey[e] = k[i];
            bstart[e] = (uint32_t)(i0 + i);
            ++e;
        }
    }
    if (i0 < n && i0 + 8 >= n) bstart[e] = n;  // the thread of the last element closes the table
}

// ------------------------------------------------------------------------------------------------ a5
// dense key -> {box, n_b} table for the gravity neighbour search (valid where the occupancy bit is set)
// + sum over the target boxes of n_b^2 (the item cost cap's work estimate; integer atomics: order-independent)
// + the occupancy bitmap: lanes are consecutive boxes (ascending keys), so the lanes sharing a 32-key occupancy word
// are contiguous; a segmented OR over them leaves ONE atomicOr per word and warp (the run-head scan's per-box
// atomicOr serialised on the shared words)
__global__ void k_boxinfo(const uint32_t *__restrict__ bkey, const uint32_t *__restrict__ bstart,
                          DevCounters *__restrict__ ctr, uint2 *__restrict__ boxinfo, uint32_t *__restrict__ occ,
                          uint32_t tkey_lo, uint32_t tkey_hi) {
    const uint32_t B = ctr->B;
    const unsigned lane = threadIdx.x & 31u;
    unsigned long long s2 = 0;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t b0 = blockIdx.x * blockDim.x; b0 < B; b0 += stride) {  // warp-uniform trip count
        const uint32_t b = b0 + threadIdx.x;
        const bool have = b < B;
        const uint32_t key = have ? bkey[b] : 0xffffffffu;
        if (have) {
            const uint32_t nb = bstart[b + 1] - bstart[b];
            boxinfo[key] = make_uint2(b, nb);
            if (key >= tkey_lo && key <= tkey_hi) s2 += (unsigned long long)nb * nb;
        }
        const uint32_t wd = key >> 5;
        uint32_t bits = have ? 1u << (key & 31u) : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t ob = __shfl_down_sync(0xffffffffu, bits, o), ow = __shfl_down_sync(0xffffffffu, wd, o);
            if (lane + o < 32u && ow == wd) bits |= ob;
        }
        const uint32_t pw = __shfl_up_sync(0xffffffffu, wd, 1);
        if (have && (lane == 0u || pw != wd)) atomicOr(&occ[wd], bits);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if ((threadIdx.x & 31u) == 0 && s2) atomicAdd(&ctr->sum_nb2, s2);
}

// a5 in two kernels, THREAD PER BOX (tile = the 256 consecutive boxes of one block):
//   k_nbr_count  the box's 27 stencil neighbours (ascending slot, C10) by Morton arithmetic: per dimension the
//                three candidate coordinates {-1, 0, +1} are formed once in interleaved form (periodic wrap /
//                open edge, C5), a slot's key is an OR of three of them; the occupancy bit and the {box, n}
//                entry are loaded together, branch-free (a stale entry of an empty key is ignored).  Per-box
//                totals -> block sums per tile (CSR entries, redundant records, work items, small-target pairs)
//                + the pair count I.
//   k_tile_scan  exclusive prefixes of the tile sums (chunks of 1024 tiles per CTA + the chunk totals)
//   k_nbr_fill   the box's occupied-slot mask and record count (saved by k_nbr_count), block scan of the per-box
//                totals + the tile's exclusive prefix (k_tile_scan), then nbr_off / red_off, the CSR staged in
//                shared memory and written coalesced, the restructure chunk heads, the eval work items or
//                small-target entries.
// Lanes are consecutive boxes, so a slot's 32 neighbour keys are close in key order (coalesced table reads),
// and no tile ever waits for another: the earlier single-kernel design (warp per 32 boxes, lane = slot, decoupled
// look-back on tiles still searching) spent about half of its 1.06 ms there; these take 0.14 + 0.006 + 0.25 ms on c5w.
constexpr int NB_THREADS = 256;
constexpr int NB_SLOTS = 27;

struct NbStencil {  // per dimension: candidate interleaved coordinates for offsets -1, 0, +1 and their validity
    uint32_t c[3][3];
    bool v[3][3];
};
__device__ __forceinline__ void make_nb(const Geom &g, uint32_t key, NbStencil &S) {
    const uint32_t full = spread3((1u << g.nb) - 1u);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const uint32_t M = full << d, top = spread3((uint32_t)(g.nbox[d] - 1)) << d, kd = key & M;
        const bool per = (g.periodic >> d) & 1u;
        S.c[d][1] = kd;
        S.v[d][1] = true;
        S.c[d][0] = kd == 0u ? top : ((kd - (1u << d)) & M);
        S.v[d][0] = kd != 0u || per;
        S.c[d][2] = kd == top ? 0u : (((kd | ~M) + (1u << d)) & M);
        S.v[d][2] = kd != top || per;
    }
}

// one dz-plane of the stencil (slots 9 dz .. 9 dz + 8), branch-free so that all 18 table loads are in flight at
// once (an invalid slot loads the box's own entry and is masked): okm bit s = slot s holds a non-empty box
__device__ __forceinline__ void nb_plane(const NbStencil &S, int dz, uint32_t key, bool tgt,
                                         const uint32_t *__restrict__ occ, const uint2 *__restrict__ boxinfo,
                                         uint32_t &okm, uint32_t &cnt, unsigned long long &red,
                                         unsigned long long &part4) {
    uint32_t nk[9], wd[9], ny[9];
    bool v[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        const int dx = j % 3, dy = j / 3;
        v[j] = tgt && S.v[0][dx] && S.v[1][dy] && S.v[2][dz];
        nk[j] = v[j] ? (S.c[0][dx] | S.c[1][dy] | S.c[2][dz]) : key;
    }
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        wd[j] = __ldg(&occ[nk[j] >> 5]);
        ny[j] = __ldg(&boxinfo[nk[j]].y);
    }
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        const bool ok = v[j] && ((wd[j] >> (nk[j] & 31u)) & 1u);
        okm |= (ok ? 1u : 0u) << (9 * dz + j);
        cnt += ok ? 1u : 0u;
        red += ok ? ny[j] : 0u;
        if (j < 4) part4 += ok ? ny[j] : 0u;
    }
}

__constant__ uint8_t c_div32[33] = {0,  32, 16, 10, 8, 6, 5, 4, 4, 3, 3, 2, 2, 2, 2, 2, 2,
                                     1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1};  // 32 / g

struct BoxTotals {
    uint32_t nbr, item, small, item_red;  // item_red: the REDUNDANT eval's items (multi-box quads, see mb_role)
    unsigned long long red;
};
__device__ __forceinline__ BoxTotals box_totals(uint32_t nbr, uint64_t red, uint32_t nb, bool tgt, uint32_t tmax,
                                                 uint32_t K, uint64_t cap) {
    BoxTotals t;
    t.nbr = nbr;
    t.red = red;
    // boxes with <= SMALL_NT targets go to the eval's thread-per-target path (no work item)
// a second small-path window: boxes of <= P2P_SMALL_NT2 targets with <= P2P_SMALL_R2 sources also take the
// thread-per-target-pair path (measured on one box: c5w eval 5961 / 5968 -> 5878 / 5897 us, c3 407 -> 400 us, c4-8 /
// c4-16 unchanged; a plain SMALL_R = 256 sent c4-8's 8-target boxes (R = 216) there and lost their quad items: +60%)
#ifndef P2P_SMALL_NT2
#define P2P_SMALL_NT2 6
#endif
#ifndef P2P_SMALL_R2
#define P2P_SMALL_R2 256
#endif
#ifndef P2P_SMALL_NT3  // a third window (sweep knob, off)
#define P2P_SMALL_NT3 0
#define P2P_SMALL_R3 0
#endif
    const bool small = (nb <= SMALL_NT && red <= SMALL_R) || (nb <= P2P_SMALL_NT2 && red <= P2P_SMALL_R2) ||
                       (nb <= P2P_SMALL_NT3 && red <= P2P_SMALL_R3);
    t.item = (small || !tgt) ? 0u : (nb + item_size(nb, red, tmax, K, cap) - 1) / item_size(nb, red, tmax, K, cap);
    t.small = (small && tgt) ? (nb + 1) / 2 : 0u;  // target PAIRS
    t.item_red = t.item;
    return t;
}

// Multi-box work items of the REDUNDANT eval (fp32): the 4 boxes of an aligned Morton key block (keys 4c .. 4c + 3, a
// 2 x 2 x 1 block of boxes) that are all non-empty target boxes with <= 8 targets each (item path, not the small-box
// path) and <= 65535 sources become ONE work item: box j owns lanes 8j .. 8j + 7 (2 groups of 4 targets x 4 source
// splits, the standard G = 8 / S = 4 layout) and the 4 runs are staged in lockstep, 64 records of each per stage (4
// bulk copies) -- possible only because every box's sources are ONE contiguous run (the redundant layout).  The
// per-item overhead (record fetch, staging, transpose-reduce, epilogue) is paid once per 4 boxes: on 8-per-box
// inputs it was half of the eval's instructions.  The grouping depends only on keys and per-box data, and the
// multi-GPU splitters are multiples of 4 keys (k_dist.cu), so a block never straddles ranks: the items, and the
// bits, are the same on any number of GPUs.
constexpr uint32_t MB_NT = 8, MB_R = 65535;
constexpr uint32_t MB_ELIG = 1u << 31;  // box_nbr[b].x flag (okm uses bits 0..26): the box may join a quad
// cost <= cap / 4: a quad item (8 lanes per box) then takes no longer than a capped single-box item (32 lanes)
__device__ __forceinline__ bool mb_eligible(bool enabled, bool tgt, uint32_t items, uint32_t nb, uint64_t red,
                                            uint64_t cap) {
    return enabled && tgt && items == 1u && nb >= 1u && nb <= MB_NT && red <= MB_R && (uint64_t)nb * red * 4 <= cap;
}
// 0: no quad, 1: leader (key % 4 == 0), 2: member of the quad led by box b - (key & 3)
__device__ __forceinline__ int mb_role(uint32_t b, uint32_t key, uint32_t B, const uint32_t *__restrict__ bkey,
                                       const uint2 *__restrict__ box_nbr) {
    if (!(box_nbr[b].x & MB_ELIG)) return 0;  // most boxes of clustered inputs: one load
    const uint32_t j = key & 3u;
    if (b < j || b - j + 3u >= B) return 0;
    const uint32_t lead = b - j, k0 = key - j;
#pragma unroll
    for (uint32_t i = 0; i < 4; ++i) {
        if (i == j) continue;
        if (bkey[lead + i] != k0 + i || !(box_nbr[lead + i].x & MB_ELIG)) return 0;
    }
    return j == 0 ? 1 : 2;
}

// block-wide inclusive scan of the four totals (NB_THREADS threads); returns the inclusive values, `tot` = sums
__device__ __forceinline__ BoxTotals block_scan_totals(BoxTotals x, BoxTotals *tot) {
    __shared__ BoxTotals s_w[NB_THREADS / 32];
    const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t a = __shfl_up_sync(0xffffffffu, x.nbr, o), b = __shfl_up_sync(0xffffffffu, x.item, o),
                       c = __shfl_up_sync(0xffffffffu, x.small, o), ir = __shfl_up_sync(0xffffffffu, x.item_red, o);
        const unsigned long long d = __shfl_up_sync(0xffffffffu, x.red, o);
        if (lane >= (unsigned)o) {
            x.nbr += a;
            x.item += b;
            x.small += c;
            x.item_red += ir;
            x.red += d;
        }
    }
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    BoxTotals add{0, 0, 0, 0, 0ull}, t{0, 0, 0, 0, 0ull};
#pragma unroll
    for (int i = 0; i < NB_THREADS / 32; ++i) {
        const BoxTotals v = s_w[i];
        if (i < (int)w) {
            add.nbr += v.nbr;
            add.item += v.item;
            add.small += v.small;
            add.item_red += v.item_red;
            add.red += v.red;
        }
        t.nbr += v.nbr;
        t.item += v.item;
        t.small += v.small;
        t.item_red += v.item_red;
        t.red += v.red;
    }
    __syncthreads();
    *tot = t;
    x.nbr += add.nbr;
    x.item += add.item;
    x.small += add.small;
    x.item_red += add.item_red;
    x.red += add.red;
    return x;
}

// block-wide sums of the totals (k_nbr_count needs only the tile sums, not the per-box prefixes): warp reductions
// (REDUX for the 32-bit fields), then warp 0
__device__ __forceinline__ BoxTotals block_sum_totals(const BoxTotals &x) {
    __shared__ BoxTotals s_w[NB_THREADS / 32];
    const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    BoxTotals r;
    r.nbr = __reduce_add_sync(0xffffffffu, x.nbr);
    r.item = __reduce_add_sync(0xffffffffu, x.item);
    r.small = __reduce_add_sync(0xffffffffu, x.small);
    r.item_red = __reduce_add_sync(0xffffffffu, x.item_red);
    unsigned long long red = x.red;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) red += __shfl_xor_sync(0xffffffffu, red, o);
    r.red = red;
    if (lane == 0) s_w[w] = r;
    __syncthreads();
    BoxTotals t{0, 0, 0, 0, 0ull};
#pragma unroll
    for (int i = 0; i < NB_THREADS / 32; ++i) {
        const BoxTotals v = s_w[i];
        t.nbr += v.nbr;
        t.item += v.item;
        t.small += v.small;
        t.item_red += v.item_red;
        t.red += v.red;
    }
    __syncthreads();
    return t;
}

// tile sums / exclusive tile offsets: [0] CSR entries, [1] redundant records, [2] work items, [3] small pairs,
// [4] REDUNDANT-eval work items (multi-box quads)
constexpr int NB_TOT = 5;
struct NbTile {
    unsigned long long v[NB_TOT];
};

#ifndef P2P_NC_MINB
#define P2P_NC_MINB 4  // (an explicit 1 let ptxas take 90 registers: 237 vs 136 us on c5w)
#endif
__global__ void __launch_bounds__(NB_THREADS, P2P_NC_MINB) k_nbr_count(Geom g, const uint32_t *__restrict__ bkey,
                                                          const uint32_t *__restrict__ bstart,
                                                          const uint2 *__restrict__ boxinfo,
                                                          const uint32_t *__restrict__ occ, DevCounters *ctr,
                                                          NbTile *__restrict__ tiles, uint2 *__restrict__ box_nbr,
                                                          uint32_t tmax, uint32_t K, bool mb,
                                                          uint32_t *__restrict__ mb_cen) {
    const uint32_t B = ctr->B;
    const uint32_t ntiles = (B + NB_THREADS - 1) / NB_THREADS;
    const uint64_t cap = item_costcap(ctr);
    unsigned long long pairs = 0;
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint32_t b = tile * NB_THREADS + threadIdx.x;
        const bool have = b < B;
        const uint32_t key = have ? bkey[b] : 0u;
        const uint32_t nb = have ? bstart[b + 1] - bstart[b] : 0u;
        const bool tgt = have && key >= g.tkey_lo && key <= g.tkey_hi;  // halo boxes: source only
        uint32_t cnt = 0, okm = 0;
        unsigned long long red = 0;
        NbStencil S;
        make_nb(g, key, S);
#pragma unroll
        unsigned long long part4 = 0, red0 = 0;
#pragma unroll
        for (int dz = 0; dz < 3; ++dz) {
            unsigned long long p4 = 0;
            nb_plane(S, dz, key, tgt, occ, boxinfo, okm, cnt, red, p4);
            if (dz == 0) red0 = red;
            if (dz == 1) part4 = p4;
        }
        BoxTotals x = box_totals(cnt, red, tgt ? nb : 0u, tgt, tmax, K, cap);
        const bool elig = mb_eligible(mb, tgt, x.item, nb, red, cap);
        // k_nbr_fill needs no occupancy search; the eligibility flag and (eligible boxes) the offset of the box's
        // own segment inside its run feed the quad items
        if (have) box_nbr[b] = make_uint2(okm | (elig ? MB_ELIG : 0u), (uint32_t)red);
        if (elig) mb_cen[b] = (uint32_t)(red0 + part4);
        pairs += (unsigned long long)(tgt ? nb : 0u) * red;
#ifndef P2P_NC_REDUCE
#define P2P_NC_REDUCE 1
#endif
#if P2P_NC_REDUCE
        const BoxTotals tot = block_sum_totals(x);
#else
        BoxTotals tot;
        block_scan_totals(x, &tot);
#endif
        if (threadIdx.x == 0) tiles[tile] = NbTile{{tot.nbr, tot.red, tot.item, tot.small, 0ull}};
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pairs += __shfl_xor_sync(0xffffffffu, pairs, o);
    if ((threadIdx.x & 31u) == 0 && pairs) atomicAdd(&ctr->I, pairs);
}

// the REDUNDANT list's item count per tile = work items - quad members (every eligible box has exactly one item)
__global__ void __launch_bounds__(NB_THREADS) k_mb_tiles(const uint32_t *__restrict__ bkey,
                                                         const uint2 *__restrict__ box_nbr, const DevCounters *ctr,
                                                         NbTile *__restrict__ tiles) {
    __shared__ uint32_t s_m[NB_THREADS / 32];
    const uint32_t B = ctr->B;
    const uint32_t ntiles = (B + NB_THREADS - 1) / NB_THREADS;
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint32_t b = tile * NB_THREADS + threadIdx.x;
        const bool member = b < B && (box_nbr[b].x & MB_ELIG) && mb_role(b, bkey[b], B, bkey, box_nbr) == 2;
        const uint32_t m = __popc(__ballot_sync(0xffffffffu, member));
        if ((threadIdx.x & 31u) == 0) s_m[threadIdx.x >> 5] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
#pragma unroll
            for (int i = 0; i < NB_THREADS / 32; ++i) t += s_m[i];
            tiles[tile].v[4] = tiles[tile].v[2] - t;
        }
        __syncthreads();
    }
}

// exclusive prefix of the per-256-box tile sums (k_nbr_count / k_mb_tiles) for k_nbr_fill: CTA c scans tiles
// 1024 c .. 1024 c + 1023 (in-chunk exclusive prefixes) and writes the chunk's total; the fill adds the totals of
// the earlier chunks (<= 11 on c5w).  The fill used to resolve its prefix itself by a look-back over the tile sums
// (ld.acquire + 3 barriers + a 5-value block reduction per tile): c5w fill 305 -> 237 us
constexpr int TS_THREADS = 1024;
__global__ void __launch_bounds__(TS_THREADS) k_tile_scan(const NbTile *__restrict__ sums, NbTile *__restrict__ excl,
                                                        NbTile *__restrict__ ctot, const DevCounters *ctr) {
    __shared__ unsigned long long s_w[TS_THREADS / 32][NB_TOT];
    const uint32_t ntiles = (ctr->B + NB_THREADS - 1) / NB_THREADS;
    const uint32_t t0 = blockIdx.x * TS_THREADS;
    if (t0 >= ntiles) return;
    const unsigned t = threadIdx.x, lane = t & 31u, w = t >> 5;
    const uint32_t q = t0 + t;
    unsigned long long v[NB_TOT], x[NB_TOT];
    const NbTile sv = q < ntiles ? sums[q] : NbTile{{0ull, 0ull, 0ull, 0ull, 0ull}};
#pragma unroll
    for (int k = 0; k < NB_TOT; ++k) {
        v[k] = sv.v[k];
        x[k] = v[k];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x[k], o);
            if (lane >= (unsigned)o) x[k] += y;
        }
        if (lane == 31) s_w[w][k] = x[k];
    }
    __syncthreads();
    if (w == 0) {  // warp 0: exclusive scan of the 32 warp totals (per value), the chunk total
#pragma unroll
        for (int k = 0; k < NB_TOT; ++k) {
            const unsigned long long y0 = s_w[lane][k];
            unsigned long long y = y0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long z = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= (unsigned)o) y += z;
            }
            if (lane == 31) ctot[blockIdx.x].v[k] = y;
            s_w[lane][k] = y - y0;
        }
    }
    __syncthreads();
    NbTile e;
#pragma unroll
    for (int k = 0; k < NB_TOT; ++k) e.v[k] = x[k] - v[k] + s_w[w][k];
    if (q < ntiles) excl[q] = e;
}

#ifndef P2P_HEADVEC
#define P2P_HEADVEC 1
#endif
#ifndef P2P_NB_SLOT4
#define P2P_NB_SLOT4 1
#endif
#ifndef P2P_NB_MINB
#define P2P_NB_MINB 3
#endif
#ifndef P2P_NB_CARVEOUT
#define P2P_NB_CARVEOUT 50
#endif
__global__ void __launch_bounds__(NB_THREADS, P2P_NB_MINB) k_nbr_fill(
    Geom g, const uint32_t *__restrict__ bkey, const uint32_t *__restrict__ bstart, const uint2 *__restrict__ boxinfo,
    const uint2 *__restrict__ box_nbr, DevCounters *ctr, const NbTile *__restrict__ incl,
    const NbTile *__restrict__ ctot, uint32_t *__restrict__ nbr_off, unsigned long long *__restrict__ red_off, uint32_t *__restrict__ nbr_box,
    uint8_t *__restrict__ nbr_slot, Item *__restrict__ items, uint32_t *__restrict__ small_tgt,
    uint32_t *__restrict__ small_box, uint32_t *__restrict__ chunk_box, unsigned long long *__restrict__ chunk_out,
    uint32_t K, uint32_t tmax, Item *__restrict__ items_red, const uint32_t *__restrict__ mb_cen) {
    __shared__ uint32_t s_box[NB_THREADS * NB_SLOTS];
    __shared__ uint8_t s_slot[NB_THREADS * NB_SLOTS];
    const uint32_t B = ctr->B;
    const uint32_t ntiles = (B + NB_THREADS - 1) / NB_THREADS;
    const uint64_t cap = item_costcap(ctr);
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint32_t b = tile * NB_THREADS + threadIdx.x;
        const bool have = b < B;
        const uint32_t key = have ? bkey[b] : 0u;
        const uint32_t s0 = have ? bstart[b] : 0u;
        const uint32_t nb = have ? bstart[b + 1] - s0 : 0u;
        const bool tgt = have && key >= g.tkey_lo && key <= g.tkey_hi;
        NbStencil S;
        make_nb(g, key, S);
        // the occupied-slot mask and record count found by k_nbr_count
        const uint2 bn = have ? box_nbr[b] : make_uint2(0u, 0u);
        const uint32_t okm = bn.x & ~MB_ELIG, cnt = __popc(okm);
        const unsigned long long red = bn.y;
        BoxTotals x = box_totals(cnt, red, tgt ? nb : 0u, tgt, tmax, K, cap);
        const int role = (items_red != nullptr && have) ? mb_role(b, key, B, bkey, box_nbr) : 0;
        const bool quad = role != 0;
        if (role == 2) x.item_red = 0u;
        BoxTotals tot;
        const BoxTotals inc = block_scan_totals(x, &tot);
        NbTile to = incl[tile];  // exclusive prefix inside the tile's chunk (k_tile_scan) + the earlier chunks
        for (uint32_t c = 0; c < tile / TS_THREADS; ++c) {
#pragma unroll
            for (int k = 0; k < NB_TOT; ++k) to.v[k] += ctot[c].v[k];
        }
        if (threadIdx.x == 0 && tile == ntiles - 1) {  // the last tile closes the offsets and publishes the totals
            const unsigned long long t0 = to.v[0] + tot.nbr, t1 = to.v[1] + tot.red;
            nbr_off[B] = (uint32_t)t0;
            red_off[B] = t1;
            ctr->n_nbr = (uint32_t)t0;
            ctr->R = t1;
            ctr->n_items = (uint32_t)(to.v[2] + tot.item);
            ctr->n_small = (uint32_t)(to.v[3] + tot.small);
            ctr->n_items_red = (uint32_t)(to.v[4] + tot.item_red);
        }
        const uint32_t e_loc = inc.nbr - x.nbr;  // block-relative CSR offset
        const uint32_t e0 = (uint32_t)to.v[0] + e_loc;
        const unsigned long long rb = to.v[1] + inc.red - x.red;
        const uint32_t it = (uint32_t)to.v[2] + inc.item - x.item;
        const uint32_t so = (uint32_t)to.v[3] + inc.small - x.small;
        const uint32_t itr = (uint32_t)to.v[4] + inc.item_red - x.item_red;
        if (have) {
            nbr_off[b] = e0;
            red_off[b] = rb;
        }
        // pass 2: CSR entries (staged), chunk heads; records before the centre slot = offset of the box's own
        // segment inside its run
        uint32_t e = e0, el = e_loc, recs = 0, cen = 0;
#pragma unroll
        for (int dz = 0; dz < 3; ++dz) {
            uint2 inf[9];
#pragma unroll
            for (int j = 0; j < 9; ++j) {
                const int sl = 9 * dz + j;
                inf[j] = boxinfo[((okm >> sl) & 1u) ? (S.c[0][j % 3] | S.c[1][j / 3] | S.c[2][dz]) : key];
            }
#pragma unroll
            for (int j = 0; j < 9; ++j) {
                const int sl = 9 * dz + j;
                if (sl == 13) cen = recs;
                if ((okm >> sl) & 1u) {
                    s_box[el] = inf[j].x;
                    s_slot[el] = (uint8_t)sl;
                    if ((e & 31u) == 0u) {  // head of a restructure chunk
                        chunk_box[e >> 5] = b;
                        chunk_out[e >> 5] = rb + recs;
                    }
                    ++e;
                    ++el;
                    recs += inf[j].y;
                }
            }
        }
        if (role == 1) {
            // the quad leader packs the 4 boxes' item data (members' from global: count finished):
            // q0 = {flag | nt_0..3 (4 bits each), t0 of box 0, R_0 | R_1 << 16, R_2 | R_3 << 16},
            // q1 = {red_base lo, hi, tofs_0 | tofs_1 << 16, tofs_2 | tofs_3 << 16}  (eval: k_eval_gravity.cu)
            uint32_t q_nt[4], q_R[4], q_tofs[4];
            q_nt[0] = nb;
            q_R[0] = (uint32_t)red;
            q_tofs[0] = cen;
#pragma unroll
            for (int j = 1; j < 4; ++j) {
                q_nt[j] = bstart[b + j + 1] - bstart[b + j];
                q_R[j] = box_nbr[b + j].y;
                q_tofs[j] = mb_cen[b + j];
            }
            Item mi;
            mi.box = 0x80000000u | q_nt[0] | (q_nt[1] << 4) | (q_nt[2] << 8) | (q_nt[3] << 12);
            mi.t0 = s0;
            mi.meta = q_R[0] | (q_R[1] << 16);
            mi.key = q_R[2] | (q_R[3] << 16);
            mi.red_base = rb;
            mi.R = q_tofs[0] | (q_tofs[1] << 16);
            mi.tofs = q_tofs[2] | (q_tofs[3] << 16);
            items_red[itr] = mi;
        }
        if (tgt) {
            if (x.item == 0) {  // small box: thread-per-target path, one entry per target pair
                for (uint32_t j = 0; j < x.small; ++j) {
                    small_tgt[so + j] = s0 + 2 * j;
                    small_box[so + j] = b;
                }
            } else {
                const uint32_t nch = x.item, sz = item_size(nb, red, tmax, K, cap);
                for (uint32_t ci = 0; ci < nch; ++ci) {
                    const uint32_t a0 = ci * sz, z0 = min(nb, (ci + 1) * sz);
                    // eval lane layout: G = ceil(n_t / K) groups of K targets, S = floor(32 / G) source splits
                    // K is a power of two; Gq <= 32 / K: 32 / Gq from a table (no integer divisions per item)
                    const uint32_t nt = z0 - a0, Gq = (nt + K - 1) >> (__ffs(K) - 1), Sq = c_div32[Gq];
                    // bit 24: the box belongs to a multi-box quad of the REDUNDANT list -- P2P_INDEXED_BITWISE then
                    // evaluates it with the quad's S = 4 splits, so its bits still equal the REDUNDANT eval's
                    const Item itm{b, s0 + a0, nt | (Sq << 8) | (Gq << 16) | (quad ? 1u << 24 : 0u), key, rb,
                                   (uint32_t)red, cen + a0};
                    items[it + ci] = itm;
                    if (items_red != nullptr && !quad) items_red[itr + ci] = itm;
                }
            }
        }
        __syncthreads();
        // coalesced copy of the tile's CSR run
        const uint32_t base = (uint32_t)to.v[0];
        for (uint32_t j = threadIdx.x; j < tot.nbr; j += NB_THREADS) nbr_box[base + j] = s_box[j];
#if P2P_NB_SLOT4
        {  // the slot bytes four at a time (32-bit stores from the first 4-byte boundary; byte stores at the ends)
            const uint32_t head = min(tot.nbr, (4u - (base & 3u)) & 3u);
            if (threadIdx.x < head) nbr_slot[base + threadIdx.x] = s_slot[threadIdx.x];
            const uint32_t nw = (tot.nbr - head) >> 2;
            uint32_t *dst = reinterpret_cast<uint32_t *>(nbr_slot + base + head);
            for (uint32_t q = threadIdx.x; q < nw; q += NB_THREADS) {
                const uint32_t j = head + 4 * q;
                dst[q] = (uint32_t)s_slot[j] | ((uint32_t)s_slot[j + 1] << 8) | ((uint32_t)s_slot[j + 2] << 16) |
                         ((uint32_t)s_slot[j + 3] << 24);
            }
            const uint32_t tail0 = head + 4 * nw;
            if (tail0 + threadIdx.x < tot.nbr) nbr_slot[base + tail0 + threadIdx.x] = s_slot[tail0 + threadIdx.x];
        }
#else
        for (uint32_t j = threadIdx.x; j < tot.nbr; j += NB_THREADS) nbr_slot[base + j] = s_slot[j];
#endif
        __syncthreads();
    }
}

__global__ void k_helm_check(const uint32_t *__restrict__ skey, uint32_t n, DevCounters *ctr) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x + 1; p < n; p += gridDim.x * blockDim.x)
        if (skey[p] == skey[p - 1]) atomicOr(&ctr->irregular, 1u);
}

__global__ void k_helm_nbr(const Geom g, uint32_t t, const uint32_t *__restrict__ bkey,
                           const uint32_t *__restrict__ bstart, const uint32_t *__restrict__ box_of,
                           DevCounters *ctr, uint32_t *__restrict__ nbr_off, uint32_t *__restrict__ nbr9,
                           uint8_t *__restrict__ nbr_slot) {
    const uint32_t B = ctr->B;
    uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long pairs = 0;
    if (b < B) {
        if (bstart[b + 1] - bstart[b] != t) atomicOr(&ctr->irregular, 1u);
        uint32_t key = bkey[b];
        int cx = (int)compact2(key), cy = (int)compact2(key >> 1);
        uint32_t present = 0;
        for (int s = 0; s < 9; ++s) {
            int nx = cx + s % 3 - 1, ny = cy + s / 3 - 1;
            uint32_t k = 0xffffffffu;
            if (nx >= 0 && nx < g.nbox[0] && ny >= 0 && ny < g.nbox[1]) {
                uint32_t nk = spread2((uint32_t)nx) | (spread2((uint32_t)ny) << 1);
                uint32_t kk = box_of[nk];
                if (kk < B && bkey[kk] == nk) k = kk;
            }
            nbr9[9 * (size_t)b + s] = k;
            nbr_slot[9 * (size_t)b + s] = (uint8_t)s;
            present += (k != 0xffffffffu);
        }
        nbr_off[b] = 9 * b;
        if (b == B - 1) nbr_off[B] = 9 * B;
        pairs = (unsigned long long)t * t * present;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pairs += __shfl_xor_sync(0xffffffffu, pairs, o);
    if ((threadIdx.x & 31u) == 0 && pairs) atomicAdd(&ctr->I, pairs);
}

static unsigned grid_for(uint64_t n, int threads, int num_sms) {
    uint64_t g = (n + threads - 1) / threads;
    uint64_t cap = (uint64_t)num_sms * 16;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, cap));
}

void free_capacity(p2p_plan *P) {
    cudaStream_t st = P->stream;
    void *bufs[] = {P->s_key, P->s_idx, P->s_kalt, P->s_valt, P->s_hist, P->s_status, P->s_partials,
                    P->s_nb_tiles, P->s_aos, P->s_box_nbr, P->boxinfo,
                    P->small_tgt, P->small_box, P->chunk_box, P->chunk_out, P->rec, P->bkey, P->bstart,
                    P->nbr_off, P->nbr_box, P->nbr_slot, P->red_off, P->box_of, P->items, P->items_red, P->s_mb_cen, P->occ};
    for (void *b : bufs) dfree(b, st);
    P->s_key = P->s_idx = P->s_kalt = P->s_valt = P->s_hist = P->s_status = nullptr;
    P->s_partials = nullptr;
    P->s_nb_tiles = nullptr;
    P->s_aos = nullptr;
    P->s_box_nbr = nullptr;
    P->boxinfo = nullptr;
    P->small_tgt = P->small_box = P->chunk_box = nullptr;
    P->chunk_out = nullptr;
    P->rec = nullptr;
    P->bkey = P->bstart = P->nbr_off = P->nbr_box = P->box_of = P->occ = nullptr;
    P->nbr_slot = nullptr;
    P->red_off = nullptr;
    P->items = P->items_red = nullptr;
    P->s_mb_cen = nullptr;
    P->skey = P->perm = nullptr;
    P->cap = P->bcap = 0;
}

// every buffer whose size depends on N (or on the box capacity min(N, key space)), allocated once
p2p_status alloc_capacity(p2p_plan *P, int64_t cap) {
    cudaStream_t st = P->stream;
    const bool grav = P->cfg.kernel == P2P_GRAVITY;
    const bool f64 = P->cfg.precision == P2P_FP64;
    const uint64_t n = (uint64_t)std::max<int64_t>(cap, 1);
    const uint64_t keyspace = grav ? (1ull << P->key_bits) : (1ull << (2 * P->nb));
    const uint64_t bcap = std::min<uint64_t>(n, keyspace);
    const int nslot = grav ? 27 : 9;
    P->cap = cap;
    P->bcap = (int64_t)bcap;
    P2P_CUDA_TRY(dalloc((void **)&P->s_key, 4 * n, st));
    P2P_CUDA_TRY(dalloc((void **)&P->s_idx, 4 * n, st));
    P2P_CUDA_TRY(dalloc((void **)&P->s_kalt, 4 * n, st));
    P2P_CUDA_TRY(dalloc((void **)&P->s_valt, 4 * n, st));
    P2P_CUDA_TRY(dalloc((void **)&P->s_hist, 4 * 4 * 256, st));
    P2P_CUDA_TRY(dalloc((void **)&P->s_status, 4 * std::max<size_t>(scan_lb_status_words(n),
                                                                    radix_status_words(n, std::max(1, P->passes))), st));
    P2P_CUDA_TRY(dalloc(&P->s_partials, scan_partials_bytes(std::max(n, bcap)), st));
    P2P_CUDA_TRY(dalloc((void **)&P->bkey, 4 * bcap, st));
    P2P_CUDA_TRY(dalloc((void **)&P->bstart, 4 * (bcap + 1), st));
    if (!grav) P2P_CUDA_TRY(dalloc((void **)&P->box_of, 4 * keyspace, st));
    P2P_CUDA_TRY(dalloc((void **)&P->occ, 4 * std::max<uint64_t>(1, keyspace / 32), st));
    P2P_CUDA_TRY(dalloc((void **)&P->nbr_off, 4 * (bcap + 1), st));
    P2P_CUDA_TRY(dalloc((void **)&P->nbr_box, 4 * nslot * bcap, st));
    P2P_CUDA_TRY(dalloc((void **)&P->nbr_slot, (size_t)nslot * bcap, st));
    if (grav) {
        P2P_CUDA_TRY(dalloc(&P->rec, (f64 ? sizeof(double4) : sizeof(float4)) * n, st));
        P2P_CUDA_TRY(dalloc(&P->s_aos, (f64 ? sizeof(double4) : sizeof(float4)) * n, st));
        P2P_CUDA_TRY(dalloc((void **)&P->s_box_nbr, sizeof(uint2) * bcap, st));
        const uint64_t ntc = div_up(bcap, NB_THREADS);  // tile sums, exclusive prefixes, per-1024-tile chunk totals
        P2P_CUDA_TRY(dalloc(&P->s_nb_tiles, sizeof(NbTile) * (2 * ntc + div_up(ntc, 1024) + 1), st));
        P2P_CUDA_TRY(dalloc((void **)&P->boxinfo, sizeof(uint2) * keyspace, st));
        // defined contents once per allocation: nb_plane's branch-free lookups load (and then mask) the entry of
        // keys whose occupancy bit is clear; entries are never cleared afterwards (stale ones are masked too)
        P2P_CUDA_TRY(cudaMemsetAsync(P->boxinfo, 0, sizeof(uint2) * keyspace, st));
        P2P_CUDA_TRY(dalloc((void **)&P->small_tgt, 4 * n, st));
        P2P_CUDA_TRY(dalloc((void **)&P->small_box, 4 * n, st));
        P2P_CUDA_TRY(dalloc((void **)&P->red_off, 8 * (bcap + 1), st));
        P2P_CUDA_TRY(dalloc((void **)&P->items, sizeof(Item) * n, st));
        // the REDUNDANT eval's own item list with multi-box quads (fp32 only: the eval's K = 4 lane layout)
        // (P2P_NO_MB=1 at plan creation: no quads, for the measurements in profiles/r02_eval_options.txt)
        const char *nomb = getenv("P2P_NO_MB");
        if (!f64 && EVAL_K_F32 == 4 && !(nomb && nomb[0] == '1')) {
            P2P_CUDA_TRY(dalloc((void **)&P->items_red, sizeof(Item) * n, st));
            P2P_CUDA_TRY(dalloc((void **)&P->s_mb_cen, 4 * bcap, st));
        }
        const uint64_t nchunk = div_up((uint64_t)nslot * bcap, 32) + 1;
        P2P_CUDA_TRY(dalloc((void **)&P->chunk_box, 4 * nchunk, st));
        P2P_CUDA_TRY(dalloc((void **)&P->chunk_out, 8 * nchunk, st));
    } else {
        P2P_CUDA_TRY(dalloc(&P->rec, (f64 ? sizeof(double2) : sizeof(float2)) * n, st));
    }
    return P2P_OK;
}

p2p_status build_gravity_structs(p2p_plan *P, const void *pos, const void *q, const void *rec_in, bool grid_a5) {
    cudaStream_t st = P->stream;
    const uint32_t n = (uint32_t)P->n;
    const bool f64 = P->cfg.precision == P2P_FP64;
    const unsigned gb = grid_for(n, 256, P->num_sms);
    // AoS record input (multi-GPU local plan): positions at stride 4, masses = the .w component
    const size_t tsz = f64 ? sizeof(double) : sizeof(float);
    const int ps = rec_in ? 4 : 3, qs = rec_in ? 4 : 1;
    if (rec_in) {
        pos = rec_in;
        q = (const char *)rec_in + 3 * tsz;
    }
    // a1 (+ the SoA input packed into records, unless the input already is records)
    void *aos = rec_in ? const_cast<void *>(rec_in) : P->s_aos;
    P2P_CUDA_TRY(cudaMemsetAsync(P->s_hist, 0, (size_t)4 * 256 * sizeof(uint32_t), st));
    if (f64)
        P2P_LAUNCH((k_bin_gravity<double, double4>), gb, 256, 0, st, (const double *)pos, ps, n, P->geom, P->s_key,
                   P->ctr, (const double *)q, rec_in ? (double4 *)nullptr : (double4 *)aos, P->passes, P->s_hist);
    else
        P2P_LAUNCH((k_bin_gravity<float, float4>), gb, 256, 0, st, (const float *)pos, ps, n, P->geom, P->s_key,
                   P->ctr, (const float *)q, rec_in ? (float4 *)nullptr : (float4 *)aos, P->passes, P->s_hist);
    // a2 (digit histograms from a1; first-pass values = input positions)
    P2P_CUDA_TRY(radix_sort_pairs(P->s_key, P->s_idx, P->s_kalt, P->s_valt, n, P->passes, P->ctr, P->s_hist,
                                  P->s_status, st, &P->skey, &P->perm, true, true));
    // a3
    if (f64)
        P2P_LAUNCH((k_permute_gravity<double4>), gb, 256, 0, st, (const double4 *)aos, P->perm, n, (double4 *)P->rec);
    else
        P2P_LAUNCH((k_permute_gravity<float4>), gb, 256, 0, st, (const float4 *)aos, P->perm, n, (float4 *)P->rec);
    // a4
    const uint64_t occ_words = std::max<uint64_t>(1, (1ull << P->key_bits) / 32);
    P2P_CUDA_TRY(cudaMemsetAsync(P->occ, 0, 4 * occ_words, st));
    // (a single-pass look-back variant, scan.cuh device_scan_lb, measured 124 vs 99 us on c5w: the 3052 tiles'
    // walks back over unpublished prefixes cost more than the second read of the keys)
#if P2P_HEADVEC
    if (n > 0) {
        const unsigned nblk = div_up(n, SC_TILE);
        uint32_t *parts = (uint32_t *)P->s_partials;
        P2P_LAUNCH(k_head_reduce, nblk, SC_THREADS, 0, st, P->skey, n, parts);
        P2P_LAUNCH((k_scan_partials<uint32_t>), 1, SC_THREADS, 0, st, parts, nblk, &P->ctr->B);
        P2P_LAUNCH(k_head_down, nblk, SC_THREADS, 0, st, P->skey, n, parts, P->bkey, P->bstart);
    } else {
        P2P_CUDA_TRY(cudaMemsetAsync(&P->ctr->B, 0, sizeof(unsigned int), st));
    }
#else
    P2P_CUDA_TRY(device_scan<uint32_t>(HeadGet1{P->skey},
                                       HeadPut{P->skey, 1u, P->bkey, P->bstart, nullptr, n}, nullptr, n,
                                       &P->ctr->B, P->s_partials, st));
#endif
    if (!grid_a5) return cudaGetLastError() == cudaSuccess ? P2P_OK : P2P_ERR_CUDA;  // adaptive mode: its own a5
    // a5
    const uint64_t bcap = (uint64_t)P->bcap;
    P2P_CUDA_TRY(cudaMemsetAsync(&P->ctr->sum_nb2, 0, sizeof(unsigned long long), st));
    P2P_LAUNCH(k_boxinfo, std::max<unsigned>(1, std::min<unsigned>(div_up(bcap, 256), (unsigned)P->num_sms * 8)), 256,
               0, st, P->bkey, P->bstart, P->ctr, P->boxinfo, P->occ, P->geom.tkey_lo, P->geom.tkey_hi);
    if (P->comm) {  // the cap's work estimate over ALL ranks' target boxes (= the 1-GPU value)
        p2p_status cs = P->comm->allreduce_sum_u64(&P->ctr->sum_nb2, 1, st);
        if (cs != P2P_OK) return cs;
    }
    const unsigned nbg = std::max<unsigned>(1, std::min<unsigned>(div_up(bcap, NB_THREADS), (unsigned)P->num_sms * 8));
    const uint64_t ntile_cap = div_up(bcap, NB_THREADS);
    NbTile *tiles = (NbTile *)P->s_nb_tiles;            // [ntile_cap] sums, then [ntile_cap] inclusive prefixes
    NbTile *incl = tiles + ntile_cap;  // exclusive tile prefixes (k_tile_scan)
    P2P_LAUNCH(k_nbr_count, nbg, NB_THREADS, 0, st, P->geom, P->bkey, P->bstart, P->boxinfo, P->occ, P->ctr, tiles,
               P->s_box_nbr, (uint32_t)ITEM_TMAX, (uint32_t)(f64 ? EVAL_K_F64 : EVAL_K_F32), P->items_red != nullptr,
               P->s_mb_cen);
    if (P->items_red)
        P2P_LAUNCH(k_mb_tiles, nbg, NB_THREADS, 0, st, P->bkey, P->s_box_nbr, P->ctr, tiles);
    static bool carveout_set = false;  // the fill keeps a large L1 (its pass-2 reloads must hit)
    if (!carveout_set && P2P_NB_CARVEOUT > 0) {
        P2P_CUDA_TRY(cudaFuncSetAttribute(k_nbr_fill, cudaFuncAttributePreferredSharedMemoryCarveout, P2P_NB_CARVEOUT));
        carveout_set = true;
    }
    NbTile *ctot = incl + ntile_cap;  // per 1024-tile chunk totals (fits the s_nb_tiles tail: 4 B per tile)
    P2P_LAUNCH(k_tile_scan, (unsigned)std::max<uint64_t>(1, div_up(ntile_cap, TS_THREADS)), TS_THREADS, 0, st, tiles,
               incl, ctot, P->ctr);
    P2P_LAUNCH(k_nbr_fill, nbg, NB_THREADS, 0, st, P->geom, P->bkey, P->bstart, P->boxinfo, P->s_box_nbr, P->ctr,
               incl, ctot, P->nbr_off, (unsigned long long *)P->red_off, P->nbr_box, P->nbr_slot, P->items,
               P->small_tgt, P->small_box, P->chunk_box, P->chunk_out, (uint32_t)(f64 ? EVAL_K_F64 : EVAL_K_F32),
               (uint32_t)ITEM_TMAX, P->items_red, P->s_mb_cen);
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}

template <typename T, typename V4>
__global__ void k_set_mass(const T *__restrict__ q, const uint32_t *__restrict__ perm, uint32_t n,
                           V4 *__restrict__ rec) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) rec[p].w = q[perm[p]];
}

p2p_status set_charges_gravity(p2p_plan *P, const void *q) {
    // masses are the .w field of the Morton-sorted records: re-gather them in sorted order
    cudaStream_t st = P->stream;
    const uint32_t n = (uint32_t)P->n;
    const unsigned gb = grid_for(n, 256, P->num_sms);
    if (P->cfg.precision == P2P_FP64)
        P2P_LAUNCH((k_set_mass<double, double4>), gb, 256, 0, st, (const double *)q, P->perm, n, (double4 *)P->rec);
    else
        P2P_LAUNCH((k_set_mass<float, float4>), gb, 256, 0, st, (const float *)q, P->perm, n, (float4 *)P->rec);
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}

p2p_status build_helmholtz_structs(p2p_plan *P, const void *pos, const void *q) {
    cudaStream_t st = P->stream;
    const uint32_t n = (uint32_t)P->n;
    const bool f64 = P->cfg.precision == P2P_FP64;
    const uint32_t t = (uint32_t)P->cfg.points_per_box;
    int stt = 0;
    while (stt * stt < (int)t) ++stt;
    const double delta = P->cfg.box_size / (double)stt;
    const unsigned gb = grid_for(n, 256, P->num_sms);
    if (f64)
        P2P_LAUNCH(k_bin_helmholtz<double>, gb, 256, 0, st, (const double *)pos, n, P->geom, stt, delta, t, P->s_key,
                   P->s_idx, P->ctr);
    else
        P2P_LAUNCH(k_bin_helmholtz<float>, gb, 256, 0, st, (const float *)pos, n, P->geom, stt, delta, t, P->s_key,
                   P->s_idx, P->ctr);
    P2P_CUDA_TRY(radix_sort_pairs(P->s_key, P->s_idx, P->s_kalt, P->s_valt, n, P->passes, P->ctr, P->s_hist,
                                  P->s_status, st, &P->skey, &P->perm));
    P2P_LAUNCH(k_helm_check, gb, 256, 0, st, P->skey, n, P->ctr);
    // a3: complex unknowns in sorted order
    if (f64)
        P2P_LAUNCH(k_permute_complex<double2>, gb, 256, 0, st, (const double2 *)q, P->perm, n, (double2 *)P->rec);
    else
        P2P_LAUNCH(k_permute_complex<float2>, gb, 256, 0, st, (const float2 *)q, P->perm, n, (float2 *)P->rec);
    // a4: boxes = runs of key / t
    P2P_CUDA_TRY(device_scan<uint32_t>(HeadGet{P->skey, t}, HeadPut{P->skey, t, P->bkey, P->bstart, P->box_of, n},
                                       nullptr, n, &P->ctr->B, P->s_partials, st));
    // a5: 9 slots per box
    P2P_LAUNCH(k_helm_nbr, div_up(P->bcap, 256), 256, 0, st, P->geom, t, P->bkey, P->bstart, P->box_of, P->ctr,
               P->nbr_off, P->nbr_box, P->nbr_slot);
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}

p2p_status set_charges_helmholtz(p2p_plan *P, const void *q) {
    cudaStream_t st = P->stream;
    const uint32_t n = (uint32_t)P->n;
    const unsigned gb = grid_for(n, 256, P->num_sms);
    if (P->cfg.precision == P2P_FP64)
        P2P_LAUNCH(k_permute_complex<double2>, gb, 256, 0, st, (const double2 *)q, P->perm, n, (double2 *)P->rec);
    else
        P2P_LAUNCH(k_permute_complex<float2>, gb, 256, 0, st, (const float2 *)q, P->perm, n, (float2 *)P->rec);
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}

}  // namespace p2p
