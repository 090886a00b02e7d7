// k_adaptive.cu -- SURVEY §8f NEXT-1 on the GPU: the adaptive binary-tree leaves (DESIGN C22), their closed
// neighbour lists (C23) and the redundant runs + REDUNDANT eval over them (C24), from a gravity plan's Morton-sorted
// box table and records.
//
// The paper's PhotoNs tree is "an irregular binary MLFMA tree" split by a clustering threshold t (P:L330,
// Fig 8).  Reading C22: longest-axis MIDPOINT splits of the periodic cube with ties z, y, x, i.e. a cell is a prefix
// of the finest-level Morton key (C7) of any length l; a cell is split while it holds more than t particles or while
// l < min_bits; finest cells are leaves whatever their count.  So the leaf of a finest box is its SHORTEST prefix
// l >= min_bits whose cell holds <= t particles (counts are non-increasing in l: a binary search over l, each count
// two binary searches over the box keys), and the leaves are the runs of consecutive boxes sharing (l, prefix):
// a head-flag scan (scan.cuh) numbers them in Morton order.  Every leaf is one contiguous run of the sorted records.
#include <vector>

#include "items.cuh"
#include "plan.hpp"
#include "restructure.cuh"
#include "scan.cuh"

namespace p2p {

// device-side sizes of the persistent (asynchronous) adaptive path: kernels read the leaf / entry counts from device
// memory (no host sync) and do nothing after a capacity overflow (null pointers: the synchronous entry points)
struct DevN {
    const uint32_t *L = nullptr, *E = nullptr, *ovf = nullptr;
    __device__ __forceinline__ bool stop() const { return ovf && *ovf; }
    __device__ __forceinline__ uint32_t l(uint32_t v) const { return L ? *L : v; }
    __device__ __forceinline__ uint32_t e(uint32_t v) const { return E ? *E : v; }
};

namespace {
// first box whose key is >= k (B boxes, ascending keys)
__device__ __forceinline__ uint32_t lower_bound_key(const uint32_t *__restrict__ bkey, uint32_t B, uint64_t k) {
    uint32_t lo = 0, hi = B;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if ((uint64_t)bkey[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// particles in the cell of the l-bit prefix of `key`
__device__ __forceinline__ uint32_t cell_count(const uint32_t *__restrict__ bkey, const uint32_t *__restrict__ bstart,
                                               uint32_t B, uint32_t key, int bits, int l) {
    const int s = bits - l;
    const uint64_t c0 = ((uint64_t)key >> s) << s, c1 = c0 + (1ull << s);
    return bstart[lower_bound_key(bkey, B, c1)] - bstart[lower_bound_key(bkey, B, c0)];
}

__global__ void k_leaf_len(const uint32_t *__restrict__ bkey, const uint32_t *__restrict__ bstart,
                           const DevCounters *__restrict__ ctr, int bits, uint32_t t, int min_bits,
                           uint8_t *__restrict__ len) {
    const uint32_t B = ctr->B;
    for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
        const uint32_t key = bkey[b];
        int lo = min_bits, hi = bits;  // the smallest l in [min_bits, bits] with count <= t; bits if none
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (cell_count(bkey, bstart, B, key, bits, mid) <= t) hi = mid;
            else lo = mid + 1;
        }
        len[b] = (uint8_t)lo;
    }
}

struct LeafHeadGet {
    const uint32_t *bkey;
    const uint8_t *len;
    int bits;
    __device__ uint32_t operator()(uint64_t p) const {
        if (p == 0) return 1u;
        const int l = len[p];
        return (l != len[p - 1] || (bkey[p] >> (bits - l)) != (bkey[p - 1] >> (bits - l))) ? 1u : 0u;
    }
};
struct LeafHeadPut {
    const uint32_t *bkey, *bstart;
    const uint8_t *len;
    int bits;
    uint32_t *leaf_len, *leaf_prefix, *leaf_start;
    __device__ void operator()(uint64_t p, uint32_t e, uint32_t v) const {
        if (v) {
            const int l = len[p];
            leaf_len[e] = (uint32_t)l;
            leaf_prefix[e] = (uint32_t)((uint64_t)bkey[p] >> (bits - l));
            leaf_start[e] = bstart[p];
        }
    }
};

// ---- C23 adjacency (dilation by the target leaf's extent + symmetric closure) ----
// dil(A) = the leaves of prefix length >= l_A inside A's 27 same-shape cells: per neighbour cell the contiguous range
// of the Morton-ordered leaf table whose cells start inside the cell's key range (minus a coarser leaf starting
// exactly at it).  With aligned cells the closed list of B is dil(B) u {(A, -S) : (B, S) in dil(A), l_A < l_B}: a
// coarser leaf overlapping D(B) contains one of B's 27 cells and so has B in its own dilation (the range
// construction of oracle/adaptive.py, pinned against the O(L^2) definition).  So: dilation counts (+ per target the
// number of transposed entries it receives), a scan, the dilation entries in order plus the transposed ones appended
// by atomic cursors, then per leaf a sort of the (few) transposed entries merged with the sorted dilation run:
// entries in (leaf, image code) order.  code = 9(s_z+1)+3(s_y+1)+(s_x+1), image +1 past the upper face (C5).
__device__ __forceinline__ void halvings_of(int l, uint32_t sh[3]) {
    sh[0] = (uint32_t)(l / 3);
    sh[1] = (uint32_t)((l + 1) / 3);
    sh[2] = (uint32_t)((l + 2) / 3);
}
// first finest key of the cell with coordinates c at halvings sh (m bits per dimension)
__device__ __forceinline__ uint32_t cell_key(const uint32_t c[3], const uint32_t sh[3], int m) {
    return spread3(c[0] << (m - sh[0])) | (spread3(c[1] << (m - sh[1])) << 1) | (spread3(c[2] << (m - sh[2])) << 2);
}
__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t *__restrict__ a, uint32_t n, uint32_t k) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
// neighbour cell of c (code), wrapped over 2^sh cells per dimension; returns the image code
__device__ __forceinline__ uint32_t nbr_cell(const uint32_t c[3], const uint32_t sh[3], int code, uint32_t out[3]) {
    const int dd[3] = {code % 3 - 1, (code / 3) % 3 - 1, code / 9 - 1};
    int img[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const int cells = 1 << sh[d];
        int v = (int)c[d] + dd[d];
        img[d] = v < 0 ? -1 : (v >= cells ? 1 : 0);
        out[d] = (uint32_t)(v - img[d] * cells);
    }
    return (uint32_t)(9 * (img[2] + 1) + 3 * (img[1] + 1) + (img[0] + 1));
}

// pass 1: thread per (leaf a, neighbour cell): the dilation range of the cell (two binary searches), its length
// added to a's count, one transposed entry counted for every finer leaf in it
__global__ void k_dil_ranges(const uint32_t *__restrict__ lkey, const uint32_t *__restrict__ llen, uint32_t L, int m,
                             uint2 *__restrict__ rng, uint8_t *__restrict__ rcode, unsigned int *__restrict__ dcnt,
                             unsigned int *__restrict__ tcnt, DevN dn = DevN()) {
    if (dn.stop()) return;
    L = dn.l(L);
    const int bits = 3 * m;
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < 27ull * L;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t a = (uint32_t)(x / 27), code = (uint32_t)(x - 27ull * a);
        const int la = (int)llen[a];
        uint32_t sh[3];
        halvings_of(la, sh);
        const uint32_t k0 = lkey[a];
        const uint32_t c[3] = {compact3(k0) >> (m - sh[0]), compact3(k0 >> 1) >> (m - sh[1]),
                               compact3(k0 >> 2) >> (m - sh[2])};
        uint32_t cc[3];
        const uint32_t ic = nbr_cell(c, sh, (int)code, cc);
        const uint32_t lo = cell_key(cc, sh, m);
        const uint64_t hi = (uint64_t)lo + (1ull << (bits - la));
        uint32_t i0 = lower_bound_u32(lkey, L, lo);
        const uint32_t i1 = hi > 0xffffffffull ? L : lower_bound_u32(lkey, L, (uint32_t)hi);
        if (i0 < i1 && (int)llen[i0] < la) ++i0;
        rng[x] = make_uint2(i0, i1);
        rcode[x] = (uint8_t)ic;
        if (i1 > i0) atomicAdd(&dcnt[a], i1 - i0);
        for (uint32_t i = i0; i < i1; ++i)
            if ((int)llen[i] > la) atomicAdd(&tcnt[i], 1u);
    }
}

// pass 2: warp per leaf, lane per neighbour cell: a range's output position is the total length of the ranges that
// start before it (the ranges are disjoint), so the dilation entries land in (leaf) order without sorting; the
// transposed entries are appended to the finer leaves' lists (atomic cursors)
__global__ void k_dil_fill(const uint32_t *__restrict__ llen, uint32_t L, const uint2 *__restrict__ rng,
                           const uint8_t *__restrict__ rcode, const uint32_t *__restrict__ off,
                           const unsigned int *__restrict__ dcnt, unsigned int *__restrict__ tcur,
                           uint32_t *__restrict__ nbr, uint8_t *__restrict__ code, DevN dn = DevN()) {
    if (dn.stop()) return;
    L = dn.l(L);
    constexpr unsigned FULL = 0xffffffffu;
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < L; a += nw) {
        uint32_t i0 = 0, i1 = 0, c = 0;
        if (lane < 27) {
            const uint2 v = rng[27ull * a + lane];
            i0 = v.x;
            i1 = v.y;
            c = rcode[27ull * a + lane];
        }
        const uint32_t n = i1 - i0;
        uint32_t pos = 0;
        for (int q = 0; q < 27; ++q) {
            const uint32_t sq = __shfl_sync(FULL, i0, q), nq = __shfl_sync(FULL, n, q);
            if (sq < i0) pos += nq;
        }
        const uint32_t la = llen[a];
        uint32_t o = off[a] + pos;
        for (uint32_t i = i0; i < i1; ++i) {
            nbr[o] = i;
            code[o++] = (uint8_t)c;
            if (llen[i] > la) {
                const uint32_t slot = off[i] + dcnt[i] + atomicAdd(&tcur[i], 1u);
                nbr[slot] = a;
                code[slot] = (uint8_t)(26u - c);
            }
        }
    }
}

// pass 3: warp per leaf: the transposed tail (coarser leaves, distinct from the dilation's) merged into the sorted
// dilation run -- every entry's final position is its rank among the tail plus its rank among the dilation run
__global__ void k_dil_merge(const uint32_t *__restrict__ off, const unsigned int *__restrict__ dcnt, uint32_t L,
                            const uint32_t *__restrict__ nbr, const uint8_t *__restrict__ code,
                            uint32_t *__restrict__ nbr_out, uint8_t *__restrict__ code_out, DevN dn = DevN()) {
    if (dn.stop()) return;
    L = dn.l(L);
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t a = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < L; a += nw) {
        const uint32_t o = off[a], d = dcnt[a], e = off[a + 1], T = e - o - d;
        for (uint32_t t = lane; t < T; t += 32) {
            const uint32_t tv = nbr[o + d + t];
            uint32_t rank = 0;  // tail entries below tv
            for (uint32_t k = 0; k < T; ++k) rank += nbr[o + d + k] < tv ? 1u : 0u;
            uint32_t lo = 0, hi = d;  // dilation entries below tv
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (nbr[o + mid] < tv) lo = mid + 1;
                else hi = mid;
            }
            nbr_out[o + rank + lo] = tv;
            code_out[o + rank + lo] = code[o + d + t];
        }
        for (uint32_t i = lane; i < d; i += 32) {
            const uint32_t v = nbr[o + i];
            uint32_t below = 0;  // tail entries below v
            for (uint32_t k = 0; k < T; ++k) below += nbr[o + d + k] < v ? 1u : 0u;
            nbr_out[o + i + below] = v;
            code_out[o + i + below] = code[o + i];
        }
    }
}

// ---- C24: per target leaf, its run length, the offset of its own (self, image 0) segment, its work items ----
__global__ void k_adapt_count(const uint32_t *__restrict__ off, const uint32_t *__restrict__ nbr,
                              const uint8_t *__restrict__ code, const uint32_t *__restrict__ lstart, uint32_t L,
                              unsigned long long *__restrict__ R, uint32_t *__restrict__ tself, DevN dn,
                              unsigned long long *__restrict__ pairs, uint32_t *__restrict__ ch_leaf = nullptr,
                              unsigned long long *__restrict__ ch_rel = nullptr) {
    if (dn.stop()) return;
    L = dn.l(L);
    unsigned long long ip = 0;
    for (uint32_t a = blockIdx.x * blockDim.x + threadIdx.x; a < L; a += gridDim.x * blockDim.x) {
        unsigned long long sum = 0, ts = 0;
        for (uint32_t e = off[a]; e < off[a + 1]; ++e) {
            const uint32_t b = nbr[e];
            if ((e & 31u) == 0u) {  // head of restructure chunk e / 32: its owner leaf and offset inside the run
                ch_leaf[e >> 5] = a;
                ch_rel[e >> 5] = sum;
            }
            if (b == a && code[e] == 13) ts = sum;
            sum += lstart[b + 1] - lstart[b];
        }
        R[a] = sum;
        tself[a] = (uint32_t)ts;
        ip += sum * (lstart[a + 1] - lstart[a]);
    }
    {  // I = sum over leaves of n_targets x run length (the pair count of the step; it sizes the work items)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ip += __shfl_xor_sync(0xffffffffu, ip, o);
        if ((threadIdx.x & 31u) == 0 && ip) atomicAdd(pairs, ip);
    }
}

// Multi-leaf quad items of the REDUNDANT eval (fp32): the grid path's multi-box quads (k_structs.cu mb_role) over
// leaves.  The 4 leaves of an aligned leaf-index block 4q .. 4q + 3 that each hold 1 .. 8 targets and <= 65535 run
// records become ONE work item: leaf j owns lanes 8j .. 8j + 7 (2 groups of 4 targets x 4 source splits) and the 4
// runs -- adjacent in red[], like their targets in the sorted records -- are staged in lockstep, so the per-item
// cost (fetch, staging, transpose-reduce, epilogue) is paid once per 4 small leaves.  Leaves are Morton-ordered: a
// block is 4 neighbouring cells; adaptive mode is single-GPU, no rank boundary constrains the blocks.
constexpr uint32_t AQ_NT = 8, AQ_R = 65535;
// the leaf's work items: ITEM_TMAX targets each, fewer when n_t x R exceeds the work-scaled cost cap (items.cuh,
// the grid path's rule with the exact pair count I)
__device__ __forceinline__ uint32_t adapt_nitems(uint32_t nt, uint64_t R, uint32_t K, uint64_t cap) {
    const uint32_t sz = item_size(nt, R, ITEM_TMAX, K, cap);
    return (nt + sz - 1) / sz;
}
// a quad member: one item, <= 8 targets, a 16-bit run, and cost <= cap / 4 (a quad item -- 8 lanes per leaf -- then
// takes no longer than a capped single-leaf item: k_structs.cu mb_eligible)
__device__ __forceinline__ bool aq_elig(const uint32_t *__restrict__ lstart, const unsigned long long *__restrict__ R,
                                        uint32_t a, uint32_t K, uint64_t cap) {
    const uint32_t nt = lstart[a + 1] - lstart[a];
    const uint64_t r = R[a];
    return nt >= 1u && nt <= AQ_NT && r <= AQ_R && (uint64_t)nt * r * 4 <= cap && adapt_nitems(nt, r, K, cap) == 1u;
}
// 0: no quad, 1: leader (a % 4 == 0), 2: member
__device__ __forceinline__ int aq_role(const uint32_t *__restrict__ lstart, const unsigned long long *__restrict__ R,
                                       uint32_t a, uint32_t L, uint32_t K, uint64_t cap) {
    const uint32_t q = a & ~3u;
    if (q + 3u >= L) return 0;
#pragma unroll
    for (uint32_t i = 0; i < 4; ++i)
        if (!aq_elig(lstart, R, q + i, K, cap)) return 0;
    return a == q ? 1 : 2;
}
// the cost cap from the device pair count; I == nullptr: uncapped (ITEM_TMAX-target items)
__device__ __forceinline__ uint64_t adapt_cap(const unsigned long long *I) { return I ? item_costcap_of(*I) : ~0ull; }
// per leaf: its work items (INDEXED list) / its items in the REDUNDANT list (quad leader 1, member 0, else its own);
// L and the pair count I from the device
struct ItemCntGet {
    const uint32_t *lstart;
    const unsigned long long *R, *I;
    uint32_t K;
    __device__ uint32_t operator()(uint64_t p) const {
        const uint32_t a = (uint32_t)p;
        return adapt_nitems(lstart[a + 1] - lstart[a], R[a], K, adapt_cap(I));
    }
};
struct RedCntGet {
    const uint32_t *lstart;
    const unsigned long long *R, *I;
    const uint32_t *Lp;
    uint32_t Lh, K;
    bool quads;
    __device__ uint32_t operator()(uint64_t p) const {
        const uint32_t a = (uint32_t)p;
        const uint64_t cap = adapt_cap(I);
        const int role = quads ? aq_role(lstart, R, a, Lp ? *Lp : Lh, K, cap) : 0;
        return role == 0 ? adapt_nitems(lstart[a + 1] - lstart[a], R[a], K, cap) : (role == 1 ? 1u : 0u);
    }
};

// eval work items of every leaf: full ITEM_TMAX-target items + a remainder (the eval's lane layout, K targets per
// lane: G = ceil(n_t / K) groups x S = floor(32 / G) source splits); targets staged from the self segment.
// items_red (optional): the REDUNDANT list at ioff_red -- a quad leader's multi-leaf item (packed like the grid's:
// k_structs.cu k_nbr_fill), nothing for a member, the leaf's own items otherwise
__global__ void k_adapt_items(const uint32_t *__restrict__ lstart, const unsigned long long *__restrict__ red_off,
                              const unsigned long long *__restrict__ R, const uint32_t *__restrict__ tself,
                              const uint32_t *__restrict__ item_off, uint32_t L, uint32_t K,
                              const unsigned long long *__restrict__ I_idx, Item *__restrict__ items, DevN dn = DevN(),
                              Item *__restrict__ items_red = nullptr, const uint32_t *__restrict__ ioff_red = nullptr,
                              const unsigned long long *__restrict__ I_red = nullptr, bool quads = false) {
    if (dn.stop()) return;
    L = dn.l(L);
    const uint64_t cap_i = adapt_cap(I_idx), cap_r = adapt_cap(I_red);
    for (uint32_t a = blockIdx.x * blockDim.x + threadIdx.x; a < L; a += gridDim.x * blockDim.x) {
        const uint32_t nt_all = lstart[a + 1] - lstart[a];
        for (int list = 0; list < (items_red ? 2 : 1); ++list) {
            const uint64_t cap = list ? cap_r : cap_i;
            if (list && quads && aq_role(lstart, R, a, L, K, cap) != 0) continue;  // written by the quad's leader
            const uint32_t sz = item_size(nt_all, R[a], ITEM_TMAX, K, cap);
            uint32_t it = list ? ioff_red[a] : item_off[a];
            for (uint32_t a0 = 0; a0 < nt_all; a0 += sz, ++it) {
                const uint32_t nt = min(sz, nt_all - a0), G = (nt + K - 1) / K, S = 32u / G;
                (list ? items_red : items)[it] = Item{a, lstart[a] + a0, nt | (S << 8) | (G << 16), 0u, red_off[a],
                                                      (uint32_t)R[a], tself[a] + a0};
            }
        }
        const int role = (items_red && quads) ? aq_role(lstart, R, a, L, K, cap_r) : 0;
        if (role == 1) {
            uint32_t q_nt[4], q_R[4], q_tofs[4];
#pragma unroll
            for (uint32_t j = 0; j < 4; ++j) {
                q_nt[j] = lstart[a + j + 1] - lstart[a + j];
                q_R[j] = (uint32_t)R[a + j];
                q_tofs[j] = tself[a + j];
            }
            Item mi;
            mi.box = 0x80000000u | q_nt[0] | (q_nt[1] << 4) | (q_nt[2] << 8) | (q_nt[3] << 12);
            mi.t0 = lstart[a];
            mi.meta = q_R[0] | (q_R[1] << 16);
            mi.key = q_R[2] | (q_R[3] << 16);
            mi.red_base = red_off[a];
            mi.R = q_tofs[0] | (q_tofs[1] << 16);
            mi.tofs = q_tofs[2] | (q_tofs[3] << 16);
            items_red[ioff_red[a]] = mi;
        }
    }
}

// Item sizes per layout, each its measured best (profiles/r02_adaptive_items.txt, c3): the REDUNDANT list is
// cost-capped like the grid's (items.cuh: the dynamic queue's tail; t = 4 / 16 / 64: -5% / -7% / -1.5% eval), the
// INDEXED list is not (its per-item CSR setup makes smaller items cost more: +6% / +7% / 0).  P2P_ADAPT_CAP=0:
// REDUNDANT uncapped too.
static bool adapt_capped() {
    const char *e = getenv("P2P_ADAPT_CAP");
    return !(e && e[0] == '0');
}
// multi-leaf quads: OPT-IN (P2P_ADAPT_QUADS=1), fp32 only.  Measured on c3 (profiles/r02_adaptive_items.txt): on
// the adaptive leaves they do not pay -- t = 4: +7% REDUNDANT eval (most quad leaves hold <= 4 targets, so half of
// every leaf's 8 lanes idle), t = 16 / 64: within noise -- unlike the grid's 8-per-box c4-8
static bool adapt_quads(const p2p_plan *P) {
    const char *e = getenv("P2P_ADAPT_QUADS");
    return P->cfg.precision != P2P_FP64 && e && e[0] == '1';
}

// the redundant runs (C24): each target leaf's entries' source runs in CSR order, rebased in fp64 to the target
// leaf's origin o_d = fma(c_d, w_d, lo_d) (w_d = L / 2^s_d) with the entry's image shift, one final rounding:
//     red = { fl_p(((double)x_j + S_d) - o_d), .., m_j },  S_d = (image digit d - 1) L   (C24, P:L197 + C11)
// Warp per CHUNK of 32 consecutive CSR entries (the grid restructure's scheme, restructure.cuh): a chunk's segments
// are one contiguous output range starting at roff[owner of its first entry] + ch_rel (both recorded by
// k_adapt_count: no entry-offset scan, no owner search), its <= 32 entries belong to <= 32 consecutive leaves (every
// leaf lists itself).  The chunk's level-1 values are loaded one chunk ahead; lanes copy windows of 32 records,
// UNR windows with all loads in flight before the first store, each lane finding its segment by ballot / OR-reduce
// over the segment starts; streaming stores (the runs are read back by the next kernel only).
// EXACT32 (host-checked: every cell origin of the 2^m lattice is an fp32 value, so every leaf origin -- a lattice
// cell origin -- is too): chunks without an image shift take the fp32 subtraction, which rounds like the fp64
// sequence (restructure.cuh).
template <typename T, typename V4, bool EXACT32>
__global__ void __launch_bounds__(256) k_adapt_restructure_chunks(
    const V4 *__restrict__ rec, const uint32_t *__restrict__ lkey, const uint32_t *__restrict__ len,
    const uint32_t *__restrict__ lstart, const uint32_t *__restrict__ off, const uint32_t *__restrict__ nbr,
    const uint8_t *__restrict__ code, const uint32_t *__restrict__ ch_leaf,
    const unsigned long long *__restrict__ ch_rel, const unsigned long long *__restrict__ roff, uint32_t L, uint32_t E,
    int m, double Lbox, double lo0, double lo1, double lo2, V4 *__restrict__ red, DevN dn = DevN()) {
    if (dn.stop()) return;
    L = dn.l(L);
    E = dn.e(E);
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int UNR = 4;
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5, nchunk = (E + 31u) >> 5;
    uint32_t n_o0 = 0, n_b = 0, n_cd = 13;
    unsigned long long n_rel = 0;
    auto load1 = [&](uint32_t c) {
        if (c < nchunk) {
            n_o0 = ch_leaf[c];
            n_rel = ch_rel[c];
            const uint32_t ee = (c << 5) + lane;
            if (ee < E) {
                n_b = nbr[ee];
                n_cd = code[ee];
            }
        }
    };
    uint32_t ch = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    load1(ch);
    for (; ch < nchunk; ch += nw) {
        const uint32_t o0 = n_o0, b = n_b, cd = n_cd;
        const unsigned long long rel = n_rel;
        load1(ch + nw);
        const uint32_t e = (ch << 5) + lane;
        const bool seg = e < E;
        uint32_t src = 0, cnt = 0;
        if (seg) {
            src = lstart[b];
            cnt = lstart[b + 1] - src;
        }
        const uint32_t ol = o0 + lane;
        uint32_t boff = FULL, keyl = 0, lenl = 0;
        if (ol < L) {
            boff = off[ol];
            keyl = lkey[ol];
            lenl = len[ol];
        }
        V4 *__restrict__ out = red + (roff[o0] + rel);
        // owner of entry e: the largest i with off[o0 + i] <= e
        uint32_t i = 0;
#pragma unroll
        for (uint32_t step = 16; step > 0; step >>= 1) {
            const uint32_t t = __shfl_sync(FULL, boff, i + step);
            if (t <= e) i += step;
        }
        const uint32_t k0 = __shfl_sync(FULL, keyl, i), ln = __shfl_sync(FULL, lenl, i);
        uint32_t sh[3];
        halvings_of((int)ln, sh);
        const double o0d = __fma_rn((double)(compact3(k0) >> (m - sh[0])), ldexp(Lbox, -(int)sh[0]), lo0);
        const double o1d = __fma_rn((double)(compact3(k0 >> 1) >> (m - sh[1])), ldexp(Lbox, -(int)sh[1]), lo1);
        const double o2d = __fma_rn((double)(compact3(k0 >> 2) >> (m - sh[2])), ldexp(Lbox, -(int)sh[2]), lo2);
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= (unsigned)o) incl += y;
        }
        const uint32_t st = incl - cnt, Rc = __shfl_sync(FULL, incl, 31);
        const uint32_t le = lane == 31 ? FULL : ((2u << lane) - 1u);
        const bool wrap = __any_sync(FULL, seg && cd != 13u);
        const bool fast32 = EXACT32 && !wrap;
        const float f0o = (float)o0d, f1o = (float)o1d, f2o = (float)o2d;
        for (uint32_t rb = 0; rb < Rc; rb += 32 * UNR) {
            V4 x[UNR];
            uint32_t xe[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const uint32_t r0 = rb + 32u * u;
                if (r0 >= Rc) break;  // warp-uniform
                // segment of record r0 + lane: segments starting before r0 - 1 + segment starts in [r0, r0 + lane]
                const uint32_t before = __popc(__ballot_sync(FULL, seg && st < r0));
                const uint32_t in_win = (seg && st >= r0 && st < r0 + 32) ? (1u << (st - r0)) : 0u;
                const uint32_t starts = __reduce_or_sync(FULL, in_win);
                xe[u] = (before - 1u + __popc(starts & le)) & 31u;
                const uint32_t e_src = __shfl_sync(FULL, src, xe[u]), e_st = __shfl_sync(FULL, st, xe[u]);
                const uint32_t r = r0 + lane;
                if (r < Rc) x[u] = rec[e_src + (r - e_st)];
            }
            if (fast32) {
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const uint32_t r0 = rb + 32u * u;
                    if (r0 >= Rc) break;
                    const float eo0 = __shfl_sync(FULL, f0o, xe[u]), eo1 = __shfl_sync(FULL, f1o, xe[u]),
                                eo2 = __shfl_sync(FULL, f2o, xe[u]);
                    const uint32_t r = r0 + lane;
                    if (r < Rc) {
                        V4 v;
                        v.x = (T)__fsub_rn(__fadd_rn((float)x[u].x, 0.0f), eo0);
                        v.y = (T)__fsub_rn(__fadd_rn((float)x[u].y, 0.0f), eo1);
                        v.z = (T)__fsub_rn(__fadd_rn((float)x[u].z, 0.0f), eo2);
                        v.w = x[u].w;
                        rs::st_cs(out + r, v);
                    }
                }
                continue;
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const uint32_t r0 = rb + 32u * u;
                if (r0 >= Rc) break;
                const uint32_t e_cd = __shfl_sync(FULL, cd, xe[u]);
                const double eo0 = __shfl_sync(FULL, o0d, xe[u]), eo1 = __shfl_sync(FULL, o1d, xe[u]),
                             eo2 = __shfl_sync(FULL, o2d, xe[u]);
                const uint32_t r = r0 + lane;
                if (r < Rc) {
                    const double S0 = (double)((int)(e_cd % 3) - 1) * Lbox,
                                 S1 = (double)((int)((e_cd / 3) % 3) - 1) * Lbox,
                                 S2 = (double)((int)(e_cd / 9) - 1) * Lbox;
                    V4 v;
                    v.x = (T)__dsub_rn(__dadd_rn((double)x[u].x, S0), eo0);
                    v.y = (T)__dsub_rn(__dadd_rn((double)x[u].y, S1), eo1);
                    v.z = (T)__dsub_rn(__dadd_rn((double)x[u].z, S2), eo2);
                    v.w = x[u].w;
                    rs::st_cs(out + r, v);
                }
            }
        }
    }
}


// INDEXED over the leaves: per leaf, bit d = its cell touches the upper face of dim d (frame -L), bit 3 + d the lower
__global__ void k_leaf_frame(const uint32_t *__restrict__ lkey, const uint32_t *__restrict__ len, uint32_t L, int m,
                             uint8_t *__restrict__ fr, DevN dn = DevN()) {
    if (dn.stop()) return;
    L = dn.l(L);
    for (uint32_t a = blockIdx.x * blockDim.x + threadIdx.x; a < L; a += gridDim.x * blockDim.x) {
        uint32_t sh[3];
        halvings_of((int)len[a], sh);
        const uint32_t k0 = lkey[a];
        uint32_t f = 0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const uint32_t c = compact3(k0 >> d) >> (m - sh[d]);
            if (c == (1u << sh[d]) - 1u) f |= 1u << d;
            if (c == 0u) f |= 8u << d;
        }
        fr[a] = (uint8_t)f;
    }
}

// every cell origin fma(c, L 2^-m, lo_d), c < 2^m, of the leaves' lattice is an fp32 value -- then so is every
// leaf origin fma(c_l, L 2^-s, lo_d): the same real number as the origin of the leaf's first cell, one rounding
static bool adapt_origins_exact_fp32(const Geom &G, int m) {
    const double w = std::ldexp(G.L[0], -m);
    for (int d = 0; d < 3; ++d)
        for (int c = 0; c < (1 << m); ++c) {
            const double o = std::fma((double)c, w, G.lo[d]);
            if ((double)(float)o != o) return false;
        }
    return true;
}

// a6 over the leaves: the chunk kernel in the plan's precision (EXACT32 when the lattice allows it)
static p2p_status launch_adapt_runs(p2p_plan *P, const uint32_t *lkey, const uint32_t *len, const uint32_t *lstart,
                                    const uint32_t *off, const uint32_t *nbr, const uint8_t *code,
                                    const uint32_t *ch_leaf, const unsigned long long *ch_rel,
                                    const unsigned long long *roff, uint32_t L, uint32_t E, uint64_t egrid, void *red,
                                    DevN dn) {
    const int m = P->key_bits / 3;
    const Geom &G = P->geom;
    cudaStream_t st = P->stream;
    unsigned gw = std::max<unsigned>(1, std::min<unsigned>(div_up(egrid, 256), (unsigned)P->num_sms * 16));
    // P2P_RS_MAXGRID=<blocks> (tests): fewer warps than chunks, so that every warp walks several chunks
    if (const char *e = getenv("P2P_RS_MAXGRID")) gw = std::max(1u, std::min(gw, (unsigned)atoi(e)));
    if (P->cfg.precision == P2P_FP64)
        P2P_LAUNCH((k_adapt_restructure_chunks<double, double4, false>), gw, 256, 0, st, (const double4 *)P->rec, lkey,
                   len, lstart, off, nbr, code, ch_leaf, ch_rel, roff, L, E, m, G.L[0], G.lo[0], G.lo[1], G.lo[2],
                   (double4 *)red, dn);
    else if (adapt_origins_exact_fp32(G, m))
        P2P_LAUNCH((k_adapt_restructure_chunks<float, float4, true>), gw, 256, 0, st, (const float4 *)P->rec, lkey,
                   len, lstart, off, nbr, code, ch_leaf, ch_rel, roff, L, E, m, G.L[0], G.lo[0], G.lo[1], G.lo[2],
                   (float4 *)red, dn);
    else
        P2P_LAUNCH((k_adapt_restructure_chunks<float, float4, false>), gw, 256, 0, st, (const float4 *)P->rec, lkey,
                   len, lstart, off, nbr, code, ch_leaf, ch_rel, roff, L, E, m, G.L[0], G.lo[0], G.lo[1], G.lo[2],
                   (float4 *)red, dn);
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}

struct U64Get {
    const unsigned long long *v;
    __device__ unsigned long long operator()(uint64_t p) const { return v[p]; }
};
struct U64Put {
    unsigned long long *off;
    __device__ void operator()(uint64_t p, unsigned long long e, unsigned long long) const { off[p] = e; }
};

struct SumGet {
    const unsigned int *a;
    const unsigned int *b;
    __device__ uint32_t operator()(uint64_t p) const { return a[p] + b[p]; }
};
struct CntGet {
    const uint32_t *cnt;
    __device__ uint32_t operator()(uint64_t p) const { return cnt[p]; }
};
struct OffPut {
    uint32_t *off;
    __device__ void operator()(uint64_t p, uint32_t e, uint32_t) const { off[p] = e; }
};
__global__ void k_leaf_keys(const uint32_t *__restrict__ len, const uint32_t *__restrict__ prefix, uint32_t L,
                            int bits, uint32_t *__restrict__ lkey, DevN dn = DevN()) {
    L = dn.l(L);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < L; i += gridDim.x * blockDim.x)
        lkey[i] = (uint32_t)((uint64_t)prefix[i] << (bits - (int)len[i]));
}
}  // namespace

p2p_status adaptive_leaves(p2p_plan *P, uint32_t t, int min_bits, uint32_t *len_h, uint32_t *prefix_h,
                           uint32_t *start_h, int64_t cap, int64_t *n_leaves) {
    cudaStream_t st = P->stream;
    const uint32_t B = (uint32_t)P->B;
    const int bits = P->key_bits;
    if (min_bits > bits) min_bits = bits;
    *n_leaves = 0;
    if (B == 0) return P2P_OK;
    uint8_t *len = nullptr;
    uint32_t *out = nullptr, *cnt = nullptr;
    P2P_CUDA_TRY(dalloc((void **)&len, B, st));
    P2P_CUDA_TRY(dalloc((void **)&out, 4 * 3 * (size_t)B, st));
    P2P_CUDA_TRY(dalloc((void **)&cnt, 4, st));
    P2P_LAUNCH(k_leaf_len, std::max<unsigned>(1, std::min<unsigned>(div_up(B, 256), (unsigned)P->num_sms * 8)), 256, 0,
               st, P->bkey, P->bstart, P->ctr, bits, t, min_bits, len);
    P2P_CUDA_TRY(device_scan<uint32_t>(LeafHeadGet{P->bkey, len, bits},
                                       LeafHeadPut{P->bkey, P->bstart, len, bits, out, out + B, out + 2 * (size_t)B},
                                       &P->ctr->B, B, cnt, P->s_partials, st));
    uint32_t L = 0;
    P2P_CUDA_TRY(cudaMemcpyAsync(&L, cnt, 4, cudaMemcpyDeviceToHost, st));
    P2P_CUDA_TRY(cudaStreamSynchronize(st));
    if ((int64_t)L > cap) {
        dfree(len, st);
        dfree(out, st);
        dfree(cnt, st);
        set_error("output capacity below the leaf count");
        return P2P_ERR_INVALID_ARGUMENT;
    }
    P2P_CUDA_TRY(cudaMemcpyAsync(len_h, out, 4 * (size_t)L, cudaMemcpyDeviceToHost, st));
    P2P_CUDA_TRY(cudaMemcpyAsync(prefix_h, out + B, 4 * (size_t)L, cudaMemcpyDeviceToHost, st));
    P2P_CUDA_TRY(cudaMemcpyAsync(start_h, out + 2 * (size_t)B, 4 * (size_t)L, cudaMemcpyDeviceToHost, st));
    P2P_CUDA_TRY(cudaStreamSynchronize(st));
    dfree(len, st);
    dfree(out, st);
    dfree(cnt, st);
    *n_leaves = L;
    return P2P_OK;
}

}  // namespace p2p

namespace p2p {

// ---- the device-side adaptive structures: leaves (C22) + closed neighbour CSR (C23) ----
struct AdaptiveDev {
    int64_t L = 0, E = 0;
    uint32_t *len = nullptr, *lkey = nullptr, *lstart = nullptr, *off = nullptr, *nbr = nullptr;
    uint8_t *code = nullptr;
    void release(cudaStream_t st) {
        void *bufs[] = {len, lkey, lstart, off, nbr, code};
        for (void *p : bufs) dfree(p, st);
        len = lkey = lstart = off = nbr = nullptr;
        code = nullptr;
    }
};

static p2p_status build_adaptive(p2p_plan *P, uint32_t t, int min_bits, AdaptiveDev &A) {
    cudaStream_t st = P->stream;
    const int bits = P->key_bits, m = bits / 3;
    if (min_bits > bits) min_bits = bits;
    const int64_t B = P->B;
    std::vector<uint32_t> ln((size_t)B + 1), px((size_t)B + 1), stt((size_t)B + 1);
    int64_t L = 0;
    p2p_status s = adaptive_leaves(P, t, min_bits, ln.data(), px.data(), stt.data(), B, &L);
    if (s != P2P_OK || L == 0) return s;
    stt[(size_t)L] = (uint32_t)P->n;
    uint32_t *dpre = nullptr, *tot = nullptr;
    unsigned int *dcnt = nullptr, *tcnt = nullptr, *tcur = nullptr;
    uint2 *rng = nullptr;
    uint8_t *rcode = nullptr;
    void *scratch = nullptr;
    P2P_CUDA_TRY(dalloc((void **)&A.len, 4 * L, st));
    P2P_CUDA_TRY(dalloc((void **)&dpre, 4 * L, st));
    P2P_CUDA_TRY(dalloc((void **)&A.lkey, 4 * L, st));
    P2P_CUDA_TRY(dalloc((void **)&A.lstart, 4 * (L + 1), st));
    P2P_CUDA_TRY(dalloc((void **)&dcnt, 4 * L, st));
    P2P_CUDA_TRY(dalloc((void **)&tcnt, 4 * L, st));
    P2P_CUDA_TRY(dalloc((void **)&tcur, 4 * L, st));
    P2P_CUDA_TRY(dalloc((void **)&rng, 8 * 27 * (size_t)L, st));
    P2P_CUDA_TRY(dalloc((void **)&rcode, 27 * (size_t)L, st));
    P2P_CUDA_TRY(dalloc((void **)&A.off, 4 * (L + 1), st));
    P2P_CUDA_TRY(dalloc((void **)&tot, 4, st));
    P2P_CUDA_TRY(dalloc(&scratch, scan_partials_bytes(L), st));
    P2P_CUDA_TRY(cudaMemsetAsync(dcnt, 0, 4 * L, st));
    P2P_CUDA_TRY(cudaMemsetAsync(tcnt, 0, 4 * L, st));
    P2P_CUDA_TRY(cudaMemsetAsync(tcur, 0, 4 * L, st));
    P2P_CUDA_TRY(cudaMemcpyAsync(A.len, ln.data(), 4 * L, cudaMemcpyHostToDevice, st));
    P2P_CUDA_TRY(cudaMemcpyAsync(dpre, px.data(), 4 * L, cudaMemcpyHostToDevice, st));
    P2P_CUDA_TRY(cudaMemcpyAsync(A.lstart, stt.data(), 4 * (L + 1), cudaMemcpyHostToDevice, st));
    const unsigned g = std::max<unsigned>(1, std::min<unsigned>(div_up(L, 128), (unsigned)P->num_sms * 8));
    const unsigned g27 = std::max<unsigned>(1, std::min<unsigned>(div_up(27 * (uint64_t)L, 256), (unsigned)P->num_sms * 16));
    P2P_LAUNCH(k_leaf_keys, g, 128, 0, st, A.len, dpre, (uint32_t)L, bits, A.lkey);
    P2P_LAUNCH(k_dil_ranges, g27, 256, 0, st, A.lkey, A.len, (uint32_t)L, m, rng, rcode, dcnt, tcnt);
    P2P_CUDA_TRY(device_scan<uint32_t>(SumGet{dcnt, tcnt}, OffPut{A.off}, nullptr, (uint64_t)L, tot, scratch, st));
    uint32_t E = 0;
    P2P_CUDA_TRY(cudaMemcpyAsync(&E, tot, 4, cudaMemcpyDeviceToHost, st));
    P2P_CUDA_TRY(cudaMemcpyAsync(A.off + L, tot, 4, cudaMemcpyDeviceToDevice, st));
    P2P_CUDA_TRY(cudaStreamSynchronize(st));
    A.L = L;
    A.E = E;
    uint32_t *nbr_t = nullptr;
    uint8_t *code_t = nullptr;
    const size_t e1 = std::max<uint32_t>(E, 1);
    P2P_CUDA_TRY(dalloc((void **)&A.nbr, 4 * e1, st));
    P2P_CUDA_TRY(dalloc((void **)&A.code, e1, st));
    P2P_CUDA_TRY(dalloc((void **)&nbr_t, 4 * e1, st));
    P2P_CUDA_TRY(dalloc((void **)&code_t, e1, st));
    const unsigned gwl = std::max<unsigned>(1, std::min<unsigned>(div_up(32 * (uint64_t)L, 256), (unsigned)P->num_sms * 16));
    P2P_LAUNCH(k_dil_fill, gwl, 256, 0, st, A.len, (uint32_t)L, rng, rcode, (const uint32_t *)A.off,
               (const unsigned int *)dcnt, tcur, nbr_t, code_t);
    P2P_LAUNCH(k_dil_merge, gwl, 256, 0, st, (const uint32_t *)A.off, (const unsigned int *)dcnt, (uint32_t)L,
               (const uint32_t *)nbr_t, (const uint8_t *)code_t, A.nbr, A.code);
    void *bufs[] = {dpre, dcnt, tcnt, tcur, rng, rcode, tot, scratch, nbr_t, code_t};
    for (void *p : bufs) dfree(p, st);
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}

// leaves (as adaptive_leaves) and their closed neighbour CSR; host outputs, synchronous
p2p_status adaptive_neighbours(p2p_plan *P, uint32_t t, int min_bits, uint32_t *off_h, uint32_t *nbr_h,
                               uint8_t *code_h, int64_t cap_leaves, int64_t cap_entries, int64_t *n_leaves,
                               int64_t *n_entries) {
    cudaStream_t st = P->stream;
    *n_leaves = *n_entries = 0;
    if (P->B == 0) return P2P_OK;
    AdaptiveDev A;
    p2p_status s = build_adaptive(P, t, min_bits, A);
    if (s == P2P_OK) {
        *n_leaves = A.L;
        *n_entries = A.E;
        if (A.L + 1 > cap_leaves || A.E > cap_entries) {
            set_error("output capacity below the leaf / entry count");
            s = P2P_ERR_INVALID_ARGUMENT;
        } else if (A.L > 0) {
            P2P_CUDA_TRY(cudaMemcpyAsync(off_h, A.off, 4 * (A.L + 1), cudaMemcpyDeviceToHost, st));
            P2P_CUDA_TRY(cudaMemcpyAsync(nbr_h, A.nbr, 4 * (size_t)A.E, cudaMemcpyDeviceToHost, st));
            P2P_CUDA_TRY(cudaMemcpyAsync(code_h, A.code, (size_t)A.E, cudaMemcpyDeviceToHost, st));
            P2P_CUDA_TRY(cudaStreamSynchronize(st));
        }
    }
    A.release(st);
    return s;
}

}  // namespace p2p

namespace p2p {

// a6 + a7 + a9 over the adaptive leaves: leaves, CSR, redundant runs (optionally copied out), items, the REDUNDANT
// eval over them; synchronous (sizes are read back)
p2p_status adaptive_eval(p2p_plan *P, uint32_t t, int min_bits, bool indexed, void *phi, void *field, void *red_h,
                         int64_t cap_red, int64_t *n_red, int64_t *n_items) {
    cudaStream_t st = P->stream;
    const bool f64 = P->cfg.precision == P2P_FP64;
    *n_red = 0;
    if (P->B == 0) return P2P_OK;
    AdaptiveDev A;
    p2p_status s = build_adaptive(P, t, min_bits, A);
    if (s != P2P_OK || A.L == 0) {
        A.release(st);
        return s;
    }
    const uint32_t L = (uint32_t)A.L;
    unsigned long long *R = nullptr, *roff = nullptr, *rtot = nullptr;
    uint32_t *tself = nullptr, *ioff = nullptr, *itot = nullptr, *zero = nullptr;
    unsigned long long *ptot = nullptr;  // the pair count I (sizes the work items)
    void *scr = nullptr;
    P2P_CUDA_TRY(dalloc((void **)&R, 8 * (size_t)L, st));
    P2P_CUDA_TRY(dalloc((void **)&roff, 8 * (size_t)L, st));
    P2P_CUDA_TRY(dalloc((void **)&rtot, 8, st));
    P2P_CUDA_TRY(dalloc((void **)&tself, 4 * (size_t)L, st));
    P2P_CUDA_TRY(dalloc((void **)&ptot, 8, st));
    P2P_CUDA_TRY(cudaMemsetAsync(ptot, 0, 8, st));
    P2P_CUDA_TRY(dalloc((void **)&ioff, 4 * (size_t)L, st));
    P2P_CUDA_TRY(dalloc((void **)&itot, 4, st));
    P2P_CUDA_TRY(dalloc((void **)&zero, 4, st));
    P2P_CUDA_TRY(dalloc(&scr, scan_partials_bytes(L), st));
    const uint32_t E = (uint32_t)A.E, nch = (E + 31u) / 32u + 1u;
    uint32_t *ch_leaf = nullptr;
    unsigned long long *ch_rel = nullptr;
    P2P_CUDA_TRY(dalloc((void **)&ch_leaf, 4 * (size_t)nch, st));
    P2P_CUDA_TRY(dalloc((void **)&ch_rel, 8 * (size_t)nch, st));
    P2P_CUDA_TRY(cudaMemsetAsync(zero, 0, 4, st));
    const unsigned g = std::max<unsigned>(1, std::min<unsigned>(div_up(L, 128), (unsigned)P->num_sms * 8));
    P2P_LAUNCH(k_adapt_count, g, 128, 0, st, A.off, A.nbr, A.code, A.lstart, L, R, tself, DevN(), ptot,
               ch_leaf, ch_rel);
    P2P_CUDA_TRY(device_scan<unsigned long long>(U64Get{R}, U64Put{roff}, nullptr, (uint64_t)L, rtot, scr, st));
    const uint32_t K = (uint32_t)(f64 ? EVAL_K_F64 : EVAL_K_F32);
    P2P_CUDA_TRY(device_scan<uint32_t>(ItemCntGet{A.lstart, R, nullptr, K}, OffPut{ioff}, nullptr, (uint64_t)L, itot, scr,
                                       st));
    // the REDUNDANT list (multi-leaf quads) -- built whatever the layout, so both paths' items are the same
    const bool quads = adapt_quads(P);
    uint32_t *ioff_red = nullptr, *itot_red = nullptr;
    P2P_CUDA_TRY(dalloc((void **)&ioff_red, 4 * (size_t)L, st));
    P2P_CUDA_TRY(dalloc((void **)&itot_red, 4, st));
    P2P_CUDA_TRY(device_scan<uint32_t>(RedCntGet{A.lstart, R, adapt_capped() ? ptot : nullptr, nullptr, L, K, quads}, OffPut{ioff_red}, nullptr,
                                       (uint64_t)L, itot_red, scr, st));
    unsigned long long Rtot = 0;
    uint32_t Itot = 0, Itot_red = 0;
    P2P_CUDA_TRY(cudaMemcpyAsync(&Rtot, rtot, 8, cudaMemcpyDeviceToHost, st));
    P2P_CUDA_TRY(cudaMemcpyAsync(&Itot, itot, 4, cudaMemcpyDeviceToHost, st));
    P2P_CUDA_TRY(cudaMemcpyAsync(&Itot_red, itot_red, 4, cudaMemcpyDeviceToHost, st));
    P2P_CUDA_TRY(cudaStreamSynchronize(st));
    void *red = nullptr;
    Item *items = nullptr, *items_red = nullptr;
    const size_t rsz = f64 ? sizeof(double4) : sizeof(float4);
    P2P_CUDA_TRY(dalloc(&red, rsz * std::max<unsigned long long>(Rtot, 1), st));
    P2P_CUDA_TRY(dalloc((void **)&items, sizeof(Item) * std::max<uint32_t>(Itot, 1), st));
    P2P_CUDA_TRY(dalloc((void **)&items_red, sizeof(Item) * std::max<uint32_t>(Itot_red, 1), st));
    const int m = P->key_bits / 3;
    uint8_t *lframe = nullptr;
    P2P_CUDA_TRY(dalloc((void **)&lframe, std::max<uint32_t>(L, 1), st));
    P2P_LAUNCH(k_leaf_frame, g, 128, 0, st, A.lkey, A.len, L, m, lframe);
    // INDEXED: the non-redundant baseline, no runs (the eval stages the neighbour segments of the sorted records)
    if (!indexed) {
        s = launch_adapt_runs(P, A.lkey, A.len, A.lstart, A.off, A.nbr, A.code, ch_leaf, ch_rel, roff, L, E, E, red,
                              DevN());
        if (s != P2P_OK) return s;
    }
    P2P_LAUNCH(k_adapt_items, g, 128, 0, st, A.lstart, roff, R, tself, ioff, L, K, nullptr, items, DevN(), items_red,
               ioff_red, adapt_capped() ? ptot : nullptr, quads);
    P2P_CUDA_TRY(cudaGetLastError());
    s = P2P_OK;
    if (phi) {
        EvalItems it = indexed ? EvalItems{items, itot, (int64_t)Itot, red, zero}
                               : EvalItems{items_red, itot_red, (int64_t)Itot_red, red, zero};
        if (indexed) {
            it.csr_off = A.off;
            it.csr_nbr = A.nbr;
            it.csr_code = A.code;
            it.lstart = A.lstart;
            it.lframe = lframe;
        }
        s = eval_gravity_items(P, it, phi, field);
    }
    *n_red = (int64_t)Rtot;
    if (n_items) *n_items = (int64_t)std::max(Itot, Itot_red);
    if (s == P2P_OK && red_h && !indexed) {
        if ((int64_t)Rtot > cap_red) {
            set_error("red capacity below the record count");
            s = P2P_ERR_INVALID_ARGUMENT;
        } else {
            P2P_CUDA_TRY(cudaMemcpyAsync(red_h, red, rsz * Rtot, cudaMemcpyDeviceToHost, st));
        }
    }
    P2P_CUDA_TRY(cudaStreamSynchronize(st));
    void *bufs[] = {R,   roff,  rtot,    tself,  ptot,     ioff,     itot,     zero,     scr,
                    red, items, ch_leaf, ch_rel, lframe, ioff_red, itot_red, items_red};
    for (void *p : bufs) dfree(p, st);
    A.release(st);
    return s;
}

}  // namespace p2p

// ======================================================================================================================
// The persistent, asynchronous adaptive path (SURVEY NEXT-1 on the per-step path; "p2p_plan_update
// builds adaptive leaves, CSR, runs and items in place, with no host sync").  p2p_adaptive_enable measures the
// current input once (synchronous, like p2p_plan_create) and allocates capacities with headroom: leaves <= boxes,
// entries <= ecap = 2 E, records <= rcap = 2 R, items <= boxes + N / 32.  Every later p2p_plan_update runs a1-a4
// and the leaves + closed CSR with all counts device-side (the kernels read L / E from device memory); p2p_restructure
// builds the runs and items, p2p_eval runs the unchanged eval over them.  A step that exceeds a capacity sets a
// device overflow flag: its kernels do nothing and p2p_get_info reports P2P_ERR_OUT_OF_MEMORY (call
// p2p_adaptive_enable again to re-measure).
namespace p2p {

namespace {
__global__ void k_adapt_tail(AdaptCtr *ac, uint32_t *__restrict__ lstart, uint32_t n) { lstart[ac->L] = n; }
// after the entry scan: off[L] = E and the entry capacity check
__global__ void k_adapt_check_e(AdaptCtr *ac, uint32_t *__restrict__ off, uint64_t ecap) {
    if (ac->E > ecap) ac->overflow = 1u;
    off[ac->L] = ac->E;
}
__global__ void k_adapt_check_r(AdaptCtr *ac, uint64_t rcap, uint64_t icap) {
    if (ac->R > rcap || ac->n_items > icap || ac->n_items_red > icap) ac->overflow = 1u;
    if (ac->overflow) ac->n_items = ac->n_items_red = 0;  // the eval then does nothing (its items were not built)
}
}  // namespace

void adaptive_free(p2p_plan *P) {
    AdaptState *A = P->ad;
    if (!A) return;
    cudaStream_t st = P->stream;
    void *bufs[] = {A->ac,    A->len8, A->rcode, A->code, A->code_t, A->lframe, A->llen, A->lprefix, A->lstart,
                    A->lkey,  A->off,  A->nbr,   A->nbr_t, A->tself, A->ioff, A->zero,    A->dcnt,
                    A->tcnt,  A->tcur, A->rng,   A->R,    A->roff,   A->ch_rel, A->red,  A->scr,     A->items,
                    A->ch_leaf, A->items_red, A->ioff_red};
    for (void *b : bufs) dfree(b, st);
    delete A;
    P->ad = nullptr;
}

p2p_status adaptive_enable(p2p_plan *P, uint32_t t, int min_bits) {
    cudaStream_t st = P->stream;
    adaptive_free(P);
    // measure the current input (synchronous, once): entries and records of its leaves
    int64_t E = 0, R = 0, I = 0;
    if (P->B > 0) {
        AdaptiveDev D;
        p2p_status s = build_adaptive(P, t, min_bits, D);
        E = D.E;
        D.release(st);
        if (s != P2P_OK) return s;
        s = adaptive_eval(P, t, min_bits, false, nullptr, nullptr, nullptr, 0, &R, &I);
        if (s != P2P_OK) return s;
    }
    AdaptState *A = new AdaptState();
    P->ad = A;
    A->t = t;
    A->min_bits = std::min(min_bits, P->key_bits);
    A->bcap = std::max<int64_t>(P->bcap, 1);
    A->ecap = std::max<int64_t>(2 * E, 64);
    A->rcap = std::max<int64_t>(2 * R, std::max<int64_t>(P->cap, 1));
    A->icap = std::max<int64_t>(2 * I, A->bcap + P->cap / 32 + 1);  // cost-capped items: measured, with headroom
    const int64_t L = A->bcap, Ec = A->ecap;
    const size_t rsz = P->cfg.precision == P2P_FP64 ? sizeof(double4) : sizeof(float4);
#define ADA(ptr, bytes)                                                                   \
    do {                                                                                  \
        if (dalloc((void **)&(ptr), (size_t)(bytes), st) != cudaSuccess) {             \
            adaptive_free(P);                                                             \
            set_error("cannot allocate the adaptive-leaf buffers");                       \
            return P2P_ERR_OUT_OF_MEMORY;                                                 \
        }                                                                                 \
    } while (0)
    ADA(A->ac, sizeof(AdaptCtr));
    ADA(A->len8, L);
    ADA(A->llen, 4 * L);
    ADA(A->lprefix, 4 * L);
    ADA(A->lstart, 4 * (L + 1));
    ADA(A->lkey, 4 * L);
    ADA(A->dcnt, 4 * L);
    ADA(A->tcnt, 4 * L);
    ADA(A->tcur, 4 * L);
    ADA(A->rng, 8 * 27 * L);
    ADA(A->rcode, 27 * L);
    ADA(A->off, 4 * (L + 1));
    ADA(A->nbr, 4 * Ec);
    ADA(A->code, Ec);
    ADA(A->nbr_t, 4 * Ec);
    ADA(A->code_t, Ec);
    ADA(A->R, 8 * L);
    ADA(A->roff, 8 * L);
    ADA(A->tself, 4 * L);
    ADA(A->ioff, 4 * L);
    ADA(A->ch_leaf, 4 * (Ec / 32 + 1));
    ADA(A->ch_rel, 8 * (Ec / 32 + 1));
    ADA(A->lframe, L);
    ADA(A->zero, 4);
    ADA(A->red, rsz * A->rcap);
    ADA(A->items, sizeof(Item) * A->icap);
    ADA(A->items_red, sizeof(Item) * A->icap);
    ADA(A->ioff_red, 4 * L);
    ADA(A->scr, std::max(scan_partials_bytes(L), scan_partials_bytes(Ec)));
#undef ADA
    P2P_CUDA_TRY(cudaMemsetAsync(A->zero, 0, 4, st));
    return adaptive_build_async(P);
}

// a5 of adaptive mode: leaves (C22) + closed CSR (C23) of the current sorted boxes, all counts device-side
p2p_status adaptive_build_async(p2p_plan *P) {
    AdaptState *A = P->ad;
    cudaStream_t st = P->stream;
    A->built = true;
    A->runs_valid = false;
    P2P_CUDA_TRY(cudaMemsetAsync(A->ac, 0, sizeof(AdaptCtr), st));
    if (P->n == 0) return P2P_OK;
    const int bits = P->key_bits, m = bits / 3;
    const uint32_t Lc = (uint32_t)A->bcap;
    const DevN dn{&A->ac->L, &A->ac->E, &A->ac->overflow};
    const unsigned gb = std::max<unsigned>(1, std::min<unsigned>(div_up(Lc, 256), (unsigned)P->num_sms * 8));
    const unsigned g27 = std::max<unsigned>(1, std::min<unsigned>(div_up(27ull * Lc, 256), (unsigned)P->num_sms * 16));
    const unsigned gw = std::max<unsigned>(1, std::min<unsigned>(div_up(32ull * Lc, 256), (unsigned)P->num_sms * 16));
    // leaves: length per box, head-flag scan -> Morton-ordered leaf table (device L)
    P2P_LAUNCH(k_leaf_len, gb, 256, 0, st, P->bkey, P->bstart, P->ctr, bits, A->t, A->min_bits, A->len8);
    P2P_CUDA_TRY(device_scan<uint32_t>(LeafHeadGet{P->bkey, A->len8, bits},
                                       LeafHeadPut{P->bkey, P->bstart, A->len8, bits, A->llen, A->lprefix, A->lstart},
                                       &P->ctr->B, Lc, &A->ac->L, A->scr, st));
    P2P_LAUNCH(k_adapt_tail, 1, 1, 0, st, A->ac, A->lstart, (uint32_t)P->n);
    P2P_LAUNCH(k_leaf_keys, gb, 256, 0, st, A->llen, A->lprefix, Lc, bits, A->lkey, dn);
    // closed neighbour CSR: dilation ranges, counts, scan (device E), fill, merge
    P2P_CUDA_TRY(cudaMemsetAsync(A->dcnt, 0, 4 * (size_t)Lc, st));
    P2P_CUDA_TRY(cudaMemsetAsync(A->tcnt, 0, 4 * (size_t)Lc, st));
    P2P_CUDA_TRY(cudaMemsetAsync(A->tcur, 0, 4 * (size_t)Lc, st));
    P2P_LAUNCH(k_dil_ranges, g27, 256, 0, st, A->lkey, A->llen, Lc, m, A->rng, A->rcode, A->dcnt, A->tcnt, dn);
    P2P_CUDA_TRY(device_scan<uint32_t>(SumGet{A->dcnt, A->tcnt}, OffPut{A->off}, &A->ac->L, Lc, &A->ac->E, A->scr, st));
    P2P_LAUNCH(k_adapt_check_e, 1, 1, 0, st, A->ac, A->off, (uint64_t)A->ecap);
    P2P_LAUNCH(k_dil_fill, gw, 256, 0, st, A->llen, Lc, A->rng, A->rcode, (const uint32_t *)A->off,
               (const unsigned int *)A->dcnt, A->tcur, A->nbr_t, A->code_t, dn);
    P2P_LAUNCH(k_dil_merge, gw, 256, 0, st, (const uint32_t *)A->off, (const unsigned int *)A->dcnt, Lc,
               (const uint32_t *)A->nbr_t, (const uint8_t *)A->code_t, A->nbr, A->code, dn);
    // per leaf: run length, self offset, items (scans: device R, items) + the restructure chunk heads, the leaf
    // frames and the work items -- what BOTH layouts' evals need (the grid path's a5 builds the same), so that
    // p2p_restructure is the redundant runs alone
    const bool f64 = P->cfg.precision == P2P_FP64;
    const unsigned g = std::max<unsigned>(1, std::min<unsigned>(div_up(Lc, 128), (unsigned)P->num_sms * 8));
    P2P_LAUNCH(k_adapt_count, g, 128, 0, st, A->off, A->nbr, A->code, A->lstart, Lc, A->R, A->tself, dn,
               &A->ac->I, A->ch_leaf, A->ch_rel);
    P2P_CUDA_TRY(device_scan<unsigned long long>(U64Get{A->R}, U64Put{A->roff}, &A->ac->L, Lc, &A->ac->R, A->scr, st));
    const uint32_t K = (uint32_t)(f64 ? EVAL_K_F64 : EVAL_K_F32);
    P2P_CUDA_TRY(device_scan<uint32_t>(ItemCntGet{A->lstart, A->R, nullptr, K}, OffPut{A->ioff}, &A->ac->L, Lc,
                                       &A->ac->n_items, A->scr, st));
    const bool quads = adapt_quads(P);
    P2P_CUDA_TRY(device_scan<uint32_t>(RedCntGet{A->lstart, A->R, adapt_capped() ? &A->ac->I : nullptr, &A->ac->L, 0u, K, quads}, OffPut{A->ioff_red},
                                       &A->ac->L, Lc, &A->ac->n_items_red, A->scr, st));
    P2P_LAUNCH(k_adapt_check_r, 1, 1, 0, st, A->ac, (uint64_t)A->rcap, (uint64_t)A->icap);
    P2P_LAUNCH(k_leaf_frame, g, 128, 0, st, A->lkey, A->llen, Lc, m, A->lframe, dn);
    P2P_LAUNCH(k_adapt_items, g, 128, 0, st, A->lstart, A->roff, A->R, A->tself, A->ioff, Lc, K, nullptr, A->items,
               dn, A->items_red, A->ioff_red, adapt_capped() ? &A->ac->I : nullptr, quads);
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}

// a6 of adaptive mode: the redundant runs (C24) over the chunk heads the update recorded
p2p_status adaptive_restructure_async(p2p_plan *P) {
    AdaptState *A = P->ad;
    if (P->n == 0) {
        A->runs_valid = true;
        return P2P_OK;
    }
    const DevN dn{&A->ac->L, &A->ac->E, &A->ac->overflow};
    p2p_status s = launch_adapt_runs(P, A->lkey, A->llen, A->lstart, A->off, A->nbr, A->code, A->ch_leaf, A->ch_rel,
                                     A->roff, (uint32_t)A->bcap, (uint32_t)A->ecap, (uint64_t)A->ecap, A->red, dn);
    if (s == P2P_OK) A->runs_valid = true;
    return s;
}

// a7 + a9 of adaptive mode: REDUNDANT over the runs, or INDEXED over the leaves' CSR segments (the baseline)
p2p_status adaptive_eval_async(p2p_plan *P, p2p_layout layout, void *phi, void *field) {
    AdaptState *A = P->ad;
    if (P->n == 0) return P2P_OK;
    EvalItems it{A->items_red, &A->ac->n_items_red, A->icap, A->red, A->zero};
    if (layout == P2P_INDEXED) {
        it.items = A->items;
        it.n_items = &A->ac->n_items;
        it.csr_off = A->off;
        it.csr_nbr = A->nbr;
        it.csr_code = A->code;
        it.lstart = A->lstart;
        it.lframe = A->lframe;
    }
    return eval_gravity_items(P, it, phi, field);  // after an overflow n_items = 0: nothing is evaluated
}

p2p_status adaptive_info(p2p_plan *P, AdaptCtr *out) {
    P2P_CUDA_TRY(cudaMemcpyAsync(out, P->ad->ac, sizeof(AdaptCtr), cudaMemcpyDeviceToHost, P->stream));
    P2P_CUDA_TRY(cudaStreamSynchronize(P->stream));
    return P2P_OK;
}

}  // namespace p2p
