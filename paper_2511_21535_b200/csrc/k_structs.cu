// k_structs.cu -- method steps a1..a5 on the device:
//   a1 bin + Morton key (fp64 IEEE binning, DESIGN C6/C7), a2 stable radix sort (k_sort.cu),
//   a3 permute into Morton-ordered AoS records, a4 box-offset scan (run heads -> compact box table),
//   a5 neighbour CSR (ascending stencil slot, C10) + redundant offsets red_off + eval work items.
// Bit-exactness with the oracle: every fp64 operation that decides an integer (box index, sub-cell) is an
// explicit IEEE intrinsic (__dsub_rn, __ddiv_rn, __fma_rn) so no contraction or reassociation can change
// a rounding.
#include <algorithm>

#include "plan.hpp"
#include "scan.cuh"

namespace p2p {

// ------------------------------------------------------------------------------------------------
// eval work items: a box's targets are split into ceil(n_b / ITEM_TMAX) chunks, more if the chunk cost
// n_t * R_b exceeds ITEM_COSTCAP interactions (bounds the tail of the dynamic work queue on clustered
// inputs).  Chunks are balanced: chunk c = [n_b c / nch, n_b (c+1) / nch).
// ITEM_TMAX (plan.hpp): at most 32 targets per item -> G <= 8 groups of K = 4 (fp32), >= 28 busy lanes
constexpr uint64_t ITEM_COSTCAP = 1ull << 17;

__device__ __forceinline__ uint32_t item_chunks(uint32_t nb_b, uint64_t nsrc, uint32_t tmax) {
    uint64_t a = (nb_b + tmax - 1) / tmax;
    uint64_t c = ((uint64_t)nb_b * nsrc + ITEM_COSTCAP - 1) / ITEM_COSTCAP;
    uint64_t m = a > c ? a : c;
    if (m > nb_b) m = nb_b;
    if (m < 1) m = 1;
    return (uint32_t)m;
}

// ------------------------------------------------------------------------------------------------ a1
// positions at pos[i * ps + d] (ps = 3: the caller's [N][3] array; ps = 4: {x,y,z,m} records)
template <typename T>
__global__ void k_bin_gravity(const T *__restrict__ pos, int ps, uint32_t n, Geom g, uint32_t *__restrict__ key,
                              uint32_t *__restrict__ idx, DevCounters *ctr) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t c[3];
        bool bad = false;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            double x = (double)pos[(size_t)ps * i + d];
            double f = floor(__ddiv_rn(__dsub_rn(x, g.lo[d]), g.h));
            if (!(f >= 0.0 && f < (double)g.nbox[d])) {
                bad = true;
                f = 0.0;
            }
            c[d] = (uint32_t)f;
        }
        if (bad) atomicMin(&ctr->err_index, (unsigned long long)i);
        key[i] = spread3(c[0]) | (spread3(c[1]) << 1) | (spread3(c[2]) << 2);
        idx[i] = i;
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
// random gather (input order is arbitrary): 4 particles per thread iteration, all loads issued before the
// stores (memory-level parallelism for the latency-bound gather)
template <typename T, typename V4>
__global__ void k_permute_gravity(const T *__restrict__ pos, int ps, const T *__restrict__ q, int qs,
                                  const uint32_t *__restrict__ perm, uint32_t n, V4 *__restrict__ rec) {
    constexpr int U = 4;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t p0 = blockIdx.x * blockDim.x + threadIdx.x; p0 < n; p0 += U * stride) {
        uint32_t i[U];
#pragma unroll
        for (int u = 0; u < U; ++u) i[u] = p0 + u * stride < n ? perm[p0 + u * stride] : 0u;
        V4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (p0 + u * stride < n) {
                r[u].x = pos[(size_t)ps * i[u] + 0];
                r[u].y = pos[(size_t)ps * i[u] + 1];
                r[u].z = pos[(size_t)ps * i[u] + 2];
                r[u].w = q[(size_t)qs * i[u]];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (p0 + u * stride < n) rec[p0 + u * stride] = r[u];
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

// ------------------------------------------------------------------------------------------------ a5
// Neighbour keys by Morton arithmetic (no decode / re-encode): lane = stencil slot with offsets dd in {-1,0,1}^3;
// a +-1 step in dimension d is a masked add / subtract on that dimension's interleaved bits, the periodic wrap
// (C5) replaces the bits by 0 or by nbox_d - 1.  Slots in ascending order (C10): slot = (dx+1) + 3 (dy+1) + 9 (dz+1).
struct MortonStencil {
    uint32_t M[3], top[3];  // dimension-d bit mask of the key space, bits of coordinate nbox_d - 1
    int dd[3];
    bool live;
};
__device__ __forceinline__ MortonStencil make_stencil(const Geom &g, unsigned lane) {
    MortonStencil s;
    s.live = lane < 27;
    const uint32_t full = spread3((1u << g.nb) - 1u);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        s.M[d] = full << d;
        s.top[d] = spread3((uint32_t)(g.nbox[d] - 1)) << d;
    }
    s.dd[0] = (int)(lane % 3) - 1;
    s.dd[1] = (int)((lane / 3) % 3) - 1;
    s.dd[2] = (int)(lane / 9) - 1;
    return s;
}
__device__ __forceinline__ bool morton_nbr(const Geom &g, const MortonStencil &s, uint32_t key, uint32_t &nk) {
    if (!s.live) return false;
    nk = key;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const uint32_t M = s.M[d], kd = key & M;
        if (s.dd[d] > 0) {
            if (kd == s.top[d]) {
                if (!((g.periodic >> d) & 1u)) return false;
                nk &= ~M;
            } else {
                nk = (((nk | ~M) + (1u << d)) & M) | (nk & ~M);
            }
        } else if (s.dd[d] < 0) {
            if (kd == 0u) {
                if (!((g.periodic >> d) & 1u)) return false;
                nk = (nk & ~M) | s.top[d];
            } else {
                nk = (((nk & M) - (1u << d)) & M) | (nk & ~M);
            }
        }
    }
    return true;
}

// dense key -> {box, n_b} table for the gravity neighbour search (valid where the occupancy bit is set)
__global__ void k_boxinfo(const uint32_t *__restrict__ bkey, const uint32_t *__restrict__ bstart,
                          const DevCounters *__restrict__ ctr, uint2 *__restrict__ boxinfo) {
    const uint32_t B = ctr->B;
    for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x)
        boxinfo[bkey[b]] = make_uint2(b, bstart[b + 1] - bstart[b]);
}

// a5 (count pass): lane = stencil slot.  Two dependent load levels per box: the box key, then the neighbour's
// occupancy word and its {box, n} entry, issued together (a stale entry of an empty key is ignored).  The
// per-slot result goes to a slot table that k_nbr_fill reads back instead of repeating the search.
__global__ void __launch_bounds__(256) k_nbr_count(Geom g, const uint32_t *__restrict__ bkey,
                                                   const uint2 *__restrict__ boxinfo,
                                                   const uint32_t *__restrict__ occ, DevCounters *ctr,
                                                   uint32_t *__restrict__ nbr_cnt, uint64_t *__restrict__ red_cnt,
                                                   uint32_t *__restrict__ item_cnt, uint32_t *__restrict__ small_cnt,
                                                   uint2 *__restrict__ slot_tab, uint32_t tmax) {
    const uint32_t B = ctr->B;
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const MortonStencil stc = make_stencil(g, lane);
    unsigned long long pairs = 0;
    constexpr int NB = 4;  // boxes per warp iteration: their lookups are in flight together
    for (uint32_t b0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * NB; b0 < B; b0 += nwarps * NB) {
        bool ok[NB];
        uint32_t kk[NB], cn[NB], key[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) key[u] = b0 + u < B ? bkey[b0 + u] : 0u;
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            ok[u] = false;
            kk[u] = 0;
            cn[u] = 0;
            uint32_t nk;
            // non-target (multi-GPU halo) boxes get no neighbour list and no work
            if (b0 + u < B && key[u] >= g.tkey_lo && key[u] <= g.tkey_hi && morton_nbr(g, stc, key[u], nk)) {
                const uint32_t w = __ldg(&occ[nk >> 5]);
                const uint2 inf = boxinfo[nk];
                ok[u] = (w >> (nk & 31u)) & 1u;
                kk[u] = inf.x;
                cn[u] = inf.y;
            }
        }
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const uint32_t b = b0 + u;
            if (b < B && lane < 27) slot_tab[27 * (size_t)b + lane] = ok[u] ? make_uint2(kk[u], cn[u]) : make_uint2(~0u, 0u);
            const uint32_t nk = __reduce_add_sync(0xffffffffu, ok[u] ? cn[u] : 0u);
            const uint32_t cnt = __popc(__ballot_sync(0xffffffffu, ok[u]));
            const uint32_t own = __shfl_sync(0xffffffffu, ok[u] ? cn[u] : 0u, 13);  // centre slot = the box itself
            if (lane == 0 && b < B) {
                const bool target = key[u] >= g.tkey_lo && key[u] <= g.tkey_hi;
                const uint32_t nb_b = target ? own : 0u;
                nbr_cnt[b] = cnt;
                red_cnt[b] = nk;
                // boxes with <= SMALL_NT targets go to the eval's thread-per-target path (no work item)
                const bool small = nb_b <= SMALL_NT && nk <= SMALL_R;
                item_cnt[b] = (small || !target) ? 0u : item_chunks(nb_b, nk, tmax);
                small_cnt[b] = small ? (nb_b + 1) / 2 : 0u;  // target PAIRS (eval small path)
                pairs += (unsigned long long)nb_b * nk;
            }
        }
    }
    if (lane == 0 && pairs) atomicAdd(&ctr->I, pairs);
}

__global__ void __launch_bounds__(256) k_nbr_fill(Geom g, const uint32_t *__restrict__ bkey,
                                                  const uint32_t *__restrict__ bstart,
                                                  const uint2 *__restrict__ slot_tab, const DevCounters *ctr,
                                                  const uint32_t *__restrict__ nbr_off,
                                                  const uint32_t *__restrict__ item_off,
                                                  const uint32_t *__restrict__ item_cnt, uint32_t *__restrict__ nbr_box,
                                                  uint8_t *__restrict__ nbr_slot, Item *__restrict__ items,
                                                  const uint32_t *__restrict__ small_off,
                                                  uint32_t *__restrict__ small_tgt, uint32_t *__restrict__ small_box,
                                                  const unsigned long long *__restrict__ red_off,
                                                  uint32_t *__restrict__ chunk_box,
                                                  unsigned long long *__restrict__ chunk_out, uint32_t K) {
    const uint32_t B = ctr->B;
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    constexpr int NB = 4;  // boxes per warp iteration (memory-level parallelism, as in k_nbr_count)
    for (uint32_t b0 = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * NB; b0 < B; b0 += nwarps * NB) {
        bool ok[NB];
        uint32_t k[NB], cn[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            // k_nbr_count's slot table (halo boxes: all ~0u, no neighbour list and no work)
            const uint2 t = (b0 + u < B && lane < 27) ? slot_tab[27 * (size_t)(b0 + u) + lane] : make_uint2(~0u, 0u);
            k[u] = t.x;
            cn[u] = t.y;
            ok[u] = k[u] != 0xffffffffu;
        }
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            const uint32_t b = b0 + u;
            const uint32_t m = __ballot_sync(0xffffffffu, ok[u]);
            if (b >= B) continue;
            // segment lengths in slot (= CSR) order; exclusive prefix = segment offset inside the box's run
            const uint32_t cnt_l = ok[u] ? cn[u] : 0u;
            uint32_t incl = cnt_l;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= (unsigned)o) incl += y;
            }
            // records of the slots before the centre (13) = offset of the box's own segment in its run
            const uint32_t cen = __shfl_sync(0xffffffffu, incl - cnt_l, 13);
            if (ok[u]) {
                const uint32_t e = nbr_off[b] + __popc(m & ((1u << lane) - 1u));
                nbr_box[e] = k[u];
                nbr_slot[e] = (uint8_t)lane;
                if ((e & 31u) == 0u) {  // head of a restructure chunk
                    chunk_box[e >> 5] = b;
                    chunk_out[e >> 5] = red_off[b] + (incl - cnt_l);
                }
            }
            const uint32_t key = bkey[b];
            if (key < g.tkey_lo || key > g.tkey_hi) continue;  // halo box: source only
            const uint32_t s0 = bstart[b], nb_b = bstart[b + 1] - s0;
            const uint32_t nch = item_cnt[b];
            if (nch == 0) {  // small box (k_nbr_count): thread-per-target path
                if (lane < (nb_b + 1) / 2) {  // one entry per target pair
                    small_tgt[small_off[b] + lane] = s0 + 2 * lane;
                    small_box[small_off[b] + lane] = b;
                }
                continue;
            }
            const uint32_t it = item_off[b];
            const unsigned long long rb = red_off[b];
            const uint32_t Rb = (uint32_t)(red_off[b + 1] - rb);
            for (uint32_t ci = lane; ci < nch; ci += 32) {
                const uint32_t a0 = (uint32_t)(((uint64_t)nb_b * ci) / nch);
                const uint32_t z0 = (uint32_t)(((uint64_t)nb_b * (ci + 1)) / nch);
                // eval lane layout: G = ceil(n_t / K) groups of K targets, S = floor(32 / G) source splits
                const uint32_t nt = z0 - a0, G = (nt + K - 1) / K, S = 32u / G;
                items[it + ci] = Item{b, s0 + a0, nt | (S << 8) | (G << 16), key, rb, Rb, cen + a0};
            }
        }
    }
}

// Helmholtz: 9-slot table, missing -> 0xffffffff (C10); boxes must be full (t samples, distinct sub-cells)
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

// ------------------------------------------------------------------------------------------------
// scan functors over plain arrays
template <typename T>
struct ArrGet {
    const T *a;
    __device__ T operator()(uint64_t i) const { return a[i]; }
};
template <typename T>
struct OffPut {
    T *off;
    const uint32_t *nptr;
    __device__ void operator()(uint64_t i, T e, T v) const {
        off[i] = e;
        if (i == (uint64_t)*nptr - 1) off[i + 1] = e + v;
    }
};

static unsigned grid_for(uint64_t n, int threads, int num_sms) {
    uint64_t g = (n + threads - 1) / threads;
    uint64_t cap = (uint64_t)num_sms * 16;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(g, cap));
}

// ------------------------------------------------------------------------------------------------
static unsigned warp_grid(uint64_t nwork, int num_sms) {
    // one warp per work unit, 8 warps per block, at most 16 resident blocks per SM (grid-stride beyond)
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(div_up(nwork, 8), (uint64_t)num_sms * 8));  // one full-occupancy wave
}

void free_capacity(p2p_plan *P) {
    cudaStream_t st = P->stream;
    void *bufs[] = {P->s_key, P->s_idx, P->s_kalt, P->s_valt, P->s_hist, P->s_status, P->s_partials,
                    P->s_nbr_cnt, P->s_item_cnt, P->s_item_off, P->s_red_cnt, P->s_small_cnt, P->s_small_off,
                    P->s_slot_tab, P->boxinfo,
                    P->small_tgt, P->small_box, P->chunk_box, P->chunk_out, P->rec, P->bkey, P->bstart,
                    P->nbr_off, P->nbr_box, P->nbr_slot, P->red_off, P->box_of, P->items, P->occ};
    for (void *b : bufs) dfree(b, st);
    P->s_key = P->s_idx = P->s_kalt = P->s_valt = P->s_hist = P->s_status = nullptr;
    P->s_partials = nullptr;
    P->s_nbr_cnt = P->s_item_cnt = P->s_item_off = nullptr;
    P->s_slot_tab = nullptr;
    P->boxinfo = nullptr;
    P->s_small_cnt = P->s_small_off = P->small_tgt = P->small_box = P->chunk_box = nullptr;
    P->chunk_out = nullptr;
    P->s_red_cnt = nullptr;
    P->rec = nullptr;
    P->bkey = P->bstart = P->nbr_off = P->nbr_box = P->box_of = P->occ = nullptr;
    P->nbr_slot = nullptr;
    P->red_off = nullptr;
    P->items = nullptr;
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
    P2P_CUDA_TRY(dalloc((void **)&P->s_status, 4 * std::max<size_t>(1, radix_status_words(n, std::max(1, P->passes))), st));
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
        P2P_CUDA_TRY(dalloc((void **)&P->s_nbr_cnt, 4 * bcap, st));
        P2P_CUDA_TRY(dalloc((void **)&P->s_slot_tab, sizeof(uint2) * 27 * bcap, st));
        P2P_CUDA_TRY(dalloc((void **)&P->boxinfo, sizeof(uint2) * keyspace, st));
        P2P_CUDA_TRY(dalloc((void **)&P->s_item_cnt, 4 * bcap, st));
        P2P_CUDA_TRY(dalloc((void **)&P->s_item_off, 4 * (bcap + 1), st));
        P2P_CUDA_TRY(dalloc((void **)&P->s_small_cnt, 4 * bcap, st));
        P2P_CUDA_TRY(dalloc((void **)&P->s_small_off, 4 * (bcap + 1), st));
        P2P_CUDA_TRY(dalloc((void **)&P->small_tgt, 4 * n, st));
        P2P_CUDA_TRY(dalloc((void **)&P->small_box, 4 * n, st));
        P2P_CUDA_TRY(dalloc((void **)&P->s_red_cnt, 8 * bcap, st));
        P2P_CUDA_TRY(dalloc((void **)&P->red_off, 8 * (bcap + 1), st));
        P2P_CUDA_TRY(dalloc((void **)&P->items, sizeof(Item) * n, st));
        const uint64_t nchunk = div_up((uint64_t)nslot * bcap, 32) + 1;
        P2P_CUDA_TRY(dalloc((void **)&P->chunk_box, 4 * nchunk, st));
        P2P_CUDA_TRY(dalloc((void **)&P->chunk_out, 8 * nchunk, st));
    } else {
        P2P_CUDA_TRY(dalloc(&P->rec, (f64 ? sizeof(double2) : sizeof(float2)) * n, st));
    }
    return P2P_OK;
}

p2p_status build_gravity_structs(p2p_plan *P, const void *pos, const void *q, const void *rec_in) {
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
    // a1
    if (f64)
        P2P_LAUNCH(k_bin_gravity<double>, gb, 256, 0, st, (const double *)pos, ps, n, P->geom, P->s_key, P->s_idx,
                   P->ctr);
    else
        P2P_LAUNCH(k_bin_gravity<float>, gb, 256, 0, st, (const float *)pos, ps, n, P->geom, P->s_key, P->s_idx,
                   P->ctr);
    // a2
    P2P_CUDA_TRY(radix_sort_pairs(P->s_key, P->s_idx, P->s_kalt, P->s_valt, n, P->passes, P->ctr, P->s_hist,
                                  P->s_status, st, &P->skey, &P->perm));
    // a3
    if (f64)
        P2P_LAUNCH((k_permute_gravity<double, double4>), gb, 256, 0, st, (const double *)pos, ps, (const double *)q,
                   qs, P->perm, n, (double4 *)P->rec);
    else
        P2P_LAUNCH((k_permute_gravity<float, float4>), gb, 256, 0, st, (const float *)pos, ps, (const float *)q, qs,
                   P->perm, n, (float4 *)P->rec);
    // a4
    const uint64_t occ_words = std::max<uint64_t>(1, (1ull << P->key_bits) / 32);
    P2P_CUDA_TRY(cudaMemsetAsync(P->occ, 0, 4 * occ_words, st));
    P2P_CUDA_TRY(device_scan<uint32_t>(HeadGet{P->skey, 1u},
                                       HeadPut{P->skey, 1u, P->bkey, P->bstart, nullptr, n, P->occ}, nullptr, n,
                                       &P->ctr->B, P->s_partials, st));
    // a5
    const uint64_t bcap = (uint64_t)P->bcap;
    const unsigned gw = warp_grid(bcap, P->num_sms);
    const uint32_t tmax = ITEM_TMAX;
    P2P_LAUNCH(k_boxinfo, std::max<unsigned>(1, std::min<unsigned>(div_up(bcap, 256), (unsigned)P->num_sms * 8)), 256,
               0, st, P->bkey, P->bstart, P->ctr, P->boxinfo);
    P2P_LAUNCH(k_nbr_count, gw, 256, 0, st, P->geom, P->bkey, P->boxinfo, P->occ, P->ctr, P->s_nbr_cnt,
               P->s_red_cnt, P->s_item_cnt, P->s_small_cnt, P->s_slot_tab, tmax);
    P2P_CUDA_TRY(device_scan<uint32_t>(ArrGet<uint32_t>{P->s_nbr_cnt}, OffPut<uint32_t>{P->nbr_off, &P->ctr->B},
                                       &P->ctr->B, bcap, &P->ctr->n_nbr, P->s_partials, st));
    P2P_CUDA_TRY(device_scan<unsigned long long>(
        ArrGet<unsigned long long>{(const unsigned long long *)P->s_red_cnt},
        OffPut<unsigned long long>{(unsigned long long *)P->red_off, &P->ctr->B}, &P->ctr->B, bcap, &P->ctr->R,
        P->s_partials, st));
    P2P_CUDA_TRY(device_scan<uint32_t>(ArrGet<uint32_t>{P->s_item_cnt}, OffPut<uint32_t>{P->s_item_off, &P->ctr->B},
                                       &P->ctr->B, bcap, &P->ctr->n_items, P->s_partials, st));
    P2P_CUDA_TRY(device_scan<uint32_t>(ArrGet<uint32_t>{P->s_small_cnt}, OffPut<uint32_t>{P->s_small_off, &P->ctr->B},
                                       &P->ctr->B, bcap, &P->ctr->n_small, P->s_partials, st));
    P2P_LAUNCH(k_nbr_fill, gw, 256, 0, st, P->geom, P->bkey, P->bstart, P->s_slot_tab, P->ctr, P->nbr_off,
               P->s_item_off, P->s_item_cnt, P->nbr_box, P->nbr_slot, P->items, P->s_small_off, P->small_tgt,
               P->small_box, (const unsigned long long *)P->red_off, P->chunk_box, P->chunk_out,
               (uint32_t)(f64 ? EVAL_K_F64 : EVAL_K_F32));
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
