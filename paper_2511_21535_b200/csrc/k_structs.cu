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

// a5, one pass: neighbour search, the four exclusive scans (CSR offsets, redundant offsets, work items, small
// target pairs) and all writes of the CSR / items / small lists / restructure chunk heads.
// One warp per tile of 32 consecutive boxes; tiles are claimed from an atomic counter in launch order, so the
// decoupled look-back (NbTileStatus) only ever waits on tiles that are already running.
//   phase A  lane = stencil slot, 4 boxes in flight: neighbour key by Morton arithmetic, then the occupancy
//            word and the {box, n} entry together (a stale entry of an empty key is ignored); per-slot results
//            to shared memory, per-box totals to lane i
//   phase B  warp scans of the per-box totals, look-back for the tile's exclusive prefix, nbr_off / red_off
//   phase C  lane = stencil slot again, per box: ballot-compacted CSR in ascending slot order (C10), the
//            restructure chunk heads, the eval work items or small-target entries
constexpr int NBB_WARPS = 4;
constexpr int NBB_TILE = 32;

__device__ __forceinline__ unsigned long long ld_vol64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_vol64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(NBB_WARPS * 32) k_nbr_build(
    Geom g, const uint32_t *__restrict__ bkey, const uint32_t *__restrict__ bstart, const uint2 *__restrict__ boxinfo,
    const uint32_t *__restrict__ occ, DevCounters *ctr, NbTileStatus *status, uint32_t *__restrict__ nbr_off,
    unsigned long long *__restrict__ red_off, uint32_t *__restrict__ nbr_box, uint8_t *__restrict__ nbr_slot,
    Item *__restrict__ items, uint32_t *__restrict__ small_tgt, uint32_t *__restrict__ small_box,
    uint32_t *__restrict__ chunk_box, unsigned long long *__restrict__ chunk_out, uint32_t K, uint32_t tmax) {
    __shared__ uint32_t s_k[NBB_WARPS][NBB_TILE][27];
    __shared__ uint32_t s_c[NBB_WARPS][NBB_TILE][27];
    constexpr unsigned FULL = 0xffffffffu;
    const uint32_t B = ctr->B;
    const uint32_t ntiles = (B + NBB_TILE - 1) / NBB_TILE;
    const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    const MortonStencil stc = make_stencil(g, lane);
    unsigned long long pairs = 0;
    while (true) {
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(&ctr->nbr_tile, 1u);
        t = __shfl_sync(FULL, t, 0);
        if (t >= ntiles) break;
        const uint32_t tb = t * NBB_TILE;
        // lane i: box tb + i
        const uint32_t mb = tb + lane;
        const bool have = mb < B;
        const uint32_t mkey = have ? bkey[mb] : 0u;
        const uint32_t ms0 = have ? bstart[mb] : 0u;
        const bool mtarget = have && mkey >= g.tkey_lo && mkey <= g.tkey_hi;  // halo boxes: source only
        uint32_t my_nbr = 0, my_item = 0, my_small = 0, my_nb = 0;
        unsigned long long my_red = 0;

        // ---- phase A ----
        constexpr int NB = 4;
        for (int i0 = 0; i0 < NBB_TILE; i0 += NB) {
            if (tb + i0 >= B) break;  // warp-uniform
            bool ok[NB];
            uint32_t kk[NB], cn[NB];
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                const int i = i0 + u;
                const uint32_t key = __shfl_sync(FULL, mkey, i);
                const bool tgt = __shfl_sync(FULL, (uint32_t)mtarget, i) != 0u;
                ok[u] = false;
                kk[u] = 0;
                cn[u] = 0;
                uint32_t nk;
                if (tgt && morton_nbr(g, stc, key, nk)) {
                    const uint32_t wd = __ldg(&occ[nk >> 5]);
                    const uint2 inf = boxinfo[nk];
                    ok[u] = (wd >> (nk & 31u)) & 1u;
                    kk[u] = inf.x;
                    cn[u] = inf.y;
                }
            }
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                const int i = i0 + u;
                if (lane < 27) {
                    s_k[w][i][lane] = ok[u] ? kk[u] : 0xffffffffu;
                    s_c[w][i][lane] = ok[u] ? cn[u] : 0u;
                }
                const uint32_t nk = __reduce_add_sync(FULL, ok[u] ? cn[u] : 0u);
                const uint32_t cnt = __popc(__ballot_sync(FULL, ok[u]));
                const uint32_t own = __shfl_sync(FULL, ok[u] ? cn[u] : 0u, 13);  // centre slot = the box itself
                if (lane == (unsigned)i && have) {
                    my_nbr = cnt;
                    my_red = nk;
                    my_nb = mtarget ? own : 0u;
                    // boxes with <= SMALL_NT targets go to the eval's thread-per-target path (no work item)
                    const bool small = my_nb <= SMALL_NT && nk <= SMALL_R;
                    my_item = (small || !mtarget) ? 0u : item_chunks(my_nb, nk, tmax);
                    my_small = (small && mtarget) ? (my_nb + 1) / 2 : 0u;  // target PAIRS
                    pairs += (unsigned long long)my_nb * nk;
                }
            }
        }
        __syncwarp();

        // ---- phase B: tile scans + decoupled look-back ----
        uint32_t in_nbr = my_nbr, in_item = my_item, in_small = my_small;
        unsigned long long in_red = my_red;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t a = __shfl_up_sync(FULL, in_nbr, o), b2 = __shfl_up_sync(FULL, in_item, o),
                           c = __shfl_up_sync(FULL, in_small, o);
            const unsigned long long d = __shfl_up_sync(FULL, in_red, o);
            if (lane >= (unsigned)o) {
                in_nbr += a;
                in_item += b2;
                in_small += c;
                in_red += d;
            }
        }
        // tile aggregates (lane 31's inclusive values); items | small << 31 share one word
        constexpr unsigned long long VMASK = (1ull << 62) - 1ull, F_AGG = 1ull << 62, F_INC = 2ull << 62;
        unsigned long long agg[3];
        agg[0] = __shfl_sync(FULL, (unsigned long long)in_nbr, 31);
        agg[1] = __shfl_sync(FULL, in_red, 31);
        agg[2] = __shfl_sync(FULL, (unsigned long long)in_item | ((unsigned long long)in_small << 31), 31);
        unsigned long long pre[3] = {0ull, 0ull, 0ull};
        NbTileStatus *me = status + t;
        const unsigned long long my_agg = lane == 0 ? agg[0] : (lane == 1 ? agg[1] : agg[2]);
        if (t == 0) {
            if (lane < 3) st_vol64(&me->w[lane], F_INC | my_agg);
        } else {
            if (lane < 3) st_vol64(&me->w[lane], F_AGG | my_agg);
            // warp-parallel look-back, per word: lane j inspects tile base - j (a window of 32 predecessors per
            // step) until the nearest inclusive prefix
#pragma unroll
            for (int wd = 0; wd < 3; ++wd) {
                for (int64_t base = (int64_t)t - 1;;) {
                    const int64_t q = base - (int64_t)lane;
                    unsigned long long x = F_INC;  // tiles before 0 act as an inclusive zero
                    if (q >= 0) {
                        do {
                            x = ld_vol64(&status[q].w[wd]);
                        } while ((x >> 62) == 0ull);
                    }
                    const uint32_t incm = __ballot_sync(FULL, (x >> 62) == 2ull);
                    const int jstop = incm ? __ffs(incm) - 1 : 31;  // nearest inclusive predecessor
                    unsigned long long v = (int)lane <= jstop ? (x & VMASK) : 0ull;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
                    pre[wd] += v;
                    if (incm) break;
                    base -= 32;
                }
            }
            if (lane < 3) {
                const unsigned long long mine = (lane == 0 ? pre[0] : (lane == 1 ? pre[1] : pre[2])) + my_agg;
                st_vol64(&me->w[lane], F_INC | mine);
            }
        }
        const unsigned long long p_nbr = pre[0], p_red = pre[1], p_is = pre[2];
        const uint32_t o_nbr = (uint32_t)p_nbr + in_nbr - my_nbr;
        const unsigned long long o_red = p_red + in_red - my_red;
        const uint32_t o_item = (uint32_t)(p_is & 0x7fffffffull) + in_item - my_item;
        const uint32_t o_small = (uint32_t)(p_is >> 31) + in_small - my_small;
        if (have) {
            nbr_off[mb] = o_nbr;
            red_off[mb] = o_red;
        }
        if (mb == B - 1) {  // the last box closes the offsets and publishes the totals
            nbr_off[B] = o_nbr + my_nbr;
            red_off[B] = o_red + my_red;
            ctr->n_nbr = o_nbr + my_nbr;
            ctr->R = o_red + my_red;
            ctr->n_items = o_item + my_item;
            ctr->n_small = o_small + my_small;
        }

        // ---- phase C: CSR, chunk heads, items / small entries (lane = stencil slot) ----
        for (int i = 0; i < NBB_TILE; ++i) {
            const uint32_t b = tb + i;
            if (b >= B) break;  // warp-uniform
            const uint32_t k = lane < 27 ? s_k[w][i][lane] : 0xffffffffu;
            const uint32_t cl = lane < 27 ? s_c[w][i][lane] : 0u;
            const bool ok = k != 0xffffffffu;
            const uint32_t m = __ballot_sync(FULL, ok);
            const uint32_t e0 = __shfl_sync(FULL, o_nbr, i);
            const unsigned long long rb = __shfl_sync(FULL, o_red, i);
            uint32_t incl = cl;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, incl, o);
                if (lane >= (unsigned)o) incl += y;
            }
            // records of the slots before the centre (13) = offset of the box's own segment in its run
            const uint32_t cen = __shfl_sync(FULL, incl - cl, 13);
            if (ok) {
                const uint32_t e = e0 + __popc(m & ((1u << lane) - 1u));
                nbr_box[e] = k;
                nbr_slot[e] = (uint8_t)lane;
                if ((e & 31u) == 0u) {  // head of a restructure chunk
                    chunk_box[e >> 5] = b;
                    chunk_out[e >> 5] = rb + (incl - cl);
                }
            }
            const bool tgt = __shfl_sync(FULL, (uint32_t)mtarget, i) != 0u;
            if (!tgt) continue;
            const uint32_t s0 = __shfl_sync(FULL, ms0, i), nb_b = __shfl_sync(FULL, my_nb, i);
            const uint32_t nch = __shfl_sync(FULL, my_item, i);
            if (nch == 0) {  // small box: thread-per-target path, one entry per target pair
                const uint32_t so = __shfl_sync(FULL, o_small, i);
                if (lane < (nb_b + 1) / 2) {
                    small_tgt[so + lane] = s0 + 2 * lane;
                    small_box[so + lane] = b;
                }
                continue;
            }
            const uint32_t it = __shfl_sync(FULL, o_item, i);
            const uint32_t key = __shfl_sync(FULL, mkey, i);
            const uint32_t Rb = (uint32_t)__shfl_sync(FULL, my_red, i);
            for (uint32_t ci = lane; ci < nch; ci += 32) {
                const uint32_t a0 = (uint32_t)(((uint64_t)nb_b * ci) / nch);
                const uint32_t z0 = (uint32_t)(((uint64_t)nb_b * (ci + 1)) / nch);
                // eval lane layout: G = ceil(n_t / K) groups of K targets, S = floor(32 / G) source splits
                const uint32_t nt = z0 - a0, G = (nt + K - 1) / K, S = 32u / G;
                items[it + ci] = Item{b, s0 + a0, nt | (S << 8) | (G << 16), key, rb, Rb, cen + a0};
            }
        }
        __syncwarp();  // phase C's shared-memory reads before the next tile's phase A writes
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pairs += __shfl_xor_sync(FULL, pairs, o);
    if (lane == 0 && pairs) atomicAdd(&ctr->I, pairs);
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
                    P->s_nb_status, P->boxinfo,
                    P->small_tgt, P->small_box, P->chunk_box, P->chunk_out, P->rec, P->bkey, P->bstart,
                    P->nbr_off, P->nbr_box, P->nbr_slot, P->red_off, P->box_of, P->items, P->occ};
    for (void *b : bufs) dfree(b, st);
    P->s_key = P->s_idx = P->s_kalt = P->s_valt = P->s_hist = P->s_status = nullptr;
    P->s_partials = nullptr;
    P->s_nb_status = nullptr;
    P->boxinfo = nullptr;
    P->small_tgt = P->small_box = P->chunk_box = nullptr;
    P->chunk_out = nullptr;
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
        P2P_CUDA_TRY(dalloc((void **)&P->s_nb_status, sizeof(NbTileStatus) * div_up(bcap, NBB_TILE), st));
        P2P_CUDA_TRY(dalloc((void **)&P->boxinfo, sizeof(uint2) * keyspace, st));
        P2P_CUDA_TRY(dalloc((void **)&P->small_tgt, 4 * n, st));
        P2P_CUDA_TRY(dalloc((void **)&P->small_box, 4 * n, st));
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
    const uint64_t ntile_cap = div_up(bcap, NBB_TILE);
    P2P_LAUNCH(k_boxinfo, std::max<unsigned>(1, std::min<unsigned>(div_up(bcap, 256), (unsigned)P->num_sms * 8)), 256,
               0, st, P->bkey, P->bstart, P->ctr, P->boxinfo);
    P2P_CUDA_TRY(cudaMemsetAsync(P->s_nb_status, 0, sizeof(NbTileStatus) * ntile_cap, st));
    P2P_CUDA_TRY(cudaMemsetAsync(&P->ctr->nbr_tile, 0, sizeof(unsigned int), st));
    P2P_LAUNCH(k_nbr_build, std::max<unsigned>(1, std::min<unsigned>(div_up(ntile_cap, NBB_WARPS), (unsigned)P->num_sms * 8)),
               NBB_WARPS * 32, 0, st, P->geom, P->bkey, P->bstart, P->boxinfo, P->occ, P->ctr, P->s_nb_status,
               P->nbr_off, (unsigned long long *)P->red_off, P->nbr_box, P->nbr_slot, P->items, P->small_tgt,
               P->small_box, P->chunk_box, P->chunk_out, (uint32_t)(f64 ? EVAL_K_F64 : EVAL_K_F32),
               (uint32_t)ITEM_TMAX);
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
