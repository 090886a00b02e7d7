// k_eval_gravity.cu -- method steps a7 (softened-gravity P2P evaluation) + a9 (scatter to input order).
//
// What it computes (DESIGN C1-C3, C12-C14; SPEC S:L253 kernel form):
//   phi_i = - sum_{j != i} m_j (r^2 + eps^2)^{-1/2},   a_i = sum_j m_j d_ij (r^2 + eps^2)^{-3/2}
// over the sources of target i's box neighbourhood, in one of three source layouts:
//   P2P_REDUNDANT        sources = the box's contiguous run red[red_off[b] .. red_off[b+1]) built by
//                        p2p_restructure (the paper's redundant layout, §5.2.1): ONE 1D TMA bulk copy
//                        (cp.async.bulk, SASS UBLKCP) per chunk of the run.
//   P2P_INDEXED          non-redundant baseline (§5.2.1): the <= 27 neighbour segments of the
//                        Morton-sorted records rec[], located through the CSR, one bulk copy per segment piece;
//                        absolute fp32 coordinates, periodic images applied as exact +-L shifts.
//   P2P_INDEXED_BITWISE  as INDEXED, then each staged record is rebased in shared memory exactly like a red[]
//                        record, so the arithmetic and the outputs equal P2P_REDUNDANT bit for bit.
//
// B200 design (the paper's GTX 1050 thread-per-particle kernel is prior art, not the blueprint):
//   * persistent CTAs (EV_WARPS warps each); every warp pulls work items (box, target chunk) from a global
//     atomic queue and runs its own 2-stage producer/consumer pipeline: while it computes chunk c from one
//     shared-memory stage, the bulk copy of chunk c+1 (possibly the next item's first chunk) lands in the
//     other stage, completion tracked by an mbarrier with expect_tx.
//   * targets live in registers: lane (g, s) holds K targets (group g) and walks the staged sources
//     j = s, s+S, ... (S = floor(32/G) source splits, G = ceil(n_t/K) groups), so a box of any occupancy keeps
//     (almost) all 32 lanes busy; the S partial sums are combined by a fixed shuffle tree (deterministic).
//   * inner loop per (source, target): 3 FADD + 3 FFMA + MUFU.RSQ + FMUL + FADD + 2 FMUL + 3 FFMA = 13 FP32-pipe
//     instructions + 1 MUFU (fp32) -> the FP32 pipe is the roofline.  The self pair
//     (d = 0, r^2 = eps^2) is evaluated like any other and its potential term subtracted bit-exactly after
//     the loop (DESIGN C3).
#include "plan.hpp"

namespace p2p {

namespace {
template <typename T> struct V4T;
template <> struct V4T<float> { using type = float4; };
template <> struct V4T<double> { using type = double4; };

constexpr int EV_WARPS = 4;              // warps per CTA
constexpr int EV_STAGE_BYTES = 4096;     // one pipeline stage per warp (256 fp32 / 128 fp64 records)

template <typename T>
struct EvalArgs {
    Geom g;
    const typename V4T<T>::type *rec;
    const typename V4T<T>::type *red;
    const uint32_t *bkey, *bstart, *nbr_off, *nbr_box;
    const uint8_t *nbr_slot;
    const uint64_t *red_off;
    const uint32_t *perm;
    const Item *items;
    uint32_t n_items;
    unsigned int *item_head;
    T *phi;
    T *field;
};

template <typename T>
__device__ __forceinline__ T rinv_of(T r2);
template <>
__device__ __forceinline__ float rinv_of<float>(float r2) { return rsqrt_ftz(r2); }
template <>
__device__ __forceinline__ double rinv_of<double>(double r2) { return 1.0 / sqrt(r2); }

template <typename T>
__device__ __forceinline__ T fma_(T a, T b, T c);
template <>
__device__ __forceinline__ float fma_<float>(float a, float b, float c) { return __fmaf_rn(a, b, c); }
template <>
__device__ __forceinline__ double fma_<double>(double a, double b, double c) { return __fma_rn(a, b, c); }

// image shift of stencil slot seen from box c (DESIGN C5)
__device__ __forceinline__ double slot_shift(const Geom &g, const uint32_t c[3], int slot, int d) {
    const int dd = d == 0 ? slot % 3 - 1 : (d == 1 ? (slot / 3) % 3 - 1 : slot / 9 - 1);
    const int v = (int)c[d] + dd;
    if (v >= g.nbox[d]) return g.L[d];
    if (v < 0) return -g.L[d];
    return 0.0;
}

// INDEXED frame of box c in dim d: boxes in the top layer of a periodic dim work in coordinates shifted by
// -L, so every image shift applied to a staged source is 0 or -L and (for lo = 0) every shift is exact
// (Sterbenz), see DESIGN §5.
__device__ __forceinline__ double frame_shift(const Geom &g, const uint32_t c[3], int d) {
    return (((g.periodic >> d) & 1u) && (int)c[d] == g.nbox[d] - 1) ? -g.L[d] : 0.0;
}

template <typename T, int LAYOUT, int K>
__global__ void __launch_bounds__(EV_WARPS * 32) k_eval_gravity(const EvalArgs<T> a) {
    using V4 = typename V4T<T>::type;
    constexpr int CH = EV_STAGE_BYTES / (int)sizeof(V4);
    constexpr unsigned FULL = 0xffffffffu;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[EV_WARPS][2];

    const int w = threadIdx.x >> 5;
    const unsigned lane = threadIdx.x & 31u;
    V4 *stage_base = reinterpret_cast<V4 *>(smem_raw + (size_t)w * 2 * EV_STAGE_BYTES);
    uint64_t *bar = bars[w];
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncwarp();

    const T eps2 = (T)a.g.eps2;

    // ---------------- producer state (item whose chunks are being copied in) ----------------
    uint32_t p_item, p_box = 0, p_R = 0, p_nch = 0;
    uint64_t p_base = 0;
    uint32_t p_src = 0, p_st = 0, p_cnt = 0, p_slot = 0, p_ne = 0;  // INDEXED: lane = segment

    auto fetch = [&]() -> uint32_t {
        uint32_t v = 0;
        if (lane == 0) v = atomicAdd(a.item_head, 1u);
        return __shfl_sync(FULL, v, 0);
    };
    auto load_item = [&](uint32_t idx) {
        const Item it = a.items[idx];
        p_box = it.box;
        if (LAYOUT == P2P_REDUNDANT) {
            p_base = a.red_off[p_box];
            p_R = (uint32_t)(a.red_off[p_box + 1] - p_base);
        } else {
            const uint32_t e0 = a.nbr_off[p_box];
            p_ne = a.nbr_off[p_box + 1] - e0;
            p_cnt = 0;
            if (lane < p_ne) {
                const uint32_t k = a.nbr_box[e0 + lane];
                p_src = a.bstart[k];
                p_cnt = a.bstart[k + 1] - p_src;
                p_slot = a.nbr_slot[e0 + lane];
            }
            uint32_t incl = p_cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(FULL, incl, o);
                if (lane >= (unsigned)o) incl += y;
            }
            p_st = incl - p_cnt;
            p_R = __shfl_sync(FULL, incl, 31);
        }
        p_nch = (p_R + CH - 1) / CH;
    };
    auto issue = [&](uint32_t chunk, int s) {
        const uint32_t c0 = chunk * CH;
        const uint32_t cnt = min((uint32_t)CH, p_R - c0);
        V4 *dst = stage_base + s * CH;
        if (lane == 0) {
            fence_proxy_async_smem();  // order earlier generic smem accesses of this stage before the async write
            mbar_arrive_expect_tx(&bar[s], cnt * (uint32_t)sizeof(V4));
        }
        __syncwarp();
        if (LAYOUT == P2P_REDUNDANT) {
            if (lane == 0) bulk_g2s(dst, a.red + p_base + c0, cnt * (uint32_t)sizeof(V4), &bar[s]);
        } else {
            const uint32_t ov0 = max(c0, p_st), ov1 = min(c0 + cnt, p_st + p_cnt);
            if (lane < p_ne && ov1 > ov0)
                bulk_g2s(dst + (ov0 - c0), a.rec + p_src + (ov0 - p_st), (ov1 - ov0) * (uint32_t)sizeof(V4), &bar[s]);
        }
    };

    p_item = fetch();
    if (p_item >= a.n_items) return;
    load_item(p_item);
    issue(0, 0);
    int s = 0;
    uint32_t phases = 0u;  // bit s = parity of stage s's mbarrier

    while (true) {
        // ---------------- adopt the producer's item as the current (consumer) item ----------------
        const Item it = a.items[p_item];
        const uint32_t c_box = p_box, c_R = p_R, c_nch = p_nch;
        const uint32_t c_st = p_st, c_cnt = p_cnt, c_slot = p_slot, c_ne = p_ne;
        const uint32_t key = a.bkey[c_box];
        const uint32_t cc[3] = {compact3(key), compact3(key >> 1), compact3(key >> 2)};
        double org[3];
#pragma unroll
        for (int d = 0; d < 3; ++d)
            org[d] = (LAYOUT == P2P_INDEXED) ? frame_shift(a.g, cc, d) : __fma_rn((double)cc[d], a.g.h, a.g.lo[d]);
        bool needs_fix = false;
        if (LAYOUT == P2P_INDEXED) {
#pragma unroll
            for (int d = 0; d < 3; ++d)
                needs_fix |= ((a.g.periodic >> d) & 1u) && (cc[d] == 0 || (int)cc[d] == a.g.nbox[d] - 1);
        }

        // lane layout: G groups of K targets, S source splits
        const uint32_t nt = it.nt;
        const uint32_t G = (nt + K - 1) / K;
        const uint32_t S = max(1u, 32u / G);
        const uint32_t g = lane / S, sl = lane - g * S;
        const bool active = g < G;

        T tx[K], ty[K], tz[K], ap[K], ax[K], ay[K], az[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t ti = g * K + k;
            T x = 0, y = 0, z = 0;
            if (active && ti < nt) {
                const V4 r = a.rec[it.t0 + ti];
                if (LAYOUT == P2P_INDEXED) {
                    x = r.x + (T)org[0];
                    y = r.y + (T)org[1];
                    z = r.z + (T)org[2];
                } else {
                    x = (T)__dsub_rn((double)r.x, org[0]);
                    y = (T)__dsub_rn((double)r.y, org[1]);
                    z = (T)__dsub_rn((double)r.z, org[2]);
                }
            }
            tx[k] = x; ty[k] = y; tz[k] = z;
            ap[k] = 0; ax[k] = 0; ay[k] = 0; az[k] = 0;
        }

        bool have_next = true;
        for (uint32_t c = 0; c < c_nch; ++c) {
            // prefetch the next chunk into the other stage
            if (c + 1 < c_nch) {
                issue(c + 1, s ^ 1);
            } else {
                p_item = fetch();
                if (p_item < a.n_items) {
                    load_item(p_item);
                    issue(0, s ^ 1);
                } else {
                    have_next = false;
                }
            }
            mbar_wait(&bar[s], (phases >> s) & 1u);
            phases ^= 1u << s;
            V4 *stg = stage_base + s * CH;
            const uint32_t c0 = c * CH;
            const uint32_t cnt = min((uint32_t)CH, c_R - c0);

            // ---- layout fix-ups of the staged raw records (INDEXED variants only) ----
            if (LAYOUT == P2P_INDEXED_BITWISE || (LAYOUT == P2P_INDEXED && needs_fix)) {
                for (uint32_t e = 0; e < c_ne; ++e) {
                    const uint32_t est = __shfl_sync(FULL, c_st, e), ecnt = __shfl_sync(FULL, c_cnt, e);
                    const int eslot = (int)__shfl_sync(FULL, c_slot, e);
                    const uint32_t ov0 = max(c0, est), ov1 = min(c0 + cnt, est + ecnt);
                    if (ov1 <= ov0) continue;
                    const double S0 = slot_shift(a.g, cc, eslot, 0), S1 = slot_shift(a.g, cc, eslot, 1),
                                 S2 = slot_shift(a.g, cc, eslot, 2);
                    if (LAYOUT == P2P_INDEXED) {
                        const T h0 = (T)(S0 + org[0]), h1 = (T)(S1 + org[1]), h2 = (T)(S2 + org[2]);
                        if (h0 == (T)0 && h1 == (T)0 && h2 == (T)0) continue;
                        for (uint32_t j = ov0 - c0 + lane; j < ov1 - c0; j += 32) {
                            V4 v = stg[j];
                            v.x += h0; v.y += h1; v.z += h2;
                            stg[j] = v;
                        }
                    } else {
                        for (uint32_t j = ov0 - c0 + lane; j < ov1 - c0; j += 32) {
                            V4 v = stg[j];
                            v.x = (T)__dsub_rn(__dadd_rn((double)v.x, S0), org[0]);
                            v.y = (T)__dsub_rn(__dadd_rn((double)v.y, S1), org[1]);
                            v.z = (T)__dsub_rn(__dadd_rn((double)v.z, S2), org[2]);
                            stg[j] = v;
                        }
                    }
                }
                __syncwarp();
            }

            // ---- the hot loop: staged sources x register targets ----
            if (active && sl < cnt) {
                const uint32_t nj = (cnt - 1 - sl) / S + 1;
                const V4 *sp = stg + sl;
#pragma unroll 2
                for (uint32_t q = 0; q < nj; ++q) {
                    const V4 src = sp[q * S];
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const T dx = src.x - tx[k];
                        const T dy = src.y - ty[k];
                        const T dz = src.z - tz[k];
                        T r2 = fma_(dx, dx, eps2);
                        r2 = fma_(dy, dy, r2);
                        r2 = fma_(dz, dz, r2);
                        const T ri = rinv_of<T>(r2);
                        const T mri = src.w * ri;
                        ap[k] += mri;
                        const T mri3 = mri * ri * ri;
                        ax[k] = fma_(mri3, dx, ax[k]);
                        ay[k] = fma_(mri3, dy, ay[k]);
                        az[k] = fma_(mri3, dz, az[k]);
                    }
                }
            }
            __syncwarp();
            s ^= 1;
        }

        // ---- combine the S source splits of each group (fixed shuffle tree -> deterministic) ----
        for (uint32_t off = 1; off < S; off <<= 1) {
            const bool take = sl + off < S;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                T v0 = __shfl_down_sync(FULL, ap[k], off), v1 = __shfl_down_sync(FULL, ax[k], off);
                T v2 = __shfl_down_sync(FULL, ay[k], off), v3 = __shfl_down_sync(FULL, az[k], off);
                if (take) { ap[k] += v0; ax[k] += v1; ay[k] += v2; az[k] += v3; }
            }
        }
        // ---- a9: scatter to input order; remove the self potential term (DESIGN C3) ----
        if (active && sl == 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const uint32_t ti = g * K + k;
                if (ti < nt) {
                    const uint32_t p = it.t0 + ti;
                    const uint32_t i = a.perm[p];
                    const T m = a.rec[p].w;
                    const T self = m * rinv_of<T>(fma_((T)0, (T)0, eps2));
                    a.phi[i] = -(ap[k] - self);
                    if (a.field) {
                        a.field[3 * (size_t)i + 0] = ax[k];
                        a.field[3 * (size_t)i + 1] = ay[k];
                        a.field[3 * (size_t)i + 2] = az[k];
                    }
                }
            }
        }
        if (!have_next) break;
    }
}

template <typename T, int LAYOUT, int K>
p2p_status launch(p2p_plan *P, void *phi, void *field, int slot) {
    using V4 = typename V4T<T>::type;
    auto kern = k_eval_gravity<T, LAYOUT, K>;
    const int smem = EV_WARPS * 2 * EV_STAGE_BYTES;
    if (P->eval_blocks[slot] == 0) {
        P2P_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int per_sm = 0;
        P2P_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, EV_WARPS * 32, smem));
        P->eval_blocks[slot] = std::max(1, per_sm) * P->num_sms;
    }
    EvalArgs<T> a;
    a.g = P->geom;
    a.rec = (const V4 *)P->rec;
    a.red = (const V4 *)P->red;
    a.bkey = P->bkey;
    a.bstart = P->bstart;
    a.nbr_off = P->nbr_off;
    a.nbr_box = P->nbr_box;
    a.nbr_slot = P->nbr_slot;
    a.red_off = P->red_off;
    a.perm = P->perm;
    a.items = P->items;
    a.n_items = (uint32_t)P->n_items;
    a.item_head = &P->ctr->item_head;
    a.phi = (T *)phi;
    a.field = (T *)field;
    const unsigned grid =
        (unsigned)std::min<int64_t>(P->eval_blocks[slot], std::max<int64_t>(1, (P->n_items + EV_WARPS - 1) / EV_WARPS));
    P2P_CUDA_TRY(cudaMemsetAsync(&P->ctr->item_head, 0, sizeof(unsigned int), P->stream));
    P2P_LAUNCH(kern, grid, EV_WARPS * 32, smem, P->stream, a);
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}
}  // namespace

p2p_status eval_gravity(p2p_plan *P, p2p_layout layout, void *phi, void *field) {
    if (P->n_items == 0) return P2P_OK;
    const bool f64 = P->cfg.precision == P2P_FP64;
    switch (layout) {
    case P2P_REDUNDANT:
        return f64 ? launch<double, P2P_REDUNDANT, 2>(P, phi, field, 0) : launch<float, P2P_REDUNDANT, 4>(P, phi, field, 0);
    case P2P_INDEXED:
        return f64 ? launch<double, P2P_INDEXED, 2>(P, phi, field, 1) : launch<float, P2P_INDEXED, 4>(P, phi, field, 1);
    case P2P_INDEXED_BITWISE:
        return f64 ? launch<double, P2P_INDEXED_BITWISE, 2>(P, phi, field, 2)
                   : launch<float, P2P_INDEXED_BITWISE, 4>(P, phi, field, 2);
    }
    return P2P_ERR_INVALID_ARGUMENT;
}

}  // namespace p2p
