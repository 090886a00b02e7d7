// k_restructure.cu -- method step a6, the paper's data redundancy (§1.1 "duplicating neighbor data
// ... threads can access all required neighbor information from a compact, contiguous region"
// §5.2.1; restructuring cost P:L386 §5.2.3 item 1).
//
// Gravity: for every target box b and every neighbour (k, slot) in CSR order, copy box k's Morton-sorted
// records into ONE contiguous run red[red_off[b] ..), rebased to b's origin in fp64 with a single
// rounding to the working precision (DESIGN C11):
//     red = { fl_p(((double)x_j + S_x) - o_bx), ..y.., ..z.., m_j },  o_bd = fma(ib_d, h, lo_d)
// One warp per box; the warp's 32 lanes cover the run's records contiguously (coalesced 16 B stores), each
// lane finding its source segment by a shuffle binary search over the <= 27 segment starts held in lanes.
// Bound: HBM -- writes 16 R bytes (fp32), reads 16 N_src bytes compulsory (repeats hit L2 in Morton order).
//
// Helmholtz: Xg[b][s][j] = xs[bstart[nbr9[b][s]] + j] or 0 (zero-padded im2col, DESIGN C10), one thread
// per element, fully coalesced.
#include "plan.hpp"

namespace p2p {

namespace {
template <typename T> struct V4T;
template <> struct V4T<float> { using type = float4; };
template <> struct V4T<double> { using type = double4; };

// image shift of stencil slot `slot` seen from box c (DESIGN C5): +L past the upper face, -L past the lower
__device__ __forceinline__ double slot_shift(const Geom &g, const uint32_t c[3], int slot, int d) {
    const int dd = d == 0 ? slot % 3 - 1 : (d == 1 ? (slot / 3) % 3 - 1 : slot / 9 - 1);
    const int v = (int)c[d] + dd;
    if (v >= g.nbox[d]) return g.L[d];
    if (v < 0) return -g.L[d];
    return 0.0;
}

template <typename T>
__global__ void __launch_bounds__(256) k_restructure_gravity(const Geom g, const typename V4T<T>::type *__restrict__ rec,
                                                             const uint32_t *__restrict__ bkey,
                                                             const uint32_t *__restrict__ bstart,
                                                             const uint32_t *__restrict__ nbr_off,
                                                             const uint32_t *__restrict__ nbr_box,
                                                             const uint8_t *__restrict__ nbr_slot,
                                                             const uint64_t *__restrict__ red_off,
                                                             const DevCounters *__restrict__ ctr,
                                                             typename V4T<T>::type *__restrict__ red) {
    using V4 = typename V4T<T>::type;
    const uint32_t B = ctr->B;  // device-side count: no host sync needed after an async p2p_plan_update
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < B; b += nwarps) {
        const uint32_t key = bkey[b];
        const uint32_t c[3] = {compact3(key), compact3(key >> 1), compact3(key >> 2)};
        const double o0 = __fma_rn((double)c[0], g.h, g.lo[0]);
        const double o1 = __fma_rn((double)c[1], g.h, g.lo[1]);
        const double o2 = __fma_rn((double)c[2], g.h, g.lo[2]);
        const uint32_t e0 = nbr_off[b], ne = nbr_off[b + 1] - e0;
        // lane e < ne holds segment e: source start, length, and the image code of its slot
        // (2 bits per dim: 1 = +L, 2 = -L, computed once per segment instead of once per record)
        uint32_t src = 0, cnt = 0, code = 0;
        if (lane < ne) {
            const uint32_t k = nbr_box[e0 + lane];
            src = bstart[k];
            cnt = bstart[k + 1] - src;
            const int slot = nbr_slot[e0 + lane];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const double S = slot_shift(g, c, slot, d);
                code |= (S > 0.0 ? 1u : (S < 0.0 ? 2u : 0u)) << (2 * d);
            }
        }
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (unsigned)o) incl += y;
        }
        const uint32_t st = incl - cnt;
        const uint32_t Rb = __shfl_sync(0xffffffffu, incl, 31);
        V4 *__restrict__ out = red + red_off[b];
        const bool seg = lane < ne;
        const uint32_t le = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
        // UNR windows of 32 records per iteration: all loads issued before the first store (memory-level
        // parallelism: the kernel is latency-bound otherwise)
        constexpr int UNR = 4;
        for (uint32_t rb = 0; rb < Rb; rb += 32 * UNR) {
            V4 x[UNR];
            uint32_t xcode[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const uint32_t r0 = rb + 32u * u;
                if (r0 >= Rb) break;  // warp-uniform: short runs skip the empty windows
                // segment of record r0 + lane without a search (segments are non-empty and contiguous):
                // segments starting before r0 (ballot) - 1 + segment starts in [r0, r0 + lane] (OR-reduced mask)
                const uint32_t before = __popc(__ballot_sync(0xffffffffu, seg && st < r0));
                const uint32_t in_win = (seg && st >= r0 && st < r0 + 32) ? (1u << (st - r0)) : 0u;
                const uint32_t starts = __reduce_or_sync(0xffffffffu, in_win);
                const uint32_t e = (before - 1u + __popc(starts & le)) & 31u;
                const uint32_t e_src = __shfl_sync(0xffffffffu, src, e);
                const uint32_t e_st = __shfl_sync(0xffffffffu, st, e);
                xcode[u] = __shfl_sync(0xffffffffu, code, e);
                const uint32_t r = r0 + lane;
                if (r < Rb) x[u] = rec[e_src + (r - e_st)];
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const uint32_t r = rb + 32u * u + lane;
                if (r < Rb) {
                    const uint32_t cd = xcode[u];
                    const double S0 = (cd & 1u) ? g.L[0] : ((cd & 2u) ? -g.L[0] : 0.0);
                    const double S1 = (cd & 4u) ? g.L[1] : ((cd & 8u) ? -g.L[1] : 0.0);
                    const double S2 = (cd & 16u) ? g.L[2] : ((cd & 32u) ? -g.L[2] : 0.0);
                    V4 v;
                    v.x = (T)__dsub_rn(__dadd_rn((double)x[u].x, S0), o0);
                    v.y = (T)__dsub_rn(__dadd_rn((double)x[u].y, S1), o1);
                    v.z = (T)__dsub_rn(__dadd_rn((double)x[u].z, S2), o2);
                    v.w = x[u].w;
                    out[r] = v;
                }
            }
        }
    }
}

template <typename C2>
__global__ void k_restructure_helmholtz(const C2 *__restrict__ xs, const uint32_t *__restrict__ bstart,
                                        const uint32_t *__restrict__ nbr9, uint32_t B, uint32_t t,
                                        C2 *__restrict__ Xg) {
    const uint64_t total = (uint64_t)B * 9 * t;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t bs = i / t;
        const uint32_t j = (uint32_t)(i - bs * t);
        const uint32_t k = nbr9[bs];
        C2 v;
        if (k != 0xffffffffu) v = xs[bstart[k] + j];
        else { v.x = 0; v.y = 0; }
        Xg[i] = v;
    }
}
}  // namespace

p2p_status restructure_gravity(p2p_plan *P) {
    if (P->sizes_known && P->B == 0) return P2P_OK;
    const uint64_t nb = P->sizes_known ? (uint64_t)P->B : (uint64_t)P->bcap;
    const unsigned grid = std::max<unsigned>(1, std::min<unsigned>(div_up(nb * 32, 256), (unsigned)P->num_sms * 16));
    if (P->cfg.precision == P2P_FP64)
        P2P_LAUNCH(k_restructure_gravity<double>, grid, 256, 0, P->stream, P->geom, (const double4 *)P->rec, P->bkey,
                   P->bstart, P->nbr_off, P->nbr_box, P->nbr_slot, P->red_off, P->ctr, (double4 *)P->red);
    else
        P2P_LAUNCH(k_restructure_gravity<float>, grid, 256, 0, P->stream, P->geom, (const float4 *)P->rec, P->bkey,
                   P->bstart, P->nbr_off, P->nbr_box, P->nbr_slot, P->red_off, P->ctr, (float4 *)P->red);
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}

p2p_status restructure_helmholtz(p2p_plan *P) {
    if (P->B == 0) return P2P_OK;
    const uint32_t t = (uint32_t)P->cfg.points_per_box;
    const uint64_t total = (uint64_t)P->B * 9 * t;
    const unsigned grid = std::min<unsigned>(div_up(total, 256), (unsigned)P->num_sms * 16);
    if (P->cfg.precision == P2P_FP64)
        P2P_LAUNCH(k_restructure_helmholtz<double2>, grid, 256, 0, P->stream, (const double2 *)P->rec, P->bstart,
                   P->nbr_box, (uint32_t)P->B, t, (double2 *)P->red);
    else
        P2P_LAUNCH(k_restructure_helmholtz<float2>, grid, 256, 0, P->stream, (const float2 *)P->rec, P->bstart,
                   P->nbr_box, (uint32_t)P->B, t, (float2 *)P->red);
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}

}  // namespace p2p
