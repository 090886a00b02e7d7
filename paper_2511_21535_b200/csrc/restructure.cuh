// restructure.cuh -- the a6 per-chunk restructure body (§1.1, §5.2.1; DESIGN C11) of
// k_restructure_gravity (k_restructure.cu), kept callable from other kernels (the round-1 fused
// restructure+eval experiment, ran it inside the eval kernel).
//
// A chunk = 32 consecutive CSR entries e = 32 ch .. 32 ch + 31.  Their source segments are consecutive in red[]
// (CSR order = run order, runs of consecutive boxes are adjacent): one contiguous output range starting at
// chunk_out[ch], even when the chunk spans several small boxes.  The warp loads the entries' segments and the
// <= 32 owner boxes' keys, finds each entry's owner by a 5-step shuffle binary search, and copies windows of 32
// records, rebased in fp64 with one final rounding:
//     red = { fl_p(((double)x_j + S_x) - o_bx), ..y.., ..z.., m_j },  o_bd = fma(ib_d, h, lo_d)
#pragma once
#include "plan.hpp"

namespace p2p {
namespace rs {

template <typename T> struct V4T;
template <> struct V4T<float> { using type = float4; };
template <> struct V4T<double> { using type = double4; };

template <typename T>
struct Ptrs {
    const typename V4T<T>::type *rec;
    const uint32_t *bkey, *bstart, *nbr_off, *nbr_box;
    const uint8_t *nbr_slot;
    const uint32_t *chunk_box;
    const unsigned long long *chunk_out;
    typename V4T<T>::type *red;
};

// image shift of stencil slot `slot` seen from box c (DESIGN C5): +L past the upper face, -L past the lower
__device__ __forceinline__ double slot_shift(const Geom &g, const uint32_t c[3], int slot, int d) {
    const int dd = d == 0 ? slot % 3 - 1 : (d == 1 ? (slot / 3) % 3 - 1 : slot / 9 - 1);
    const int v = (int)c[d] + dd;
    if (v >= g.nbox[d]) return g.L[d];
    if (v < 0) return -g.L[d];
    return 0.0;
}

// Restructure chunk `ch` given its level-1 values (head box b0, output offset gout, lane e's CSR entry k / slot,
// loaded by the caller -- the standalone kernel one chunk ahead).  Returns the chunk's record count Rc.
// EXACT32: the host verified that every box origin of the grid is an fp32 value (fp32 fast path, see below).
// red[] records are written once and read back only by the next kernel, after a 4.75 GB stream: streaming
// (evict-first) stores keep them from evicting the rec[] lines the chunk gathers re-read from L2 (c5w: 1.27 ->
// 1.18 ms; an evict-last policy on the rec[] loads instead gained nothing)
__device__ __forceinline__ void st_cs(float4 *p, const float4 &v) { __stcs(p, v); }
__device__ __forceinline__ void st_cs(double4 *p, const double4 &v) {
    __stcs(reinterpret_cast<double2 *>(p), make_double2(v.x, v.y));
    __stcs(reinterpret_cast<double2 *>(p) + 1, make_double2(v.z, v.w));
}

#ifndef P2P_RS_PACKED
#define P2P_RS_PACKED 1
#endif
#ifndef P2P_RS_ONESHFL
#define P2P_RS_ONESHFL 1
#endif
#ifndef P2P_RS_SENT
#define P2P_RS_SENT 1
#endif
#ifndef P2P_RS_ICODE
#define P2P_RS_ICODE 1
#endif
template <typename T, bool EXACT32>
__device__ __forceinline__ uint32_t chunk(const Geom &g, const Ptrs<T> &p, uint32_t B, uint32_t n_nbr, uint32_t ch,
                                          uint32_t b0, unsigned long long gout, uint32_t n_k, uint32_t n_slot,
                                          unsigned lane) {
    using V4 = typename V4T<T>::type;
    constexpr unsigned FULL = 0xffffffffu;
    const uint32_t e = (ch << 5) + lane;
    const bool seg = e < n_nbr;
    const uint32_t k = seg ? n_k : 0u, slot = seg ? n_slot : 13u;
    // ---- level 2: boxes b0 .. b0 + 31 (CSR starts, keys) and lane e's source segment ----
    const uint32_t bl = b0 + lane;
    uint32_t boff = 0xffffffffu, keyl = 0;
    if (bl < B) {
        boff = p.nbr_off[bl];
        keyl = p.bkey[bl];
    }
    uint32_t src = 0, cnt = 0;
    if (seg) {
        src = p.bstart[k];
        cnt = p.bstart[k + 1] - src;
    }
    // owner of entry e: the largest i with nbr_off[b0 + i] <= e (non-decreasing in i; every target box owns
    // >= 1 entry, so the chunk's <= 32 entries belong to boxes b0 .. b0 + 31)
    uint32_t i = 0;
#pragma unroll
    for (uint32_t step = 16; step > 0; step >>= 1) {
        const uint32_t t = __shfl_sync(FULL, boff, i + step);
        if (t <= e) i += step;
    }
    const uint32_t key = __shfl_sync(FULL, keyl, i);
    const uint32_t c[3] = {compact3(key), compact3(key >> 1), compact3(key >> 2)};
    const double o0 = __fma_rn((double)c[0], g.h, g.lo[0]);
    const double o1 = __fma_rn((double)c[1], g.h, g.lo[1]);
    const double o2 = __fma_rn((double)c[2], g.h, g.lo[2]);
    // image code of the entry's slot (2 bits per dim: 1 = +L, 2 = -L), once per segment
    uint32_t code = 0;
#if P2P_RS_ICODE
    {  // integer form of slot_shift's sign (L > 0): +L past the upper face, -L past the lower
        const int so[3] = {(int)(slot % 3u) - 1, (int)((slot / 3u) % 3u) - 1, (int)(slot / 9u) - 1};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const int v = (int)c[d] + so[d];
            code |= (v >= g.nbox[d] ? 1u : (v < 0 ? 2u : 0u)) << (2 * d);
        }
    }
#else
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double S = slot_shift(g, c, (int)slot, d);
        code |= (S > 0.0 ? 1u : (S < 0.0 ? 2u : 0u)) << (2 * d);
    }
#endif
    // segments of consecutive CSR entries are consecutive in red[]: one contiguous output range per chunk
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= (unsigned)o) incl += y;
    }
    const uint32_t st = incl - cnt;
    const uint32_t src_m_st = src - st;
    const uint32_t stS = seg ? st : 0xffffffffu;
    const uint32_t Rc = __shfl_sync(FULL, incl, 31);
    V4 *__restrict__ out = p.red + gout;
    const uint32_t le = lane == 31 ? FULL : ((2u << lane) - 1u);
    // ---- level 3: UNR windows of 32 records per iteration, all loads issued before the first store ----
    // chunks without any periodic image (all but the boundary layers) skip the shift selection: adding the
    // +0.0 shift keeps the oracle's rounding sequence (and its -0 -> +0 behaviour) exactly
    const bool wrap = __any_sync(FULL, seg && code != 0u);
    // fp32 fast path (C11 unchanged bit for bit): with no periodic shift and every owner origin exactly an
    // fp32 value, fl32(fl64(x + 0) - o) == fl32(fl32(x + 0) - o) -- a single subtraction of two fp32
    // operands rounded through fp64 (53 >= 2*24 + 2 bits) rounds like the direct fp32 subtraction -- so the
    // conversions and fp64 operations (6 F2F on the XU pipe per record) drop out
    const float f0o = (float)o0, f1o = (float)o1, f2o = (float)o2;
    const bool fast32 = EXACT32 && !wrap;
    const double L0 = g.L[0], L1 = g.L[1], L2 = g.L[2];
#ifndef P2P_RS_UNR
#define P2P_RS_UNR 4
#endif
    constexpr int UNR = P2P_RS_UNR;
    for (uint32_t rb = 0; rb < Rc; rb += 32 * UNR) {
        V4 x[UNR];
        uint32_t xe[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint32_t r0 = rb + 32u * u;
            if (r0 >= Rc) break;  // warp-uniform: short ranges skip the empty windows
            // segment of record r0 + lane without a search (segments are non-empty and contiguous):
            // segments starting before r0 (ballot) - 1 + segment starts in [r0, r0 + lane] (OR-reduced mask)
#if P2P_RS_SENT
            // stS = st, or ~0 for lanes past the CSR end: no per-window "seg &&"; the entry index is always in
            // [0, 31] (segments are contiguous from record 0), so no mask either
            const uint32_t before = __popc(__ballot_sync(FULL, stS < r0));
            const uint32_t d0 = stS - r0;
            const uint32_t in_win = d0 < 32u ? (1u << d0) : 0u;
            const uint32_t starts = __reduce_or_sync(FULL, in_win);
            xe[u] = before - 1u + __popc(starts & le);
#else
            const uint32_t before = __popc(__ballot_sync(FULL, seg && st < r0));
            const uint32_t in_win = (seg && st >= r0 && st < r0 + 32) ? (1u << (st - r0)) : 0u;
            const uint32_t starts = __reduce_or_sync(FULL, in_win);
            xe[u] = (before - 1u + __popc(starts & le)) & 31u;
#endif
            // one shuffle: the entry's (source start - run offset), so record r of the window is rec[sd + r]
            // (mod 2^32 arithmetic: sd may wrap, the sum never exceeds the record count)
#if P2P_RS_ONESHFL
            const uint32_t sd = __shfl_sync(FULL, src_m_st, xe[u]);
#else
            const uint32_t sd = __shfl_sync(FULL, src, xe[u]) - __shfl_sync(FULL, st, xe[u]);
#endif
            const uint32_t r = r0 + lane;
            if (r < Rc) x[u] = p.rec[sd + r];
        }
        if (fast32) {
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const uint32_t r0 = rb + 32u * u;
                if (r0 >= Rc) break;
                const float eo0 = __shfl_sync(FULL, f0o, xe[u]);
                const float eo1 = __shfl_sync(FULL, f1o, xe[u]);
                const float eo2 = __shfl_sync(FULL, f2o, xe[u]);
                const uint32_t r = r0 + lane;
                if (r < Rc) {
                    V4 v;
#if P2P_RS_PACKED
                    // x, y as one FP32x2 pair (FADD2): fl(fl(x + 0) + (-o)) == fl(fl(x + 0) - o) bit for bit
                    const float2 xy = __fadd2_rn(__fadd2_rn(make_float2((float)x[u].x, (float)x[u].y),
                                                            make_float2(0.0f, 0.0f)),
                                                 make_float2(-eo0, -eo1));
                    v.x = (T)xy.x;
                    v.y = (T)xy.y;
#else
                    v.x = (T)__fsub_rn(__fadd_rn((float)x[u].x, 0.0f), eo0);
                    v.y = (T)__fsub_rn(__fadd_rn((float)x[u].y, 0.0f), eo1);
#endif
                    v.z = (T)__fsub_rn(__fadd_rn((float)x[u].z, 0.0f), eo2);
                    v.w = x[u].w;
                    st_cs(out + r, v);
                }
            }
            continue;
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint32_t r0 = rb + 32u * u;
            if (r0 >= Rc) break;
            const double eo0 = __shfl_sync(FULL, o0, xe[u]);
            const double eo1 = __shfl_sync(FULL, o1, xe[u]);
            const double eo2 = __shfl_sync(FULL, o2, xe[u]);
            double S0 = 0.0, S1 = 0.0, S2 = 0.0;
            if (wrap) {
                const uint32_t cd = __shfl_sync(FULL, code, xe[u]);
                S0 = (cd & 1u) ? L0 : ((cd & 2u) ? -L0 : 0.0);
                S1 = (cd & 4u) ? L1 : ((cd & 8u) ? -L1 : 0.0);
                S2 = (cd & 16u) ? L2 : ((cd & 32u) ? -L2 : 0.0);
            }
            const uint32_t r = r0 + lane;
            if (r < Rc) {
                V4 v;
                v.x = (T)__dsub_rn(__dadd_rn((double)x[u].x, S0), eo0);
                v.y = (T)__dsub_rn(__dadd_rn((double)x[u].y, S1), eo1);
                v.z = (T)__dsub_rn(__dadd_rn((double)x[u].z, S2), eo2);
                v.w = x[u].w;
                st_cs(out + r, v);
            }
        }
    }
    return Rc;
}

}  // namespace rs

template <typename T>
inline rs::Ptrs<T> rs_ptrs(const p2p_plan *P) {
    using V4 = typename rs::V4T<T>::type;
    return rs::Ptrs<T>{(const V4 *)P->rec, P->bkey,     P->bstart,    P->nbr_off, P->nbr_box,
                       P->nbr_slot,        P->chunk_box, P->chunk_out, (V4 *)P->red};
}

}  // namespace p2p
