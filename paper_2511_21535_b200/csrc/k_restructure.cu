// k_restructure.cu -- method step a6, the paper's data redundancy (§1.1 "duplicating neighbor data
// ... threads can access all required neighbor information from a compact, contiguous region"
// §5.2.1; restructuring cost P:L386 §5.2.3 item 1).
//
// Gravity: for every target box b and every neighbour (k, slot) in CSR order, copy box k's Morton-sorted
// records into ONE contiguous run red[red_off[b] ..), rebased to b's origin in fp64 with a single
// rounding to the working precision (DESIGN C11):
//     red = { fl_p(((double)x_j + S_x) - o_bx), ..y.., ..z.., m_j },  o_bd = fma(ib_d, h, lo_d)
// One warp per CHUNK of 32 consecutive CSR entries (not per box): the entries' segments are consecutive in
// red[] (CSR order = run order, and runs of consecutive boxes are adjacent), so a chunk is one contiguous output
// range even when it spans several small boxes.  k_nbr_fill records each chunk's owner box and output start.
// Three dependent load levels per chunk (entry -> segment / owner box -> records) instead of four per box, and
// no per-box idle lanes: the Plummer workloads' median box has R ~ 20 records.  The 32 lanes cover the range
// contiguously (coalesced 16 B stores), each lane finding its segment from a ballot / OR-reduce over the
// segment starts held in lanes.
// Bound: HBM -- writes 16 R bytes (fp32), reads 16 N_src bytes compulsory (repeats hit L2 in Morton order).
//
// Helmholtz: Xg[b][s][j] = xs[bstart[nbr9[b][s]] + j] or 0 (zero-padded im2col, DESIGN C10), one thread
// per 16-byte vector (per element when a row of t complex values is not a 16-byte multiple), fully coalesced.
#include <cmath>

#include "plan.hpp"
#include "restructure.cuh"

namespace p2p {

namespace {
template <typename T, bool EXACT32>
__global__ void __launch_bounds__(256) k_restructure_gravity(const Geom g, const rs::Ptrs<T> p,
                                                             const DevCounters *__restrict__ ctr) {
    // device-side counts: no host sync needed after an asynchronous p2p_plan_update
    const uint32_t B = ctr->B, n_nbr = ctr->n_nbr;
    const uint32_t nchunk = (n_nbr + 31u) >> 5;
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    // level 1 of a chunk: its head and lane e's CSR entry -- loaded one chunk ahead (software pipeline)
    uint32_t n_b0 = 0, n_k = 0, n_slot = 13;
    unsigned long long n_gout = 0;
    auto load1 = [&](uint32_t c) {
        if (c < nchunk) {
            n_b0 = p.chunk_box[c];
            n_gout = p.chunk_out[c];
            const uint32_t ee = (c << 5) + lane;
            if (ee < n_nbr) {
                n_k = p.nbr_box[ee];
                n_slot = p.nbr_slot[ee];
            }
        }
    };
    uint32_t ch = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    load1(ch);
    for (; ch < nchunk; ch += nw) {
        const uint32_t b0 = n_b0, k = n_k, slot = n_slot;
        const unsigned long long gout = n_gout;
        load1(ch + nw);
        rs::chunk<T, EXACT32>(g, p, B, n_nbr, ch, b0, gout, k, slot, lane);
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

// the same im2col with 16-byte vectors: thread per 16 B of Xg (rows of t complex values are 16-byte multiples when
// t * sizeof(C2) is; the lattice is regular, so bstart[k] = k t and the source rows are 16-byte aligned too);
// 32-bit indexing, a shift instead of the 64-bit division per element (c2b 0.142 -> 0.088 ms, c2a 0.044 -> 0.031)
template <bool POW2>
__global__ void __launch_bounds__(256) k_restructure_helmholtz_v(const uint4 *__restrict__ xs, uint32_t esz,
                                                                 const uint32_t *__restrict__ bstart,
                                                                 const uint32_t *__restrict__ nbr9, uint32_t rows,
                                                                 uint32_t n16, uint32_t sh, uint4 *__restrict__ Xg) {
    const uint32_t total = rows * n16;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < total; v += gridDim.x * blockDim.x) {
        const uint32_t row = POW2 ? v >> sh : v / n16;
        const uint32_t j = v - row * n16;
        const uint32_t k = __ldg(nbr9 + row);
        uint4 x = make_uint4(0u, 0u, 0u, 0u);  // missing neighbour: +0.0 real and imaginary (C10)
        if (k != 0xffffffffu) x = __ldg(xs + (size_t)__ldg(bstart + k) * esz / 16u + j);
        Xg[v] = x;
    }
}
}  // namespace

// every box origin o_d = fma(c, h, lo_d), c < nbox_d, is exactly an fp32 value (the restructure's fp32 path)
bool origins_exact_fp32(const Geom &g) {
    for (int d = 0; d < 3; ++d)
        for (int c = 0; c < g.nbox[d]; ++c) {
            const double o = std::fma((double)c, g.h, g.lo[d]);
            if ((double)(float)o != o) return false;
        }
    return true;
}

p2p_status restructure_gravity(p2p_plan *P) {
    if (P->sizes_known && (P->B == 0 || P->n_nbr == 0)) return P2P_OK;
    // one warp per chunk of 32 CSR entries; the chunk count is device-side after an asynchronous update
    const uint64_t nchunk = div_up(P->sizes_known ? (uint64_t)P->n_nbr : 27ull * (uint64_t)P->bcap, 32);
    const unsigned grid = std::max<unsigned>(1, std::min<unsigned>(div_up(nchunk * 32, 256), (unsigned)P->num_sms * 16));
    if (P->cfg.precision == P2P_FP64)
        P2P_LAUNCH((k_restructure_gravity<double, false>), grid, 256, 0, P->stream, P->geom, rs_ptrs<double>(P), P->ctr);
    else if (origins_exact_fp32(P->geom))
        P2P_LAUNCH((k_restructure_gravity<float, true>), grid, 256, 0, P->stream, P->geom, rs_ptrs<float>(P), P->ctr);
    else
        P2P_LAUNCH((k_restructure_gravity<float, false>), grid, 256, 0, P->stream, P->geom, rs_ptrs<float>(P), P->ctr);
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}

p2p_status restructure_helmholtz(p2p_plan *P) {
    if (P->B == 0) return P2P_OK;
    const uint32_t t = (uint32_t)P->cfg.points_per_box;
    const uint64_t total = (uint64_t)P->B * 9 * t;
    const uint32_t esz = P->cfg.precision == P2P_FP64 ? 16u : 8u;
    const uint64_t rows = (uint64_t)P->B * 9;
    if ((t * esz) % 16 == 0 && rows * (t * esz / 16) < (1ull << 32)) {
        const uint32_t n16 = t * esz / 16;
        const bool pow2 = (n16 & (n16 - 1)) == 0;
        const uint32_t sh = pow2 ? (uint32_t)__builtin_ctz(n16) : 0u;
        const unsigned g16 = std::min<unsigned>(div_up(rows * n16, 256), (unsigned)P->num_sms * 16);
        if (pow2)
            P2P_LAUNCH(k_restructure_helmholtz_v<true>, g16, 256, 0, P->stream, (const uint4 *)P->rec, esz, P->bstart,
                       P->nbr_box, (uint32_t)rows, n16, sh, (uint4 *)P->red);
        else
            P2P_LAUNCH(k_restructure_helmholtz_v<false>, g16, 256, 0, P->stream, (const uint4 *)P->rec, esz,
                       P->bstart, P->nbr_box, (uint32_t)rows, n16, sh, (uint4 *)P->red);
        P2P_CUDA_TRY(cudaGetLastError());
        return P2P_OK;
    }
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
