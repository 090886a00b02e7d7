// k_pairrec.cu -- SURVEY §8f NEXT-4: the paper's THREAD-level data redundancy (§5.2.1 "duplicating
// particle data for each interaction pair ... an Array-of-Structures (AoS) format, where each entry contains both
// source and target attributes"; partial results reduced "through the update process", §1.1).  A third
// point on the redundancy-granularity axis beside the box-level run (P2P_REDUNDANT) and no redundancy
// (P2P_INDEXED).
//
// Pair record of CSR entry e = (target box b, neighbour k, slot s), records in CSR order:
//     [ n_b target tuples : fl_p(((double)x_i + 0) - o_b), m_i ] [ n_k source tuples, rebased exactly like red ]
// i.e. bit for bit b's own (slot-13) segment of red followed by e's segment of red (DESIGN C11).  Record start
//     pr(e) = t_off[b] + red_off[b] + (e - nbr_off[b]) n_b + (records of b's earlier entries)
// with t_off = exclusive scan of |N(b)| n_b (= the partial-result slot base of box b).
// Eval: one lane per (record, target) reads its target tuple and the record's sources (the record is the only
// memory it touches) and writes one partial {phi, a} slot; the update sums every target's partials in ascending
// record order (deterministic) and scatters to input order (a9).
// Bound: HBM -- the records (16 (T + R) bytes, T = sum |N(b)| n_b = R by neighbour symmetry) are written once
// and streamed once, the partials (16 T bytes) written and read once; the pair math is the a7 kernel's.
#include <cmath>

#include "plan.hpp"
#include "scan.cuh"

namespace p2p {

namespace {
template <typename T> struct V4T;
template <> struct V4T<float> { using type = float4; };
template <> struct V4T<double> { using type = double4; };

constexpr int PR_THREADS = 256;

struct TgtCount {  // |N(b)| n_b
    const uint32_t *nbr_off, *bstart;
    __device__ unsigned long long operator()(uint64_t b) const {
        return (unsigned long long)(nbr_off[b + 1] - nbr_off[b]) * (bstart[b + 1] - bstart[b]);
    }
};
struct TgtPut {
    unsigned long long *t_off;
    uint32_t B;
    __device__ void operator()(uint64_t b, unsigned long long e, unsigned long long v) const {
        t_off[b] = e;
        if (b == B - 1) t_off[B] = e + v;
    }
};

__device__ __forceinline__ double slot_shift_d(const Geom &g, const uint32_t c[3], int slot, int d) {
    const int dd = d == 0 ? slot % 3 - 1 : (d == 1 ? (slot / 3) % 3 - 1 : slot / 9 - 1);
    const int v = (int)c[d] + dd;
    if (v >= g.nbox[d]) return g.L[d];
    if (v < 0) return -g.L[d];
    return 0.0;
}

// The box's records are ONE contiguous range [t_off[b] + red_off[b], + ne n_b + R_b): lanes sweep it 32 records at
// a time (coalesced stores); lane l < ne holds entry l's record start, and each output record finds its entry by a
// shuffle binary search over those starts, then whether it is a target tuple (first n_b of the record) or a source.
__device__ __forceinline__ uint32_t entry_of(uint32_t q, uint32_t my_start, uint32_t ne) {
    // largest l < ne with start(l) <= q (start non-decreasing in l; lanes >= ne hold 0xffffffff)
    uint32_t l = 0;
#pragma unroll
    for (uint32_t step = 16; step > 0; step >>= 1) {
        const uint32_t t = __shfl_sync(0xffffffffu, my_start, (l + step) & 31u);
        if (l + step < ne && t <= q) l += step;
    }
    return l;
}

// warp per target box
template <typename T>
__global__ void __launch_bounds__(PR_THREADS) k_restructure_pairs(
    const Geom g, const typename V4T<T>::type *__restrict__ rec, uint32_t B, const uint32_t *__restrict__ bkey,
    const uint32_t *__restrict__ bstart, const uint32_t *__restrict__ nbr_off, const uint32_t *__restrict__ nbr_box,
    const uint8_t *__restrict__ nbr_slot, const unsigned long long *__restrict__ red_off,
    const unsigned long long *__restrict__ t_off, typename V4T<T>::type *__restrict__ pr) {
    using V4 = typename V4T<T>::type;
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < B; b += nw) {
        const uint32_t key = bkey[b];
        const uint32_t c[3] = {compact3(key), compact3(key >> 1), compact3(key >> 2)};
        const double o[3] = {__fma_rn((double)c[0], g.h, g.lo[0]), __fma_rn((double)c[1], g.h, g.lo[1]),
                             __fma_rn((double)c[2], g.h, g.lo[2])};
        const uint32_t s0 = bstart[b], nb = bstart[b + 1] - s0;
        const uint32_t e0 = nbr_off[b], ne = nbr_off[b + 1] - e0;  // <= 27
        // lane l < ne: entry e0 + l -- source box start, image code, record start (box-relative)
        uint32_t ks = 0, nk = 0, code = 0;
        if (lane < ne) {
            const uint32_t k = nbr_box[e0 + lane];
            const int sl = nbr_slot[e0 + lane];
            ks = bstart[k];
            nk = bstart[k + 1] - ks;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const double S = slot_shift_d(g, c, sl, d);
                code |= (S > 0.0 ? 1u : (S < 0.0 ? 2u : 0u)) << (2 * d);
            }
        }
        uint32_t inc = lane < ne ? nb + nk : 0u;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= (unsigned)d) inc += y;
        }
        const uint32_t my_start = lane < ne ? inc - (nb + nk) : 0xffffffffu;
        const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
        V4 *out = pr + t_off[b] + red_off[b];
        for (uint32_t q0 = 0; q0 < total; q0 += 32) {
            const uint32_t q = q0 + lane;
            const uint32_t l = entry_of(q, my_start, ne);
            const uint32_t st = __shfl_sync(0xffffffffu, my_start, l), kl = __shfl_sync(0xffffffffu, ks, l),
                           cd = __shfl_sync(0xffffffffu, code, l);
            if (q >= total) continue;
            const uint32_t r = q - st;
            const bool tgt = r < nb;
            const V4 x = tgt ? rec[s0 + r] : rec[kl + (r - nb)];
            // targets: the slot-13 rebase (S = +0); sources: the slot's image (C5), rebased like red (C11)
            const double S0 = tgt ? 0.0 : ((cd & 1u) ? g.L[0] : ((cd & 2u) ? -g.L[0] : 0.0));
            const double S1 = tgt ? 0.0 : ((cd & 4u) ? g.L[1] : ((cd & 8u) ? -g.L[1] : 0.0));
            const double S2 = tgt ? 0.0 : ((cd & 16u) ? g.L[2] : ((cd & 32u) ? -g.L[2] : 0.0));
            V4 v;
            v.x = (T)__dsub_rn(__dadd_rn((double)x.x, S0), o[0]);
            v.y = (T)__dsub_rn(__dadd_rn((double)x.y, S1), o[1]);
            v.z = (T)__dsub_rn(__dadd_rn((double)x.z, S2), o[2]);
            v.w = x.w;
            out[q] = v;
        }
    }
}

__device__ __forceinline__ float rinv_of(float r2) { return rsqrt_ftz(r2); }  // C14
__device__ __forceinline__ double rinv_of(double r2) { return rsqrt(r2); }  // C14

// warp per target box; lane = one (record, target) slot of the box's ne x n_b partial slots (the paper's thread
// per target per pair record): the lane reads its target tuple and its record's sources -- nothing else -- and
// writes its partial.  Partial slot of (entry l, target j) = t_off[b] + l n_b + j.
template <typename T>
__global__ void __launch_bounds__(PR_THREADS) k_eval_pairrec(uint32_t B, const uint32_t *__restrict__ bstart,
                                                             const uint32_t *__restrict__ nbr_off,
                                                             const uint32_t *__restrict__ nbr_box,
                                                             const uint8_t *__restrict__ nbr_slot,
                                                             const unsigned long long *__restrict__ red_off,
                                                             const unsigned long long *__restrict__ t_off,
                                                             const typename V4T<T>::type *__restrict__ pr, T eps2,
                                                             typename V4T<T>::type *__restrict__ partial) {
    using V4 = typename V4T<T>::type;
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < B; b += nw) {
        const uint32_t nb = bstart[b + 1] - bstart[b];
        const uint32_t e0 = nbr_off[b], ne = nbr_off[b + 1] - e0;
        uint32_t nk = 0, self = 0;
        if (lane < ne) {
            const uint32_t k = nbr_box[e0 + lane];
            nk = bstart[k + 1] - bstart[k];
            self = nbr_slot[e0 + lane] == 13 ? 1u : 0u;
        }
        uint32_t inc = nk;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= (unsigned)d) inc += y;
        }
        const uint32_t srcoff = inc - nk;  // records of the box's earlier entries' sources
        const V4 *box_pr = pr + t_off[b] + red_off[b];
        V4 *box_part = partial + t_off[b];
        const uint32_t nslot = ne * nb;
        for (uint32_t s0 = 0; s0 < nslot; s0 += 32) {
            const uint32_t s = s0 + lane;
            const uint32_t l = s < nslot ? s / nb : 0u, j = s < nslot ? s - l * nb : 0u;
            const uint32_t nkl = __shfl_sync(0xffffffffu, nk, l), sol = __shfl_sync(0xffffffffu, srcoff, l);
            const bool slf = __shfl_sync(0xffffffffu, self, l) != 0u;
            if (s >= nslot) continue;
            const V4 *recd = box_pr + (unsigned long long)l * nb + sol;  // this lane's pair record
            const V4 t = recd[j];
            T ph = 0, ax = 0, ay = 0, az = 0;
            for (uint32_t q = 0; q < nkl; ++q) {
                const V4 sr = recd[nb + q];
                const T dx = sr.x - t.x, dy = sr.y - t.y, dz = sr.z - t.z;
                const T r2 = dx * dx + dy * dy + dz * dz + eps2;
                const T ri = rinv_of(r2);
                const T mr = sr.w * ri;
                const T mr3 = mr * ri * ri;
                if (!(slf && q == j)) ph -= mr;  // C3: the self pair is excluded from phi
                ax += mr3 * dx;
                ay += mr3 * dy;
                az += mr3 * dz;
            }
            V4 v;
            v.x = ph;
            v.y = ax;
            v.z = ay;
            v.w = az;
            box_part[s] = v;
        }
    }
}

// the update: every target sums its partials in ascending record order (deterministic) -> input order (a9)
template <typename T>
__global__ void __launch_bounds__(PR_THREADS) k_reduce_pairrec(uint32_t B, const uint32_t *__restrict__ bstart,
                                                               const uint32_t *__restrict__ nbr_off,
                                                               const uint32_t *__restrict__ perm,
                                                               const unsigned long long *__restrict__ t_off,
                                                               const typename V4T<T>::type *__restrict__ partial,
                                                               T *__restrict__ phi, T *__restrict__ field) {
    using V4 = typename V4T<T>::type;
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < B; b += nw) {
        const uint32_t s0 = bstart[b], nb = bstart[b + 1] - s0;
        const uint32_t ne = nbr_off[b + 1] - nbr_off[b];
        const V4 *pb = partial + t_off[b];
        for (uint32_t j = lane; j < nb; j += 32) {
            T a0 = 0, a1 = 0, a2 = 0, a3 = 0;
            for (uint32_t l = 0; l < ne; ++l) {
                const V4 v = pb[(unsigned long long)l * nb + j];
                a0 += v.x;
                a1 += v.y;
                a2 += v.z;
                a3 += v.w;
            }
            const uint32_t i = perm[s0 + j];
            phi[i] = a0;
            if (field) {
                field[3 * (size_t)i + 0] = a1;
                field[3 * (size_t)i + 1] = a2;
                field[3 * (size_t)i + 2] = a3;
            }
        }
    }
}

unsigned warp_grid(uint64_t nwarps, int num_sms) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(div_up(nwarps * 32, PR_THREADS), (uint64_t)num_sms * 16));
}
}  // namespace

void free_pairrec(p2p_plan *P) {
    void *bufs[] = {P->pr, P->pr_partial, P->pr_toff};
    for (void *b : bufs) dfree(b, P->stream);
    P->pr = P->pr_partial = nullptr;
    P->pr_toff = nullptr;
    P->pr_records = P->pr_targets = 0;
    P->pr_valid = false;
}

// needs the host copies of B / n_nbr / R (sizes_known); one more host sync for the target-slot total T
p2p_status restructure_pairs(p2p_plan *P) {
    cudaStream_t st = P->stream;
    const bool f64 = P->cfg.precision == P2P_FP64;
    const uint32_t B = (uint32_t)P->B;
    free_pairrec(P);
    if (B == 0) {
        P->pr_valid = true;
        return P2P_OK;
    }
    P2P_CUDA_TRY(dalloc((void **)&P->pr_toff, 8 * ((size_t)B + 1), st));
    void *scratch = nullptr;
    P2P_CUDA_TRY(dalloc(&scratch, scan_partials_bytes(B) * 2, st));
    p2p_status s = P2P_OK;
    {
        cudaError_t e = device_scan<unsigned long long>(TgtCount{P->nbr_off, P->bstart},
                                                        TgtPut{P->pr_toff, B}, nullptr, B, nullptr, scratch, st);
        if (e != cudaSuccess) s = P2P_ERR_CUDA;
    }
    dfree(scratch, st);
    if (s != P2P_OK) return s;
    unsigned long long T = 0;
    P2P_CUDA_TRY(cudaMemcpyAsync(&T, P->pr_toff + B, 8, cudaMemcpyDeviceToHost, st));
    P2P_CUDA_TRY(cudaStreamSynchronize(st));
    P->pr_targets = (int64_t)T;
    P->pr_records = (int64_t)T + P->R;
    const size_t rs = f64 ? sizeof(double4) : sizeof(float4);
    P2P_CUDA_TRY(dalloc(&P->pr, rs * (size_t)std::max<int64_t>(P->pr_records, 1), st));
    P2P_CUDA_TRY(dalloc(&P->pr_partial, rs * (size_t)std::max<int64_t>(P->pr_targets, 1), st));
    const unsigned grid = warp_grid(B, P->num_sms);
    if (f64)
        P2P_LAUNCH(k_restructure_pairs<double>, grid, PR_THREADS, 0, st, P->geom, (const double4 *)P->rec, B, P->bkey,
                   P->bstart, P->nbr_off, P->nbr_box, P->nbr_slot, (const unsigned long long *)P->red_off, P->pr_toff,
                   (double4 *)P->pr);
    else
        P2P_LAUNCH(k_restructure_pairs<float>, grid, PR_THREADS, 0, st, P->geom, (const float4 *)P->rec, B, P->bkey,
                   P->bstart, P->nbr_off, P->nbr_box, P->nbr_slot, (const unsigned long long *)P->red_off, P->pr_toff,
                   (float4 *)P->pr);
    P2P_CUDA_TRY(cudaGetLastError());
    P->pr_valid = true;
    return P2P_OK;
}

p2p_status eval_pairrec(p2p_plan *P, void *phi, void *field) {
    cudaStream_t st = P->stream;
    const uint32_t B = (uint32_t)P->B;
    if (B == 0) return P2P_OK;
    const unsigned grid = warp_grid(B, P->num_sms);
    const unsigned long long *ro = (const unsigned long long *)P->red_off;
    if (P->cfg.precision == P2P_FP64) {
        P2P_LAUNCH(k_eval_pairrec<double>, grid, PR_THREADS, 0, st, B, P->bstart, P->nbr_off, P->nbr_box, P->nbr_slot,
                   ro, P->pr_toff, (const double4 *)P->pr, P->geom.eps2, (double4 *)P->pr_partial);
        P2P_LAUNCH(k_reduce_pairrec<double>, grid, PR_THREADS, 0, st, B, P->bstart, P->nbr_off, P->perm, P->pr_toff,
                   (const double4 *)P->pr_partial, (double *)phi, (double *)field);
    } else {
        P2P_LAUNCH(k_eval_pairrec<float>, grid, PR_THREADS, 0, st, B, P->bstart, P->nbr_off, P->nbr_box, P->nbr_slot,
                   ro, P->pr_toff, (const float4 *)P->pr, (float)P->geom.eps2, (float4 *)P->pr_partial);
        P2P_LAUNCH(k_reduce_pairrec<float>, grid, PR_THREADS, 0, st, B, P->bstart, P->nbr_off, P->perm, P->pr_toff,
                   (const float4 *)P->pr_partial, (float *)phi, (float *)field);
    }
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}

}  // namespace p2p
