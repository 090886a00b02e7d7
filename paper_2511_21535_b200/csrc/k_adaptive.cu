// k_adaptive.cu -- SURVEY §8f NEXT-1, first GPU step: the adaptive binary-tree leaves (DESIGN C22) of a gravity
// plan's particles, computed on the device from the plan's Morton-sorted box table.
//
// The paper's PhotoNs tree is "an irregular binary MLFMA tree" split by a clustering threshold t (P:L330,
// Fig 8).  Reading C22: longest-axis MIDPOINT splits of the periodic cube with ties z, y, x, i.e. a cell is a prefix
// of the finest-level Morton key (C7) of any length l; a cell is split while it holds more than t particles or while
// l < min_bits; finest cells are leaves whatever their count.  So the leaf of a finest box is its SHORTEST prefix
// l >= min_bits whose cell holds <= t particles (counts are non-increasing in l: a binary search over l, each count
// two binary searches over the box keys), and the leaves are the runs of consecutive boxes sharing (l, prefix):
// a head-flag scan (scan.cuh) numbers them in Morton order.  Every leaf is one contiguous run of the sorted records.
#include "plan.hpp"
#include "scan.cuh"

namespace p2p {

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
