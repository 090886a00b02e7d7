// items.cuh -- sizing of the eval's work items (a5 grid boxes, k_structs.cu; adaptive leaves, k_adaptive.cu)
#pragma once
#include "plan.hpp"

namespace p2p {

// ------------------------------------------------------------------------------------------------
// eval work items: a box's targets are split into chunks of at most ITEM_TMAX targets, more chunks if the chunk cost
// n_t * R_b exceeds ITEM_COSTCAP interactions (bounds the tail of the dynamic work queue on clustered inputs).
// Chunk sizes are chosen for the eval's lane layout (G = ceil(n_t / 4) groups of 4 targets x S = floor(32 / G)
// source splits): every chunk but the box's last has ITEM_TMAX targets, or -- when the cost cap binds -- the
// largest of 24, 20, 16, 12, 8, 4 targets not above the capped balanced size (G * S = 30 or 32 busy lanes); the
// earlier balanced chunks (e.g. 25 + 25 targets: 28 lanes, 25 of 28 target slots) left up to 22% of the
// lane-slots idle (c5w eval 6.60 -> 6.16 ms).
// ITEM_TMAX (plan.hpp): at most 32 targets per item -> G <= 8 groups of K = 4 (fp32)
// The cap scales with the work: the dynamic queue's tail is bounded by its largest item, so a fixed 2^17-pair cap
// left a 1e6-particle Plummer eval (c3, 6e8 pairs: 2e5 pairs per warp) waiting on single 2^17-pair items (SMs
// active 81% of the kernel).  cap = pow2floor(I_est / (4 W)) clamped to [2^13, 2^17], I_est = 27 sum_b n_b^2 (the
// pair count of a uniform periodic grid; ~25 sum n_b^2 on the Plummer inputs) over the TARGET boxes, W = a fixed
// nominal eval warp count (148 SMs x 20) -- sum_nb2 is all-reduced over ranks, so every rank and a 1-GPU plan
// derive the same cap and the same items (bitwise results independent of the GPU count).  c3 479 -> ~390 us;
// c5w, c3dense, c4-k unchanged (their cap stays 2^17) (profiles/r02_eval_options.txt).
#ifndef P2P_ITEM_COSTCAP
#define P2P_ITEM_COSTCAP (1ull << 17)
#endif
constexpr uint64_t ITEM_COSTCAP = P2P_ITEM_COSTCAP;  // upper bound of the cap
constexpr uint64_t ITEM_COSTCAP_MIN = 1ull << 13;
constexpr uint64_t EVAL_WARPS_NOMINAL = 148 * 20;

// cap = pow2floor(pairs / (P2P_CAP_DIV W)) clamped to [ITEM_COSTCAP_MIN, ITEM_COSTCAP]
__device__ __forceinline__ uint64_t item_costcap_of(uint64_t pairs) {
#ifndef P2P_CAP_DIV
#define P2P_CAP_DIV 4  // items per nominal eval warp the cap aims at (8 / 2 / 1 / 16 measured: r02_eval_options.txt)
#endif
    const uint64_t est = pairs / ((uint64_t)P2P_CAP_DIV * EVAL_WARPS_NOMINAL);
    if (est >= ITEM_COSTCAP) return ITEM_COSTCAP;
    if (est <= ITEM_COSTCAP_MIN) return ITEM_COSTCAP_MIN;
    return 1ull << (63 - __clzll((long long)est));
}
// grid boxes: the pair count estimated before the CSR exists, 27 sum_b n_b^2
__device__ __forceinline__ uint64_t item_costcap(const DevCounters *ctr) { return item_costcap_of(27ull * ctr->sum_nb2); }

// targets per item of a box with nb_b targets and nsrc sources (its items: ceil(nb_b / size))
// K = targets per lane of the eval (the capped sizes are multiples of K: every group of K target slots full)
__device__ __forceinline__ uint32_t item_size(uint32_t nb_b, uint64_t nsrc, uint32_t tmax, uint32_t K, uint64_t cap) {
    const uint32_t a = (nb_b + tmax - 1) / tmax;
    // the cap is a power of two (item_costcap_of): a shift instead of a 64-bit division (a5 runs this per box)
    const uint64_t num = (uint64_t)nb_b * nsrc + cap - 1;
    const uint64_t c = (cap & (cap - 1)) == 0 ? num >> (__ffsll((long long)cap) - 1) : num / cap;
    if (c <= a) return tmax;
    const uint32_t ts = c > nb_b ? 0u : nb_b / (uint32_t)c;  // balanced chunk size under the cap
    if (ts < K) return ts > 1 ? ts : 1u;
    if (K == 8) return ts >= 24 ? 24u : ts >= 16 ? 16u : 8u;
    return ts >= 24 ? 24u : ts >= 20 ? 20u : ts >= 16 ? 16u : ts >= 12 ? 12u : ts >= 8 ? 8u : 4u;
}

}  // namespace p2p
