// plan.hpp -- the opaque p2p_plan object and the internal kernel entry points of libp2p.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "comm.hpp"
#include "common.cuh"
#include "p2p.h"

namespace p2p {

// device-resident counters written by the structure kernels; read back ONCE at the end of plan_create
struct DevCounters {
    unsigned long long err_index;  // min out-of-domain input index (init ~0ull)
    unsigned int irregular;        // helmholtz: non-regular lattice detected
    unsigned int B;                // non-empty boxes
    unsigned int n_nbr;            // CSR entries
    unsigned int n_items;          // eval work items
    unsigned long long R;          // redundant records
    unsigned long long I;          // pair interactions
    unsigned int item_head;        // eval work queue head (reset before every eval)
    unsigned int sort_tile_ctr[4]; // onesweep tile counters, one per pass
    unsigned int scan_tile_ctr;    // single-pass box-table scan (scan.cuh k_scan_lb)
    unsigned int rs_head;          // restructure chunk queue (P2P_RS_BATCH)
    unsigned int n_small;          // targets of small boxes (thread-per-target path of the eval)
    unsigned int small_head;       // eval small-target queue head (reset before every eval)
    unsigned int n_items_red;      // REDUNDANT-eval work items (items_red)
    unsigned long long sum_nb2;    // sum over target boxes of n_b^2 (k_boxinfo; all-reduced over ranks): item cost cap
};

// eval work item: a chunk [t0, t0 + nt) of the sorted targets of box `box`
// meta = n_t | S << 8 | G << 16: the warp lane layout (G groups of K targets x S source splits, G*S <= 32)
// key / red_base / R duplicate the box's Morton key and redundant run so the eval's one-item-ahead prefetch is a
// single 32-byte load (no dependent loads on the critical path of tiny items).  tofs = offset of the item's
// first target inside the run (the box's own slot-13 segment + the item's target offset): the REDUNDANT eval
// stages its targets already rebased from red[] instead of re-deriving them in fp64.
struct __align__(16) Item {
    uint32_t box;
    uint32_t t0;
    uint32_t meta;
    uint32_t key;
    unsigned long long red_base;
    uint32_t R;
    uint32_t tofs;
};
#ifndef P2P_EVAL_K
#define P2P_EVAL_K 4
#endif
// targets per lane in k_eval_gravity (fp32: K/2 packed FP32x2 pairs).  K = 4 or 8 (build option).  The hot
// loop alone reaches 0.83 (K = 4) / 0.86 (K = 8) of the FP32 lane-op peak (scripts/ubench_evalmix.cu,
// profiles/r02_ubench_evalmix.txt), but K = 8 needs 128 registers (16 warps per SM): c5w eval 6.00 -> 6.43 ms,
// c4-8 1.60 -> 1.78, c4-128 15.3 -> 15.6, so K = 4 stays
constexpr int EVAL_K_F32 = P2P_EVAL_K;
constexpr int EVAL_K_F64 = 2;
constexpr uint32_t ITEM_TMAX = 32;  // max targets per work item (lane utilisation)
// boxes with <= SMALL_NT targets and <= SMALL_R sources take the eval's thread-per-target path (no work item):
// their per-item overhead would exceed their work, and their runs are short enough for L1-latency-bound loads
#ifndef P2P_SMALL_NT
#define P2P_SMALL_NT 8
#endif
#ifndef P2P_SMALL_R
#define P2P_SMALL_R 128
#endif
constexpr uint32_t SMALL_NT = P2P_SMALL_NT;
constexpr uint32_t SMALL_R = P2P_SMALL_R;

// gravity geometry passed by value to kernels
struct Geom {
    double lo[3];
    double h;
    double L[3];          // periodic lengths nbox_d * h (IEEE product, C5)
    int32_t nbox[3];
    uint32_t periodic;
    int32_t nb;           // Morton bits per dim
    double eps2;          // eps^2 (fp64)
    uint32_t tkey_lo, tkey_hi;  // target boxes: keys in [tkey_lo, tkey_hi] (multi-GPU: this rank's Morton range)
};

}  // namespace p2p

namespace p2p {
// the persistent adaptive-leaf state (SURVEY NEXT-1 on the per-step path, k_adaptive.cu): capacities fixed at
// p2p_adaptive_enable, every count device-side, no host sync per step
struct AdaptCtr {
    uint32_t L, E, n_items, overflow;
    unsigned long long R, I;
    uint32_t n_items_red, pad;  // the REDUNDANT eval's items (multi-leaf quads, fp32)
};
struct AdaptState {
    uint32_t t = 0;
    int min_bits = 9;
    int64_t bcap = 0, ecap = 0, rcap = 0, icap = 0;
    AdaptCtr *ac = nullptr;
    uint8_t *len8 = nullptr, *rcode = nullptr, *code = nullptr, *code_t = nullptr, *lframe = nullptr;
    uint32_t *llen = nullptr, *lprefix = nullptr, *lstart = nullptr, *lkey = nullptr, *off = nullptr, *nbr = nullptr,
             *nbr_t = nullptr, *tself = nullptr, *ioff = nullptr, *zero = nullptr;
    unsigned int *dcnt = nullptr, *tcnt = nullptr, *tcur = nullptr;
    uint2 *rng = nullptr;
    unsigned long long *R = nullptr, *roff = nullptr, *ch_rel = nullptr;  // ch_*: per restructure chunk (32 entries)
    uint32_t *ch_leaf = nullptr;
    void *red = nullptr, *scr = nullptr;
    Item *items = nullptr;
    Item *items_red = nullptr;  // REDUNDANT list: multi-leaf quads + the other leaves' items
    uint32_t *ioff_red = nullptr;
    bool built = false;     // leaves + CSR of the current positions
    bool runs_valid = false;
};
}  // namespace p2p

struct p2p_plan {
    p2p_config cfg;
    cudaStream_t stream = nullptr;
    int device = 0;
    int num_sms = 148;
    int64_t n = 0;
    int key_bits = 0, passes = 0, nb = 0;
    p2p::Geom geom{};
    // sizes (host copies, valid after plan_create)
    int64_t B = 0, n_nbr = 0, R = 0, I = 0, n_items = 0;
    // device buffers
    void *rec = nullptr;        // gravity: float4/double4 {x,y,z,m} Morton-sorted; helmholtz: complex xs
    uint32_t *skey = nullptr, *perm = nullptr, *bkey = nullptr, *bstart = nullptr;
    uint32_t *nbr_off = nullptr, *nbr_box = nullptr;
    uint8_t *nbr_slot = nullptr;
    uint64_t *red_off = nullptr;
    uint32_t *box_of = nullptr;  // Helmholtz: dense Morton-key -> box lookup
    uint32_t *occ = nullptr;     // gravity: occupancy bitmap of the key space (cleared every build)
    p2p::Item *items = nullptr;
    p2p::Item *items_red = nullptr;
    uint32_t *s_mb_cen = nullptr;    // per eligible box: offset of its own segment in its run (quad items)  // the REDUNDANT eval's items: multi-box quads + the other boxes' items (fp32)
    void *red = nullptr;         // gravity red[R] records; helmholtz Xg[B][9][t]
    void *table = nullptr;       // helmholtz pattern table P[t][9t] complex
    void *tc_table = nullptr;    // helmholtz tensor-core operand: real W hi / lo, 2 x [2t][18t] fp32 (k_helm_tc.cu)
    int tc_rf = 1;               // copies of W (block-level redundancy factor RF)
    p2p::DevCounters *ctr = nullptr;
    // capacity-sized scratch, allocated once per plan (p2p_plan_update reuses it: no allocation, no sync)
    int64_t cap = 0, bcap = 0, red_cap = 0;
    // host-buffer entry points (p2p_plan_update_host / p2p_eval_host): plan-owned device staging
    void *stage_in = nullptr, *stage_out = nullptr;
    int64_t stage_in_cap = 0, stage_out_cap = 0;
    uint32_t *s_key = nullptr, *s_idx = nullptr, *s_kalt = nullptr, *s_valt = nullptr;
    uint32_t *s_hist = nullptr, *s_status = nullptr;
    void *s_partials = nullptr;
    void *s_aos = nullptr;       // gravity: the SoA input packed into {x,y,z,m} records (input order), a3's source
    uint2 *s_box_nbr = nullptr;  // per box: occupied-slot mask, redundant records (k_nbr_count -> k_nbr_fill)
    void *s_nb_tiles = nullptr;  // [ceil(B / 256)] k_nbr_count tile sums -> k_nbr_scan offsets
    uint2 *boxinfo = nullptr;     // gravity: dense Morton key -> {box, n_b} (valid where occ has the bit set)
    uint32_t *small_tgt = nullptr, *small_box = nullptr;  // sorted target index / its box, small boxes only
    // restructure chunks: every 32 consecutive CSR entries e = 32 c .. 32 c + 31 form one chunk; their redundant
    // segments are one contiguous range of red[] starting at chunk_out[c]; chunk_box[c] = box owning entry 32 c
    uint32_t *chunk_box = nullptr;
    unsigned long long *chunk_out = nullptr;
    bool sizes_known = false;  // host copies of B, n_nbr, R, I, n_items valid (false after an async update)
    // ---- multi-GPU: this rank owns the target boxes of one contiguous Morton range ----
    p2p::CommBase *comm = nullptr;
    int64_t n_in = 0;          // caller's particles on this rank (outputs are for these, in their input order)
    int64_t n_own = 0;         // owned (target) particles after the repartition; local plan n = n_own + halo
    uint32_t *perm_send = nullptr;          // input index of the i-th particle sent in the repartition
    std::vector<int64_t> rp_scnt, rp_soff, rp_rcnt, rp_roff;  // repartition counts / offsets (elements)
    std::vector<uint32_t> splitters;        // G + 1 key boundaries of the rank ranges
    void *phi_loc = nullptr, *field_loc = nullptr, *res_own = nullptr, *res_back = nullptr;
    void *peer_tab = nullptr;  // device PeerRes of the fused peer-memory result return (cudaMalloc)
    bool red_valid = false;
    p2p::AdaptState *ad = nullptr;  // adaptive-leaf mode (p2p_adaptive_enable)
    bool grid_stale = false;        // grid a5 not built (after adaptive-mode updates) until the next p2p_plan_update
    // SURVEY NEXT-4 pair records (k_pairrec.cu): [T + R] records, [T] partial slots, t_off[B + 1] slot bases
    void *pr = nullptr, *pr_partial = nullptr;
    unsigned long long *pr_toff = nullptr;
    int64_t pr_records = 0, pr_targets = 0;
    bool pr_valid = false;
    p2p_status sticky = P2P_OK;
    int eval_blocks[10] = {};  // persistent eval grid per layout (+ [3] / [4] the adaptive-leaf evals; +5: peer-result kernels)
};

namespace p2p {

// k_sort.cu: stable LSD radix sort of (key, value) pairs, `passes` 8-bit digits.  On return the sorted
// pairs are in (*kout, *vout) which point to either the in or the alt buffers.
// hist: [4][256] u32, status: [passes][ceil(n/4096)][256] u32 scratch (plan-owned)
cudaError_t radix_sort_pairs(uint32_t *kin, uint32_t *vin, uint32_t *kalt, uint32_t *valt, uint32_t n, int passes,
                             DevCounters *ctr, uint32_t *hist, uint32_t *status, cudaStream_t st, uint32_t **kout,
                             uint32_t **vout, bool iota_values = false, bool hist_ready = false);
size_t radix_status_words(uint64_t n, int passes);

// k_structs.cu
p2p_status alloc_capacity(p2p_plan *P, int64_t cap);   // all N-/B-sized buffers + scratch
void free_capacity(p2p_plan *P);
// pos/q: SoA caller arrays; or, if rec_in != nullptr, AoS {x,y,z,m} records (multi-GPU local plans)
p2p_status build_gravity_structs(p2p_plan *P, const void *pos, const void *q, const void *rec_in = nullptr,
                                 bool grid_a5 = true);
p2p_status build_helmholtz_structs(p2p_plan *P, const void *pos, const void *q);
p2p_status set_charges_gravity(p2p_plan *P, const void *q);
p2p_status set_charges_helmholtz(p2p_plan *P, const void *q);

// k_restructure.cu
p2p_status restructure_gravity(p2p_plan *P);
bool origins_exact_fp32(const Geom &g);  // every box origin fma(c, h, lo_d) is an fp32 value
p2p_status restructure_helmholtz(p2p_plan *P);

// k_eval_gravity.cu / k_helmholtz.cu
// the REDUNDANT eval over an explicit item list and redundant buffer (adaptive leaves, k_adaptive.cu)
struct EvalItems {
    const Item *items;
    const uint32_t *n_items;  // device
    int64_t n_items_host;     // grid sizing
    const void *red;
    const uint32_t *zero;     // device 0 (no small-box path)
    // INDEXED over adaptive leaves (csr_off != nullptr): the leaves' CSR, first sorted particle per leaf [L + 1],
    // frame / boundary flags per leaf (bit d: touches the upper face of dim d, bit 3 + d: the lower face)
    const uint32_t *csr_off = nullptr, *csr_nbr = nullptr, *lstart = nullptr;
    const uint8_t *csr_code = nullptr, *lframe = nullptr;
};
p2p_status eval_gravity_items(p2p_plan *P, const EvalItems &it, void *phi, void *field);
// multi-GPU over peer memory (comm_ipc.cu): the eval stores each owned target's {phi, fx, fy, fz} into its origin
// rank's receive buffer (device table, k_dist.cu)
constexpr int PEER_MAX = 64;
struct PeerRes {
    int G;
    uint32_t lo[PEER_MAX];   // first local slot of the run received from rank r (owned head first)
    char *dst[PEER_MAX];     // rank r's receive buffer
    int64_t off[PEER_MAX];   // where this rank's results land in it (records)
};
p2p_status eval_gravity(p2p_plan *P, p2p_layout layout, void *phi, void *field, const PeerRes *pr = nullptr);

// k_dist.cu: the distributed (multi-GPU) plan build and result return
p2p_status build_distributed(p2p_plan *P, const void *pos, const void *q);
p2p_status eval_distributed(p2p_plan *P, p2p_layout layout, void *phi, void *field);
void free_distributed(p2p_plan *P);
p2p_status eval_helmholtz(p2p_plan *P, p2p_layout layout, void *y);
p2p_status helmholtz_table(p2p_plan *P);
// k_helm_tc.cu: a8 as one 3xTF32 tcgen05 GEMM (fp32, t in {16, 64})
bool helmholtz_tc_supported(const p2p_plan *P);
p2p_status helmholtz_tc_table(p2p_plan *P, const float *Pf);
p2p_status eval_helmholtz_tc(p2p_plan *P, void *y, bool gather);  // gather: the INDEXED layout

// k_adaptive.cu: SURVEY NEXT-1 adaptive binary-tree leaves (C22) from the box table; host outputs, synchronous
p2p_status adaptive_leaves(p2p_plan *P, uint32_t t, int min_bits, uint32_t *len_h, uint32_t *prefix_h,
                           uint32_t *start_h, int64_t cap, int64_t *n_leaves);
p2p_status adaptive_neighbours(p2p_plan *P, uint32_t t, int min_bits, uint32_t *off_h, uint32_t *nbr_h,
                               uint8_t *code_h, int64_t cap_leaves, int64_t cap_entries, int64_t *n_leaves,
                               int64_t *n_entries);
// the persistent asynchronous adaptive path (p2p_adaptive_enable / update / restructure / eval in adaptive mode)
p2p_status adaptive_enable(p2p_plan *P, uint32_t t, int min_bits);
void adaptive_free(p2p_plan *P);
p2p_status adaptive_build_async(p2p_plan *P);
p2p_status adaptive_restructure_async(p2p_plan *P);
p2p_status adaptive_eval_async(p2p_plan *P, p2p_layout layout, void *phi, void *field);
p2p_status adaptive_info(p2p_plan *P, AdaptCtr *out);  // synchronises
p2p_status adaptive_eval(p2p_plan *P, uint32_t t, int min_bits, bool indexed, void *phi, void *field, void *red_h,
                         int64_t cap_red, int64_t *n_red, int64_t *n_items = nullptr);

// k_pairrec.cu: the thread-level pair-record layout (P2P_PAIRREC)
p2p_status restructure_pairs(p2p_plan *P);
p2p_status eval_pairrec(p2p_plan *P, void *phi, void *field);
void free_pairrec(p2p_plan *P);

// allocation helpers (stream-ordered, pooled)
cudaError_t dalloc(void **p, size_t bytes, cudaStream_t st);
void dfree(void *p, cudaStream_t st);

}  // namespace p2p
