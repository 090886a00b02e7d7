/*
 * include/p2p.h -- C ABI v1 of libp2p, the B200-native (sm_100a) MLFMA near-field (P2P) operator with
 * the data-redundancy layout of arXiv 2511.21535 ("Modeling the Effect of Data Redundancy on Speedup in
 * MLFMA Near-Field Computation").
 *
 * Citations: P:Lnnn = PAPER.md line nnn (section / equation / table named), S:Lnnn = SPEC.md line nnn,
 * DESIGN.md §3 C<k> = the numbered reading of a silent / garbled / ambiguous passage.
 *
 * The operator (§1: "direct particle-to-particle interactions within neighboring cells, forming a
 * stencil-like computation"): particles are binned into leaf boxes, Morton-sorted, given E2 neighbour
 * lists (27-box stencil in 3D, §5.2; 9-box in 2D, §5.1), then each target box's
 * neighbour sources are gathered into ONE contiguous redundant buffer (§1.1, §5.2.1
 * "duplicated data enables threads to access contiguous blocks") and every target accumulates its
 * direct interactions against that buffer.  Two pair kernels:
 *   P2P_GRAVITY      softened 1/r (PhotoNs-2.0-like; form fixed by S:L253, DESIGN C1-C3):
 *                    phi_i = -sum_{j!=i} m_j (r^2+eps^2)^{-1/2},  a_i = sum_j m_j d_ij (r^2+eps^2)^{-3/2}
 *   P2P_HELMHOLTZ2D  the DBIM-MLFMA pattern table ("all 9t^2 neighboring patterns ... loaded
 *                    into shared memory"): y_i = sum_s sum_j P[i][s t + j] x_j, P from
 *                    G(r) = (i/4) H0^(1)(k r) (DESIGN C15), complex.
 *
 * Pipeline of calls (SPEC's build_uniform_tree + e2_neighbors = p2p_plan_create,
 * pack_redundant = p2p_restructure, run_p2p_redundant / run_p2p_indexing = p2p_eval):
 *   p2p_plan_create -> p2p_restructure -> p2p_eval(P2P_REDUNDANT)  (-> p2p_eval ...) -> p2p_destroy
 *
 * General conventions
 *  - Every function returns p2p_status (nothing throws across the ABI); p2p_last_error() gives a
 *    thread-local message naming the violated invariant (SPEC style).
 *  - Pointers marked "device" must be CUDA device (or managed) memory of the current device; host
 *    pointers there are rejected with P2P_ERR_INVALID_ARGUMENT.  Pointers marked "host" are plain host
 *    memory.  The caller owns every buffer it passes; the plan owns every internal buffer.
 *  - All device work is stream-ordered on cfg->stream (a cudaStream_t, NULL = legacy default stream).
 *    p2p_plan_create performs exactly ONE host synchronisation (to learn the box / neighbour / buffer
 *    sizes); every other compute call only enqueues.  Asynchronous kernel faults surface as
 *    P2P_ERR_CUDA at the next call or the caller's own synchronisation; CUDA / NCCL errors are sticky
 *    and leave the plan unusable (destroy it).
 *  - Outputs are always OVERWRITTEN (never accumulated), in the caller's INPUT order (DESIGN C12).
 *  - Determinism: outputs are bitwise reproducible for a fixed input and config; P2P_REDUNDANT and
 *    P2P_INDEXED_BITWISE are bitwise equal; P2P_INDEXED agrees with them within tolerance.
 */
#ifndef P2P_H_
#define P2P_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define P2P_ABI_VERSION 1

typedef struct p2p_plan p2p_plan; /* opaque */
typedef struct p2p_comm p2p_comm; /* opaque; wraps an ncclComm_t owned by the library */

typedef enum {
    P2P_OK = 0,
    P2P_ERR_INVALID_ARGUMENT = 1, /* NULL / host pointer where device required, n < 0, h <= 0, eps <= 0,
                                     dim/kernel mismatch, periodic dim with nbox < 3, nbox < 1 */
    P2P_ERR_OUT_OF_DOMAIN = 2,    /* a position outside [lo, lo + nbox*h) in some dim (never clamped);
                                     p2p_last_error names the first offending input index */
    P2P_ERR_OUT_OF_MEMORY = 3,
    P2P_ERR_CUDA = 4,             /* sticky */
    P2P_ERR_NCCL = 5,             /* sticky */
    P2P_ERR_BAD_STATE = 6,        /* eval(REDUNDANT) before restructure / after set_charges, ... */
    P2P_ERR_UNSUPPORTED = 7       /* key overflow (> 1024 boxes per dim in 3D, > 2^32 keys in 2D),
                                     Helmholtz input that is not a regular t-per-box lattice,
                                     n_local >= 2^30 (u32 indices; the radix sort's look-back packs
                                     per-digit prefixes into 30-bit fields) */
} p2p_status;

typedef enum { P2P_GRAVITY = 0, P2P_HELMHOLTZ2D = 1 } p2p_kernel;

/* Working precision: fp32 = fp32 storage, accumulation and outputs; fp64 = fp64 throughout.  Binning,
 * keys and the rebase of redundant records are always computed in fp64 IEEE arithmetic (C6, C11). */
typedef enum { P2P_FP32 = 0, P2P_FP64 = 1 } p2p_precision;

typedef enum {
    P2P_REDUNDANT = 0,      /* stream the restructured per-target-box buffer red[] (the paper's redundant
                               layout, §5.2.1; DBIM: the zero-padded im2col Xg, §5.1.2) */
    P2P_INDEXED = 1,        /* non-redundant baseline (§5.2.1 "Particle indices are first loaded,
                               followed by data access"): neighbour segments of the Morton-sorted
                               records, located through the neighbour CSR, staged on the fly */
    P2P_INDEXED_BITWISE = 2,/* test configuration of INDEXED: stages bit-identical copies of red[]
                               records, so its outputs equal P2P_REDUNDANT bit for bit */
    P2P_PAIRREC = 3         /* SURVEY NEXT-4, the paper's THREAD-level redundancy (§5.2.1): one AoS
                               pair record [targets of b ; sources of k] per neighbour pair (b, k), one
                               partial result per (record, target), then the update sums them in record
                               order (§1.1).  Gravity, single-GPU plans; needs p2p_restructure_pairs */
} p2p_layout;

typedef struct {
    int32_t dim;                /* 3 for P2P_GRAVITY, 2 for P2P_HELMHOLTZ2D */
    p2p_kernel kernel;
    p2p_precision precision;
    double box_size;            /* h > 0: leaf box edge */
    double lo[3];               /* domain origin; the domain is lo + [0, nbox*h) per dim */
    int32_t nbox[3];            /* boxes per dim (>= 1; >= 3 where periodic); unused dims ignored */
    uint32_t periodic_mask;     /* bit d set => periodic in dim d (gravity only; DBIM is open, C5) */
    double softening;           /* gravity: eps > 0 (C2) */
    double wavenumber;          /* helmholtz: k > 0 (C15 uses k = 2 pi / (10 Delta)) */
    int32_t points_per_box;     /* helmholtz: t, a perfect square; sample spacing Delta = h / sqrt(t) */
    void *stream;               /* cudaStream_t */
    p2p_comm *comm;             /* NULL => single GPU; else every rank calls collectively */
} p2p_config;

/* Build the plan: bin (a1), Morton keys, stable radix sort (a2), permute into Morton-ordered records
 * (a3), box-offset scan (a4), neighbour CSR + redundant offsets + work items (a5).  Copies what it needs
 * from the inputs into plan-owned storage; the inputs may be reused once the stream passes this point.
 *   positions : device, [n_local][dim] row-major, float (FP32) or double (FP64)
 *   charges   : device, gravity: [n_local] masses (same type as positions);
 *               helmholtz: [n_local] complex (re, im) pairs of that type
 *   out       : host, receives the plan (NULL on failure)
 * One host synchronisation. */
p2p_status p2p_plan_create(const p2p_config *cfg, int64_t n_local, const void *positions, const void *charges,
                           p2p_plan **out);

/* Rebuild a1..a5 of an existing GRAVITY plan for new positions / charges (a PhotoNs-like time step: the
 * particles moved, the tree is rebuilt every step, §4, §5.2.3 item 1).  Same config; n_local may
 * change (buffers grow stream-ordered if n_local exceeds the capacity).  Fully ASYNCHRONOUS: no host
 * synchronisation and, in steady state, no allocation -- box / neighbour / buffer counts stay on the device
 * (the redundant buffer is sized for the worst case R <= 27 n_local).  Input errors detected on the device
 * (P2P_ERR_OUT_OF_DOMAIN) are reported by the next synchronising call (p2p_get_info / p2p_copy_out); results
 * computed in between are undefined.  Invalidates red[] (restructure again).  Helmholtz: P2P_ERR_UNSUPPORTED.
 * Multi-GPU plans (cfg->comm): COLLECTIVE, every rank calls with its new input slice; the repartition and halo
 * exchange run again (their sizes need host synchronisations for the NCCL counts), the local structures reuse
 * the plan's buffers as above. */
p2p_status p2p_plan_update(p2p_plan *plan, int64_t n_local, const void *positions, const void *charges);

/* Host-buffer variants of p2p_plan_update / p2p_eval: the end-to-end path of a time-stepping code whose
 * particle data live in host memory.  p2p_plan_update_host copies the inputs into plan-owned device staging
 * (cudaMemcpyAsync on the plan's stream: asynchronous for page-locked host memory, the caller keeps the host
 * buffers alive until the stream passes the copy) and runs p2p_plan_update on it.  p2p_eval_host evaluates
 * into plan-owned device results, copies them to the host buffers and returns after the copy completed (ONE
 * stream synchronisation): the host results are valid on return.
 *   positions_host : host, [n_local][3] (the plan's precision);  charges_host : host, [n_local] masses
 *   potential_host : host, [n_local];  field_host : host, [n_local][3] or NULL
 * Device pointers are rejected (P2P_ERR_INVALID_ARGUMENT: use the device entry points).  Gravity, single-GPU
 * plans only (else P2P_ERR_UNSUPPORTED).  Staging grows on demand (the first call per size allocates). */
p2p_status p2p_plan_update_host(p2p_plan *plan, int64_t n_local, const void *positions_host,
                                const void *charges_host);
p2p_status p2p_eval_host(p2p_plan *plan, p2p_layout layout, void *potential_host, void *field_host);

/* a6: build the redundant buffer (gravity: red[R] records {x,y,z,m} rebased to the target box origin,
 * C11; helmholtz: Xg[B][9][t], zero segments for missing neighbours, C10).  Enqueue only. */
p2p_status p2p_restructure(p2p_plan *plan);

/* build the pair-record buffer of P2P_PAIRREC ("duplicating particle data for each
 * interaction pair ... each entry contains both source and target attributes").  Record of CSR entry e =
 * (b, k, slot): b's n_b target tuples rebased to o_b, then k's n_k source tuples rebased like red (C11) -- bit for
 * bit b's own segment of red followed by e's segment.  Records in CSR order; 16 (T + R) bytes (fp64: 32), T =
 * sum_b |N(b)| n_b (= R by neighbour symmetry), plus 16 T bytes of partial results.  Gravity, single-GPU plans
 * (else P2P_ERR_UNSUPPORTED); synchronises the stream once (sizes).  Invalidated by update / set_charges. */
p2p_status p2p_restructure_pairs(p2p_plan *plan);
/* records (T + R) and partial-result slots (T) of the current pair-record buffer (BAD_STATE if not built) */
p2p_status p2p_get_pairrec_size(const p2p_plan *plan, int64_t *records, int64_t *partials);

/* SURVEY NEXT-1, first GPU step: the adaptive binary-tree leaves of the plan's particles (DESIGN C22; "an
 * irregular binary MLFMA tree", P:L330 clustering threshold): longest-axis midpoint splits with ties z, y, x, so
 * a cell is an l-bit prefix of the finest Morton key; a cell splits while it holds more than t particles or while
 * l < min_bits (9 keeps periodic images unique for the adjacency of the next step); finest cells are leaves
 * whatever their count.  Computed on the device from the sorted box table; leaves in Morton order, each one
 * contiguous run of the sorted particles.
 *   len_out[L], prefix_out[L], start_out[L] : host, u32 -- prefix length l, the l-bit prefix, the leaf's first
 *                                              sorted particle (its count = next start or n_local minus start)
 *   capacity : entries the outputs hold (n_boxes always suffices);  *n_leaves : L
 * Gravity single-GPU plans on a periodic cube of 2^m boxes per dimension (else P2P_ERR_UNSUPPORTED); t >= 1.
 * Synchronous (one stream synchronisation); the plan is unchanged. */
p2p_status p2p_adaptive_leaves(p2p_plan *plan, int32_t t, int32_t min_bits, uint32_t *len_out, uint32_t *prefix_out,
                               uint32_t *start_out, int64_t capacity, int64_t *n_leaves);

/* SURVEY NEXT-1, second GPU step: the closed neighbour lists of the adaptive leaves (DESIGN C23: B + S overlaps the
 * target leaf dilated by its own extent, then symmetric closure), built on the device by range lookups in the
 * Morton-ordered leaf table.  CSR over the leaves of p2p_adaptive_leaves(t, min_bits):
 *   off_out[L + 1] (u32), nbr_out[E] (u32 leaf index), code_out[E] (u8 image code 9(s_z+1)+3(s_y+1)+(s_x+1),
 *   S_d = +1 when the neighbour wraps past the upper face, C5); entries of a leaf in ascending (leaf, code) order.
 * min_bits >= 9 (unique periodic images); a periodic cube of 2^m >= 8 boxes per dimension; capacities in entries
 * (else P2P_ERR_INVALID_ARGUMENT, the counts are still returned).  Synchronous; the plan is unchanged. */
p2p_status p2p_adaptive_neighbours(p2p_plan *plan, int32_t t, int32_t min_bits, uint32_t *off_out, uint32_t *nbr_out,
                                   uint8_t *code_out, int64_t cap_leaves, int64_t cap_entries, int64_t *n_leaves,
                                   int64_t *n_entries);

/* SURVEY NEXT-1, a6 + a7 + a9 over the adaptive leaves: builds the leaves and closed lists as above, the redundant
 * run of every target leaf (DESIGN C24: its entries' source runs in CSR order, rebased in fp64 to the target leaf's
 * origin fma(c, w, lo) with the entry's image shift, one final rounding), and evaluates every target against its
 * run with the REDUNDANT eval kernel (C1, C3; outputs in input order, overwritten).
 *   potential, field : device, as p2p_eval (potential NULL: build only, e.g. to copy the runs out)
 *   red_out : host or NULL, [cap_records][4] records of the plan's precision, leaves in order;  *n_records : R
 *   layout : P2P_REDUNDANT (the runs above) or P2P_INDEXED (the non-redundant baseline: the same eval kernel stages the
 *            leaves' neighbour segments of the sorted records, absolute coordinates, exact -L frames; no runs built)
 * Same preconditions as p2p_adaptive_neighbours.  Synchronous (sizes are read back); the plan is unchanged. */
p2p_status p2p_adaptive_eval(p2p_plan *plan, int32_t t, int32_t min_bits, p2p_layout layout, void *potential,
                             void *field, void *red_out, int64_t cap_records, int64_t *n_records);

/* SURVEY NEXT-1 on the per-step path: ADAPTIVE-LEAF MODE of a gravity plan.  After
 * p2p_adaptive_enable(plan, t, min_bits) the plan's steps run over the adaptive leaves (C22-C24) instead of the grid
 * boxes: p2p_plan_update = a1-a4 + the leaves + their closed neighbour CSR + run lengths, work items and chunk heads
 * (what both layouts need, like the grid's a5); p2p_restructure = the leaves' redundant runs;
 * p2p_eval(P2P_REDUNDANT | P2P_INDEXED) = the eval over them (other layouts: UNSUPPORTED; P2P_REDUNDANT needs the
 * restructure of the current update, P2P_INDEXED only the update).  All
 * of it is ASYNCHRONOUS with every count on the device (no host sync, no allocation per step): enable measures the
 * current input once (synchronous, like p2p_plan_create) and sizes the buffers with headroom (neighbour entries and
 * redundant records 2x the measured, leaves <= boxes).  An update exceeding them sets a device flag: its
 * restructure / eval do nothing and p2p_get_info reports P2P_ERR_OUT_OF_MEMORY (call p2p_adaptive_enable again).
 * p2p_get_info in adaptive mode describes the leaves (n_boxes = leaves, n_nbr = entries, n_red = records,
 * n_pairs, n_items).  Same preconditions as p2p_adaptive_neighbours (single-GPU periodic cube of 2^m >= 8 boxes).
 * p2p_adaptive_disable returns to grid mode (the next restructure / eval needs a p2p_plan_update first). */
p2p_status p2p_adaptive_enable(p2p_plan *plan, int32_t t, int32_t min_bits);
p2p_status p2p_adaptive_disable(p2p_plan *plan);

/* a7/a8 + a9: evaluate every target and scatter to input order.
 *   potential : device, gravity [n_local] real; helmholtz [n_local] complex (re, im)
 *   field     : device, gravity [n_local][3] real (the acceleration, C1) or NULL; helmholtz: must be NULL
 * P2P_REDUNDANT requires a preceding p2p_restructure, P2P_PAIRREC a preceding p2p_restructure_pairs (else
 * P2P_ERR_BAD_STATE).  Enqueue only. */
p2p_status p2p_eval(p2p_plan *plan, p2p_layout layout, void *potential, void *field);

/* Replace the charges, keeping the geometry (DBIM reuses its geometry across iterations).
 * charges: device, same layout as in p2p_plan_create, INPUT order.  Invalidates red[] (restructure
 * again before eval(REDUNDANT)).  Enqueue only. */
p2p_status p2p_set_charges(p2p_plan *plan, const void *charges);

/* Free every plan-owned buffer (stream-ordered).  NULL-safe.
 * Memory: plan buffers come from a LIBRARY-OWNED stream-ordered pool per device (cudaMemPoolCreate; the device's
 * default pool and PyTorch's caching allocator are untouched).  Freed blocks stay reserved in that pool while any
 * plan on the device is alive (cheap regrowth inside a time-step loop); destroying the LAST live plan of a device
 * synchronises the plan's stream and trims the pool to zero, returning the memory to the driver. */
void p2p_destroy(p2p_plan *plan);

/* ---- introspection for bit-exact parity (copy-out only; never hands out internal pointers) ---- */
typedef enum {
    P2P_ARR_PERM = 0,        /* u32 [n_local]   perm[p] = input index of sorted slot p */
    P2P_ARR_SORTED_KEYS = 1, /* u32 [n_local]   Morton keys in sorted order (helmholtz: box*t + subcell) */
    P2P_ARR_BOX_KEYS = 2,    /* u32 [n_boxes]   ascending Morton keys of the non-empty boxes */
    P2P_ARR_BOX_START = 3,   /* u32 [n_boxes+1] first sorted slot of each box, last = n_local */
    P2P_ARR_NBR_OFF = 4,     /* u32 [n_boxes+1] neighbour CSR offsets (helmholtz: 9 b) */
    P2P_ARR_NBR_BOX = 5,     /* u32 [n_nbr]     neighbour box index (helmholtz: 0xffffffff = missing) */
    P2P_ARR_NBR_SLOT = 6,    /* u8  [n_nbr]     stencil slot 0..26 (2D 0..8), ascending per box */
    P2P_ARR_RED_OFF = 7,     /* u64 [n_boxes+1] first record of each box's redundant run */
    P2P_ARR_RED = 8,         /* gravity: [n_red][4] float/double; helmholtz: [n_boxes][9][t] complex */
    P2P_ARR_PAIRREC = 9      /* gravity pair records [T + R][4] float/double (p2p_restructure_pairs) */
} p2p_array;

typedef struct {
    int64_t n_local;   /* particles on this rank */
    int64_t n_boxes;   /* B: non-empty boxes */
    int64_t n_nbr;     /* neighbour CSR entries */
    int64_t n_red;     /* R: redundant records (helmholtz: 9 t B) */
    int64_t n_pairs;   /* I: pair interactions evaluated (gravity incl. i = j; helmholtz non-padded), C19 */
    int64_t n_items;   /* eval work items */
    int32_t key_bits;  /* Morton key width */
    int32_t sort_passes;
} p2p_info;

/* Both synchronise the plan's stream. `bytes` must equal the array's exact size. */
p2p_status p2p_get_info(const p2p_plan *plan, p2p_info *out);
p2p_status p2p_copy_out(const p2p_plan *plan, p2p_array which, void *host_dst, size_t bytes);

/* ---- multi-GPU: NCCL communicator owned by the library ----
 * The 128 id bytes are produced on rank 0 by p2p_comm_unique_id and broadcast by the caller (e.g. over
 * a torch.distributed process group); every rank then calls p2p_comm_create collectively. */
p2p_status p2p_comm_unique_id(void *id_out /* host, 128 bytes */);
p2p_status p2p_comm_create(int nranks, int rank, const void *id /* host, 128 bytes */, p2p_comm **out);
void p2p_comm_destroy(p2p_comm *comm);

/* Multi-GPU plan semantics (cfg->comm != NULL; gravity only).  Every rank calls p2p_plan_create / p2p_eval
 * collectively with ITS OWN input slice (any distribution).  The ranks repartition the particles into
 * contiguous Morton ranges of boxes, balanced by particle count on a coarse supercell histogram
 * (p2p_partition_splitters), route every particle to its owner and, as a halo source, to every other rank owning
 * one of its box's 26 neighbours (one all-to-all-v), and each rank evaluates the targets of its range;
 * p2p_eval returns every result to the rank and input slot it came from.  Results are bitwise identical to a
 * 1-GPU plan over the rank-major concatenation of the slices.  p2p_get_info / p2p_copy_out describe the rank's
 * LOCAL plan (owned + halo particles; halo boxes have empty neighbour lists and runs).  p2p_plan_update is
 * collective too (a new time step: the partition is recomputed); p2p_set_charges and the host-buffer entry
 * points return P2P_ERR_UNSUPPORTED for multi-GPU plans. */

/* The count-balanced splitters of SURVEY §8e / DESIGN C20, as computed inside the collective plan build
 * (exported for testing the host logic): hist[nbins] = global particle counts per supercell (supercell =
 * key >> shift); rank r gets keys [splitters[r], splitters[r+1]), splitters[0] = 0, splitters[nranks] =
 * 2^key_bits; splitter r = (first supercell whose exclusive prefix count >= r * total / nranks) << shift.
 *   hist: host, [nbins] u64;  splitters_out: host, [nranks + 1] u32 */
p2p_status p2p_partition_splitters(const uint64_t *hist, int64_t nbins, int shift, int key_bits, int nranks,
                                   uint32_t *splitters_out);

/* The splitters a collective plan's latest build derived ON THE DEVICE (k_splitters, from the all-reduced
 * supercell histogram, sc_bits = min(key_bits, 18)); they must equal p2p_partition_splitters of the same
 * histogram (tests).  splitters_out: host, [nranks + 1] u32.  INVALID_ARGUMENT for a 1-GPU plan or n != nranks+1. */
p2p_status p2p_get_splitters(const p2p_plan *plan, uint32_t *splitters_out, int n);

/* In-process "loopback" communicators: nranks emulated ranks = nranks host threads of ONE process sharing one
 * device; the collectives become device-to-device copies + a host barrier.  Used to run the whole multi-GPU
 * algorithm on a single GPU (tests: bit-identity against the 1-GPU plan). */
typedef struct p2p_loopback_group p2p_loopback_group;
p2p_status p2p_loopback_group_create(int nranks, p2p_loopback_group **out);
void p2p_loopback_group_destroy(p2p_loopback_group *group);
p2p_status p2p_comm_create_loopback(p2p_loopback_group *group, int rank, p2p_comm **out);

/* Multi-PROCESS communicator over CUDA IPC peer memory (SURVEY §8e "B200-native option"): one process per rank
 * on one node -- one GPU each (peer copies over NVLink / NVSwitch) or several processes sharing one GPU (NCCL
 * allows one rank per device).  Each rank exports a cudaMalloc'd device arena; the collectives stage into the
 * own arena and pull from the peers' (comm_ipc.cu).  `name` (no '/') names the POSIX shared-memory rendezvous
 * segment: rank 0 creates it (INVALID_ARGUMENT if the name exists), the others wait up to 120 s for it; use a
 * fresh random token per communicator (rank 0 draws it, the caller broadcasts it, e.g. over torch.distributed).
 * Collective over all nranks ranks; the segment name is unlinked once every rank attached.
 *   name: host NUL-terminated string;  out: receives the communicator (free with p2p_comm_destroy). */
p2p_status p2p_comm_create_ipc(int nranks, int rank, const char *name, p2p_comm **out);

/* ---- diagnostics ---- */
const char *p2p_status_string(p2p_status s);
const char *p2p_last_error(void);        /* thread-local detail of the last failing call on this thread */
uint64_t p2p_kernel_launch_count(void);   /* number of libp2p kernels launched by this process so far */
int p2p_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* P2P_H_ */
