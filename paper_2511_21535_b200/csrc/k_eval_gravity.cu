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
//                        absolute coordinates, periodic images applied as exact -L shifts.
//   P2P_INDEXED_BITWISE  as INDEXED, then each staged record is rebased in shared memory exactly like a red[]
//                        record, so the arithmetic and the outputs equal P2P_REDUNDANT bit for bit.
//
// B200 design (the paper's GTX 1050 thread-per-particle kernel is prior art, not the blueprint):
//   * persistent CTAs (EV_WARPS warps each); every warp pulls work items (box, <= 32-target chunk; a 32-byte
//     record prefetched one item ahead) from a global atomic queue (EV_BATCH = 1 item per atomic, claimed one item ahead) and runs its own
//     2-stage producer/consumer pipeline: while it computes chunk c from one shared-memory stage, the bulk
//     copies of chunk c+1 -- or of the next item's first chunk AND its targets (REDUNDANT: already rebased,
//     from the box's own segment of its run) -- land in the other stage (mbarrier + expect_tx completion).
//     Boxes with <= 8 targets and <= 128 sources (or <= 6 and <= 256) take a thread-per-target-pair path instead (one warp per CTA
//     starts with them, so their load latency hides behind the other warps' item work).
//   * targets live in registers: lane (g, s) holds K targets (group g) and walks the staged sources
//     j = s, s+S, ... (S source splits, G groups; S, G precomputed per item by k_nbr_fill), so boxes of any
//     occupancy keep (almost) all 32 lanes busy; the S partial sums are combined by a fixed transpose-reduce
//     (deterministic).
//   * fp32: targets are paired and the pair math is issued as packed FP32x2 instructions (FADD2 / FMUL2 /
//     FFMA2, sm_100a; the source component is a broadcast scalar operand), so the 13 FP32-pipe lane-ops of an
//     interaction cost only 6.5 issue slots + 1 MUFU.RSQ: the kernel is bound by the FP32 pipe
//     (128 lane-ops/clk/SM), not by instruction issue.  The rounding of every operation is the same as the
//     scalar formula (fma.rn.f32x2 == two fma.rn.f32).
//   * the hot loop is specialised on S (immediate-offset LDS, 4 sources per iteration, one ALU pointer add) and
//     holds the targets negated (d = s + (-t): no per-chunk prologue); no IMAD runs on the FMA-heavy pipe.
//   * the self pair (d = 0, r^2 = eps^2) is evaluated like any other and its potential term subtracted
//     bit-exactly after the loop (DESIGN C3).
#include <type_traits>

#include "plan.hpp"

namespace p2p {

namespace {
template <typename T> struct V4T;
template <> struct V4T<float> { using type = float4; };
template <> struct V4T<double> { using type = double4; };

#ifndef P2P_EV_WARPS
#define P2P_EV_WARPS 4
#endif
constexpr int EV_WARPS = P2P_EV_WARPS;   // warps per CTA (x 5 CTAs per SM for the fp32 REDUNDANT kernel: 20 warps)
constexpr int EV_STAGE_BYTES = 4096;     // source records per pipeline stage per warp (256 fp32 / 128 fp64)
constexpr int EV_TGT = 32;               // max targets per item (ITEM_TMAX in k_structs.cu)
// work-item records are prefetched through cp.async into a per-warp shared slot (P2P_ITEM_REGS: into registers,
// the round-1 default): c4-8 eval 1.515 -> 1.463 ms, c5w / c3 unchanged (profiles/r02_eval_options.txt)
#if !defined(P2P_ITEM_REGS) && !defined(P2P_ITEM_SMEM)
#define P2P_ITEM_SMEM
#endif
#ifndef P2P_EV_BATCH
#define P2P_EV_BATCH 1  // 1 vs 2 vs 3 per atomic (profiles/r02_eval_options.txt): c4-8 -1.3%, c5w / c3 equal
#endif
constexpr int EV_BATCH = P2P_EV_BATCH;   // work items claimed per queue atomic

// ceil(2^20 / S) for S = 0..32: x / S == (x * M20[S]) >> 20 exactly for x < 2^11 (no integer division)
__constant__ uint32_t c_m20[33] = {0,       1048576, 524288, 349526, 262144, 209716, 174763, 149797, 131072,
                                   116509,  104858,  95326,  87382,  80660,  74899,  69906,  65536,  61681,
                                   58255,   55189,   52429,  49933,  47663,  45591,  43691,  41944,  40330,
                                   38837,   37450,   36158,  34953,  33826,  32768};

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
    const uint32_t *n_items;   // device-side count (valid without a host sync after p2p_plan_update)
    unsigned int *item_head;
    const uint32_t *n_small;   // small-box targets (thread-per-target path)
    unsigned int *small_head;
    const uint32_t *small_tgt, *small_box;
    T *phi;
    T *field;
    uint32_t zero;             // always 0 (see queue_claim)
    const uint8_t *lframe;     // ADAPT: per leaf, bit d = touches the upper face of periodic dim d, bit 3 + d the lower
    const PeerRes *pr;         // multi-GPU over peer memory: results stored straight into the origin ranks' buffers
};

// a9: one result value (q = 0 potential, 1..3 field component) of local target slot i -- into the caller's arrays,
// or (multi-GPU, peer memory) into its origin rank's receive buffer: rank r = the run holding i (runs are rank-major,
// lo[] ascending), element (off[r] + i - lo[r]) of {phi, fx, fy, fz} records -- the reverse all-to-all-v of the
// results fused into the eval's epilogue
// PEER is a template parameter (only the multi-GPU peer-memory launch instantiates it): with the destination
// search compiled into every kernel the REDUNDANT eval grew from 3864 to 4672 SASS instructions and ran 5% slower
// (c5w 5.96 -> 6.26 ms on one box)
template <bool PEER, typename T>
__device__ __forceinline__ void put_result(const EvalArgs<T> &a, uint32_t i, int q, T v) {
    if constexpr (PEER) {
        const PeerRes *pr = a.pr;
        int lo = 0, hi = pr->G - 1;  // the largest r with lo[r] <= i
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (pr->lo[mid] <= i) lo = mid;
            else hi = mid - 1;
        }
        T *d = reinterpret_cast<T *>(pr->dst[lo]) + (size_t)(pr->off[lo] + (int64_t)(i - pr->lo[lo])) * 4 + q;
        *d = v;
    } else if (q == 0) {
        a.phi[i] = v;
    } else if (a.field) {
        a.field[3 * (size_t)i + (q - 1)] = v;
    }
}

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

// one lane claims `n` work items.  ptxas turns an atomic on a warp-uniform address into a warp-aggregated one
// whose result it broadcasts at once -- a wait for the atomic's round trip that the batch prefetch is meant to
// hide.  The address is made lane-dependent for the compiler by a runtime zero (EvalArgs::zero = 0):
// head + (laneid & zero) == head.
__device__ __forceinline__ uint32_t queue_claim(unsigned int *head, uint32_t n, uint32_t zero) {
    uint32_t lid, r;
    asm("mov.u32 %0, %%laneid;" : "=r"(lid));
    asm volatile("atom.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(head + (lid & zero)), "r"(n) : "memory");
    return r;
}

// ---- per-lane target block + accumulators --------------------------------------------------------
template <typename T, int K>
struct Tgt;

// fp32: K targets as K/2 packed pairs (float2 + the sm_100 packed intrinsics __fadd2_rn / __fmul2_rn /
// __ffma2_rn -> SASS FADD2 / FMUL2 / FFMA2; the broadcast source component becomes a scalar operand)
__device__ __forceinline__ float2 bc(float v) { return make_float2(v, v); }

template <int K>
struct Tgt<float, K> {
    static constexpr int P = K / 2;
    float2 tx[P], ty[P], tz[P], ap[P], ax[P], ay[P], az[P];
    // the targets are held NEGATED (-x, -y, -z): d = s + (-t) is then a plain FADD2 with no per-chunk negation
    // prologue (exact: negation is exact, s + (-t) == s - t bit for bit)
    __device__ __forceinline__ void set(int k, float x, float y, float z) {
        const int p = k >> 1;
        if (k & 1) { tx[p].y = -x; ty[p].y = -y; tz[p].y = -z; }
        else { tx[p].x = -x; ty[p].x = -y; tz[p].x = -z; }
    }
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int p = 0; p < P; ++p) tx[p] = ty[p] = tz[p] = ap[p] = ax[p] = ay[p] = az[p] = make_float2(0.f, 0.f);
    }
    __device__ __forceinline__ void interact(const float4 &s, float2 E) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const float2 dx = __fadd2_rn(bc(s.x), tx[p]);
            const float2 dy = __fadd2_rn(bc(s.y), ty[p]);
            const float2 dz = __fadd2_rn(bc(s.z), tz[p]);
            float2 r2 = __ffma2_rn(dx, dx, E);
            r2 = __ffma2_rn(dy, dy, r2);
            r2 = __ffma2_rn(dz, dz, r2);
            const float2 ri = make_float2(rsqrt_ftz(r2.x), rsqrt_ftz(r2.y));
            const float2 mri = __fmul2_rn(bc(s.w), ri);
            ap[p] = __fadd2_rn(ap[p], mri);
            const float2 m3 = __fmul2_rn(mri, __fmul2_rn(ri, ri));  // ri*ri in parallel with m*ri: one FMUL shorter chain
            ax[p] = __ffma2_rn(m3, dx, ax[p]);
            ay[p] = __ffma2_rn(m3, dy, ay[p]);
            az[p] = __ffma2_rn(m3, dz, az[p]);
        }
    }
    // Transpose-reduce of the S source splits of a group: every lane holds V = 4K values (f = K q + k with q = 0
    // potential, 1..3 field, k = target) as NW = 2K packed pairs.  Each level exchanges HALF of the remaining
    // values with the partner split and keeps the other half, so log2(S) levels cost NW/2 + NW/4 + ... shuffles
    // of pairs instead of NW per level.  A non-power-of-two S first folds its tail splits [Sp, S) onto [0, S - Sp).
    // Afterwards split sl < Sp (lg = log2 Sp, Lh = min(lg, log2 V)) holds the cnt = V >> Lh consecutive values
    // f0 .. f0 + cnt - 1 in v[], f0 = (sl >> (lg - Lh)) * cnt; when lg > log2 V only the splits whose low
    // lg - Lh bits are 0 hold unique values.  Fixed exchange pattern -> deterministic.
    static constexpr int NW = 2 * K;
    static constexpr int LOGV = K == 4 ? 4 : 5;  // log2(4K)
    template <int H>
    static __device__ __forceinline__ void tr_level(float2 (&w)[NW], uint32_t sl, uint32_t gbase, uint32_t o) {
        const bool up = (sl & o) != 0u;
        const uint32_t src = (gbase + (sl ^ o)) & 31u;
#pragma unroll
        for (int i = 0; i < H; ++i) {
            const float2 snd = up ? w[i] : w[i + H];
            const float2 kp = up ? w[i + H] : w[i];
            const float2 r = make_float2(__shfl_sync(0xffffffffu, snd.x, src), __shfl_sync(0xffffffffu, snd.y, src));
            w[i] = __fadd2_rn(kp, r);
        }
    }
    __device__ __forceinline__ void treduce(uint32_t S, uint32_t sl, uint32_t gbase, float (&v)[4]) const {
        static_assert(K == 4 || K == 8, "transpose-reduce is written for K = 4 or 8");
        float2 w[NW];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            w[p] = ap[p];
            w[P + p] = ax[p];
            w[2 * P + p] = ay[p];
            w[3 * P + p] = az[p];
        }
        uint32_t Sp = S;
        if (S & (S - 1u)) {
            Sp = 1u << (31 - __clz(S));
            const uint32_t src = (gbase + sl + Sp) & 31u;
            const bool take = sl + Sp < S;
#pragma unroll
            for (int i = 0; i < NW; ++i) {
                const float2 r = make_float2(__shfl_sync(0xffffffffu, w[i].x, src),
                                             __shfl_sync(0xffffffffu, w[i].y, src));
                if (take) w[i] = __fadd2_rn(w[i], r);
            }
        }
        const uint32_t lg = 31u - __clz(Sp);  // S >= 4 -> lg in 2..5
        // packed levels: keep NW/2, NW/4, ..., 1 pairs (level l runs when lg > l)
        if (lg >= 1) tr_level<NW / 2>(w, sl, gbase, Sp >> 1);
        if (lg >= 2) tr_level<NW / 4>(w, sl, gbase, Sp >> 2);
        if (lg >= 3) tr_level<NW / 8>(w, sl, gbase, Sp >> 3);
        if constexpr (NW >= 16) {
            if (lg >= 4) tr_level<NW / 16>(w, sl, gbase, Sp >> 4);
        }
        constexpr int LP = NW == 8 ? 3 : 4;  // packed levels available (log2 NW)
        if (lg >= (uint32_t)LP + 1u) {  // scalar level: split the last pair
            const uint32_t o = Sp >> (LP + 1);
            const bool up = (sl & o) != 0u;
            const float snd = up ? w[0].x : w[0].y, kp = up ? w[0].y : w[0].x;
            w[0].x = kp + __shfl_sync(0xffffffffu, snd, (gbase + (sl ^ o)) & 31u);
        }
        if (lg >= (uint32_t)LOGV + 1u) w[0].x += __shfl_xor_sync(0xffffffffu, w[0].x, 1);  // K = 4, S = 32 only
        v[0] = w[0].x;
        v[1] = w[0].y;
        v[2] = w[1].x;
        v[3] = w[1].y;
    }
    __device__ __forceinline__ void get(int k, float &p_, float &x, float &y, float &z) const {
        const int p = k >> 1;
        p_ = (k & 1) ? ap[p].y : ap[p].x;
        x = (k & 1) ? ax[p].y : ax[p].x;
        y = (k & 1) ? ay[p].y : ay[p].x;
        z = (k & 1) ? az[p].y : az[p].x;
    }
    static __device__ __forceinline__ float self_rinv(float eps2) { return rsqrt_ftz(__fmaf_rn(0.f, 0.f, eps2)); }
    static __device__ __forceinline__ float2 eps_pack(float e2) { return make_float2(e2, e2); }
};

// fp64: scalar
template <int K>
struct Tgt<double, K> {
    double tx[K], ty[K], tz[K], ap[K], ax[K], ay[K], az[K];
    __device__ __forceinline__ void set(int k, double x, double y, double z) {
#pragma unroll
        for (int q = 0; q < K; ++q)
            if (q == k) { tx[q] = x; ty[q] = y; tz[q] = z; }
    }
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int k = 0; k < K; ++k) tx[k] = ty[k] = tz[k] = ap[k] = ax[k] = ay[k] = az[k] = 0.0;
    }
    __device__ __forceinline__ void interact(const double4 &s, double E) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const double dx = s.x - tx[k], dy = s.y - ty[k], dz = s.z - tz[k];
            double r2 = __fma_rn(dx, dx, E);
            r2 = __fma_rn(dy, dy, r2);
            r2 = __fma_rn(dz, dz, r2);
            const double ri = rsqrt(r2);  // C14: MUFU.RSQ64H seed + one 2nd-order Newton step (<= 1 ulp)
            const double mri = s.w * ri;
            ap[k] += mri;
            const double m3 = mri * (ri * ri);
            ax[k] = __fma_rn(m3, dx, ax[k]);
            ay[k] = __fma_rn(m3, dy, ay[k]);
            az[k] = __fma_rn(m3, dz, az[k]);
        }
    }
    __device__ __forceinline__ void reduce(uint32_t S, uint32_t sl) {
        for (uint32_t off = 1; off < S; off <<= 1) {
            const bool take = sl + off < S;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const double v0 = __shfl_down_sync(0xffffffffu, ap[k], off), v1 = __shfl_down_sync(0xffffffffu, ax[k], off);
                const double v2 = __shfl_down_sync(0xffffffffu, ay[k], off), v3 = __shfl_down_sync(0xffffffffu, az[k], off);
                if (take) { ap[k] += v0; ax[k] += v1; ay[k] += v2; az[k] += v3; }
            }
        }
    }
    __device__ __forceinline__ void get(int k, double &p_, double &x, double &y, double &z) const {
        p_ = ap[k]; x = ax[k]; y = ay[k]; z = az[k];
    }
    static __device__ __forceinline__ double self_rinv(double eps2) { return rsqrt(__fma_rn(0.0, 0.0, eps2)); }
    static __device__ __forceinline__ double eps_pack(double e2) { return e2; }
};

// ---- thread-per-target path for the targets of small boxes (n_b <= SMALL_NT) ----------------------------
// One lane = one target; the lane walks its box's source sequence in run order (REDUNDANT: the contiguous
// red[] run through the read-only L1 path; INDEXED: the CSR segments of rec[]), so there is no per-item
// staging, no source split and no reduction -- the per-item overhead that dominates tiny boxes disappears.
// Lanes of one warp are consecutive targets in Morton order, so lanes of the same box read the same
// addresses (one L1 wavefront).  Same formula and rounding sequence as Tgt::interact.
// shared-memory record load from a 32-bit shared address
template <typename V4>
__device__ __forceinline__ V4 lds_rec(uint32_t a);
template <>
__device__ __forceinline__ float4 lds_rec<float4>(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a)
                 : "memory");
    return v;
}
template <>
__device__ __forceinline__ double4 lds_rec<double4>(uint32_t a) {
    double4 v;
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2+16];" : "=d"(v.z), "=d"(v.w) : "r"(a) : "memory");
    return v;
}

// shared-memory record load at a compile-time byte offset from a 32-bit shared address
template <int OFF>
__device__ __forceinline__ float4 lds_rec_off(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4+%5];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(a), "n"(OFF) : "memory");
    return v;
}

// the eval hot loop: nj sources at shared addresses sa, sa + ST, sa + 2 ST, ... (ST = S records), two per
// iteration with one remainder step; the accumulators stay in the same registers (no IMAD.MOV copies on the
// FMA-heavy pipe the FFMA2s run on)
template <typename T, int K, int SS, typename TG, typename EP>
__device__ __forceinline__ void hot_loop(TG &tg, uint32_t sa, uint32_t nj, const EP &E) {
    constexpr int ST = SS * 16;
    const uint32_t end4 = sa + (nj & ~3u) * (uint32_t)ST;
#pragma unroll 1
    for (; sa != end4; sa += 4 * ST) {
        const float4 s0 = lds_rec<float4>(sa), s1 = lds_rec_off<ST>(sa), s2 = lds_rec_off<2 * ST>(sa),
                     s3 = lds_rec_off<3 * ST>(sa);
        tg.interact(s0, E);
        tg.interact(s1, E);
        tg.interact(s2, E);
        tg.interact(s3, E);
    }
#pragma unroll 1
    for (uint32_t r = nj & 3u; r; --r, sa += ST) tg.interact(lds_rec<float4>(sa), E);
}
// the same loop with the split stride in a register (one loop body for every S): the S-specialised copies are 7 x
// 2 KB of hot code, and when a CTA's warps run different S the instruction cache misses (c3 ncu: 13% of the stall
// samples "no instruction"); this costs 3 more ALU adds per 4 sources on the otherwise FMA-bound loop
template <int K, typename TG, typename EP>
__device__ __forceinline__ void hot_loop_rt4(TG &tg, uint32_t sa, uint32_t nj, uint32_t stride, const EP &E) {
    uint32_t a1 = sa + stride, a2 = sa + 2 * stride, a3 = sa + 3 * stride;
    const uint32_t st4 = 4 * stride;
    const uint32_t end4 = sa + (nj & ~3u) * stride;
#pragma unroll 1
    for (; sa != end4; sa += st4, a1 += st4, a2 += st4, a3 += st4) {
        const float4 s0 = lds_rec<float4>(sa), s1 = lds_rec<float4>(a1), s2 = lds_rec<float4>(a2),
                     s3 = lds_rec<float4>(a3);
        tg.interact(s0, E);
        tg.interact(s1, E);
        tg.interact(s2, E);
        tg.interact(s3, E);
    }
#pragma unroll 1
    for (uint32_t r = nj & 3u; r; --r, sa += stride) tg.interact(lds_rec<float4>(sa), E);
}
template <typename T, int K, typename TG, typename EP>
__device__ __forceinline__ void hot_loop_rt(TG &tg, uint32_t sa, uint32_t nj, uint32_t stride, const EP &E) {
    using V4 = typename V4T<T>::type;
    const uint32_t end2 = sa + (nj & ~1u) * stride;
#pragma unroll 1
    for (; sa != end2; sa += 2 * stride) {
        const V4 s0 = lds_rec<V4>(sa), s1 = lds_rec<V4>(sa + stride);
        tg.interact(s0, E);
        tg.interact(s1, E);
    }
    if (nj & 1u) tg.interact(lds_rec<V4>(sa), E);
}

__device__ __forceinline__ float4 ldro(const float4 *p) { return __ldg(p); }
__device__ __forceinline__ double4 ldro(const double4 *p) {
    const double2 a = __ldg(reinterpret_cast<const double2 *>(p)), b = __ldg(reinterpret_cast<const double2 *>(p) + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

template <typename T, int LAYOUT, bool PEER>
__device__ __forceinline__ void small_phase(const EvalArgs<T> &a, unsigned lane) {
    using V4 = typename V4T<T>::type;
    const uint32_t n_small = *a.n_small;
    const T eps2 = (T)a.g.eps2;
    while (true) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(a.small_head, 32u);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= n_small) break;
        const uint32_t i = base + lane;
        if (i < n_small) {
        // lane = a PAIR of targets of one small box (the second may not exist: b_end), so the pair math is the
        // same packed FP32x2 code as the item path (Tgt<T,2>), one broadcast source per step
        const uint32_t p = a.small_tgt[i], b = a.small_box[i];
        const uint32_t b_end = a.bstart[b + 1];
        const bool two = p + 1 < b_end;
        const uint32_t key = a.bkey[b];
        const uint32_t cc[3] = {compact3(key), compact3(key >> 1), compact3(key >> 2)};
        double org[3];
#pragma unroll
        for (int d = 0; d < 3; ++d)
            org[d] = (LAYOUT == P2P_INDEXED) ? frame_shift(a.g, cc, d) : __fma_rn((double)cc[d], a.g.h, a.g.lo[d]);
        Tgt<T, 2> tg;
        tg.zero();
        T tm[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const V4 t = a.rec[(k == 1 && two) ? p + 1 : p];
            tm[k] = t.w;
            if (LAYOUT == P2P_INDEXED)
                tg.set(k, t.x + (T)org[0], t.y + (T)org[1], t.z + (T)org[2]);
            else
                tg.set(k, (T)__dsub_rn((double)t.x, org[0]), (T)__dsub_rn((double)t.y, org[1]),
                       (T)__dsub_rn((double)t.z, org[2]));
        }
        const auto E = Tgt<T, 2>::eps_pack(eps2);
        if (LAYOUT == P2P_REDUNDANT) {
            const uint64_t r0 = a.red_off[b], r1 = a.red_off[b + 1];
            const V4 *run = a.red + r0;
            const uint32_t R = (uint32_t)(r1 - r0);
            uint32_t j = 0;
            // four loads in flight per lane (the path is L1/L2-latency bound, not FP32 bound)
#pragma unroll 1
            for (; j + 4 <= R; j += 4) {
                const V4 s0 = ldro(run + j), s1 = ldro(run + j + 1), s2 = ldro(run + j + 2), s3 = ldro(run + j + 3);
                tg.interact(s0, E);
                tg.interact(s1, E);
                tg.interact(s2, E);
                tg.interact(s3, E);
            }
#pragma unroll 1
            for (; j < R; ++j) tg.interact(ldro(run + j), E);
        } else {
            const uint32_t e0 = a.nbr_off[b], e1 = a.nbr_off[b + 1];
            for (uint32_t e = e0; e < e1; ++e) {
                const uint32_t k = a.nbr_box[e];
                const int slot = a.nbr_slot[e];
                const double S0 = slot_shift(a.g, cc, slot, 0), S1 = slot_shift(a.g, cc, slot, 1),
                             S2 = slot_shift(a.g, cc, slot, 2);
                const uint32_t q0 = a.bstart[k], q1 = a.bstart[k + 1];
                if (LAYOUT == P2P_INDEXED) {
                    const T h0 = (T)(S0 + org[0]), h1 = (T)(S1 + org[1]), h2 = (T)(S2 + org[2]);
#pragma unroll 2
                    for (uint32_t q = q0; q < q1; ++q) {
                        V4 s = ldro(a.rec + q);
                        s.x += h0;
                        s.y += h1;
                        s.z += h2;
                        tg.interact(s, E);
                    }
                } else {
                    for (uint32_t q = q0; q < q1; ++q) {
                        V4 s = ldro(a.rec + q);
                        s.x = (T)__dsub_rn(__dadd_rn((double)s.x, S0), org[0]);
                        s.y = (T)__dsub_rn(__dadd_rn((double)s.y, S1), org[1]);
                        s.z = (T)__dsub_rn(__dadd_rn((double)s.z, S2), org[2]);
                        tg.interact(s, E);
                    }
                }
            }
        }
        const T rs = Tgt<T, 2>::self_rinv(eps2);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            if (k == 1 && !two) break;
            T pot, fx, fy, fz;
            tg.get(k, pot, fx, fy, fz);
            const uint32_t idx = a.perm[p + k];
            put_result<PEER>(a, idx, 0, -(pot - tm[k] * rs));
            put_result<PEER>(a, idx, 1, fx);
            put_result<PEER>(a, idx, 2, fy);
            put_result<PEER>(a, idx, 3, fz);
        }
        }
    }
}

// ADAPT (P2P_INDEXED over adaptive leaves, k_adaptive.cu): the CSR's slot is the image code itself, a leaf's frame /
// boundary flags come from a.lframe instead of the uniform grid's box coordinates, and a leaf may list more than 32
// neighbour segments (the lane-per-segment registers then cover groups of 32, re-read from the CSR per chunk)
template <typename T, int LAYOUT, int K, bool ADAPT = false, bool PEER = false>
__global__ void __launch_bounds__(EV_WARPS * 32, sizeof(T) == 4 ? (K == 8 ? 16 : (LAYOUT == P2P_REDUNDANT ? 20 : 16)) / EV_WARPS : 1) k_eval_gravity(const EvalArgs<T> a) {
    using V4 = typename V4T<T>::type;
    constexpr int CH = EV_STAGE_BYTES / (int)sizeof(V4);
    constexpr int STAGE_RECS = CH + EV_TGT;  // source chunk + the item's targets
    constexpr unsigned FULL = 0xffffffffu;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bars[EV_WARPS][2];
    __shared__ __align__(16) uint4 qslot[EV_WARPS][2];  // the warp's next Item record (cp.async prefetch)

    const int w = threadIdx.x >> 5;
    const unsigned lane = threadIdx.x & 31u;
    V4 *stage_base = reinterpret_cast<V4 *>(smem_raw) + (size_t)w * 2 * STAGE_RECS;
    uint64_t *bar = bars[w];
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncwarp();

    const T eps2 = (T)a.g.eps2;
    const auto E = Tgt<T, K>::eps_pack(eps2);
    const uint32_t n_items = *a.n_items;

    // ---------------- producer state (item whose chunks are being copied in) ----------------
    uint32_t p_box = 0, p_t0 = 0, p_meta = 0, p_key = 0, p_R = 0, p_nch = 0, p_tofs = 0;
    uint64_t p_base = 0;
    uint32_t p_src = 0, p_st = 0, p_cnt = 0, p_slot = 0, p_ne = 0;  // INDEXED: lane = segment
    uint32_t p_e0 = 0;  // ADAPT: the item's first CSR entry
    // multi-box items (k_structs.cu mb_quad; REDUNDANT fp32): 4 boxes, 8 lanes each, runs staged in lockstep
    constexpr bool MBK = LAYOUT == P2P_REDUNDANT && sizeof(T) == 4 && K == 4 && !ADAPT;
    constexpr uint32_t MBP = 64;  // records of each box's run per stage (4 x 64 = CH)
    bool p_mb = false;
    uint32_t p_mbnt = 0, p_R01 = 0, p_R23 = 0, p_tofs01 = 0, p_tofs23 = 0;
    // ADAPT: segment group g0 .. g0 + 31 of the CSR row at e0 (ne entries), starts offset by `base`
    auto seg_group = [&](uint32_t e0, uint32_t ne, uint32_t g0, uint32_t base, uint32_t &src, uint32_t &st,
                         uint32_t &cntl, uint32_t &code, uint32_t &tot) {
        const bool valid = g0 + lane < ne;
        src = 0;
        cntl = 0;
        code = 13;
        if (valid) {
            const uint32_t k = a.nbr_box[e0 + g0 + lane];
            src = a.bstart[k];
            cntl = a.bstart[k + 1] - src;
            code = a.nbr_slot[e0 + g0 + lane];
        }
        uint32_t incl = cntl;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (unsigned)o) incl += y;
        }
        st = base + incl - cntl;
        tot = __shfl_sync(0xffffffffu, incl, 31);
    };

    // work-queue pipeline: each atomicAdd claims EV_BATCH consecutive items (fewer atomics on the one queue
    // counter) and its result is consumed by shfl a whole batch later; item n+1's 32-byte Item record is already
    // in shared memory when its first chunk is issued -- no dependent load on the per-item critical path
    // (REDUNDANT).  Default P2P_ITEM_SMEM: the record goes through cp.async into a per-warp shared slot instead of
    // registers (with registers the compiler copies the 128-bit loads into the loop-carried registers at once,
    // waiting for them): c4-8 eval -3.4%, c5w / c3 unchanged (profiles/r02_eval_options.txt).
    uint32_t pend = 0;  // lane 0: result of the last issued atomicAdd
    uint32_t nb_idx = 0, nb_left = 0;
    auto next_index = [&]() -> uint32_t {
        if (nb_left == 0) {
            nb_idx = __shfl_sync(FULL, pend, 0);
            nb_left = EV_BATCH;
            if (lane == 0) pend = queue_claim(a.item_head, (uint32_t)EV_BATCH, a.zero);
        }
        --nb_left;
        return nb_idx++;
    };
    // unconditional (index clamped; only called with n_items >= 1): a predicated load made the compiler copy the
    // prefetched registers right away (a predicated MOV on the load result), stalling on the load it was hiding
#ifndef P2P_ITEM_SMEM
    uint4 q0 = make_uint4(0, 0, 0, 0), q1 = make_uint4(0, 0, 0, 0);
    auto prefetch = [&](uint32_t idx) {
        const uint4 *src = reinterpret_cast<const uint4 *>(a.items + min(idx, n_items - 1u));
        q0 = __ldg(src);
        q1 = __ldg(src + 1);
    };
    auto load_item = [&]() {
#else
    auto prefetch = [&](uint32_t idx) {
        const uint4 *src = reinterpret_cast<const uint4 *>(a.items + min(idx, n_items - 1u));
        if (lane < 2)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&qslot[w][lane])), "l"(src + lane)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto load_item = [&]() {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        const uint4 q0 = qslot[w][0], q1 = qslot[w][1];
#endif
        p_box = q0.x;
        p_t0 = q0.y;
        p_meta = q0.z;
        p_key = q0.w;
        if (LAYOUT == P2P_REDUNDANT) {
            p_base = (uint64_t)q1.x | ((uint64_t)q1.y << 32);
            p_R = q1.z;
            p_tofs = q1.w;
            if constexpr (MBK) {
                p_mb = (q0.x >> 31) != 0u;
                if (p_mb) {
                    p_mbnt = q0.x & 0xffffu;
                    p_R01 = q0.z;
                    p_R23 = q0.w;
                    p_tofs01 = q1.z;
                    p_tofs23 = q1.w;
                    p_meta = 32u | (4u << 8) | (8u << 16);  // G = 8 groups (2 per box) x S = 4 splits
                    p_R = max(max(p_R01 & 0xffffu, p_R01 >> 16), max(p_R23 & 0xffffu, p_R23 >> 16));
                }
            }
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
            if constexpr (ADAPT) {
                p_e0 = e0;
                for (uint32_t g0 = 32; g0 < p_ne; g0 += 32) {  // rows longer than a warp: the remaining groups
                    uint32_t src, st, cntl, code, tot;
                    seg_group(e0, p_ne, g0, p_R, src, st, cntl, code, tot);
                    p_R += tot;
                }
            }
        }
        p_nch = (MBK && p_mb) ? (p_R + MBP - 1) / MBP : (p_R + CH - 1) / CH;
    };
    // copy chunk `chunk` of the producer item into stage s (+ the item's targets when chunk == 0)
    auto issue = [&](uint32_t chunk, int s) {
        if constexpr (MBK) {
            if (p_mb) {  // box j = lane & 3: piece `chunk` of its run (lanes 0..3), its targets (lanes 4..7)
                V4 *dst = stage_base + s * STAGE_RECS;
                const uint32_t j = lane & 3u;
                const uint32_t R0 = p_R01 & 0xffffu, R1 = p_R01 >> 16, R2 = p_R23 & 0xffffu, R3 = p_R23 >> 16;
                const uint32_t Rj = j == 0 ? R0 : (j == 1 ? R1 : (j == 2 ? R2 : R3));
                const uint32_t pre = (j > 0 ? R0 : 0u) + (j > 1 ? R1 : 0u) + (j > 2 ? R2 : 0u);
                const uint32_t ntj = (p_mbnt >> (4 * j)) & 0xfu;
                const uint32_t tofj = j < 2 ? (j == 0 ? p_tofs01 & 0xffffu : p_tofs01 >> 16)
                                            : (j == 2 ? p_tofs23 & 0xffffu : p_tofs23 >> 16);
                const uint32_t c0 = chunk * MBP;
                const uint32_t cntj = Rj > c0 ? min(MBP, Rj - c0) : 0u;
                uint32_t bytes = (lane < 4u ? cntj : 0u) + ((chunk == 0 && lane >= 4u && lane < 8u) ? ntj : 0u);
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) bytes += __shfl_xor_sync(FULL, bytes, o);
                if (lane == 0) mbar_arrive_expect_tx(&bar[s], bytes * (uint32_t)sizeof(V4));
                __syncwarp();
                if (lane < 4u && cntj > 0u)
                    bulk_g2s(dst + MBP * j, a.red + p_base + pre + c0, cntj * (uint32_t)sizeof(V4), &bar[s]);
                if (chunk == 0 && lane >= 4u && lane < 8u && ntj > 0u)
                    bulk_g2s(dst + CH + 8u * j, a.red + p_base + pre + tofj, ntj * (uint32_t)sizeof(V4), &bar[s]);
                return;
            }
        }
        const uint32_t c0 = chunk * CH;
        const uint32_t cnt = min((uint32_t)CH, p_R - c0);
        const uint32_t nt = p_meta & 0xffu;
        V4 *dst = stage_base + s * STAGE_RECS;
        if (lane == 0) {
            // the INDEXED variants WRITE the staged records (frame fix-ups, rebase): order those generic writes
            // before the next async (TMA) write of the stage.  REDUNDANT only reads the stage, and every read has
            // retired into the registers the hot loop consumed before the __syncwarp that precedes this issue
#ifndef P2P_EV_FENCE_ALL
            if (LAYOUT != P2P_REDUNDANT)
#endif
                fence_proxy_async_smem();
            mbar_arrive_expect_tx(&bar[s], (cnt + (chunk == 0 ? nt : 0u)) * (uint32_t)sizeof(V4));
        }
        __syncwarp();
        if (LAYOUT == P2P_REDUNDANT) {
            if (lane == 0) bulk_g2s(dst, a.red + p_base + c0, cnt * (uint32_t)sizeof(V4), &bar[s]);
        } else {
            const uint32_t ov0 = max(c0, p_st), ov1 = min(c0 + cnt, p_st + p_cnt);
            if (lane < p_ne && ov1 > ov0)
                bulk_g2s(dst + (ov0 - c0), a.rec + p_src + (ov0 - p_st), (ov1 - ov0) * (uint32_t)sizeof(V4), &bar[s]);
            if constexpr (ADAPT) {
                uint32_t base = __shfl_sync(FULL, p_st + p_cnt, 31);
                for (uint32_t g0 = 32; g0 < p_ne && base < c0 + cnt; g0 += 32) {
                    uint32_t src, st, cntl, code, tot;
                    seg_group(p_e0, p_ne, g0, base, src, st, cntl, code, tot);
                    const uint32_t v0 = max(c0, st), v1 = min(c0 + cnt, st + cntl);
                    if (v1 > v0)
                        bulk_g2s(dst + (v0 - c0), a.rec + src + (v0 - st), (v1 - v0) * (uint32_t)sizeof(V4), &bar[s]);
                    base += tot;
                }
            }
        }
        // targets: REDUNDANT takes them already rebased from the box's own segment of its run
        if (chunk == 0 && lane == 31)
            bulk_g2s(dst + CH, LAYOUT == P2P_REDUNDANT ? a.red + p_base + p_tofs : a.rec + p_t0,
                     nt * (uint32_t)sizeof(V4), &bar[s]);
    };

    // the small boxes' targets (thread per target, L1/L2-latency bound) are taken first by one warp of every
    // CTA, so their latency hides behind the FP32-bound item work of the CTA's other warps (run last by all
    // warps, they would form a latency-bound tail)
#ifndef P2P_SMALL_WARPS
#define P2P_SMALL_WARPS 1  // warps per CTA that start on the small boxes
#endif
    const bool small_first = w >= EV_WARPS - P2P_SMALL_WARPS;
    if (small_first) small_phase<T, LAYOUT, PEER>(a, lane);
    if (lane == 0) pend = queue_claim(a.item_head, (uint32_t)EV_BATCH, a.zero);
    const uint32_t first = next_index();
    if (first < n_items) {
    prefetch(first);
    load_item();
    issue(0, 0);
    uint32_t nxt = next_index();
    prefetch(nxt);
    int s = 0;
    uint32_t phases = 0u;  // bit s = parity of stage s's mbarrier

    while (true) {
        // ---------------- adopt the producer's item as the current (consumer) item ----------------
        const uint32_t c_t0 = p_t0, c_meta = p_meta, c_R = p_R, c_nch = p_nch;
        const uint32_t c_st = p_st, c_cnt = p_cnt, c_slot = p_slot, c_ne = p_ne, c_e0 = p_e0;
        const bool c_mb = MBK && p_mb;
        const uint32_t c_mbnt = p_mbnt, c_R01 = p_R01, c_R23 = p_R23;
        const uint32_t cc[3] = {compact3(p_key), compact3(p_key >> 1), compact3(p_key >> 2)};
        double org[3];
        bool needs_fix = false;
        if constexpr (ADAPT) {  // leaf frame: -L in the dims where the leaf touches the upper face (bits 0..2)
            const uint32_t fr = a.lframe[p_box];
#pragma unroll
            for (int d = 0; d < 3; ++d) org[d] = ((fr >> d) & 1u) ? -a.g.L[d] : 0.0;
            needs_fix = fr != 0u;  // touches an upper (bits 0..2) or lower (bits 3..5) face
        } else {
#pragma unroll
            for (int d = 0; d < 3; ++d)
                org[d] = (LAYOUT == P2P_INDEXED) ? frame_shift(a.g, cc, d) : __fma_rn((double)cc[d], a.g.h, a.g.lo[d]);
            if (LAYOUT == P2P_INDEXED) {
#pragma unroll
                for (int d = 0; d < 3; ++d)
                    needs_fix |= ((a.g.periodic >> d) & 1u) && (cc[d] == 0 || (int)cc[d] == a.g.nbox[d] - 1);
            }
        }
        // lane layout (precomputed by k_nbr_fill): G groups of K targets x S source splits
        uint32_t S = (c_meta >> 8) & 0xffu, G = (c_meta >> 16) & 0xffu;
        const uint32_t nt = c_meta & 0xffu;
        if (LAYOUT == P2P_INDEXED_BITWISE && sizeof(T) == 4 && ((c_meta >> 24) & 1u)) {
            S = 4u;  // a multi-box-quad member: the REDUNDANT eval's lane layout (G <= 2 groups x 4 splits)
            G = (nt + K - 1) / K;
        }
        const uint32_t m20 = c_m20[S];
        const uint32_t g = (lane * m20) >> 20, sl = lane - g * S;
        const bool active = g < G;
        // a9: the output slot of target `lane` of the item (one coalesced load, issued now and used in the
        // epilogue -- the load latency was exposed there on small items: c4-8); the epilogue fetches target ti's
        // slot and mass from lane ti by shuffle (2 registers instead of 2 K)
        // target slot ti holds a real target iff bit ti of vmask (multi-box items: slot 8 j + l = target l of box j)
        uint32_t vmask = nt >= 32u ? 0xffffffffu : ((1u << nt) - 1u);
        uint32_t my_t = c_t0 + lane;
        if (c_mb) {
            vmask = 0u;
            uint32_t pre = 0u;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t ntj = (c_mbnt >> (4 * j)) & 0xfu;
                vmask |= ((1u << ntj) - 1u) << (8 * j);
                if ((lane >> 3) == (uint32_t)j) my_t = c_t0 + pre + (lane & 7u);
                pre += ntj;
            }
        }
        const bool my_valid = (vmask >> lane) & 1u;
        const uint32_t my_slot = my_valid ? __ldg(a.perm + my_t) : 0u;
        T my_m = 0;

        Tgt<T, K> tg;
        tg.zero();

        bool have_next = true;
        for (uint32_t c = 0; c < c_nch; ++c) {
            // prefetch the next chunk (or the next item's first chunk + targets) into the other stage
            if (c + 1 < c_nch) {
                issue(c + 1, s ^ 1);
            } else if (nxt < n_items) {
                load_item();
                issue(0, s ^ 1);
                nxt = next_index();
                prefetch(nxt);
            } else {
                have_next = false;
            }
            mbar_wait(&bar[s], (phases >> s) & 1u);
            phases ^= 1u << s;
            V4 *stg = stage_base + s * STAGE_RECS;
            const uint32_t c0 = c * CH;
            const uint32_t cnt = min((uint32_t)CH, c_R - c0);

            if (c == 0) {  // targets landed with the first chunk
                if (my_valid) my_m = stg[CH + lane].w;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const uint32_t ti = g * K + k;
                    T x = 0, y = 0, z = 0;
                    if (active && ((vmask >> ti) & 1u)) {
                        const V4 r = stg[CH + ti];
                        if (LAYOUT == P2P_INDEXED) {
                            x = r.x + (T)org[0];
                            y = r.y + (T)org[1];
                            z = r.z + (T)org[2];
                        } else if (LAYOUT == P2P_REDUNDANT) {
                            x = r.x;
                            y = r.y;
                            z = r.z;
                        } else {  // INDEXED_BITWISE: k_restructure's formula with S = 0
                            x = (T)__dsub_rn(__dadd_rn((double)r.x, 0.0), org[0]);
                            y = (T)__dsub_rn(__dadd_rn((double)r.y, 0.0), org[1]);
                            z = (T)__dsub_rn(__dadd_rn((double)r.z, 0.0), org[2]);
                        }
                    }
                    tg.set(k, x, y, z);
                }
            }

            // ---- layout fix-ups of the staged raw records (INDEXED variants only) ----
            if (LAYOUT == P2P_INDEXED_BITWISE || (LAYOUT == P2P_INDEXED && needs_fix)) {
                // segment groups of 32 (one group unless ADAPT rows are longer than a warp)
                uint32_t gbase = 0;
                for (uint32_t g0 = 0; g0 < c_ne; g0 += 32) {
                uint32_t g_st = c_st, g_cnt = c_cnt, g_slot = c_slot, g_tot = 0;
                if (ADAPT && g0 > 0) {
                    uint32_t src;
                    seg_group(c_e0, c_ne, g0, gbase, src, g_st, g_cnt, g_slot, g_tot);
                } else {
                    g_tot = __shfl_sync(FULL, c_st + c_cnt, 31);
                }
                const uint32_t gne = min(32u, c_ne - g0);
                for (uint32_t e = 0; e < gne; ++e) {
                    const uint32_t est = __shfl_sync(FULL, g_st, e), ecnt = __shfl_sync(FULL, g_cnt, e);
                    const int eslot = (int)__shfl_sync(FULL, g_slot, e);
                    const uint32_t ov0 = max(c0, est), ov1 = min(c0 + cnt, est + ecnt);
                    if (ov1 <= ov0) continue;
                    const double S0 = ADAPT ? (double)(eslot % 3 - 1) * a.g.L[0] : slot_shift(a.g, cc, eslot, 0);
                    const double S1 = ADAPT ? (double)((eslot / 3) % 3 - 1) * a.g.L[1] : slot_shift(a.g, cc, eslot, 1);
                    const double S2 = ADAPT ? (double)(eslot / 9 - 1) * a.g.L[2] : slot_shift(a.g, cc, eslot, 2);
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
                gbase = (ADAPT && g0 > 0) ? gbase + g_tot : g_tot;
                if (!ADAPT) break;
                }
                __syncwarp();
            }

            // ---- the hot loop: staged sources x register targets ----
            if (c_mb) {  // group g = box g / 2's targets over its own piece of this stage (S = 4)
                const uint32_t j = g >> 1;
                const uint32_t Rj = (j < 2 ? c_R01 : c_R23) >> (16 * (j & 1u)) & 0xffffu;
                const uint32_t cj = c * MBP, cntj = Rj > cj ? min(MBP, Rj - cj) : 0u;
                if (sl < cntj) {
                    if constexpr (sizeof(T) == 4)
                        hot_loop<T, K, 4>(tg, smem_u32(stg + MBP * j + sl), ((cntj - 1u - sl) >> 2) + 1u, E);
                }
            } else if (active && sl < cnt) {
                // two sources per iteration with one remainder step: the accumulators stay in the same
                // registers (no IMAD.MOV copies, which would occupy the FMA-heavy pipe the FFMA2s run on), and
                // the addresses advance by pointer increments (ALU pipe) instead of IMAD
                const uint32_t nj = (((cnt - 1 - sl) * m20) >> 20) + 1;
                const uint32_t sa = smem_u32(stg + sl);
                // the split stride S as a compile-time constant: the second source of an iteration is an
                // immediate-offset LDS and the pointer advances once per two sources
                if constexpr (sizeof(T) == 4) {
#ifdef P2P_EV_HOT_RT
                    hot_loop_rt4<K>(tg, sa, nj, S * 16u, E);
#else
                    switch (S) {
                    case 32: hot_loop<T, K, 32>(tg, sa, nj, E); break;
                    case 16: hot_loop<T, K, 16>(tg, sa, nj, E); break;
                    case 10: hot_loop<T, K, 10>(tg, sa, nj, E); break;
                    case 8: hot_loop<T, K, 8>(tg, sa, nj, E); break;
                    case 6: hot_loop<T, K, 6>(tg, sa, nj, E); break;
                    case 5: hot_loop<T, K, 5>(tg, sa, nj, E); break;
                    default: hot_loop<T, K, 4>(tg, sa, nj, E); break;  // S >= 4 always (G <= 8)
                    }
#endif
                } else {
                    hot_loop_rt<T, K>(tg, sa, nj, S * (uint32_t)sizeof(V4), E);
                }
            }
            __syncwarp();
            s ^= 1;
        }

        // ---- combine the S source splits of each group (fixed shuffle pattern -> deterministic) and
        // ---- a9: scatter to input order; remove the self potential term (DESIGN C3) ----
        if constexpr (sizeof(T) == 4) {
            float v[4];
            tg.treduce(S, sl, g * S, v);
            // the lane's values after the transpose-reduce (see Tgt::treduce): f0 .. f0 + vcnt - 1 (vcnt <= 4:
            // S >= 4 for K = 4, S >= 8 for K = 8, as ITEM_TMAX = 32 bounds G)
            constexpr uint32_t LOGV = Tgt<T, K>::LOGV, LOGK = K == 4 ? 2u : 3u;
            const uint32_t lg = 31u - __clz(S);  // log2 of the power-of-two part of S
            const uint32_t Lh = lg < LOGV ? lg : LOGV, vcnt = (1u << LOGV) >> Lh, f0 = (sl >> (lg - Lh)) * vcnt;
            const bool own = active && sl < (1u << lg) && (lg <= LOGV || (sl & 1u) == 0u);
            const T rs = Tgt<T, K>::self_rinv(eps2);
#pragma unroll
            for (int j = 0; j < 4; ++j) {  // all lanes run the shuffles (no divergence around them)
                const uint32_t f = f0 + j, q = f >> LOGK, k = f & (K - 1u), ti = g * K + k;
                const uint32_t i = __shfl_sync(FULL, my_slot, ti & 31u);
                const T mk = __shfl_sync(FULL, my_m, ti & 31u);
                if ((uint32_t)j < vcnt && own && ((vmask >> ti) & 1u))
                    put_result<PEER>(a, i, (int)q, q == 0 ? -(v[j] - mk * rs) : v[j]);
            }
        } else {
        tg.reduce(S, sl);
        {
            const T rs = Tgt<T, K>::self_rinv(eps2);
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const uint32_t ti = g * K + k;
                const uint32_t i = __shfl_sync(FULL, my_slot, ti & 31u);
                const T mk = __shfl_sync(FULL, my_m, ti & 31u);
                if (active && sl == 0 && ((vmask >> ti) & 1u)) {
                    T pot, fx, fy, fz;
                    tg.get(k, pot, fx, fy, fz);
                    put_result<PEER>(a, i, 0, -(pot - mk * rs));
                    put_result<PEER>(a, i, 1, fx);
                    put_result<PEER>(a, i, 2, fy);
                    put_result<PEER>(a, i, 3, fz);
                }
            }
        }
        }
        if (!have_next) break;
    }
    }
    // the remaining small boxes' targets, if any (fills the tail of the item queue)
    if (!small_first) small_phase<T, LAYOUT, PEER>(a, lane);
}

template <typename T, int LAYOUT, int K, bool ADAPT = false, bool PEER = false>
p2p_status launch(p2p_plan *P, void *phi, void *field, int slot, const EvalItems *ov = nullptr,
                  const PeerRes *pr = nullptr) {
    using V4 = typename V4T<T>::type;
    auto kern = k_eval_gravity<T, LAYOUT, K, ADAPT, PEER>;
    const int smem = EV_WARPS * 2 * (EV_STAGE_BYTES + EV_TGT * (int)sizeof(V4));
    if (PEER) slot += 5;  // own occupancy record
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
    a.n_items = &P->ctr->n_items;
    if constexpr (LAYOUT == P2P_REDUNDANT && sizeof(T) == 4 && K == 4 && !ADAPT) {
        if (P->items_red) {  // the REDUNDANT item list with multi-box quads (k_structs.cu mb_quad)
            a.items = P->items_red;
            a.n_items = &P->ctr->n_items_red;
        }
    }
    a.item_head = &P->ctr->item_head;
    a.n_small = &P->ctr->n_small;
    a.small_head = &P->ctr->small_head;
    a.small_tgt = P->small_tgt;
    a.small_box = P->small_box;
    a.phi = (T *)phi;
    a.field = (T *)field;
    a.zero = 0u;
    a.lframe = nullptr;
    a.pr = pr;
    if (ov) {  // an explicit item list over an explicit redundant buffer / CSR (adaptive leaves), no small-box path
        a.red = (const V4 *)ov->red;
        a.items = ov->items;
        a.n_items = ov->n_items;
        a.n_small = ov->zero;
        if (ov->csr_off) {
            a.nbr_off = ov->csr_off;
            a.nbr_box = ov->csr_nbr;
            a.nbr_slot = ov->csr_code;
            a.bstart = ov->lstart;
            a.lframe = ov->lframe;
        }
    }
    const int64_t nit = ov ? ov->n_items_host : (P->sizes_known ? P->n_items + (P->n + 31) / 32 : P->cap);
    const unsigned grid =
        (unsigned)std::min<int64_t>(P->eval_blocks[slot], std::max<int64_t>(1, (nit + EV_WARPS - 1) / EV_WARPS));
    P2P_CUDA_TRY(cudaMemsetAsync(&P->ctr->item_head, 0, sizeof(unsigned int), P->stream));
    P2P_CUDA_TRY(cudaMemsetAsync(&P->ctr->small_head, 0, sizeof(unsigned int), P->stream));
    P2P_LAUNCH(kern, grid, EV_WARPS * 32, smem, P->stream, a);
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}
}  // namespace

p2p_status eval_gravity_items(p2p_plan *P, const EvalItems &it, void *phi, void *field) {
    if (it.csr_off) {  // INDEXED over the adaptive leaves' CSR (the non-redundant baseline)
        if (P->cfg.precision == P2P_FP64) return launch<double, P2P_INDEXED, EVAL_K_F64, true>(P, phi, field, 4, &it);
        return launch<float, P2P_INDEXED, EVAL_K_F32, true>(P, phi, field, 4, &it);
    }
    if (P->cfg.precision == P2P_FP64) return launch<double, P2P_REDUNDANT, EVAL_K_F64>(P, phi, field, 3, &it);
    return launch<float, P2P_REDUNDANT, EVAL_K_F32>(P, phi, field, 3, &it);
}

p2p_status eval_gravity(p2p_plan *P, p2p_layout layout, void *phi, void *field, const PeerRes *pr) {
    if (P->sizes_known && P->n == 0) return P2P_OK;
    const bool f64 = P->cfg.precision == P2P_FP64;
    if (pr) {  // multi-GPU over peer memory: results stored into the origin ranks' buffers
        switch (layout) {
        case P2P_REDUNDANT:
            return f64 ? launch<double, P2P_REDUNDANT, EVAL_K_F64, false, true>(P, phi, field, 0, nullptr, pr)
                       : launch<float, P2P_REDUNDANT, EVAL_K_F32, false, true>(P, phi, field, 0, nullptr, pr);
        case P2P_INDEXED:
            return f64 ? launch<double, P2P_INDEXED, EVAL_K_F64, false, true>(P, phi, field, 1, nullptr, pr)
                       : launch<float, P2P_INDEXED, EVAL_K_F32, false, true>(P, phi, field, 1, nullptr, pr);
        case P2P_INDEXED_BITWISE:
            return f64 ? launch<double, P2P_INDEXED_BITWISE, EVAL_K_F64, false, true>(P, phi, field, 2, nullptr, pr)
                       : launch<float, P2P_INDEXED_BITWISE, EVAL_K_F32, false, true>(P, phi, field, 2, nullptr, pr);
        }
        return P2P_ERR_INVALID_ARGUMENT;
    }
    switch (layout) {
    case P2P_REDUNDANT:
        return f64 ? launch<double, P2P_REDUNDANT, EVAL_K_F64>(P, phi, field, 0)
                   : launch<float, P2P_REDUNDANT, EVAL_K_F32>(P, phi, field, 0);
    case P2P_INDEXED:
        return f64 ? launch<double, P2P_INDEXED, EVAL_K_F64>(P, phi, field, 1)
                   : launch<float, P2P_INDEXED, EVAL_K_F32>(P, phi, field, 1);
    case P2P_INDEXED_BITWISE:
        return f64 ? launch<double, P2P_INDEXED_BITWISE, EVAL_K_F64>(P, phi, field, 2)
                   : launch<float, P2P_INDEXED_BITWISE, EVAL_K_F32>(P, phi, field, 2);
    }
    return P2P_ERR_INVALID_ARGUMENT;
}

}  // namespace p2p
