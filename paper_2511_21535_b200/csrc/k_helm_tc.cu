// k_helm_tc.cu -- method step a8 (§5.1) on the 5th-generation tensor cores: Y = Xg P^T as ONE
// real GEMM, fp32-accurate through 3xTF32 ("a 3xTF32 tensor-core variant of Y = X P^T under
// the 1e-5 tolerance").
//
// Real form.  Xg[b] (9t complex, interleaved re/im) is a real row of K = 18t floats as stored -- the restructure
// output is the A operand without any copy.  The pattern table becomes a real N x K matrix W (N = 2t):
//   row i      (Re y_i):  W[i][2c] =  Re P[i][c],  W[i][2c+1]   = -Im P[i][c]
//   row t + i  (Im y_i):  W[t+i][2c] = Im P[i][c],  W[t+i][2c+1] =  Re P[i][c]
// so D[b][n] = sum_k Xg[b][k] W[n][k] holds Re y in columns < t and Im y in columns >= t.
//
// 3xTF32.  x = hi(x) + lo(x) with hi(x) = x rounded to the nearest TF32 value (low 13 mantissa bits zero, so the
// tensor core reads it exactly) and lo(x) = x - hi(x) (exact in fp32, |lo| <= 2^-11 |x|); D = Xhi Whi + Xhi Wlo +
// Xlo Whi, the dropped Xlo Wlo term and the TF32 reading of the lo parts are ~2^-22 relative per product.  W's parts are built once on the host (plan create); X is split
// in shared memory after each TMA load (hi in place, lo into a second buffer with the same swizzled offsets).
//
// Kernel: one CTA per 128 boxes (M = 128), all N = 2t outputs in one TMEM accumulator (N fp32 columns).
//   warp SW, one lane     TMA producer: 2D tensor loads (128-byte swizzle) of the X tile and both W tiles of
//                         each 32-float K slice into a 3-stage ring (mbarrier full / empty)
//   warps 0..SW-1         split X of each landed slice (mbarrier split, 32 SW arrivals; SW = 4, or 8 at t = 64)
//   warp SW+1, one lane   MMA issuer: 4 K-steps x 3 tcgen05.mma per slice (kind::tf32, M = 128, N = 2t, K = 8,
//                         both operands K-major from shared memory descriptors), committed to the stage's empty
//                         barrier (and, after the last slice, to the accumulator barrier)
//   epilogue (warps 0-3)  tcgen05.ld of the accumulator rows (TMEM lane = box), scatter to input order
//
// GATHER = true is the non-redundant (INDEXED) layout on the same tensor cores -- the like-for-like DBIM comparison
// of the paper's block-level redundancy (§5.1.2): no Xg; each split thread gathers its box row's K slice
// straight from the Morton-sorted unknowns, xs[t * nbr9[b][s] ..] (slot s = the slice's stencil segment, a missing
// neighbour zero-filled), by cp.async 16-byte copies into its own row of the stage, D = TC_STAGES - 1 slices ahead
// (private rows: no barrier), then splits as above.  Only W goes through TMA.  Same A values, same MMA sequence:
// the outputs equal the REDUNDANT tensor-core path bit for bit.
#include <cuda.h>

#include <cstdlib>
#include <cstring>
#include <vector>

#include "plan.hpp"

namespace p2p {

namespace {
constexpr int TC_BM = 128;        // boxes per CTA (MMA M, TMEM lanes)
constexpr int TC_BK = 32;         // floats per K slice = one 128-byte swizzle row
constexpr int TC_STAGES = 4;      // smem ring of X + W hi + W lo slices (48 KB each at t = 64)
// threads per CTA: split / epilogue warps (4 at t = 16, 8 at t = 64) + 1 TMA producer warp + 1 MMA issuer warp
// split warps per CTA (P2P_HELM_SPLITW, t = 64): the X split into TF32 hi / lo (smem -> registers -> tcgen05.st) paces
// the kernel, so at t = 64 (one CTA per SM) 8 warps split, two per TMEM lane quarter, 16 of a slice's 32 columns each
#ifndef P2P_HELM_SPLITW
#define P2P_HELM_SPLITW 8
#endif
template <int T>
constexpr int tc_splitw() { return T == 64 ? P2P_HELM_SPLITW : 4; }
template <int T>
constexpr int tc_threads() { return 32 * (tc_splitw<T>() + 2); }
// TMEM accumulators (K slices round-robin, summed in fp32 at the end): as many as fit the 512 TMEM columns, at
// most 8 -- the tensor core's internal fp32 accumulation loses ~2^-23 of the running sum per step (measured: one
// accumulator 7.8e-6, four 2.0e-6 relative L2 at t = 64 vs the fp64 oracle)
// (the remaining columns hold >= 2 stages of the X hi / lo operand, 64 columns each)
template <int N>
constexpr int tc_nacc() { return (N < 32 ? 32 : N) * 8 <= 256 ? 8 : (512 - 128) / (N < 32 ? 32 : N); }

__device__ __forceinline__ uint32_t cvta_smem(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// the nearest TF32 value (ties away from zero on the magnitude bits): |x - hi| <= 2^-11 |x|, and x - hi is exact
// in fp32; finite inputs of this path never reach the exponent limit
__device__ __forceinline__ float tf32_rn(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart (SBO), sm_100 version 1
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(1024u >> 4) << 32) |
           ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int x, int y, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(map), "r"(x), "r"(y), "r"(bar)
        : "memory");
}

// the same 2D load delivered to every CTA of `mask` in the cluster (same shared offset, each CTA's own mbarrier)
__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap *map, int x, int y, uint32_t bar,
                                               uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, "
        "%3}], [%4], %5;" ::"r"(dst),
        "l"(map), "r"(x), "r"(y), "r"(bar), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void mma_commit_mc(uint32_t bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::
                     "r"(bar), "h"(mask)
                 : "memory");
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(cvta_smem(bar)) : "memory");
}

// A from TMEM (X hi / lo written by the split warps), B from a shared-memory descriptor
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// 32 consecutive 32-bit TMEM columns of this thread's lane <- registers
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
        "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
        "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

// 16 consecutive 32-bit TMEM columns of this thread's lane <- registers
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// t = 16: half the TMEM (256 columns: 4 accumulators + 2 operand stages) and 96 KB of shared memory per CTA, so two
// CTAs share an SM (the grid of 512 small tiles was 3.5 waves of one CTA per SM); t = 64: the whole TMEM
template <int T>
constexpr uint32_t tc_tcols() { return T == 16 ? 256u : 512u; }

__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void *src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}

// NSPLIT = 2 (t = 64, P2P_HELM_NSPLIT): the N = 2t outputs of a 128-box tile are split over two CTAs (half 0: the
// Re y columns, 1: the Im y columns; each loads X and its half of W; the two are adjacent in launch order, so the
// second X read hits L2): 1024 units of work instead of 512, so the last of the 148-SM waves is nearly full (512
// tiles were 3.46 waves of one CTA per SM: 13.5% idle)
// CL > 1 (P2P_HELM_CLUSTER): clusters of CL CTAs share every W slice through TMA MULTICAST ("RF copies
// of the pattern table ... as B200 cluster TMA multicast"): CTA r of the cluster loads rows [r N/CL, (r+1) N/CL) of
// the W hi / lo slice into the same shared offset of all CL CTAs, so each W byte crosses L2 -> SM once per cluster
// instead of once per CTA (W was 2/3 of the kernel's 48 KB per slice of TMA traffic).  A stage is refilled only
// after all CL MMA issuers released it: their commits arrive on every CTA's `empty` barrier (multicast commit).
template <int T, bool GATHER = false, int NSPLIT = 1, int CL = 1>
__global__ void __launch_bounds__(tc_threads<T>(), T == 16 ? 2 : 1)
    k_helm_tc(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmWhi,
              const __grid_constant__ CUtensorMap tmWlo, uint32_t rf, const uint32_t *__restrict__ bstart,
              const uint32_t *__restrict__ perm, uint32_t B, float2 *__restrict__ y,
              const float *__restrict__ xs, const uint32_t *__restrict__ nbr9) {
    constexpr int NF = 2 * T, N = NF / NSPLIT, K = 18 * T, NKT = K / TC_BK;  // NF: all outputs, N: this CTA's
    static_assert(NSPLIT == 1 || (NSPLIT == 2 && T >= 32), "split into the Re / Im halves only");
    constexpr uint32_t X_BYTES = TC_BM * TC_BK * 4, W_BYTES = N * TC_BK * 4;
    constexpr uint32_t STAGE_BYTES = X_BYTES + 2 * W_BYTES;  // X (raw fp32), W hi, W lo
    constexpr uint32_t AST = N < 32 ? 32 : N;                 // TMEM columns per accumulator
    constexpr uint32_t TCOLS = tc_tcols<T>();
    constexpr int NACC = T == 16 ? 4 : tc_nacc<N>();
    constexpr uint32_t ACOL = NACC * AST;                       // first TMEM column of the A stages
    constexpr int ASTAGES = (int)((TCOLS - ACOL) / (2 * TC_BK)); // X hi + X lo = 64 columns per stage
    static_assert(ASTAGES >= 2, "TMEM budget");
    // instruction descriptor: D fp32, A/B TF32, both K-major, N >> 3, M >> 4
    constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                               ((uint32_t)(TC_BM >> 4) << 24);
    static_assert(K % TC_BK == 0 && N % 16 == 0 && N <= 256, "unsupported t");
    constexpr int SW = tc_splitw<T>();           // split warps: 4 or 8 (two per TMEM lane quarter)
    constexpr int NCH = 8 / (SW / 4);            // 16-byte chunks of a 128-byte row per split thread
    static_assert(SW == 4 || SW == 8, "4 or 8 split warps");

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[TC_STAGES], empty[TC_STAGES], tsplit[8], tfree[8], accum;
    __shared__ uint32_t tmem_base;
    // 1024-byte alignment of the stage ring (128-byte swizzle atoms)
    const uint32_t ring = (cvta_smem(smem_raw) + 1023u) & ~1023u;
    unsigned char *ring_gen = smem_raw + (ring - cvta_smem(smem_raw));

    const unsigned tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    const uint32_t half = NSPLIT == 2 ? (blockIdx.x & 1u) : 0u, tile = NSPLIT == 2 ? (blockIdx.x >> 1) : blockIdx.x;
    const uint32_t m0 = tile * TC_BM;
    if (tid == 0) {
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CL);  // one commit from each MMA issuer of the cluster
        }
        for (int a = 0; a < ASTAGES; ++a) {
            mbar_init(&tsplit[a], 32 * SW);
            mbar_init(&tfree[a], 1);
        }
        mbar_init(&accum, 1);
        fence_mbar_init();
    }
    if (warp == 0) {  // TCOLS TMEM columns: NACC accumulators + ASTAGES (X hi, X lo) operand stages
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(cvta_smem(&tmem_base)),
                     "r"(TCOLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if constexpr (CL > 1) cluster_sync();  // every CTA's barriers initialised before any multicast lands
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base;
    const uint32_t crank = CL > 1 ? cluster_rank() : 0u;
    constexpr uint16_t CMASK = (uint16_t)((1u << CL) - 1u);

    if (warp == SW) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            for (int kt = 0; kt < NKT; ++kt) {
                const int s = kt % TC_STAGES;
                if (kt >= TC_STAGES) mbar_wait(&empty[s], (uint32_t)((kt / TC_STAGES - 1) & 1));
                const uint32_t st = ring + s * STAGE_BYTES;
                mbar_arrive_expect_tx(&full[s], GATHER ? 2 * W_BYTES : STAGE_BYTES);
                if (!GATHER) tma_load_2d(st, &tmX, kt * TC_BK, (int)m0, cvta_smem(&full[s]));
                // block-level redundancy (RF copies of the pattern table): CTA b reads copy b mod RF
                // (clusters: the cluster's index mod RF -- its CTAs share one copy)
                const int wrow = (int)(((CL > 1 ? tile / CL : tile) % rf) * NF + half * N);
                if constexpr (CL > 1) {
                    constexpr int RP = N / CL;  // W rows this CTA multicasts (a multiple of 8: whole swizzle atoms)
                    const uint32_t off = crank * RP * (TC_BK * 4);
                    tma_load_2d_mc(st + X_BYTES + off, &tmWhi, kt * TC_BK, wrow + (int)(crank * RP),
                                   cvta_smem(&full[s]), CMASK);
                    tma_load_2d_mc(st + X_BYTES + W_BYTES + off, &tmWlo, kt * TC_BK, wrow + (int)(crank * RP),
                                   cvta_smem(&full[s]), CMASK);
                } else {
                    tma_load_2d(st + X_BYTES, &tmWhi, kt * TC_BK, wrow, cvta_smem(&full[s]));
                    tma_load_2d(st + X_BYTES + W_BYTES, &tmWlo, kt * TC_BK, wrow, cvta_smem(&full[s]));
                }
            }
        }
    } else if (warp == SW + 1) {
        // ---------------- MMA issuer (one lane): A = X hi / lo from TMEM, B = W hi / lo from shared memory ----
        if (lane == 0) {
            for (int kt = 0; kt < NKT; ++kt) {
                const int s = kt % TC_STAGES, a = kt % ASTAGES;
                mbar_wait(&full[s], (uint32_t)((kt / TC_STAGES) & 1));
                mbar_wait(&tsplit[a], (uint32_t)((kt / ASTAGES) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t st = ring + s * STAGE_BYTES;
                const uint32_t b_hi = st + X_BYTES, b_lo = b_hi + W_BYTES;
                const uint32_t a_hi = tmem + ACOL + (uint32_t)a * (2 * TC_BK), a_lo = a_hi + TC_BK;
                const uint32_t d = tmem + (uint32_t)((kt % NACC) * AST);
#pragma unroll
                for (int k = 0; k < TC_BK / 8; ++k) {  // 4 K-steps of 8 TF32: 8 TMEM columns / 32 smem bytes
                    const uint32_t acc0 = (kt >= NACC || k > 0) ? 1u : 0u;
                    mma_tf32_ts(d, a_hi + 8 * k, sdesc_sw128(b_hi + 32 * k), IDESC, acc0);
                    mma_tf32_ts(d, a_hi + 8 * k, sdesc_sw128(b_lo + 32 * k), IDESC, 1u);
                    mma_tf32_ts(d, a_lo + 8 * k, sdesc_sw128(b_hi + 32 * k), IDESC, 1u);
                }
                if constexpr (CL > 1)
                    mma_commit_mc(cvta_smem(&empty[s]), CMASK);  // stage s consumed: tell every producer of the cluster
                else
                    mma_commit(cvta_smem(&empty[s]));  // W of smem stage s consumed
                mma_commit(cvta_smem(&tfree[a]));  // X hi / lo of TMEM stage a consumed
            }
            mma_commit(cvta_smem(&accum));
        }
    } else {
        // ---------------- split X rows into TF32 hi / lo, straight into TMEM ----------------
        // thread = one X row (TMEM lane 32 warp + lane); its 128-byte row sits 16-byte-chunk-swizzled in smem
        const uint32_t rq = warp & 3u, hh = warp >> 2;  // TMEM lane quarter; which NCH chunks of the row
        const uint32_t r = rq * 32 + lane;
        const uint32_t lane_cols = (rq * 32u) << 16;
        const uint32_t c0 = hh * NCH;
        // GATHER: this row's K slice kt = 32 floats of stencil segment s = 32 kt / 2t (2t is a multiple of 32)
        constexpr int GD = TC_STAGES - 1;  // slices gathered ahead
        const uint32_t gb = m0 + r;
        auto gather = [&](int kt) {
            const uint32_t f0 = (uint32_t)kt * TC_BK, slot = f0 / (2 * T), off = f0 - slot * 2 * T;
            const uint32_t k = gb < B ? __ldg(nbr9 + (size_t)gb * 9 + slot) : 0xffffffffu;
            const bool ok = k != 0xffffffffu;
            const float *src = xs + (ok ? (size_t)k * 2 * T + off : 0);
            const uint32_t dst = ring + (uint32_t)(kt % TC_STAGES) * STAGE_BYTES + r * 128;
#pragma unroll
            for (int c = (int)c0; c < (int)c0 + NCH; ++c) cp_async16_zfill(dst + 16 * c, src + 4 * c, ok ? 16u : 0u);
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        if constexpr (GATHER) {
            for (int kt = 0; kt < GD; ++kt) {
                if (kt < NKT) gather(kt);
                else asm volatile("cp.async.commit_group;" ::: "memory");
            }
        }
        for (int kt = 0; kt < NKT; ++kt) {
            const int s = kt % TC_STAGES, a = kt % ASTAGES;
            if constexpr (GATHER) {
                // stage (kt + GD) % TC_STAGES was last read by this thread at slice kt - 1 (its own row)
                if (kt + GD < NKT) gather(kt + GD);
                else asm volatile("cp.async.commit_group;" ::: "memory");
                asm volatile("cp.async.wait_group %0;" ::"n"(GD) : "memory");
            } else {
                mbar_wait(&full[s], (uint32_t)((kt / TC_STAGES) & 1));
            }
            if (kt >= ASTAGES) mbar_wait(&tfree[a], (uint32_t)((kt / ASTAGES - 1) & 1));
            const unsigned char *row = ring_gen + s * STAGE_BYTES + r * 128;
            uint32_t hi[4 * NCH], lo[4 * NCH];
#pragma unroll
            for (int j = 0; j < NCH; ++j) {
                const uint32_t c = c0 + (uint32_t)j;
                const float4 v = *reinterpret_cast<const float4 *>(row + ((GATHER ? c : (c ^ (r & 7))) << 4));
                const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float h = tf32_rn(e[q]);
                    hi[4 * j + q] = __float_as_uint(h);
                    lo[4 * j + q] = __float_as_uint(__fsub_rn(e[q], h));
                }
            }
            const uint32_t ta = tmem + lane_cols + ACOL + (uint32_t)a * (2 * TC_BK) + 4 * c0;
            if constexpr (NCH == 8) {
                tmem_st32(ta, hi);
                tmem_st32(ta + TC_BK, lo);
            } else {
                tmem_st16(ta, hi);
                tmem_st16(ta + TC_BK, lo);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            mbar_arrive(&tsplit[a]);
        }
        // ---------------- epilogue: TMEM -> registers -> y in input order (lane quarters: warps 0..3) ----------------
        if (hh == 0) {
        mbar_wait(&accum, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t b = m0 + r;  // this thread's TMEM lane = box
        const uint32_t lane_addr = tmem + lane_cols;
        const uint32_t s0 = b < B ? bstart[b] : 0u;
        if constexpr (T < 32) {  // t = 16: Re in columns 0..15, Im in 16..31 of one 32-column load
            float v[32];
            tmem_ld32(lane_addr, v);
#pragma unroll
            for (int ac = 1; ac < NACC; ++ac) {
                float w[32];
                tmem_ld32(lane_addr + ac * AST, w);
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] += w[i];
            }
            if (b < B) {
#pragma unroll
                for (int i = 0; i < T; ++i) y[perm[s0 + i]] = make_float2(v[i], v[T + i]);
            }
        } else if constexpr (NSPLIT == 2) {  // this CTA's half: Re (half 0) or Im (1) of outputs 0 .. t-1
            float *yf = reinterpret_cast<float *>(y) + half;
#pragma unroll
            for (int c0 = 0; c0 < T; c0 += 32) {
                float v[32];
                tmem_ld32(lane_addr + c0, v);
#pragma unroll
                for (int ac = 1; ac < NACC; ++ac) {
                    float w[32];
                    tmem_ld32(lane_addr + ac * AST + c0, w);
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] += w[i];
                }
                if (b < B) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) yf[2 * (size_t)perm[s0 + c0 + i]] = v[i];
                }
            }
        } else {
#pragma unroll
            for (int c0 = 0; c0 < T; c0 += 32) {  // outputs c0 .. c0 + 31
                float re[32], im[32];
                tmem_ld32(lane_addr + c0, re);
                tmem_ld32(lane_addr + T + c0, im);
#pragma unroll
                for (int ac = 1; ac < NACC; ++ac) {
                    float w[32];
                    tmem_ld32(lane_addr + ac * AST + c0, w);
#pragma unroll
                    for (int i = 0; i < 32; ++i) re[i] += w[i];
                    tmem_ld32(lane_addr + ac * AST + T + c0, w);
#pragma unroll
                    for (int i = 0; i < 32; ++i) im[i] += w[i];
                }
                if (b < B) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) y[perm[s0 + c0 + i]] = make_float2(re[i], im[i]);
                }
            }
        }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    __syncthreads();
    if constexpr (CL > 1) cluster_sync();  // no CTA exits while a cluster peer may still multicast into it
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS) : "memory");
    }
}

// ---------------------------------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

// 2D fp32 tensor [rows][cols] row-major, box [box_rows][32 floats], 128-byte swizzle
bool make_map(CUtensorMap *m, const void *base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 4};
    const cuuint32_t box[2] = {(cuuint32_t)TC_BK, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int T, bool GATHER, int NSPLIT = 1, int CL = 1>
p2p_status launch_tc(p2p_plan *P, void *y) {
    constexpr int N = 2 * T, K = 18 * T, NC = N / NSPLIT;
    constexpr uint32_t STAGE_BYTES = TC_BM * TC_BK * 4 + 2 * NC * TC_BK * 4;
    const int smem = (int)(TC_STAGES * STAGE_BYTES + 1024);
    CUtensorMap mx, mwh, mwl;
    const float *W = (const float *)P->tc_table;  // [RF] copies of W hi, then [RF] copies of W lo
    const uint32_t rf = (uint32_t)P->tc_rf;
    if (!make_map(&mx, GATHER ? (const void *)W : P->red, GATHER ? (uint64_t)rf * N : (uint64_t)P->B, K,
                  GATHER ? NC : TC_BM) || !make_map(&mwh, W, (uint64_t)rf * N, K, NC / CL) ||
        !make_map(&mwl, W + (size_t)rf * N * K, (uint64_t)rf * N, K, NC / CL)) {
        set_error("cuTensorMapEncodeTiled unavailable or rejected the Helmholtz operands");
        return P2P_ERR_CUDA;
    }
    auto kern = k_helm_tc<T, GATHER, NSPLIT, CL>;
    P2P_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const unsigned tiles = (unsigned)div_up((uint64_t)P->B, TC_BM);
    const unsigned grid = div_up(tiles, CL) * CL * NSPLIT;  // whole clusters (CTAs past B load zeros, store nothing)
    if constexpr (CL > 1) {
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(grid);
        lc.blockDim = dim3(tc_threads<T>());
        lc.dynamicSmemBytes = (size_t)smem;
        lc.stream = P->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        P2P_CUDA_TRY(cudaLaunchKernelEx(&lc, kern, mx, mwh, mwl, rf, (const uint32_t *)P->bstart,
                                        (const uint32_t *)P->perm, (uint32_t)P->B, (float2 *)y,
                                        (const float *)P->rec, (const uint32_t *)P->nbr_box));
        g_launches.fetch_add(1, std::memory_order_relaxed);
    } else {
        P2P_LAUNCH(kern, grid, tc_threads<T>(), smem, P->stream, mx, mwh, mwl, rf, P->bstart, P->perm, (uint32_t)P->B,
                   (float2 *)y, (const float *)P->rec, P->nbr_box);
    }
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}
}  // namespace

bool helmholtz_tc_supported(const p2p_plan *P) {
    const int t = P->cfg.points_per_box;
    return P->cfg.precision == P2P_FP32 && (t == 16 || t == 64) && encode_fn() != nullptr;
}

// W hi / lo (2 x [2t][18t] fp32, K-major) from the fp32 pattern table P[t][9t] (complex)
p2p_status helmholtz_tc_table(p2p_plan *P, const float *Pf /* host, [t][9t] complex */) {
    const int t = P->cfg.points_per_box, N = 2 * t, K = 18 * t;
    std::vector<float> w((size_t)2 * N * K);
    float *hi = w.data(), *lo = w.data() + (size_t)N * K;
    auto split = [](float x, float &h, float &l) {
        uint32_t u;
        std::memcpy(&u, &x, 4);
        u = (u + 0x1000u) & 0xFFFFE000u;  // nearest TF32 value (as tf32_rn on the device)
        std::memcpy(&h, &u, 4);
        l = x - h;  // exact
    };
    for (int i = 0; i < t; ++i)
        for (int c = 0; c < 9 * t; ++c) {
            const float pr = Pf[2 * ((size_t)i * 9 * t + c)], pi = Pf[2 * ((size_t)i * 9 * t + c) + 1];
            const float v[4] = {pr, -pi, pi, pr};  // W[i][2c], W[i][2c+1], W[t+i][2c], W[t+i][2c+1]
            const size_t q[4] = {(size_t)i * K + 2 * c, (size_t)i * K + 2 * c + 1, (size_t)(t + i) * K + 2 * c,
                                 (size_t)(t + i) * K + 2 * c + 1};
            for (int e = 0; e < 4; ++e) split(v[e], hi[q[e]], lo[q[e]]);
        }
    // RF copies (P2P_HELM_RF, default 1: measured no gain): [RF] x W hi, then [RF] x W lo
    const char *e = getenv("P2P_HELM_RF");
    const int rf = e ? std::max(1, std::min(8, atoi(e))) : 1;
    P->tc_rf = rf;
    std::vector<float> wr((size_t)2 * rf * N * K);
    for (int r = 0; r < rf; ++r) {
        std::memcpy(wr.data() + (size_t)r * N * K, hi, sizeof(float) * N * K);
        std::memcpy(wr.data() + (size_t)(rf + r) * N * K, lo, sizeof(float) * N * K);
    }
    P2P_CUDA_TRY(dalloc(&P->tc_table, wr.size() * 4, P->stream));
    P2P_CUDA_TRY(cudaMemcpyAsync(P->tc_table, wr.data(), wr.size() * 4, cudaMemcpyHostToDevice, P->stream));
    P2P_CUDA_TRY(cudaStreamSynchronize(P->stream));
    return P2P_OK;
}

p2p_status eval_helmholtz_tc(p2p_plan *P, void *y, bool gather) {
    if (P->B == 0) return P2P_OK;
    // measured options (profiles/r02_helm_tc_variants.txt), both bit-identical to the default and slower on B200:
    //   P2P_HELM_NSPLIT=2     t = 64 outputs split over two CTAs per 128-box tile (better wave fill, 2x the X split)
    //   P2P_HELM_CLUSTER=2|4  W slices multicast over clusters of 2 / 4 CTAs (W's L2 -> SM traffic / CL)
    const char *e = getenv("P2P_HELM_NSPLIT");  // read per call (tests switch them within one process)
    const int nsplit = (e && atoi(e) == 2) ? 2 : 1;
    const char *c = getenv("P2P_HELM_CLUSTER");
    int cl = c ? atoi(c) : 1;
    if (cl != 1 && cl != 2 && cl != 4) cl = 1;
    if (P->cfg.points_per_box == 16) {
        if (cl == 4) return gather ? launch_tc<16, true, 1, 4>(P, y) : launch_tc<16, false, 1, 4>(P, y);
        if (cl == 2) return gather ? launch_tc<16, true, 1, 2>(P, y) : launch_tc<16, false, 1, 2>(P, y);
        return gather ? launch_tc<16, true>(P, y) : launch_tc<16, false>(P, y);
    }
    if (nsplit == 2) return gather ? launch_tc<64, true, 2>(P, y) : launch_tc<64, false, 2>(P, y);
    if (cl == 4) return gather ? launch_tc<64, true, 1, 4>(P, y) : launch_tc<64, false, 1, 4>(P, y);
    if (cl == 2) return gather ? launch_tc<64, true, 1, 2>(P, y) : launch_tc<64, false, 1, 2>(P, y);
    return gather ? launch_tc<64, true>(P, y) : launch_tc<64, false>(P, y);
}

}  // namespace p2p
