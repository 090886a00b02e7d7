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
#include <cstdlib>
#include <string>

#include "plan.hpp"
#include "restructure.cuh"

namespace p2p {

namespace {

// ---- pipelined restructure (round 2): cp.async gathers into a per-warp 2-stage shared-memory ring ----------
// The round-1 kernel (below, P2P_RS_LEGACY) ran three dependent load levels per chunk (entry -> segment / owner ->
// records) with at most 4 windows of gathered records in flight in REGISTERS, so every warp waited ~3 memory
// latencies per chunk (ncu: 45% long-scoreboard stalls, 0.63 of the HBM copy peak).  Here a warp streams PIECES
// of <= 4 KB of one chunk's output range: the records of piece p+1 are gathered by cp.async (LDGSTS, no registers
// held) into one shared stage while the warp rebases and stores piece p from the other, and the next chunk's
// metadata (level 1 two chunks ahead, level 2 one chunk ahead) is loaded while the current chunk's pieces run.
// Same records, same fp64 rebase, same bits as rs::chunk (tests: red[] byte-equal to the oracle).
namespace rsp {
constexpr int WARPS = 8;
constexpr int DATA_BYTES = 4096;                // records of one piece (256 fp32 / 128 fp64)
constexpr int STAGE_BYTES = DATA_BYTES + 256;   // + the owning entry (lane) of every record, one byte each

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

struct L1 {  // level 1 of a chunk: owner of its first entry, output start, lane e's entry
    uint32_t b0, k, slot;
    unsigned long long gout;
};
struct L2 {  // level 2: lane i's box b0 + i (CSR start, key), lane e's source segment
    uint32_t boff, keyl, src, cnt;
};
struct Meta {  // a chunk, derived from L1 + L2 (per lane = entry 32 ch + lane)
    uint32_t src, st, code, Rc;
    double o0, o1, o2;
    unsigned long long gout;
    bool seg, wrap;
};

template <typename T>
__device__ __forceinline__ L1 load_l1(const rs::Ptrs<T> &p, uint32_t c, uint32_t nchunk, uint32_t n_nbr,
                                      unsigned lane) {
    L1 a{0u, 0u, 13u, 0ull};
    if (c < nchunk) {
        a.b0 = p.chunk_box[c];
        a.gout = p.chunk_out[c];
        const uint32_t e = (c << 5) + lane;
        if (e < n_nbr) {
            a.k = p.nbr_box[e];
            a.slot = p.nbr_slot[e];
        }
    }
    return a;
}
template <typename T>
__device__ __forceinline__ L2 load_l2(const rs::Ptrs<T> &p, const L1 &a, uint32_t c, uint32_t nchunk, uint32_t B,
                                      uint32_t n_nbr, unsigned lane) {
    L2 b{0xffffffffu, 0u, 0u, 0u};
    if (c < nchunk) {
        const uint32_t bl = a.b0 + lane;
        if (bl < B) {
            b.boff = p.nbr_off[bl];
            b.keyl = p.bkey[bl];
        }
        if ((c << 5) + lane < n_nbr) {
            b.src = p.bstart[a.k];
            b.cnt = p.bstart[a.k + 1] - b.src;
        }
    }
    return b;
}
__device__ __forceinline__ Meta derive(const Geom &g, const L1 &a, const L2 &b, uint32_t c, uint32_t n_nbr,
                                       unsigned lane) {
    constexpr unsigned FULL = 0xffffffffu;
    Meta m;
    const uint32_t e = (c << 5) + lane;
    m.seg = e < n_nbr;
    uint32_t i = 0;  // owner of entry e: the largest i with nbr_off[b0 + i] <= e
#pragma unroll
    for (uint32_t step = 16; step > 0; step >>= 1) {
        const uint32_t t = __shfl_sync(FULL, b.boff, i + step);
        if (t <= e) i += step;
    }
    const uint32_t key = __shfl_sync(FULL, b.keyl, i);
    const uint32_t cc[3] = {compact3(key), compact3(key >> 1), compact3(key >> 2)};
    m.o0 = __fma_rn((double)cc[0], g.h, g.lo[0]);
    m.o1 = __fma_rn((double)cc[1], g.h, g.lo[1]);
    m.o2 = __fma_rn((double)cc[2], g.h, g.lo[2]);
    const int slot = m.seg ? (int)a.slot : 13;
    uint32_t code = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double S = rs::slot_shift(g, cc, slot, d);
        code |= (S > 0.0 ? 1u : (S < 0.0 ? 2u : 0u)) << (2 * d);
    }
    m.code = code;
    const uint32_t cnt = m.seg ? b.cnt : 0u;
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= (unsigned)o) incl += y;
    }
    m.st = incl - cnt;
    m.src = b.src;
    m.Rc = __shfl_sync(FULL, incl, 31);
    m.gout = a.gout;
    m.wrap = __any_sync(FULL, m.seg && code != 0u);
    return m;
}
// the entry (lane index) owning record r0 + lane of the chunk: segments starting before r0 (ballot) - 1 + segment
// starts inside [r0, r0 + lane] (OR-reduced bit mask); segments are non-empty and contiguous
__device__ __forceinline__ uint32_t entry_of(const Meta &m, uint32_t r0, uint32_t le) {
    const uint32_t before = __popc(__ballot_sync(0xffffffffu, m.seg && m.st < r0));
    const uint32_t in_win = (m.seg && m.st >= r0 && m.st < r0 + 32) ? (1u << (m.st - r0)) : 0u;
    const uint32_t starts = __reduce_or_sync(0xffffffffu, in_win);
    return (before - 1u + __popc(starts & le)) & 31u;
}

template <typename T, bool EXACT32>
__global__ void __launch_bounds__(WARPS * 32, 3) k_restructure_pipe(const Geom g, const rs::Ptrs<T> p,
                                                                    const DevCounters *__restrict__ ctr) {
    using V4 = typename rs::V4T<T>::type;
    constexpr int PIECE = DATA_BYTES / (int)sizeof(V4);  // records per stage (256 fp32, 128 fp64)
    constexpr int WIN = PIECE / 32;
    constexpr unsigned FULL = 0xffffffffu;
    extern __shared__ __align__(128) unsigned char rsp_smem[];  // [WARPS][2][STAGE_BYTES]
    auto smem = reinterpret_cast<unsigned char (*)[2][STAGE_BYTES]>(rsp_smem);
    const uint32_t B = ctr->B, n_nbr = ctr->n_nbr;
    const uint32_t nchunk = (n_nbr + 31u) >> 5;
    const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t le = lane == 31 ? FULL : ((2u << lane) - 1u);
    const uint32_t sbase = smem_u32(&smem[w][0][0]);

    uint32_t ci = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (ci >= nchunk) return;
    // issue side: chunk ci (meta mi, next piece qi); prefetched: level 1 + 2 of ci + nw, level 1 of ci + 2 nw
    Meta mi;
    {
        const L1 a = load_l1(p, ci, nchunk, n_nbr, lane);
        mi = derive(g, a, load_l2(p, a, ci, nchunk, B, n_nbr, lane), ci, n_nbr, lane);
    }
    L1 pre1 = load_l1(p, ci + nw, nchunk, n_nbr, lane);
    L1 pre1b = load_l1(p, ci + 2 * nw, nchunk, n_nbr, lane);
    L2 pre2 = load_l2(p, pre1, ci + nw, nchunk, B, n_nbr, lane);
    uint32_t qi = 0;

    auto issue_piece = [&](const Meta &m, uint32_t q, int s) {
        const uint32_t dst = sbase + (uint32_t)s * STAGE_BYTES;
#pragma unroll
        for (int u = 0; u < WIN; ++u) {
            const uint32_t r0 = q * PIECE + 32u * u;
            if (r0 >= m.Rc) break;  // warp-uniform
            const uint32_t xe = entry_of(m, r0, le);
            const uint32_t e_src = __shfl_sync(FULL, m.src, xe), e_st = __shfl_sync(FULL, m.st, xe);
            const uint32_t r = r0 + lane;
            // the record's entry for the consume side (found once, here)
            asm volatile("st.shared.u8 [%0], %1;" ::"r"(dst + DATA_BYTES + 32u * u + lane), "r"(xe) : "memory");
            if (r < m.Rc) {
                const V4 *srcp = p.rec + e_src + (r - e_st);
                const uint32_t d = dst + (32u * u + lane) * (uint32_t)sizeof(V4);
#pragma unroll
                for (int h = 0; h < (int)sizeof(V4) / 16; ++h)
                    cp_async16(d + 16u * h, reinterpret_cast<const unsigned char *>(srcp) + 16 * h);
            }
        }
    };
    // one more piece on the issue side into stage s (false when everything is issued)
    auto advance_issue = [&](int s) -> bool {
        if (qi * PIECE >= mi.Rc) {
            ci += nw;
            if (ci >= nchunk) return false;
            mi = derive(g, pre1, pre2, ci, n_nbr, lane);
            pre1 = pre1b;
            pre2 = load_l2(p, pre1, ci + nw, nchunk, B, n_nbr, lane);
            pre1b = load_l1(p, ci + 2 * nw, nchunk, n_nbr, lane);
            qi = 0;
        }
        issue_piece(mi, qi, s);
        ++qi;
        return true;
    };

    issue_piece(mi, 0, 0);
    qi = 1;
    cp_commit();
    Meta mc = mi;  // consume side
    uint32_t qc = 0;
    int s = 0;
    const double L0 = g.L[0], L1v = g.L[1], L2v = g.L[2];
    while (true) {
        const bool more = advance_issue(s ^ 1);
        cp_commit();
        cp_wait1();
        __syncwarp();
        // ---- rebase + store piece qc of chunk mc from stage s ----
        const uint32_t src_s = sbase + (uint32_t)s * STAGE_BYTES;
        V4 *__restrict__ out = p.red + mc.gout;
        const bool fast32 = EXACT32 && !mc.wrap;
        const float f0o = (float)mc.o0, f1o = (float)mc.o1, f2o = (float)mc.o2;
#pragma unroll
        for (int u = 0; u < WIN; ++u) {
            const uint32_t r0 = qc * PIECE + 32u * u;
            if (r0 >= mc.Rc) break;
            uint32_t xe;
            asm volatile("ld.shared.u8 %0, [%1];" : "=r"(xe) : "r"(src_s + DATA_BYTES + 32u * u + lane) : "memory");
            const uint32_t r = r0 + lane;
            const uint32_t a = src_s + (32u * u + lane) * (uint32_t)sizeof(V4);
            if (fast32) {
                const float eo0 = __shfl_sync(FULL, f0o, xe), eo1 = __shfl_sync(FULL, f1o, xe),
                            eo2 = __shfl_sync(FULL, f2o, xe);
                if (r < mc.Rc) {
                    float4 x;
                    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                                 : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "r"(a) : "memory");
                    V4 v;
                    v.x = (T)__fsub_rn(__fadd_rn(x.x, 0.0f), eo0);
                    v.y = (T)__fsub_rn(__fadd_rn(x.y, 0.0f), eo1);
                    v.z = (T)__fsub_rn(__fadd_rn(x.z, 0.0f), eo2);
                    v.w = (T)x.w;
                    rs::st_cs(out + r, v);
                }
            } else {
                const double eo0 = __shfl_sync(FULL, mc.o0, xe), eo1 = __shfl_sync(FULL, mc.o1, xe),
                             eo2 = __shfl_sync(FULL, mc.o2, xe);
                double S0 = 0.0, S1 = 0.0, S2 = 0.0;
                if (mc.wrap) {
                    const uint32_t cd = __shfl_sync(FULL, mc.code, xe);
                    S0 = (cd & 1u) ? L0 : ((cd & 2u) ? -L0 : 0.0);
                    S1 = (cd & 4u) ? L1v : ((cd & 8u) ? -L1v : 0.0);
                    S2 = (cd & 16u) ? L2v : ((cd & 32u) ? -L2v : 0.0);
                }
                if (r < mc.Rc) {
                    const V4 x = *reinterpret_cast<const V4 *>(&smem[w][s][(32u * u + lane) * sizeof(V4)]);  // 16-B aligned
                    V4 v;
                    v.x = (T)__dsub_rn(__dadd_rn((double)x.x, S0), eo0);
                    v.y = (T)__dsub_rn(__dadd_rn((double)x.y, S1), eo1);
                    v.z = (T)__dsub_rn(__dadd_rn((double)x.z, S2), eo2);
                    v.w = x.w;
                    rs::st_cs(out + r, v);
                }
            }
        }
        __syncwarp();  // stage s is refilled by the next iteration's issue
        ++qc;
        if (qc * PIECE >= mc.Rc) {
            if (!more) break;
            mc = mi;
            qc = 0;
        }
        s ^= 1;
    }
}
}  // namespace rsp

#ifndef P2P_RS_BATCH
#define P2P_RS_BATCH 0
#endif
#ifndef P2P_RS_MINB
#define P2P_RS_MINB 0  // 0: no register cap (ptxas picks 62)
#endif
#if P2P_RS_MINB > 0
#define P2P_RS_LB __launch_bounds__(256, P2P_RS_MINB)
#else
#define P2P_RS_LB __launch_bounds__(256)
#endif
template <typename T, bool EXACT32>
__global__ void P2P_RS_LB k_restructure_gravity(const Geom g, const rs::Ptrs<T> p,
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
#if P2P_RS_BATCH > 0
    // dynamic batches of P2P_RS_BATCH consecutive chunks per queue atomic (the next batch claimed a batch ahead):
    // the static stride left the SMs 7% idle at the end (ncu: active cycles min / avg / max 1.98 / 2.14 / 2.27 M of
    // 2.29 M on c5w -- the Plummer core's chunks carry more records); one atomic per chunk serialised on the counter
    (void)nw;
    unsigned int *head = const_cast<unsigned int *>(&ctr->rs_head);
    uint32_t cur = 0, nxt = 0;
    if (lane == 0) cur = atomicAdd(head, (unsigned)P2P_RS_BATCH);
    cur = __shfl_sync(0xffffffffu, cur, 0);
    while (cur < nchunk) {
        if (lane == 0) nxt = atomicAdd(head, (unsigned)P2P_RS_BATCH);
        const uint32_t end = min(nchunk, cur + (uint32_t)P2P_RS_BATCH);
        load1(cur);
        for (uint32_t c = cur; c < end; ++c) {
            const uint32_t b0 = n_b0, k = n_k, slot = n_slot;
            const unsigned long long gout = n_gout;
            if (c + 1 < end) load1(c + 1);
            rs::chunk<T, EXACT32>(g, p, B, n_nbr, c, b0, gout, k, slot, lane);
        }
        cur = __shfl_sync(0xffffffffu, nxt, 0);
    }
#else
    uint32_t ch = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    load1(ch);
    for (; ch < nchunk; ch += nw) {
        const uint32_t b0 = n_b0, k = n_k, slot = n_slot;
        const unsigned long long gout = n_gout;
        load1(ch + nw);
        rs::chunk<T, EXACT32>(g, p, B, n_nbr, ch, b0, gout, k, slot, lane);
    }
#endif
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
    // 4 vectors per thread per step, loads first (4 independent nbr9 -> xs chains in flight)
    const uint32_t stride = gridDim.x * blockDim.x;
    uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    for (; v + 3 * stride < total; v += 4 * stride) {
        uint4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t w = v + u * stride;
            const uint32_t row = POW2 ? w >> sh : w / n16;
            const uint32_t k = __ldg(nbr9 + row);
            x[u] = make_uint4(0u, 0u, 0u, 0u);
            if (k != 0xffffffffu) x[u] = __ldg(xs + (size_t)k * n16 + (w - row * n16));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) __stcs(Xg + v + u * stride, x[u]);
    }
    for (; v < total; v += stride) {
        const uint32_t row = POW2 ? v >> sh : v / n16;
        const uint32_t j = v - row * n16;
        const uint32_t k = __ldg(nbr9 + row);
        uint4 x = make_uint4(0u, 0u, 0u, 0u);  // missing neighbour: +0.0 real and imaginary (C10)
        // the lattice is regular (every box holds exactly t samples, else UNSUPPORTED at plan creation), so box k's
        // samples start at k t: no dependent bstart load; Xg is written once and read by the next kernel -- streaming
        // stores keep the L2 for the xs rows every Xg row re-reads
        if (k != 0xffffffffu) x = __ldg(xs + (size_t)k * n16 + j);
        __stcs(Xg + v, x);
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
#ifndef P2P_RS_CTAS_PER_SM
#define P2P_RS_CTAS_PER_SM 16
#endif
    const unsigned grid =
        std::max<unsigned>(1, std::min<unsigned>(div_up(nchunk * 32, 256), (unsigned)P->num_sms * P2P_RS_CTAS_PER_SM));
    static const bool legacy = [] {
        // the pipelined kernel (rsp::k_restructure_pipe) measured SLOWER than the chunk kernel on every workload
        // (c5w 1.38 vs 1.18 ms, c4-8 1.23 vs 1.11, c3 0.126 vs 0.097: ncu -- long-scoreboard stalls 46% -> 13%,
        // but 55% more instructions and 24 instead of 32 warps per SM leave it issue-bound at 70%); it stays
        // available as P2P_RS=pipe for the record (profiles/r02_restructure_variants.txt)
        const char *e = getenv("P2P_RS");
        return !(e && std::string(e) == "pipe");
    }();
    if (!legacy) {
        // pipelined kernel: 3 CTAs of 8 warps per SM (64 KB of stages each), a warp per chunk stride
        const unsigned g2 = std::max<unsigned>(
            1, std::min<unsigned>(div_up(nchunk, rsp::WARPS), (unsigned)P->num_sms * 3));
        constexpr int smem = rsp::WARPS * 2 * rsp::STAGE_BYTES;
        auto kd = rsp::k_restructure_pipe<double, false>;
        auto kf1 = rsp::k_restructure_pipe<float, true>;
        auto kf0 = rsp::k_restructure_pipe<float, false>;
        if (P->cfg.precision == P2P_FP64) {
            P2P_CUDA_TRY(cudaFuncSetAttribute(kd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            P2P_LAUNCH(kd, g2, rsp::WARPS * 32, smem, P->stream, P->geom, rs_ptrs<double>(P), P->ctr);
        } else {
            auto kf = origins_exact_fp32(P->geom) ? kf1 : kf0;
            P2P_CUDA_TRY(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            P2P_LAUNCH(kf, g2, rsp::WARPS * 32, smem, P->stream, P->geom, rs_ptrs<float>(P), P->ctr);
        }
        P2P_CUDA_TRY(cudaGetLastError());
        return P2P_OK;
    }
    if (P2P_RS_BATCH > 0) P2P_CUDA_TRY(cudaMemsetAsync(&P->ctr->rs_head, 0, sizeof(unsigned int), P->stream));
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
