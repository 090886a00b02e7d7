// k_helmholtz.cu -- the DBIM-MLFMA-like case (§5.1): the 9t^2 pattern table and method step a8.
//
// Pattern table ("all 9t^2 neighboring patterns ... calculated once before algorithm execution and
// used later by loading into sharing-memory"): P[i][s t + j] = weight between target sub-cell i of a box and
// source sub-cell j of its stencil neighbour s = 3(dy+1) + (dx+1), sub-cell q = qy sqrt(t) + qx.  Weights
// (DESIGN C15): G(r) Delta^2 with G(r) = (i/4) H0^(1)(k r) off the diagonal, the Richmond equal-area-disk self
// term (i pi a / 2k) H1^(1)(k a) - 1/k^2, a = Delta / sqrt(pi), on the diagonal.  Built ONCE per plan on the
// host in fp64 with libstdc++'s std::cyl_bessel_j / std::cyl_neumann (an implementation independent of the
// oracle's), rounded once to the working precision and copied to the device.
//
// a8: y_b = P Xg_b for every box b -- a batched complex matrix-vector product, i.e. one GEMM
// Y[B x t] = Xg[B x 9t] P^T.  Round-1 kernel: CUDA-core FP32 (4 FFMA per complex MAC), CTA tile of BM boxes x
// t outputs, register micro-tile RB boxes x RO outputs per thread, K streamed through shared memory in KT
// slices.  REDUNDANT reads the im2col buffer Xg (restructure output); INDEXED gathers the same values from
// the Morton-sorted unknowns through the 9-slot neighbour table on the fly (zero for missing neighbours).
#include <cmath>
#include <cstdlib>
#include <complex>
#include <vector>

#include "plan.hpp"

namespace p2p {

namespace {
template <typename T> struct C2T;
template <> struct C2T<float> { using type = float2; };
template <> struct C2T<double> { using type = double2; };

void weight(double r, double delta, double k, double *re, double *im) {
    if (r == 0.0) {
        const double a = delta / std::sqrt(M_PI);
        const double c = M_PI * a / (2.0 * k);
        // i c H1(ka) - 1/k^2, H1 = J1 + i Y1
        *re = -c * std::cyl_neumann(1.0, k * a) - 1.0 / (k * k);
        *im = c * std::cyl_bessel_j(1.0, k * a);
    } else {
        const double kr = k * r;
        *re = -0.25 * std::cyl_neumann(0.0, kr) * delta * delta;
        *im = 0.25 * std::cyl_bessel_j(0.0, kr) * delta * delta;
    }
}

constexpr int HZ_THREADS = 256;
constexpr int HZ_KT = 16;

// tiled kernel for a compile-time t (16 or 64)
template <typename T, int LAYOUT, int TT, int RB, int RO>
__global__ void __launch_bounds__(HZ_THREADS) k_eval_helm_tiled(const typename C2T<T>::type *__restrict__ Pt,
                                                                 const typename C2T<T>::type *__restrict__ Xg,
                                                                 const typename C2T<T>::type *__restrict__ xs,
                                                                 const uint32_t *__restrict__ nbr9,
                                                                 const uint32_t *__restrict__ bstart,
                                                                 const uint32_t *__restrict__ perm, uint32_t B,
                                                                 typename C2T<T>::type *__restrict__ y) {
    using C2 = typename C2T<T>::type;
    constexpr int TO = TT / RO;                 // threads along outputs
    constexpr int TB = HZ_THREADS / TO;         // threads along boxes
    constexpr int BM = TB * RB;                 // boxes per CTA
    constexpr int KK = 9 * TT;
    __shared__ C2 Xs[BM][HZ_KT + 1];
    __shared__ C2 Ps[TT][HZ_KT + 1];
    const int tid = threadIdx.x;
    const int to = tid % TO, tb = tid / TO;
    const uint32_t b0 = blockIdx.x * BM;
    T accr[RB][RO], acci[RB][RO];
#pragma unroll
    for (int i = 0; i < RB; ++i)
#pragma unroll
        for (int j = 0; j < RO; ++j) accr[i][j] = acci[i][j] = 0;

    for (int m0 = 0; m0 < KK; m0 += HZ_KT) {
        for (int e = tid; e < BM * HZ_KT; e += HZ_THREADS) {
            const int bi = e / HZ_KT, kk = e % HZ_KT;
            const uint32_t b = b0 + bi;
            C2 v;
            v.x = 0;
            v.y = 0;
            if (b < B) {
                const int m = m0 + kk;
                if (LAYOUT == P2P_REDUNDANT) {
                    v = Xg[(size_t)b * KK + m];
                } else {
                    const int s = m / TT, j = m % TT;
                    const uint32_t k = nbr9[(size_t)b * 9 + s];
                    if (k != 0xffffffffu) v = xs[bstart[k] + j];
                }
            }
            Xs[bi][kk] = v;
        }
        for (int e = tid; e < TT * HZ_KT; e += HZ_THREADS) {
            const int i = e / HZ_KT, kk = e % HZ_KT;
            Ps[i][kk] = Pt[(size_t)i * KK + m0 + kk];
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < HZ_KT; ++kk) {
            C2 xv[RB], pv[RO];
#pragma unroll
            for (int i = 0; i < RB; ++i) xv[i] = Xs[tb * RB + i][kk];
#pragma unroll
            for (int j = 0; j < RO; ++j) pv[j] = Ps[to * RO + j][kk];
#pragma unroll
            for (int i = 0; i < RB; ++i)
#pragma unroll
                for (int j = 0; j < RO; ++j) {
                    accr[i][j] = fma(pv[j].x, xv[i].x, accr[i][j]);
                    accr[i][j] = fma(-pv[j].y, xv[i].y, accr[i][j]);
                    acci[i][j] = fma(pv[j].x, xv[i].y, acci[i][j]);
                    acci[i][j] = fma(pv[j].y, xv[i].x, acci[i][j]);
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < RB; ++i) {
        const uint32_t b = b0 + tb * RB + i;
        if (b >= B) continue;
#pragma unroll
        for (int j = 0; j < RO; ++j) {
            const uint32_t o = bstart[b] + to * RO + j;
            C2 v;
            v.x = accr[i][j];
            v.y = acci[i][j];
            y[perm[o]] = v;
        }
    }
}

// generic kernel for any t: one thread per (box, output)
template <typename T, int LAYOUT>
__global__ void k_eval_helm_generic(const typename C2T<T>::type *__restrict__ Pt,
                                    const typename C2T<T>::type *__restrict__ Xg,
                                    const typename C2T<T>::type *__restrict__ xs, const uint32_t *__restrict__ nbr9,
                                    const uint32_t *__restrict__ bstart, const uint32_t *__restrict__ perm, uint32_t B,
                                    uint32_t t, typename C2T<T>::type *__restrict__ y) {
    using C2 = typename C2T<T>::type;
    const uint64_t total = (uint64_t)B * t;
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t b = (uint32_t)(q / t), i = (uint32_t)(q % t);
        T yr = 0, yi = 0;
        for (uint32_t s = 0; s < 9; ++s) {
            const uint32_t k = nbr9[(size_t)b * 9 + s];
            for (uint32_t j = 0; j < t; ++j) {
                C2 xv;
                if (LAYOUT == P2P_REDUNDANT) xv = Xg[((size_t)b * 9 + s) * t + j];
                else if (k != 0xffffffffu) xv = xs[bstart[k] + j];
                else { xv.x = 0; xv.y = 0; }
                const C2 pv = Pt[(size_t)i * 9 * t + s * t + j];
                yr = fma(pv.x, xv.x, yr);
                yr = fma(-pv.y, xv.y, yr);
                yi = fma(pv.x, xv.y, yi);
                yi = fma(pv.y, xv.x, yi);
            }
        }
        C2 v;
        v.x = yr;
        v.y = yi;
        y[perm[bstart[b] + i]] = v;
    }
}

// fp32 kernel with packed FP32x2 complex MACs: acc = (re, im); per complex MAC (a+ib)(c+id):
//   acc = fma2((a, a), (c, d), acc); acc = fma2((-b, b), (d, c), acc)      -> 2 FFMA2 (4 lane-ops)
// so the FP32 work issues in half the slots.  Shared tiles hold X as (c, d, d, c) and P as (a, a, -b, b) float4
// so one LDS.128 yields both operand pairs.  Warp tile 32 boxes x 16 outputs, lane = (box group bg, output
// group og), boxes bg + 8r / outputs og + 4r' interleaved (conflict-free LDS.128); CTA = 8 warps.
// Rounding sequence per component identical to k_eval_helm_tiled (fp64) (same two fmas in the same order).
constexpr int HF_KT = 8;

template <int LAYOUT, int TT>
__global__ void __launch_bounds__(256) k_eval_helm_f2(const float2 *__restrict__ Pt, const float2 *__restrict__ Xg,
                                                       const float2 *__restrict__ xs, const uint32_t *__restrict__ nbr9,
                                                       const uint32_t *__restrict__ bstart,
                                                       const uint32_t *__restrict__ perm, uint32_t B,
                                                       float2 *__restrict__ y) {
    constexpr int WO = TT / 16, WB = 8 / WO, BM = 32 * WB, KK = 9 * TT;
    constexpr int RB = 4, RO = 4;
    __shared__ float4 Xs[BM][HF_KT + 1];
    __shared__ float4 Ps[TT][HF_KT + 1];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int wb = w / WO, wo = w % WO;
    const int bg = lane >> 2, og = lane & 3;
    const uint32_t b0 = blockIdx.x * BM;
    float2 acc[RB][RO];
#pragma unroll
    for (int i = 0; i < RB; ++i)
#pragma unroll
        for (int j = 0; j < RO; ++j) acc[i][j] = make_float2(0.f, 0.f);

    // register double buffering: the global loads of chunk m0 + KT are issued before chunk m0 is computed
    constexpr int XE = BM * HF_KT / 256, PE = (TT * HF_KT + 255) / 256;
    float2 xr[XE], pr[PE];
    auto gload = [&](int m0) {
#pragma unroll
        for (int q = 0; q < XE; ++q) {
            const int e = tid + 256 * q, bi = e / HF_KT, kk = e % HF_KT;
            const uint32_t b = b0 + bi;
            float2 v = make_float2(0.f, 0.f);
            if (b < B) {
                const int m = m0 + kk;
                if (LAYOUT == P2P_REDUNDANT) {
                    v = Xg[(size_t)b * KK + m];
                } else {
                    const uint32_t k = nbr9[(size_t)b * 9 + m / TT];
                    if (k != 0xffffffffu) v = xs[bstart[k] + m % TT];
                }
            }
            xr[q] = v;
        }
#pragma unroll
        for (int q = 0; q < PE; ++q) {
            const int e = tid + 256 * q;
            if (e < TT * HF_KT) pr[q] = Pt[(size_t)(e / HF_KT) * KK + m0 + e % HF_KT];
        }
    };
    gload(0);
    for (int m0 = 0; m0 < KK; m0 += HF_KT) {
#pragma unroll
        for (int q = 0; q < XE; ++q) {
            const int e = tid + 256 * q;
            Xs[e / HF_KT][e % HF_KT] = make_float4(xr[q].x, xr[q].y, xr[q].y, xr[q].x);
        }
#pragma unroll
        for (int q = 0; q < PE; ++q) {
            const int e = tid + 256 * q;
            if (e < TT * HF_KT) Ps[e / HF_KT][e % HF_KT] = make_float4(pr[q].x, pr[q].x, -pr[q].y, pr[q].y);
        }
        __syncthreads();
        if (m0 + HF_KT < KK) gload(m0 + HF_KT);
#pragma unroll
        for (int kk = 0; kk < HF_KT; ++kk) {
            float4 xv[RB], pv[RO];
#pragma unroll
            for (int r = 0; r < RB; ++r) xv[r] = Xs[wb * 32 + bg + 8 * r][kk];
#pragma unroll
            for (int r = 0; r < RO; ++r) pv[r] = Ps[wo * 16 + og + 4 * r][kk];
#pragma unroll
            for (int i = 0; i < RB; ++i)
#pragma unroll
                for (int j = 0; j < RO; ++j) {
                    acc[i][j] = __ffma2_rn(make_float2(pv[j].x, pv[j].y), make_float2(xv[i].x, xv[i].y), acc[i][j]);
                    acc[i][j] = __ffma2_rn(make_float2(pv[j].z, pv[j].w), make_float2(xv[i].z, xv[i].w), acc[i][j]);
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < RB; ++i) {
        const uint32_t b = b0 + wb * 32 + bg + 8 * i;
        if (b >= B) continue;
        const uint32_t s0 = bstart[b];
#pragma unroll
        for (int j = 0; j < RO; ++j) y[perm[s0 + wo * 16 + og + 4 * j]] = acc[i][j];
    }
}

template <typename T, int LAYOUT>
p2p_status launch_helm(p2p_plan *P, void *y) {
    using C2 = typename C2T<T>::type;
    const uint32_t t = (uint32_t)P->cfg.points_per_box, B = (uint32_t)P->B;
    const C2 *Pt = (const C2 *)P->table, *Xg = (const C2 *)P->red, *xs = (const C2 *)P->rec;
    bool done = false;
    if constexpr (sizeof(T) == 4) {
        if (t == 16) {
            P2P_LAUNCH((k_eval_helm_f2<LAYOUT, 16>), div_up(B, 256), 256, 0, P->stream, (const float2 *)Pt,
                       (const float2 *)Xg, (const float2 *)xs, P->nbr_box, P->bstart, P->perm, B, (float2 *)y);
            done = true;
        } else if (t == 64) {
            P2P_LAUNCH((k_eval_helm_f2<LAYOUT, 64>), div_up(B, 64), 256, 0, P->stream, (const float2 *)Pt,
                       (const float2 *)Xg, (const float2 *)xs, P->nbr_box, P->bstart, P->perm, B, (float2 *)y);
            done = true;
        }
    }
    if (!done) {
        const unsigned grid = std::min<unsigned>(div_up((uint64_t)B * t, 256), (unsigned)P->num_sms * 16);
        P2P_LAUNCH((k_eval_helm_generic<T, LAYOUT>), grid, 256, 0, P->stream, Pt, Xg, xs, P->nbr_box, P->bstart,
                   P->perm, B, t, (C2 *)y);
    }
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}
}  // namespace

p2p_status helmholtz_table(p2p_plan *P) {
    const int t = P->cfg.points_per_box;
    int st = 0;
    while (st * st < t) ++st;
    const double delta = P->cfg.box_size / (double)st;
    const double k = P->cfg.wavenumber;
    const size_t ne = (size_t)t * 9 * t;
    std::vector<double> tab(2 * ne);
    for (int i = 0; i < t; ++i) {
        const int ix = i % st, iy = i / st;
        for (int s = 0; s < 9; ++s) {
            const int dx = s % 3 - 1, dy = s / 3 - 1;
            for (int j = 0; j < t; ++j) {
                const int jx = j % st, jy = j / st;
                const double rx = (double)(dx * st + jx - ix) * delta, ry = (double)(dy * st + jy - iy) * delta;
                double re, im;
                weight(std::sqrt(rx * rx + ry * ry), delta, k, &re, &im);
                const size_t q = (size_t)i * 9 * t + s * t + j;
                tab[2 * q] = re;
                tab[2 * q + 1] = im;
            }
        }
    }
    const bool f64 = P->cfg.precision == P2P_FP64;
    const size_t bytes = ne * (f64 ? sizeof(double2) : sizeof(float2));
    P2P_CUDA_TRY(dalloc(&P->table, bytes, P->stream));
    if (f64) {
        P2P_CUDA_TRY(cudaMemcpyAsync(P->table, tab.data(), bytes, cudaMemcpyHostToDevice, P->stream));
        P2P_CUDA_TRY(cudaStreamSynchronize(P->stream));
    } else {
        std::vector<float> f(2 * ne);
        for (size_t q = 0; q < 2 * ne; ++q) f[q] = (float)tab[q];
        P2P_CUDA_TRY(cudaMemcpyAsync(P->table, f.data(), bytes, cudaMemcpyHostToDevice, P->stream));
        P2P_CUDA_TRY(cudaStreamSynchronize(P->stream));
        if (helmholtz_tc_supported(P)) return helmholtz_tc_table(P, f.data());
    }
    return P2P_OK;
}

p2p_status eval_helmholtz(p2p_plan *P, p2p_layout layout, void *y) {
    if (P->B == 0) return P2P_OK;
    const bool f64 = P->cfg.precision == P2P_FP64;
    // REDUNDANT fp32 with t in {16, 64}: the tensor-core GEMM; P2P_HELM_SIMT=1 keeps the CUDA-core kernel
    // (diagnostics / comparison only)
    static const bool force_simt = [] {
        const char *e = getenv("P2P_HELM_SIMT");
        return e && e[0] == '1';
    }();
    // fp32 t in {16, 64}: BOTH layouts on the tensor cores (the like-for-like DBIM comparison): REDUNDANT streams Xg
    // by TMA, INDEXED gathers the neighbour segments of xs by cp.async (k_helm_tc.cu GATHER); P2P_HELM_SIMT=1 runs
    // both on the CUDA cores instead
    if ((layout == P2P_REDUNDANT || layout == P2P_INDEXED) && P->tc_table && !force_simt)
        return eval_helmholtz_tc(P, y, layout == P2P_INDEXED);
    if (layout == P2P_REDUNDANT) return f64 ? launch_helm<double, P2P_REDUNDANT>(P, y) : launch_helm<float, P2P_REDUNDANT>(P, y);
    return f64 ? launch_helm<double, P2P_INDEXED>(P, y) : launch_helm<float, P2P_INDEXED>(P, y);
}

}  // namespace p2p
