// k_dist.cu -- the multi-GPU path: Morton-range sharding with a halo exchange.
//
// Collective plan build on every rank (all steps stream-ordered; a few host syncs for exchange sizes):
//   1. bin + key the rank's input particles (the same k_bin_gravity as the 1-GPU path);
//   2. coarse histogram over 2^sc_bits Morton "supercells" (key >> shift), all-reduced (sum);
//   3. identical count-balanced splitters on every rank: rank r owns keys [spl[r], spl[r+1]) -- contiguous
//      Morton ranges aligned to supercells (C20);
//   4. repartition: owner of every input particle, stable counting order by owner, all-to-all-v of
//      {x,y,z,m} records -> the owned particles, arranged by (source rank, source input order);
//   5. halo: every owned box whose 26-neighbourhood touches another rank's range is sent whole to that rank
//      (box-level ownership makes the halo symmetric, so no request round is needed);
//   6. the local plan = the ordinary a1..a5 over [owned ; halo] with target boxes restricted to the owned range
//      (halo boxes are sources only).
// Within every box the particles keep increasing GLOBAL input order (owned: rank-major concatenation; halo: the
// owner's sorted order), so every target's redundant run -- records, order and rebased bits -- is identical to
// the 1-GPU plan on the concatenated input: results are bitwise independent of the GPU count.
// Eval: the local eval into owned-order buffers, then the reverse all-to-all-v returns each result to the rank
// and input slot it came from.
#include <algorithm>
#include <vector>

#include "plan.hpp"
#include "scan.cuh"

namespace p2p {

namespace {
template <typename T> struct V4T;
template <> struct V4T<float> { using type = float4; };
template <> struct V4T<double> { using type = double4; };

// positions at pos[i*ps + d] (same binning arithmetic as k_structs.cu k_bin_gravity, DESIGN C6)
template <typename T>
__global__ void k_keys(const T *__restrict__ pos, int ps, uint32_t n, Geom g, uint32_t *__restrict__ key,
                       uint32_t *__restrict__ idx, unsigned long long *err) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t c[3];
        bool bad = false;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            double f = floor(__ddiv_rn(__dsub_rn((double)pos[(size_t)ps * i + d], g.lo[d]), g.h));
            if (!(f >= 0.0 && f < (double)g.nbox[d])) {
                bad = true;
                f = 0.0;
            }
            c[d] = (uint32_t)f;
        }
        if (bad) atomicMin(err, (unsigned long long)i);
        key[i] = spread3(c[0]) | (spread3(c[1]) << 1) | (spread3(c[2]) << 2);
        idx[i] = i;
    }
}

__global__ void k_sc_hist(const uint32_t *__restrict__ key, uint32_t n, int shift, unsigned long long *hist) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        atomicAdd(&hist[key[i] >> shift], 1ull);
}

// hist[nbins] = 1 if this rank saw an out-of-domain input (summed over ranks by the all-reduce)
__global__ void k_err_flag(const unsigned long long *err, unsigned long long *flag) {
    *flag = *err != ~0ull ? 1ull : 0ull;
}

__device__ __forceinline__ int owner_of(uint32_t key, const uint32_t *spl, int G) {
    int lo = 0, hi = G - 1;  // largest r with spl[r] <= key
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (spl[mid] <= key) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void k_dest(const uint32_t *__restrict__ key, uint32_t n, const uint32_t *__restrict__ spl, int G,
                       uint32_t *__restrict__ dest, unsigned int *__restrict__ cnt) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int r = owner_of(key[i], spl, G);
        dest[i] = (uint32_t)r;
        atomicAdd(&cnt[r], 1u);
    }
}

template <typename T, typename V4>
__global__ void k_gather_rec(const T *__restrict__ pos, int ps, const T *__restrict__ q, int qs,
                             const uint32_t *__restrict__ order, uint32_t n, V4 *__restrict__ out) {
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const uint32_t i = order[p];
        V4 r;
        r.x = pos[(size_t)ps * i + 0];
        r.y = pos[(size_t)ps * i + 1];
        r.z = pos[(size_t)ps * i + 2];
        r.w = q[(size_t)qs * i];
        out[p] = r;
    }
}

struct HeadGetD {
    const uint32_t *skey;
    __device__ uint32_t operator()(uint64_t p) const { return (p == 0 || skey[p] != skey[p - 1]) ? 1u : 0u; }
};
struct HeadPutD {
    const uint32_t *skey;
    uint32_t *bkey, *bstart;
    uint32_t n;
    __device__ void operator()(uint64_t p, uint32_t e, uint32_t v) const {
        if (v) {
            bkey[e] = skey[p];
            bstart[e] = (uint32_t)p;
        }
        if (p == n - 1) bstart[e + v] = n;
    }
};

// ranks (other than `me`) that own a key of the box's 26-neighbourhood: they need this box as halo
__device__ unsigned long long halo_mask(const Geom &g, uint32_t key, const uint32_t *spl, int G, int me) {
    const uint32_t c[3] = {compact3(key), compact3(key >> 1), compact3(key >> 2)};
    unsigned long long m = 0ull;
    for (int slot = 0; slot < 27; ++slot) {
        if (slot == 13) continue;
        const int dd[3] = {slot % 3 - 1, (slot / 3) % 3 - 1, slot / 9 - 1};
        uint32_t nc[3];
        bool ok = true;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            int v = (int)c[d] + dd[d];
            if (v < 0 || v >= g.nbox[d]) {
                if (!((g.periodic >> d) & 1u)) ok = false;
                v = v < 0 ? v + g.nbox[d] : v - g.nbox[d];
            }
            nc[d] = (uint32_t)v;
        }
        if (!ok) continue;
        const int r = owner_of(spread3(nc[0]) | (spread3(nc[1]) << 1) | (spread3(nc[2]) << 2), spl, G);
        if (r != me) m |= 1ull << r;
    }
    return m;
}

__global__ void k_halo_count(Geom g, const uint32_t *__restrict__ bkey, const uint32_t *__restrict__ bstart,
                             const uint32_t *__restrict__ Bp, const uint32_t *__restrict__ spl, int G, int me,
                             unsigned long long *__restrict__ mask, unsigned long long *__restrict__ cnt) {
    const uint32_t B = *Bp;
    for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x) {
        const unsigned long long m = halo_mask(g, bkey[b], spl, G, me);
        mask[b] = m;
        const uint32_t nb = bstart[b + 1] - bstart[b];
        for (unsigned long long mm = m; mm; mm &= mm - 1) atomicAdd(&cnt[__ffsll((long long)mm) - 1], (unsigned long long)nb);
    }
}

// warp per box: a box bound for rank r is copied whole (sorted order) to a slot reserved with one atomic
template <typename V4>
__global__ void k_halo_pack(const uint32_t *__restrict__ bstart, const uint32_t *__restrict__ Bp,
                            const unsigned long long *__restrict__ mask, const V4 *__restrict__ sorted,
                            const long long *__restrict__ base, unsigned long long *__restrict__ cursor,
                            V4 *__restrict__ out) {
    const uint32_t B = *Bp;
    const unsigned lane = threadIdx.x & 31u;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < B; b += nwarps) {
        const uint32_t s0 = bstart[b], nb = bstart[b + 1] - s0;
        for (unsigned long long mm = mask[b]; mm; mm &= mm - 1) {
            const int r = __ffsll((long long)mm) - 1;
            unsigned long long pos = 0;
            if (lane == 0) pos = atomicAdd(&cursor[r], (unsigned long long)nb);
            pos = __shfl_sync(0xffffffffu, pos, 0);
            for (uint32_t j = lane; j < nb; j += 32) out[base[r] + pos + j] = sorted[s0 + j];
        }
    }
}

template <typename T, typename V4>
__global__ void k_pack_results(const T *__restrict__ phi, const T *__restrict__ field, uint32_t n, V4 *__restrict__ res) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        V4 r;
        r.x = phi[i];
        r.y = field[3 * (size_t)i + 0];
        r.z = field[3 * (size_t)i + 1];
        r.w = field[3 * (size_t)i + 2];
        res[i] = r;
    }
}

template <typename T, typename V4>
__global__ void k_unpack_results(const V4 *__restrict__ res, const uint32_t *__restrict__ perm_send, uint32_t n,
                                 T *__restrict__ phi, T *__restrict__ field) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const uint32_t i = perm_send[j];
        const V4 r = res[j];
        phi[i] = r.x;
        if (field) {
            field[3 * (size_t)i + 0] = r.y;
            field[3 * (size_t)i + 1] = r.z;
            field[3 * (size_t)i + 2] = r.w;
        }
    }
}

// rank r owns keys [spl[r], spl[r+1]): spl[r] = (first supercell whose exclusive prefix count >= r*total/G)
// << shift -- a pure function of the all-reduced histogram, so every rank derives the same splitters
void compute_splitters(const unsigned long long *h, int64_t nbins, int shift, int key_bits, int G, uint32_t *spl) {
    unsigned long long total = 0;
    for (int64_t b = 0; b < nbins; ++b) total += h[b];
    spl[0] = 0u;
    int r = 1;
    unsigned long long cum = 0;
    for (int64_t b = 0; b < nbins && r < G; ++b) {
        while (r < G && (unsigned __int128)cum * G >= (unsigned __int128)r * total) spl[r++] = (uint32_t)(b << shift);
        cum += h[b];
    }
    for (; r < G; ++r) spl[r] = (uint32_t)std::min<uint64_t>((uint64_t)nbins << shift, 0xffffffffull);
    spl[G] = (uint32_t)std::min<uint64_t>((uint64_t)1 << key_bits, 0xffffffffull);
}

unsigned grid1(uint64_t n, int num_sms) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(div_up(n, 256), (uint64_t)num_sms * 16));
}

struct Tmp {  // stream-ordered temporaries of the build
    cudaStream_t st;
    std::vector<void *> bufs;
    template <typename X>
    cudaError_t get(X **p, size_t bytes) {
        cudaError_t e = dalloc((void **)p, bytes, st);
        if (e == cudaSuccess) bufs.push_back(*p);
        return e;
    }
    ~Tmp() {
        for (void *b : bufs) dfree(b, st);
    }
};

template <typename T>
p2p_status build_dist_t(p2p_plan *P, const void *pos_v, const void *q_v) {
    using V4 = typename V4T<T>::type;
    free_distributed(P);  // a previous build's exchange buffers (p2p_plan_update on a collective plan)
    CommBase *C = P->comm;
    const int G = C->nranks, me = C->rank;
    cudaStream_t st = P->stream;
    const uint32_t n_in = (uint32_t)P->n_in;
    const T *pos = (const T *)pos_v, *q = (const T *)q_v;
    Tmp tmp{st, {}};
    const unsigned gb = grid1(std::max<uint32_t>(n_in, 1), P->num_sms);
    // ---- 1. keys of the input particles ----
    uint32_t *key = nullptr, *idx = nullptr, *kalt = nullptr, *valt = nullptr, *hist8 = nullptr, *status = nullptr;
    unsigned long long *err = nullptr;
    const size_t nn = std::max<uint32_t>(n_in, 1);
    P2P_CUDA_TRY(tmp.get(&key, 4 * nn));
    P2P_CUDA_TRY(tmp.get(&idx, 4 * nn));
    P2P_CUDA_TRY(tmp.get(&kalt, 4 * nn));
    P2P_CUDA_TRY(tmp.get(&valt, 4 * nn));
    P2P_CUDA_TRY(tmp.get(&hist8, 4 * 4 * 256));
    P2P_CUDA_TRY(tmp.get(&err, 8));
    P2P_CUDA_TRY(cudaMemsetAsync(err, 0xff, 8, st));
    if (n_in) P2P_LAUNCH(k_keys<T>, gb, 256, 0, st, pos, 3, n_in, P->geom, key, idx, err);
    // ---- 2. supercell histogram (+ one extra bin: ranks with an out-of-domain input), all-reduced ----
    const int sc_bits = std::min(P->key_bits, 20), shift = P->key_bits - sc_bits;
    const size_t nbins = (size_t)1 << sc_bits;
    unsigned long long *hist = nullptr;
    P2P_CUDA_TRY(tmp.get(&hist, 8 * (nbins + 1)));
    P2P_CUDA_TRY(cudaMemsetAsync(hist, 0, 8 * (nbins + 1), st));
    if (n_in) P2P_LAUNCH(k_sc_hist, gb, 256, 0, st, key, n_in, shift, hist);
    P2P_LAUNCH(k_err_flag, 1, 1, 0, st, err, hist + nbins);
    p2p_status s = C->allreduce_sum_u64(hist, nbins + 1, st);
    if (s != P2P_OK) return s;
    std::vector<unsigned long long> h(nbins + 1);
    unsigned long long herr = ~0ull;
    P2P_CUDA_TRY(cudaMemcpyAsync(h.data(), hist, 8 * (nbins + 1), cudaMemcpyDeviceToHost, st));
    P2P_CUDA_TRY(cudaMemcpyAsync(&herr, err, 8, cudaMemcpyDeviceToHost, st));
    P2P_CUDA_TRY(cudaStreamSynchronize(st));
    if (h[nbins]) {  // every rank bails out consistently
        if (herr != ~0ull) {
            char buf[160];
            snprintf(buf, sizeof buf, "position of input particle %llu is outside the domain (C6)", herr);
            set_error(buf);
        } else {
            set_error("another rank has a position outside the domain (C6)");
        }
        return P2P_ERR_OUT_OF_DOMAIN;
    }
    // ---- 3. count-balanced splitters, identical on every rank (C20) ----
    P->splitters.assign(G + 1, 0u);
    compute_splitters(h.data(), (int64_t)nbins, shift, P->key_bits, G, P->splitters.data());
    const uint32_t lo = P->splitters[me], hi = P->splitters[me + 1];
    P->geom.tkey_lo = lo;
    P->geom.tkey_hi = hi > lo ? hi - 1 : 0u;
    if (hi <= lo) P->geom.tkey_lo = 1;  // empty range: no target box
    uint32_t *spl = nullptr;
    P2P_CUDA_TRY(tmp.get(&spl, 4 * (G + 1)));
    P2P_CUDA_TRY(cudaMemcpyAsync(spl, P->splitters.data(), 4 * (G + 1), cudaMemcpyHostToDevice, st));
    // ---- 4. owners + stable order by owner (1-pass radix sort on the owner rank: stability keeps input order) ----
    uint32_t *dest = nullptr;
    unsigned int *dcnt = nullptr;
    P2P_CUDA_TRY(tmp.get(&dest, 4 * nn));
    P2P_CUDA_TRY(tmp.get(&dcnt, 4 * G));
    P2P_CUDA_TRY(cudaMemsetAsync(dcnt, 0, 4 * G, st));
    P2P_CUDA_TRY(tmp.get(&status, 4 * std::max<size_t>(1, radix_status_words(nn, 1))));
    if (n_in) P2P_LAUNCH(k_dest, gb, 256, 0, st, key, n_in, spl, G, dest, dcnt);
    uint32_t *sdest = nullptr, *order = nullptr;
    P2P_CUDA_TRY(radix_sort_pairs(dest, idx, kalt, valt, n_in, 1, P->ctr, hist8, status, st, &sdest, &order));
    P2P_CUDA_TRY(dalloc((void **)&P->perm_send, 4 * nn, st));
    P2P_CUDA_TRY(cudaMemcpyAsync(P->perm_send, order, 4 * (size_t)n_in, cudaMemcpyDeviceToDevice, st));
    std::vector<unsigned int> hc(G);
    P2P_CUDA_TRY(cudaMemcpyAsync(hc.data(), dcnt, 4 * G, cudaMemcpyDeviceToHost, st));
    P2P_CUDA_TRY(cudaStreamSynchronize(st));
    P->rp_scnt.assign(G, 0);
    P->rp_soff.assign(G, 0);
    P->rp_rcnt.assign(G, 0);
    P->rp_roff.assign(G, 0);
    for (int r = 0; r < G; ++r) {
        P->rp_scnt[r] = hc[r];
        if (r) P->rp_soff[r] = P->rp_soff[r - 1] + P->rp_scnt[r - 1];
    }
    s = C->alltoall_counts(P->rp_scnt.data(), P->rp_rcnt.data(), st);
    if (s != P2P_OK) return s;
    int64_t n_own = 0;
    for (int r = 0; r < G; ++r) {
        P->rp_roff[r] = n_own;
        n_own += P->rp_rcnt[r];
    }
    P->n_own = n_own;
    // ---- 5. repartition: all-to-all-v of {x,y,z,m} records ----
    V4 *send = nullptr, *own = nullptr;
    P2P_CUDA_TRY(tmp.get(&send, sizeof(V4) * nn));
    P2P_CUDA_TRY(tmp.get(&own, sizeof(V4) * std::max<int64_t>(n_own, 1)));
    if (n_in) P2P_LAUNCH((k_gather_rec<T, V4>), gb, 256, 0, st, pos, 3, q, 1, order, n_in, send);
    {
        std::vector<int64_t> so(G), sc(G), ro(G), rc(G);
        for (int r = 0; r < G; ++r) {
            so[r] = P->rp_soff[r] * (int64_t)sizeof(V4);
            sc[r] = P->rp_scnt[r] * (int64_t)sizeof(V4);
            ro[r] = P->rp_roff[r] * (int64_t)sizeof(V4);
            rc[r] = P->rp_rcnt[r] * (int64_t)sizeof(V4);
        }
        s = C->alltoallv(send, so.data(), sc.data(), own, ro.data(), rc.data(), st);
        if (s != P2P_OK) return s;
    }
    // ---- 6. owned boxes (sorted), halo selection and exchange ----
    const uint32_t no = (uint32_t)n_own;
    const size_t nno = std::max<uint32_t>(no, 1);
    uint32_t *okey = nullptr, *oidx = nullptr, *okalt = nullptr, *ovalt = nullptr, *ostatus = nullptr;
    uint32_t *obkey = nullptr, *obstart = nullptr, *oB = nullptr;
    void *opart = nullptr;
    P2P_CUDA_TRY(tmp.get(&okey, 4 * nno));
    P2P_CUDA_TRY(tmp.get(&oidx, 4 * nno));
    P2P_CUDA_TRY(tmp.get(&okalt, 4 * nno));
    P2P_CUDA_TRY(tmp.get(&ovalt, 4 * nno));
    P2P_CUDA_TRY(tmp.get(&ostatus, 4 * std::max<size_t>(1, radix_status_words(nno, std::max(1, P->passes)))));
    P2P_CUDA_TRY(tmp.get(&obkey, 4 * nno));
    P2P_CUDA_TRY(tmp.get(&obstart, 4 * (nno + 1)));
    P2P_CUDA_TRY(tmp.get(&oB, 4));
    P2P_CUDA_TRY(tmp.get(&opart, scan_partials_bytes(nno)));
    P2P_CUDA_TRY(cudaMemsetAsync(oB, 0, 4, st));
    const unsigned gbo = grid1(nno, P->num_sms);
    if (no) P2P_LAUNCH(k_keys<T>, gbo, 256, 0, st, (const T *)own, 4, no, P->geom, okey, oidx, err);
    uint32_t *oskey = nullptr, *operm = nullptr;
    P2P_CUDA_TRY(radix_sort_pairs(okey, oidx, okalt, ovalt, no, P->passes, P->ctr, hist8, ostatus, st, &oskey, &operm));
    P2P_CUDA_TRY(device_scan<uint32_t>(HeadGetD{oskey}, HeadPutD{oskey, obkey, obstart, no}, nullptr, no, oB, opart,
                                       st));
    V4 *osorted = nullptr;
    P2P_CUDA_TRY(tmp.get(&osorted, sizeof(V4) * nno));
    if (no)
        P2P_LAUNCH((k_gather_rec<T, V4>), gbo, 256, 0, st, (const T *)own, 4, (const T *)own + 3, 4, operm, no,
                   osorted);
    unsigned long long *omask = nullptr, *hcnt = nullptr, *cursor = nullptr;
    long long *hbase = nullptr;
    P2P_CUDA_TRY(tmp.get(&omask, 8 * nno));
    P2P_CUDA_TRY(tmp.get(&hcnt, 8 * G));
    P2P_CUDA_TRY(tmp.get(&cursor, 8 * G));
    P2P_CUDA_TRY(tmp.get(&hbase, 8 * G));
    P2P_CUDA_TRY(cudaMemsetAsync(hcnt, 0, 8 * G, st));
    P2P_CUDA_TRY(cudaMemsetAsync(cursor, 0, 8 * G, st));
    P2P_LAUNCH(k_halo_count, gbo, 256, 0, st, P->geom, obkey, obstart, oB, spl, G, me, omask, hcnt);
    std::vector<unsigned long long> hh(G);
    P2P_CUDA_TRY(cudaMemcpyAsync(hh.data(), hcnt, 8 * G, cudaMemcpyDeviceToHost, st));
    P2P_CUDA_TRY(cudaStreamSynchronize(st));
    std::vector<int64_t> hs(G), hso(G), hr(G), hro(G);
    int64_t hsend = 0;
    for (int r = 0; r < G; ++r) {
        hs[r] = (int64_t)hh[r];
        hso[r] = hsend;
        hsend += hs[r];
    }
    P2P_CUDA_TRY(cudaMemcpyAsync(hbase, hso.data(), 8 * G, cudaMemcpyHostToDevice, st));
    V4 *hsendbuf = nullptr;
    P2P_CUDA_TRY(tmp.get(&hsendbuf, sizeof(V4) * std::max<int64_t>(hsend, 1)));
    P2P_LAUNCH((k_halo_pack<V4>), gbo, 256, 0, st, obstart, oB, omask, osorted, hbase, cursor, hsendbuf);
    s = C->alltoall_counts(hs.data(), hr.data(), st);
    if (s != P2P_OK) return s;
    int64_t n_halo = 0;
    for (int r = 0; r < G; ++r) {
        hro[r] = n_halo;
        n_halo += hr[r];
    }
    // the local input = [owned (repartition order) ; halo]
    V4 *local = nullptr;
    P2P_CUDA_TRY(tmp.get(&local, sizeof(V4) * std::max<int64_t>(n_own + n_halo, 1)));
    if (n_own) P2P_CUDA_TRY(cudaMemcpyAsync(local, own, sizeof(V4) * n_own, cudaMemcpyDeviceToDevice, st));
    {
        std::vector<int64_t> so(G), sc(G), ro(G), rc(G);
        for (int r = 0; r < G; ++r) {
            so[r] = hso[r] * (int64_t)sizeof(V4);
            sc[r] = hs[r] * (int64_t)sizeof(V4);
            ro[r] = (n_own + hro[r]) * (int64_t)sizeof(V4);
            rc[r] = hr[r] * (int64_t)sizeof(V4);
        }
        s = C->alltoallv(hsendbuf, so.data(), sc.data(), local, ro.data(), rc.data(), st);
        if (s != P2P_OK) return s;
    }
    // ---- 7. the local plan over [owned ; halo], targets = this rank's Morton range ----
    // capacity buffers persist across p2p_plan_update calls (grow only); the temporaries above are released
    // stream-ordered (cudaFreeAsync), after every collective that reads them has completed on this stream
    P->n = n_own + n_halo;
    if (P->n == 0) return P2P_OK;
    if (P->n > P->cap) {
        free_capacity(P);
        s = alloc_capacity(P, P->n);
        if (s != P2P_OK) return s;
    }
    s = build_gravity_structs(P, nullptr, nullptr, local);
    if (s != P2P_OK) return s;
    P2P_CUDA_TRY(dalloc(&P->phi_loc, sizeof(T) * std::max<int64_t>(n_own, 1), st));
    P2P_CUDA_TRY(dalloc(&P->field_loc, 3 * sizeof(T) * std::max<int64_t>(n_own, 1), st));
    P2P_CUDA_TRY(dalloc(&P->res_own, sizeof(V4) * std::max<int64_t>(n_own, 1), st));
    P2P_CUDA_TRY(dalloc(&P->res_back, sizeof(V4) * nn, st));
    return P2P_OK;
}

template <typename T>
p2p_status eval_dist_t(p2p_plan *P, p2p_layout layout, void *phi, void *field) {
    using V4 = typename V4T<T>::type;
    cudaStream_t st = P->stream;
    const int G = P->comm->nranks;
    if (P->n > 0) {
        p2p_status s = eval_gravity(P, layout, P->phi_loc, P->field_loc);
        if (s != P2P_OK) return s;
    }
    const uint32_t no = (uint32_t)P->n_own, ni = (uint32_t)P->n_in;
    if (no) P2P_LAUNCH((k_pack_results<T, V4>), grid1(no, P->num_sms), 256, 0, st, (const T *)P->phi_loc,
                       (const T *)P->field_loc, no, (V4 *)P->res_own);
    std::vector<int64_t> so(G), sc(G), ro(G), rc(G);
    for (int r = 0; r < G; ++r) {  // the reverse of the repartition
        so[r] = P->rp_roff[r] * (int64_t)sizeof(V4);
        sc[r] = P->rp_rcnt[r] * (int64_t)sizeof(V4);
        ro[r] = P->rp_soff[r] * (int64_t)sizeof(V4);
        rc[r] = P->rp_scnt[r] * (int64_t)sizeof(V4);
    }
    p2p_status s = P->comm->alltoallv(P->res_own, so.data(), sc.data(), P->res_back, ro.data(), rc.data(), st);
    if (s != P2P_OK) return s;
    if (ni) P2P_LAUNCH((k_unpack_results<T, V4>), grid1(ni, P->num_sms), 256, 0, st, (const V4 *)P->res_back,
                       P->perm_send, ni, (T *)phi, (T *)field);
    P2P_CUDA_TRY(cudaGetLastError());
    return P2P_OK;
}
}  // namespace

p2p_status build_distributed(p2p_plan *P, const void *pos, const void *q) {
    return P->cfg.precision == P2P_FP64 ? build_dist_t<double>(P, pos, q) : build_dist_t<float>(P, pos, q);
}

p2p_status eval_distributed(p2p_plan *P, p2p_layout layout, void *phi, void *field) {
    return P->cfg.precision == P2P_FP64 ? eval_dist_t<double>(P, layout, phi, field)
                                        : eval_dist_t<float>(P, layout, phi, field);
}

}  // namespace p2p

extern "C" p2p_status p2p_partition_splitters(const uint64_t *hist, int64_t nbins, int shift, int key_bits,
                                              int nranks, uint32_t *splitters_out) {
    if (!hist || !splitters_out || nbins < 1 || nranks < 1 || shift < 0 || key_bits < 0 || key_bits > 32 ||
        (nbins << shift) > ((int64_t)1 << 32)) {
        p2p::set_error("invalid splitter arguments");
        return P2P_ERR_INVALID_ARGUMENT;
    }
    p2p::compute_splitters((const unsigned long long *)hist, nbins, shift, key_bits, nranks, splitters_out);
    return P2P_OK;
}

namespace p2p {

void free_distributed(p2p_plan *P) {
    void *bufs[] = {P->perm_send, P->phi_loc, P->field_loc, P->res_own, P->res_back};
    for (void *b : bufs) dfree(b, P->stream);
    P->perm_send = nullptr;
    P->phi_loc = P->field_loc = P->res_own = P->res_back = nullptr;
}

}  // namespace p2p
