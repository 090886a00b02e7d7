// p2p_api.cu -- the C ABI of libp2p (include/p2p.h): argument validation, plan life cycle, error plumbing.
// Every step of the path runs in this library's kernels (k_*.cu); this file only orchestrates.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "plan.hpp"

namespace p2p {

static thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

void set_error(const std::string &msg) { g_err = msg; }

// P2P_TRACE=1: host-side phase timestamps of p2p_plan_create on stderr (diagnostics only)
static bool trace_on() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("P2P_TRACE");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}
struct Tracer {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void at(const char *what) {
        if (!trace_on()) return;
        auto us = std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0).count();
        fprintf(stderr, "[p2p trace] %-28s %8lld us\n", what, (long long)us);
    }
};

// Library-owned stream-ordered memory pool, one per device (the device's DEFAULT pool is never touched, so
// other cudaMallocAsync users and PyTorch's caching allocator see no change).  Freed blocks stay in the pool while
// a plan is alive on the device (time steps that grow / shrink plan buffers or create and destroy plans stay
// cheap); when the last plan of the device is destroyed the pool is trimmed to zero and its memory returns to the
// driver (p2p.h: p2p_destroy).
static std::mutex g_pool_mu;
static std::map<int, cudaMemPool_t> g_pools;
static std::map<int, int> g_live_plans;

static cudaMemPool_t lib_pool(int dev) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto it = g_pools.find(dev);
    if (it != g_pools.end()) return it->second;
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    g_pools[dev] = pool;
    return pool;
}

void plan_opened(int dev) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    ++g_live_plans[dev];
}

// called after the plan's frees were enqueued; trims the pool once no plan of the device is alive
void plan_closed(int dev, cudaStream_t st) {
    cudaMemPool_t pool = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        if (--g_live_plans[dev] > 0) return;
        auto it = g_pools.find(dev);
        if (it == g_pools.end()) return;
        pool = it->second;
    }
    cudaStreamSynchronize(st);  // the stream-ordered frees must have executed before the trim can return them
    cudaMemPoolTrimTo(pool, 0);
}

cudaError_t dalloc(void **p, size_t bytes, cudaStream_t st) {
    *p = nullptr;
    if (bytes == 0) bytes = 16;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool = lib_pool(dev);
    if (!pool) return cudaMallocAsync(p, bytes, st);
    return cudaMallocFromPoolAsync(p, bytes, pool, st);
}

void dfree(void *p, cudaStream_t st) {
    if (p) cudaFreeAsync(p, st);
}

static bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

static p2p_status fail(p2p_status s, const std::string &msg) {
    set_error(msg);
    return s;
}

// entry guard: sticky state, async errors from earlier work
static p2p_status enter(p2p_plan *P) {
    if (!P) return fail(P2P_ERR_INVALID_ARGUMENT, "plan is NULL");
    if (P->sticky != P2P_OK) return fail(P->sticky, "plan is unusable after an earlier CUDA/NCCL error");
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != P->device) cudaSetDevice(P->device);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        P->sticky = P2P_ERR_CUDA;
        return fail(P2P_ERR_CUDA, std::string("asynchronous CUDA error: ") + cudaGetErrorString(e));
    }
    return P2P_OK;
}

static p2p_status mark(p2p_plan *P, p2p_status s) {
    if (s == P2P_ERR_CUDA || s == P2P_ERR_NCCL) P->sticky = s;
    return s;
}

static void free_plan_buffers(p2p_plan *P) {
    cudaStream_t st = P->stream;
    adaptive_free(P);
    free_capacity(P);
    free_distributed(P);
    free_pairrec(P);
    void *bufs[] = {P->red, P->table, P->tc_table, P->ctr, P->stage_in, P->stage_out};
    for (void *b : bufs) dfree(b, st);
    P->red = P->table = P->tc_table = P->stage_in = P->stage_out = nullptr;
    P->stage_in_cap = P->stage_out_cap = 0;
    P->ctr = nullptr;
}

// host copies of the device-side sizes after an asynchronous p2p_plan_update (synchronises the stream)
static p2p_status resolve_sizes(p2p_plan *P) {
    if (P->sizes_known) return P2P_OK;
    DevCounters h;
    cudaError_t e = cudaMemcpyAsync(&h, P->ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, P->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(P->stream);
    if (e != cudaSuccess) {
        P->sticky = P2P_ERR_CUDA;
        return fail(P2P_ERR_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e));
    }
    if (h.err_index != ~0ull) {
        char buf[200];
        snprintf(buf, sizeof buf,
                 "position of input particle %llu is outside the domain [lo, lo + nbox*h) (C6); the plan holds "
                 "no valid structures until the next successful p2p_plan_update",
                 (unsigned long long)h.err_index);
        return fail(P2P_ERR_OUT_OF_DOMAIN, buf);
    }
    P->B = h.B;
    P->n_nbr = h.n_nbr;
    P->R = (int64_t)h.R;
    P->I = (int64_t)h.I;
    P->n_items = h.n_items;
    P->sizes_known = true;
    return P2P_OK;
}

}  // namespace p2p

using namespace p2p;

extern "C" {

int p2p_abi_version(void) { return P2P_ABI_VERSION; }

uint64_t p2p_kernel_launch_count(void) { return g_launches.load(); }

const char *p2p_last_error(void) { return g_err.c_str(); }

const char *p2p_status_string(p2p_status s) {
    switch (s) {
    case P2P_OK: return "P2P_OK";
    case P2P_ERR_INVALID_ARGUMENT: return "P2P_ERR_INVALID_ARGUMENT";
    case P2P_ERR_OUT_OF_DOMAIN: return "P2P_ERR_OUT_OF_DOMAIN";
    case P2P_ERR_OUT_OF_MEMORY: return "P2P_ERR_OUT_OF_MEMORY";
    case P2P_ERR_CUDA: return "P2P_ERR_CUDA";
    case P2P_ERR_NCCL: return "P2P_ERR_NCCL";
    case P2P_ERR_BAD_STATE: return "P2P_ERR_BAD_STATE";
    case P2P_ERR_UNSUPPORTED: return "P2P_ERR_UNSUPPORTED";
    }
    return "P2P_ERR_UNKNOWN";
}

p2p_status p2p_plan_create(const p2p_config *cfg, int64_t n_local, const void *positions, const void *charges,
                           p2p_plan **out) {
    if (!out) return fail(P2P_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (!cfg) return fail(P2P_ERR_INVALID_ARGUMENT, "cfg is NULL");
    if (n_local < 0) return fail(P2P_ERR_INVALID_ARGUMENT, "n_local < 0");
    if (n_local >= (int64_t)1 << 30)
        return fail(P2P_ERR_UNSUPPORTED, "n_local >= 2^30 (the radix look-back packs digit prefixes into 30 bits)");
    const bool grav = cfg->kernel == P2P_GRAVITY;
    if (!grav && cfg->kernel != P2P_HELMHOLTZ2D) return fail(P2P_ERR_INVALID_ARGUMENT, "unknown kernel");
    if (cfg->precision != P2P_FP32 && cfg->precision != P2P_FP64)
        return fail(P2P_ERR_INVALID_ARGUMENT, "unknown precision");
    if ((grav && cfg->dim != 3) || (!grav && cfg->dim != 2))
        return fail(P2P_ERR_INVALID_ARGUMENT, "dim does not match the kernel (gravity: 3, helmholtz: 2)");
    if (!(cfg->box_size > 0.0) || !std::isfinite(cfg->box_size))
        return fail(P2P_ERR_INVALID_ARGUMENT, "box_size h must be > 0");
    for (int d = 0; d < cfg->dim; ++d) {
        if (cfg->nbox[d] < 1) return fail(P2P_ERR_INVALID_ARGUMENT, "nbox[d] must be >= 1");
        if (((cfg->periodic_mask >> d) & 1u) && cfg->nbox[d] < 3)
            return fail(P2P_ERR_INVALID_ARGUMENT, "a periodic dimension needs nbox >= 3 (27 distinct images, C5)");
        if (!std::isfinite(cfg->lo[d])) return fail(P2P_ERR_INVALID_ARGUMENT, "lo must be finite");
    }
    if (grav && !(cfg->softening > 0.0)) return fail(P2P_ERR_INVALID_ARGUMENT, "softening eps must be > 0 (C2)");
    if (!grav) {
        if (cfg->periodic_mask & 3u) return fail(P2P_ERR_INVALID_ARGUMENT, "helmholtz domain is open (C5)");
        if (!(cfg->wavenumber > 0.0)) return fail(P2P_ERR_INVALID_ARGUMENT, "wavenumber k must be > 0");
        int t = cfg->points_per_box, st = 0;
        while (st * st < t) ++st;
        if (t < 1 || st * st != t) return fail(P2P_ERR_INVALID_ARGUMENT, "points_per_box t must be a perfect square");
    }
    if (cfg->comm && !grav) return fail(P2P_ERR_UNSUPPORTED, "multi-GPU plans are gravity plans (DBIM is 1-GPU)");
    if (cfg->comm && !cfg->comm->impl) return fail(P2P_ERR_INVALID_ARGUMENT, "comm is not initialised");
    if (n_local > 0 && (!is_device_ptr(positions) || !is_device_ptr(charges)))
        return fail(P2P_ERR_INVALID_ARGUMENT, "positions / charges must be device pointers");

    Tracer tr;
    p2p_plan *P = new p2p_plan();
    P->cfg = *cfg;
    P->stream = (cudaStream_t)cfg->stream;
    cudaGetDevice(&P->device);
    cudaDeviceGetAttribute(&P->num_sms, cudaDevAttrMultiProcessorCount, P->device);
    P->n = n_local;
    // geometry
    Geom &g = P->geom;
    g.h = cfg->box_size;
    int32_t mx = 1;
    for (int d = 0; d < 3; ++d) {
        const bool used = d < cfg->dim;
        g.lo[d] = used ? cfg->lo[d] : 0.0;
        g.nbox[d] = used ? cfg->nbox[d] : 1;
        g.L[d] = (double)g.nbox[d] * g.h;  // IEEE product (C5)
        if (g.nbox[d] > mx) mx = g.nbox[d];
    }
    g.periodic = grav ? (cfg->periodic_mask & 7u) : 0u;
    int nb = 0;
    while ((1 << nb) < mx) ++nb;
    g.nb = nb;
    g.eps2 = cfg->softening * cfg->softening;
    P->nb = nb;
    if (grav) {
        if (nb > 10) {
            delete P;
            return fail(P2P_ERR_UNSUPPORTED, "more than 1024 boxes per dim (u32 Morton keys, C7)");
        }
        P->key_bits = 3 * nb;
    } else {
        if (nb > 16) {
            delete P;
            return fail(P2P_ERR_UNSUPPORTED, "more than 65536 boxes per dim");
        }
        uint64_t kmax = ((uint64_t)1 << (2 * nb)) * (uint64_t)cfg->points_per_box;
        int kb = 0;
        while (((uint64_t)1 << kb) < kmax) ++kb;
        if (kb > 32) {
            delete P;
            return fail(P2P_ERR_UNSUPPORTED, "helmholtz key (box * t + subcell) exceeds 32 bits");
        }
        P->key_bits = kb;
    }
    P->passes = (P->key_bits + 7) / 8;

    cudaStream_t st = P->stream;
    plan_opened(P->device);
    auto bail = [&](p2p_status s) {
        free_plan_buffers(P);
        cudaStreamSynchronize(st);
        plan_closed(P->device, st);
        delete P;
        return s;
    };
    if (dalloc((void **)&P->ctr, sizeof(DevCounters), st) != cudaSuccess)
        return bail(fail(P2P_ERR_OUT_OF_MEMORY, "cannot allocate counters"));
    cudaMemsetAsync(P->ctr, 0, sizeof(DevCounters), st);
    cudaMemsetAsync(&P->ctr->err_index, 0xff, sizeof(unsigned long long), st);
    g.tkey_lo = 0u;  // single GPU: every box is a target box
    g.tkey_hi = 0xffffffffu;
    p2p_status s = P2P_OK;
    if (cfg->comm) {
        // multi-GPU: collective build (repartition + halo), then the local plan over [owned ; halo] (k_dist.cu)
        P->comm = cfg->comm->impl;
        P->n_in = n_local;
        s = build_distributed(P, positions, charges);
        if (s != P2P_OK) return bail(s);
        if (P->n == 0) {
            cudaStreamSynchronize(st);
            P->sizes_known = true;
            *out = P;
            return P2P_OK;
        }
    } else {
        P->n_in = n_local;
        if (n_local == 0) {
            cudaStreamSynchronize(st);
            P->sizes_known = true;
            *out = P;
            return P2P_OK;
        }
        tr.at("validated+counters");
        if (alloc_capacity(P, n_local) != P2P_OK)
            return bail(fail(P2P_ERR_OUT_OF_MEMORY, "cannot allocate plan buffers"));
        s = grav ? build_gravity_structs(P, positions, charges) : build_helmholtz_structs(P, positions, charges);
        if (s != P2P_OK) return bail(s);
    }
    tr.at("structs enqueued");
    // the ONE host synchronisation: sizes for the redundant buffer and launch geometry
    DevCounters h;
    cudaError_t e = cudaMemcpyAsync(&h, P->ctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return bail(fail(P2P_ERR_CUDA, std::string("CUDA error in plan build: ") + cudaGetErrorString(e)));
    tr.at("synchronised");
    if (h.err_index != ~0ull) {
        char buf[160];
        snprintf(buf, sizeof buf, "position of input particle %llu is outside the domain [lo, lo + nbox*h) (C6)",
                 (unsigned long long)h.err_index);
        return bail(fail(P2P_ERR_OUT_OF_DOMAIN, buf));
    }
    if (h.irregular) return bail(fail(P2P_ERR_UNSUPPORTED, "helmholtz input is not a regular t-per-box lattice (C8)"));
    P->B = h.B;
    P->I = (int64_t)h.I;
    if (grav) {
        P->n_nbr = h.n_nbr;
        P->R = (int64_t)h.R;
        P->n_items = h.n_items;
        const size_t rec_sz = cfg->precision == P2P_FP64 ? sizeof(double4) : sizeof(float4);
        if (dalloc(&P->red, rec_sz * (size_t)std::max<int64_t>(P->R, 1), st) != cudaSuccess)
            return bail(fail(P2P_ERR_OUT_OF_MEMORY, "cannot allocate the redundant buffer"));
        P->red_cap = std::max<int64_t>(P->R, 1);
    } else {
        const int64_t t = cfg->points_per_box;
        P->n_nbr = 9 * P->B;
        P->R = 9 * t * P->B;
        P->n_items = P->B;
        const size_t c_sz = cfg->precision == P2P_FP64 ? sizeof(double2) : sizeof(float2);
        if (dalloc(&P->red, c_sz * (size_t)std::max<int64_t>(P->R, 1), st) != cudaSuccess)
            return bail(fail(P2P_ERR_OUT_OF_MEMORY, "cannot allocate the im2col buffer"));
        s = helmholtz_table(P);
        if (s != P2P_OK) return bail(s);
    }
    tr.at("red allocated");
    P->sizes_known = true;
    *out = P;
    return P2P_OK;
}

p2p_status p2p_plan_update(p2p_plan *P, int64_t n_local, const void *positions, const void *charges) {
    p2p_status s = enter(P);
    if (s != P2P_OK) return s;
    if (P->cfg.kernel != P2P_GRAVITY)
        return fail(P2P_ERR_UNSUPPORTED, "p2p_plan_update is for gravity plans (DBIM geometry is fixed: use set_charges)");
    if (n_local < 0) return fail(P2P_ERR_INVALID_ARGUMENT, "n_local < 0");
    if (n_local >= (int64_t)1 << 30)
        return fail(P2P_ERR_UNSUPPORTED, "n_local >= 2^30 (the radix look-back packs digit prefixes into 30 bits)");
    if (n_local > 0 && (!is_device_ptr(positions) || !is_device_ptr(charges)))
        return fail(P2P_ERR_INVALID_ARGUMENT, "positions / charges must be device pointers");
    cudaStream_t st = P->stream;
    if (P->comm) {
        // collective rebuild (every rank calls): the exchange sizes need the host (NCCL counts), the local
        // structures reuse the plan's capacity buffers and stay device-side like the single-GPU update
        P->n_in = n_local;
        P->sizes_known = false;
        P->red_valid = false;
        P->pr_valid = false;
        cudaMemsetAsync(P->ctr, 0, sizeof(DevCounters), st);
        cudaMemsetAsync(&P->ctr->err_index, 0xff, sizeof(unsigned long long), st);
        p2p_status bs = build_distributed(P, positions, charges);
        if (bs != P2P_OK) return mark(P, bs);
        const int64_t need = std::max<int64_t>(27 * P->n, 1);
        if (P->red_cap < need) {
            dfree(P->red, st);
            const size_t rec_sz = P->cfg.precision == P2P_FP64 ? sizeof(double4) : sizeof(float4);
            if (dalloc(&P->red, rec_sz * (size_t)need, st) != cudaSuccess) {
                P->red = nullptr;
                P->red_cap = 0;
                P->sticky = P2P_ERR_OUT_OF_MEMORY;
                return fail(P2P_ERR_OUT_OF_MEMORY, "cannot allocate the redundant buffer");
            }
            P->red_cap = need;
        }
        if (P->n == 0) {
            P->sizes_known = true;
            P->B = P->n_nbr = P->R = P->I = P->n_items = 0;
        }
        return P2P_OK;
    }
    if (n_local > P->cap) {  // grow (stream-ordered; steady-state time steps never get here)
        free_capacity(P);
        if (alloc_capacity(P, n_local) != P2P_OK) {
            P->sticky = P2P_ERR_OUT_OF_MEMORY;
            return fail(P2P_ERR_OUT_OF_MEMORY, "cannot grow plan buffers");
        }
    }
    // worst case R <= 27 N (each record is one of <= 27 images of a particle) -> no host sync needed
    const int64_t red_need = std::max<int64_t>(27 * n_local, 1);
    if (P->red_cap < red_need) {
        dfree(P->red, st);
        const size_t rec_sz = P->cfg.precision == P2P_FP64 ? sizeof(double4) : sizeof(float4);
        if (dalloc(&P->red, rec_sz * (size_t)red_need, st) != cudaSuccess) {
            P->red = nullptr;
            P->red_cap = 0;
            P->sticky = P2P_ERR_OUT_OF_MEMORY;
            return fail(P2P_ERR_OUT_OF_MEMORY, "cannot allocate the redundant buffer");
        }
        P->red_cap = red_need;
    }
    P->n = n_local;
    P->sizes_known = false;
    P->red_valid = false;
    P->pr_valid = false;
    cudaMemsetAsync(P->ctr, 0, sizeof(DevCounters), st);
    cudaMemsetAsync(&P->ctr->err_index, 0xff, sizeof(unsigned long long), st);
    if (P->ad) P->ad->runs_valid = false;
    if (n_local == 0) {
        P->sizes_known = true;
        P->B = P->n_nbr = P->R = P->I = P->n_items = 0;
        if (P->ad) return mark(P, adaptive_build_async(P));
        P->grid_stale = false;
        return P2P_OK;
    }
    if (P->ad) {  // adaptive-leaf mode: a1-a4 as always, then the leaves + closed CSR (no grid a5), asynchronous
        s = build_gravity_structs(P, positions, charges, nullptr, false);
        if (s != P2P_OK) return mark(P, s);
        if (P->bcap > P->ad->bcap) {  // the box capacity grew (rare): re-measure and re-allocate (synchronous)
            s = resolve_sizes(P);
            if (s != P2P_OK) return s;
            return mark(P, adaptive_enable(P, P->ad->t, P->ad->min_bits));
        }
        return mark(P, adaptive_build_async(P));
    }
    P->grid_stale = false;
    return mark(P, build_gravity_structs(P, positions, charges));
}

// ---- host-buffer entry points: the library stages the copies on the plan's stream ----
static bool grow_stage(p2p_plan *P, void **buf, int64_t *cap, int64_t need_bytes) {
    if (*cap >= need_bytes) return true;
    dfree(*buf, P->stream);
    *buf = nullptr;
    *cap = 0;
    if (dalloc(buf, (size_t)need_bytes, P->stream) != cudaSuccess) {
        *buf = nullptr;
        return false;
    }
    *cap = need_bytes;
    return true;
}

p2p_status p2p_plan_update_host(p2p_plan *P, int64_t n_local, const void *positions_host, const void *charges_host) {
    p2p_status s = enter(P);
    if (s != P2P_OK) return s;
    if (P->cfg.kernel != P2P_GRAVITY || P->comm)
        return fail(P2P_ERR_UNSUPPORTED, "p2p_plan_update_host: single-GPU gravity plans only");
    if (n_local < 0) return fail(P2P_ERR_INVALID_ARGUMENT, "n_local < 0");
    if (n_local > 0 && (!positions_host || !charges_host)) return fail(P2P_ERR_INVALID_ARGUMENT, "NULL argument");
    if (n_local > 0 && (is_device_ptr(positions_host) || is_device_ptr(charges_host)))
        return fail(P2P_ERR_INVALID_ARGUMENT, "positions / charges must be host pointers (use p2p_plan_update)");
    const size_t tsz = P->cfg.precision == P2P_FP64 ? sizeof(double) : sizeof(float);
    const size_t pb = 3 * tsz * (size_t)n_local, qb = tsz * (size_t)n_local;
    if (!grow_stage(P, &P->stage_in, &P->stage_in_cap, (int64_t)std::max<size_t>(pb + qb, 1)))
        return fail(P2P_ERR_OUT_OF_MEMORY, "cannot allocate the input staging buffer");
    char *d = (char *)P->stage_in;
    if (n_local > 0) {
        cudaError_t e = cudaMemcpyAsync(d, positions_host, pb, cudaMemcpyHostToDevice, P->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(d + pb, charges_host, qb, cudaMemcpyHostToDevice, P->stream);
        if (e != cudaSuccess) return fail(P2P_ERR_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e));
    }
    return p2p_plan_update(P, n_local, d, d + pb);
}

p2p_status p2p_eval_host(p2p_plan *P, p2p_layout layout, void *potential_host, void *field_host) {
    p2p_status s = enter(P);
    if (s != P2P_OK) return s;
    if (P->cfg.kernel != P2P_GRAVITY || P->comm)
        return fail(P2P_ERR_UNSUPPORTED, "p2p_eval_host: single-GPU gravity plans only");
    if (P->n > 0 && !potential_host) return fail(P2P_ERR_INVALID_ARGUMENT, "NULL potential");
    if ((potential_host && is_device_ptr(potential_host)) || (field_host && is_device_ptr(field_host)))
        return fail(P2P_ERR_INVALID_ARGUMENT, "potential / field must be host pointers (use p2p_eval)");
    const size_t tsz = P->cfg.precision == P2P_FP64 ? sizeof(double) : sizeof(float);
    const size_t ob = tsz * (size_t)P->n, fb = field_host ? 3 * tsz * (size_t)P->n : 0;
    if (!grow_stage(P, &P->stage_out, &P->stage_out_cap, (int64_t)std::max<size_t>(ob + fb, 1)))
        return fail(P2P_ERR_OUT_OF_MEMORY, "cannot allocate the output staging buffer");
    char *d = (char *)P->stage_out;
    s = p2p_eval(P, layout, d, field_host ? d + ob : nullptr);
    if (s != P2P_OK) return s;
    cudaError_t e = cudaSuccess;
    if (ob) e = cudaMemcpyAsync(potential_host, d, ob, cudaMemcpyDeviceToHost, P->stream);
    if (e == cudaSuccess && fb) e = cudaMemcpyAsync(field_host, d + ob, fb, cudaMemcpyDeviceToHost, P->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(P->stream);
    if (e != cudaSuccess) return fail(P2P_ERR_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e));
    return P2P_OK;
}

p2p_status p2p_restructure(p2p_plan *P) {
    p2p_status s = enter(P);
    if (s != P2P_OK) return s;
    if (P->n == 0) {
        P->red_valid = true;
        return P2P_OK;
    }
    if (P->ad) return mark(P, adaptive_restructure_async(P));  // adaptive mode: the leaves' runs + items
    if (P->grid_stale) return fail(P2P_ERR_BAD_STATE, "after p2p_adaptive_disable: call p2p_plan_update first");
    s = P->cfg.kernel == P2P_GRAVITY ? restructure_gravity(P) : restructure_helmholtz(P);
    if (s == P2P_OK) P->red_valid = true;
    return mark(P, s);
}

p2p_status p2p_restructure_pairs(p2p_plan *P) {
    p2p_status s = enter(P);
    if (s != P2P_OK) return s;
    if (P->cfg.kernel != P2P_GRAVITY || P->comm)
        return fail(P2P_ERR_UNSUPPORTED, "pair records are for single-GPU gravity plans");
    s = resolve_sizes(P);
    if (s != P2P_OK) return s;
    return mark(P, restructure_pairs(P));
}

p2p_status p2p_adaptive_leaves(p2p_plan *P, int32_t t, int32_t min_bits, uint32_t *len_out, uint32_t *prefix_out,
                               uint32_t *start_out, int64_t capacity, int64_t *n_leaves) {
    p2p_status s = enter(P);
    if (s != P2P_OK) return s;
    if (!len_out || !prefix_out || !start_out || !n_leaves || t < 1 || min_bits < 0 || capacity < 0)
        return fail(P2P_ERR_INVALID_ARGUMENT, "adaptive leaves: NULL output, t < 1, min_bits < 0 or capacity < 0");
    if (P->cfg.kernel != P2P_GRAVITY || P->comm)
        return fail(P2P_ERR_UNSUPPORTED, "adaptive leaves are for single-GPU gravity plans");
    const int32_t n0 = P->cfg.nbox[0];
    if (P->cfg.nbox[1] != n0 || P->cfg.nbox[2] != n0 || (n0 & (n0 - 1)) != 0 || P->cfg.periodic_mask != 7u)
        return fail(P2P_ERR_UNSUPPORTED, "adaptive leaves need a periodic cube of 2^m boxes per dimension (C22)");
    s = resolve_sizes(P);
    if (s != P2P_OK) return s;
    return mark(P, adaptive_leaves(P, (uint32_t)t, min_bits, len_out, prefix_out, start_out, capacity, n_leaves));
}

p2p_status p2p_adaptive_neighbours(p2p_plan *P, int32_t t, int32_t min_bits, uint32_t *off_out, uint32_t *nbr_out,
                                   uint8_t *code_out, int64_t cap_leaves, int64_t cap_entries, int64_t *n_leaves,
                                   int64_t *n_entries) {
    p2p_status s = enter(P);
    if (s != P2P_OK) return s;
    if (!off_out || !nbr_out || !code_out || !n_leaves || !n_entries || t < 1 || min_bits < 9 || cap_leaves < 0 ||
        cap_entries < 0)
        return fail(P2P_ERR_INVALID_ARGUMENT,
                    "adaptive neighbours: NULL output, t < 1, min_bits < 9 (unique images, C22) or capacity < 0");
    if (P->cfg.kernel != P2P_GRAVITY || P->comm)
        return fail(P2P_ERR_UNSUPPORTED, "adaptive leaves are for single-GPU gravity plans");
    const int32_t n0 = P->cfg.nbox[0];
    if (P->cfg.nbox[1] != n0 || P->cfg.nbox[2] != n0 || (n0 & (n0 - 1)) != 0 || n0 < 8 || P->cfg.periodic_mask != 7u)
        return fail(P2P_ERR_UNSUPPORTED, "adaptive leaves need a periodic cube of 2^m >= 8 boxes per dimension (C22)");
    s = resolve_sizes(P);
    if (s != P2P_OK) return s;
    return mark(P, adaptive_neighbours(P, (uint32_t)t, min_bits, off_out, nbr_out, code_out, cap_leaves, cap_entries,
                                       n_leaves, n_entries));
}

p2p_status p2p_adaptive_eval(p2p_plan *P, int32_t t, int32_t min_bits, p2p_layout layout, void *potential, void *field,
                             void *red_out, int64_t cap_records, int64_t *n_records) {
    p2p_status s = enter(P);
    if (s != P2P_OK) return s;
    if (!n_records || t < 1 || min_bits < 9 || cap_records < 0)
        return fail(P2P_ERR_INVALID_ARGUMENT, "adaptive eval: NULL n_records, t < 1, min_bits < 9 or capacity < 0");
    if (layout != P2P_REDUNDANT && layout != P2P_INDEXED)
        return fail(P2P_ERR_INVALID_ARGUMENT, "adaptive eval: layout must be P2P_REDUNDANT or P2P_INDEXED");
    if (P->cfg.kernel != P2P_GRAVITY || P->comm)
        return fail(P2P_ERR_UNSUPPORTED, "adaptive leaves are for single-GPU gravity plans");
    const int32_t n0 = P->cfg.nbox[0];
    if (P->cfg.nbox[1] != n0 || P->cfg.nbox[2] != n0 || (n0 & (n0 - 1)) != 0 || n0 < 8 || P->cfg.periodic_mask != 7u)
        return fail(P2P_ERR_UNSUPPORTED, "adaptive leaves need a periodic cube of 2^m >= 8 boxes per dimension (C22)");
    if (potential && !is_device_ptr(potential)) return fail(P2P_ERR_INVALID_ARGUMENT, "potential must be a device pointer");
    if (field && !is_device_ptr(field)) return fail(P2P_ERR_INVALID_ARGUMENT, "field must be a device pointer");
    if (field && !potential) return fail(P2P_ERR_INVALID_ARGUMENT, "field needs the potential buffer too");
    s = resolve_sizes(P);
    if (s != P2P_OK) return s;
    return mark(P, adaptive_eval(P, (uint32_t)t, min_bits, layout == P2P_INDEXED, potential, field, red_out, cap_records,
                                 n_records));
}

p2p_status p2p_get_pairrec_size(const p2p_plan *P, int64_t *records, int64_t *partials) {
    if (!P || !records || !partials) return fail(P2P_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!P->pr_valid) return fail(P2P_ERR_BAD_STATE, "pair records are not built (call p2p_restructure_pairs)");
    *records = P->pr_records;
    *partials = P->pr_targets;
    return P2P_OK;
}

p2p_status p2p_eval(p2p_plan *P, p2p_layout layout, void *potential, void *field) {
    p2p_status s = enter(P);
    if (s != P2P_OK) return s;
    if (layout != P2P_REDUNDANT && layout != P2P_INDEXED && layout != P2P_INDEXED_BITWISE && layout != P2P_PAIRREC)
        return fail(P2P_ERR_INVALID_ARGUMENT, "unknown layout");
    if (layout == P2P_PAIRREC) {
        if (P->cfg.kernel != P2P_GRAVITY || P->comm)
            return fail(P2P_ERR_UNSUPPORTED, "P2P_PAIRREC is for single-GPU gravity plans");
        if (!P->pr_valid)
            return fail(P2P_ERR_BAD_STATE, "eval(P2P_PAIRREC) needs p2p_restructure_pairs first (and after update)");
        if (P->n == 0) return P2P_OK;
        if (!is_device_ptr(potential)) return fail(P2P_ERR_INVALID_ARGUMENT, "potential must be a device pointer");
        if (field && !is_device_ptr(field)) return fail(P2P_ERR_INVALID_ARGUMENT, "field must be a device pointer");
        return mark(P, eval_pairrec(P, potential, field));
    }
    if (P->ad) {  // adaptive-leaf mode
        if (layout != P2P_REDUNDANT && layout != P2P_INDEXED)
            return fail(P2P_ERR_UNSUPPORTED, "adaptive mode evaluates P2P_REDUNDANT or P2P_INDEXED");
        if (layout == P2P_REDUNDANT && !P->ad->runs_valid)
            return fail(P2P_ERR_BAD_STATE,
                        "eval(P2P_REDUNDANT) needs p2p_restructure first in adaptive mode (and after update)");
        if (P->n == 0) return P2P_OK;
        if (!is_device_ptr(potential)) return fail(P2P_ERR_INVALID_ARGUMENT, "potential must be a device pointer");
        if (field && !is_device_ptr(field)) return fail(P2P_ERR_INVALID_ARGUMENT, "field must be a device pointer");
        return mark(P, adaptive_eval_async(P, layout, potential, field));
    }
    if (P->grid_stale) return fail(P2P_ERR_BAD_STATE, "after p2p_adaptive_disable: call p2p_plan_update first");
    if (layout == P2P_REDUNDANT && !P->red_valid)
        return fail(P2P_ERR_BAD_STATE, "eval(P2P_REDUNDANT) needs p2p_restructure first (and after set_charges)");
    if (P->comm) {  // collective: every rank calls, even with no particles
        if (P->n_in > 0 && !is_device_ptr(potential))
            return fail(P2P_ERR_INVALID_ARGUMENT, "potential must be a device pointer");
        if (field && !is_device_ptr(field)) return fail(P2P_ERR_INVALID_ARGUMENT, "field must be a device pointer");
        return mark(P, eval_distributed(P, layout, potential, field));
    }
    if (P->n == 0) return P2P_OK;
    if (!is_device_ptr(potential)) return fail(P2P_ERR_INVALID_ARGUMENT, "potential must be a device pointer");
    if (P->cfg.kernel == P2P_GRAVITY) {
        if (field && !is_device_ptr(field)) return fail(P2P_ERR_INVALID_ARGUMENT, "field must be a device pointer");
        return mark(P, eval_gravity(P, layout, potential, field));
    }
    if (field) return fail(P2P_ERR_INVALID_ARGUMENT, "helmholtz has no field output (pass NULL)");
    return mark(P, eval_helmholtz(P, layout, potential));
}

p2p_status p2p_set_charges(p2p_plan *P, const void *charges) {
    p2p_status s = enter(P);
    if (s != P2P_OK) return s;
    if (P->comm) return fail(P2P_ERR_UNSUPPORTED, "multi-GPU plans: charges move with the repartition (re-create)");
    if (P->n == 0) return P2P_OK;
    if (!is_device_ptr(charges)) return fail(P2P_ERR_INVALID_ARGUMENT, "charges must be a device pointer");
    P->red_valid = false;
    P->pr_valid = false;
    if (P->ad) P->ad->runs_valid = false;
    s = P->cfg.kernel == P2P_GRAVITY ? set_charges_gravity(P, charges) : set_charges_helmholtz(P, charges);
    return mark(P, s);
}

void p2p_destroy(p2p_plan *P) {
    if (!P) return;
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != P->device) cudaSetDevice(P->device);
    free_plan_buffers(P);
    plan_closed(P->device, P->stream);
    delete P;
}

p2p_status p2p_get_info(const p2p_plan *Pc, p2p_info *out) {
    if (!Pc || !out) return fail(P2P_ERR_INVALID_ARGUMENT, "NULL argument");
    p2p_plan *P = const_cast<p2p_plan *>(Pc);  // resolves the lazily synchronised host copies of the sizes
    if (P->sticky != P2P_OK) return fail(P->sticky, "plan is unusable after an earlier error");
    p2p_status rs = resolve_sizes(P);
    if (rs != P2P_OK) return rs;
    cudaError_t e = cudaStreamSynchronize(P->stream);
    if (e != cudaSuccess) return fail(P2P_ERR_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e));
    out->n_local = P->n;
    out->n_boxes = P->B;
    out->n_nbr = P->n_nbr;
    out->n_red = P->R;
    out->n_pairs = P->I;
    out->n_items = P->n_items;
    out->key_bits = P->key_bits;
    out->sort_passes = P->passes;
    if (P->ad) {  // adaptive mode: the leaves' counts
        AdaptCtr h;
        rs = adaptive_info(P, &h);
        if (rs != P2P_OK) return rs;
        if (h.overflow)
            return fail(P2P_ERR_OUT_OF_MEMORY, "adaptive capacities exceeded by the last update (entries / records / "
                                               "items above 2x the measured input): call p2p_adaptive_enable again");
        out->n_boxes = h.L;
        out->n_nbr = h.E;
        out->n_red = (int64_t)h.R;
        out->n_pairs = (int64_t)h.I;
        out->n_items = h.n_items;
    }
    return P2P_OK;
}

p2p_status p2p_adaptive_enable(p2p_plan *P, int32_t t, int32_t min_bits) {
    p2p_status s = enter(P);
    if (s != P2P_OK) return s;
    if (t < 1 || min_bits < 9) return fail(P2P_ERR_INVALID_ARGUMENT, "adaptive mode: t < 1 or min_bits < 9 (C22)");
    if (P->cfg.kernel != P2P_GRAVITY || P->comm)
        return fail(P2P_ERR_UNSUPPORTED, "adaptive mode is for single-GPU gravity plans");
    const int32_t n0 = P->cfg.nbox[0];
    if (P->cfg.nbox[1] != n0 || P->cfg.nbox[2] != n0 || (n0 & (n0 - 1)) != 0 || n0 < 8 || P->cfg.periodic_mask != 7u)
        return fail(P2P_ERR_UNSUPPORTED, "adaptive mode needs a periodic cube of 2^m >= 8 boxes per dimension (C22)");
    s = resolve_sizes(P);
    if (s != P2P_OK) return s;
    return mark(P, adaptive_enable(P, (uint32_t)t, min_bits));
}

p2p_status p2p_adaptive_disable(p2p_plan *P) {
    p2p_status s = enter(P);
    if (s != P2P_OK) return s;
    if (!P->ad) return P2P_OK;
    adaptive_free(P);
    // the grid a5 structures (neighbour CSR, items) are not built in adaptive mode: the next grid restructure / eval
    // needs a p2p_plan_update first
    P->grid_stale = true;
    P->red_valid = false;
    return P2P_OK;
}

p2p_status p2p_get_splitters(const p2p_plan *P, uint32_t *out, int n) {
    if (!P || !out) return fail(P2P_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!P->comm) return fail(P2P_ERR_INVALID_ARGUMENT, "not a multi-GPU plan");
    if (n != (int)P->splitters.size()) return fail(P2P_ERR_INVALID_ARGUMENT, "n != nranks + 1");
    std::copy(P->splitters.begin(), P->splitters.end(), out);
    return P2P_OK;
}

p2p_status p2p_copy_out(const p2p_plan *Pc, p2p_array which, void *host_dst, size_t bytes) {
    if (!Pc || (!host_dst && bytes)) return fail(P2P_ERR_INVALID_ARGUMENT, "NULL argument");
    p2p_plan *P = const_cast<p2p_plan *>(Pc);
    if (P->sticky != P2P_OK) return fail(P->sticky, "plan is unusable after an earlier error");
    p2p_status rs = resolve_sizes(P);
    if (rs != P2P_OK) return rs;
    const bool grav = P->cfg.kernel == P2P_GRAVITY;
    const bool f64 = P->cfg.precision == P2P_FP64;
    const void *src = nullptr;
    size_t need = 0;
    switch (which) {
    case P2P_ARR_PERM: src = P->perm; need = 4 * (size_t)P->n; break;
    case P2P_ARR_SORTED_KEYS: src = P->skey; need = 4 * (size_t)P->n; break;
    case P2P_ARR_BOX_KEYS: src = P->bkey; need = 4 * (size_t)P->B; break;
    case P2P_ARR_BOX_START: src = P->bstart; need = 4 * (size_t)(P->B + 1); break;
    case P2P_ARR_NBR_OFF: src = P->nbr_off; need = 4 * (size_t)(P->B + 1); break;
    case P2P_ARR_NBR_BOX: src = P->nbr_box; need = 4 * (size_t)P->n_nbr; break;
    case P2P_ARR_NBR_SLOT: src = P->nbr_slot; need = (size_t)P->n_nbr; break;
    case P2P_ARR_RED_OFF:
        if (!grav) return fail(P2P_ERR_UNSUPPORTED, "helmholtz runs have fixed stride 9t (no red_off array)");
        src = P->red_off; need = 8 * (size_t)(P->B + 1); break;
    case P2P_ARR_RED:
        if (!P->red_valid) return fail(P2P_ERR_BAD_STATE, "the redundant buffer is not built (call p2p_restructure)");
        src = P->red;
        need = (size_t)P->R * (grav ? (f64 ? 32 : 16) : (f64 ? 16 : 8));
        break;
    case P2P_ARR_PAIRREC:
        if (!P->pr_valid) return fail(P2P_ERR_BAD_STATE, "pair records are not built (call p2p_restructure_pairs)");
        src = P->pr;
        need = (size_t)P->pr_records * (f64 ? 32 : 16);
        break;
    default: return fail(P2P_ERR_INVALID_ARGUMENT, "unknown array");
    }
    if (P->n == 0) need = 0;
    if (bytes != need) {
        char buf[128];
        snprintf(buf, sizeof buf, "bytes = %zu but the array holds %zu bytes", bytes, need);
        return fail(P2P_ERR_INVALID_ARGUMENT, buf);
    }
    if (need == 0) return P2P_OK;
    cudaError_t e = cudaStreamSynchronize(P->stream);
    if (e == cudaSuccess) e = cudaMemcpy(host_dst, src, need, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return fail(P2P_ERR_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e));
    return P2P_OK;
}

}  // extern "C"
