// comm.cu -- communicators owned by libp2p.
//   NCCL: bootstrapped from a 128-byte ncclUniqueId that rank 0 produces and the caller broadcasts (e.g. over a
//         torch.distributed process group); NCCL 2.28 from the wheel PyTorch itself loads (soname libnccl.so.2).
//         all-to-all-v = one ncclGroupStart/End of per-peer ncclSend/ncclRecv (NVLink / NVSwitch).
//   Loopback: G emulated ranks in one process (one host thread each, one shared device) -- the distributed
//         algorithm with device-to-device copies instead of NCCL, used to test bit-identity against 1 GPU.
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "comm.hpp"
#include "plan.hpp"

namespace p2p {

namespace {
#define NCCL_TRY(expr)                                                                  \
    do {                                                                                \
        ncclResult_t r_ = (expr);                                                       \
        if (r_ != ncclSuccess) {                                                        \
            set_error(std::string("NCCL error: ") + ncclGetErrorString(r_) + " (" #expr ")"); \
            return P2P_ERR_NCCL;                                                        \
        }                                                                               \
    } while (0)

struct NcclComm : CommBase {
    ncclComm_t comm = nullptr;
    long long *dcnt = nullptr;  // 2 * nranks int64 scratch for count exchange
    ~NcclComm() override {
        if (dcnt) cudaFree(dcnt);
        if (comm) ncclCommDestroy(comm);
    }
    p2p_status allreduce_sum_u64(unsigned long long *dev, size_t count, cudaStream_t st) override {
        NCCL_TRY(ncclAllReduce(dev, dev, count, ncclUint64, ncclSum, comm, st));
        return P2P_OK;
    }
    p2p_status allgather_u64(const unsigned long long *send, unsigned long long *recv, size_t count,
                             cudaStream_t st) override {
        NCCL_TRY(ncclAllGather(send, recv, count, ncclUint64, comm, st));
        return P2P_OK;
    }
    p2p_status alltoall_counts(const int64_t *send, int64_t *recv, cudaStream_t st) override {
        P2P_CUDA_TRY(cudaMemcpyAsync(dcnt, send, sizeof(long long) * nranks, cudaMemcpyHostToDevice, st));
        NCCL_TRY(ncclGroupStart());
        for (int r = 0; r < nranks; ++r) {
            NCCL_TRY(ncclSend(dcnt + r, 1, ncclInt64, r, comm, st));
            NCCL_TRY(ncclRecv(dcnt + nranks + r, 1, ncclInt64, r, comm, st));
        }
        NCCL_TRY(ncclGroupEnd());
        P2P_CUDA_TRY(cudaMemcpyAsync(recv, dcnt + nranks, sizeof(long long) * nranks, cudaMemcpyDeviceToHost, st));
        P2P_CUDA_TRY(cudaStreamSynchronize(st));
        return P2P_OK;
    }
    p2p_status alltoallv(const void *send, const int64_t *soff, const int64_t *scnt, void *recv, const int64_t *roff,
                         const int64_t *rcnt, cudaStream_t st) override {
        // the rank's own block (in weak scaling nearly all of it: a rank keeps its own tile) is a device-local
        // copy on the stream (HBM-speed copy engine) instead of an NCCL send/recv to self
        if (scnt[rank] != rcnt[rank]) {
            set_error("alltoallv: self send / receive counts differ");
            return P2P_ERR_INVALID_ARGUMENT;
        }
        if (rcnt[rank] > 0)
            P2P_CUDA_TRY(cudaMemcpyAsync((char *)recv + roff[rank], (const char *)send + soff[rank], (size_t)rcnt[rank],
                                         cudaMemcpyDeviceToDevice, st));
        if (nranks == 1) return P2P_OK;
        NCCL_TRY(ncclGroupStart());
        for (int r = 0; r < nranks; ++r) {
            if (r == rank) continue;
            if (scnt[r] > 0) NCCL_TRY(ncclSend((const char *)send + soff[r], (size_t)scnt[r], ncclChar, r, comm, st));
            if (rcnt[r] > 0) NCCL_TRY(ncclRecv((char *)recv + roff[r], (size_t)rcnt[r], ncclChar, r, comm, st));
        }
        NCCL_TRY(ncclGroupEnd());
        return P2P_OK;
    }
};

struct LoopbackComm : CommBase {
    LoopbackGroup *g = nullptr;
    p2p_status allreduce_sum_u64(unsigned long long *dev, size_t count, cudaStream_t st) override {
        std::vector<unsigned long long> mine(count), sum(count, 0ull);
        P2P_CUDA_TRY(cudaMemcpyAsync(mine.data(), dev, count * 8, cudaMemcpyDeviceToHost, st));
        P2P_CUDA_TRY(cudaStreamSynchronize(st));
        g->red_ptr[rank] = mine.data();
        g->barrier();
        for (int r = 0; r < nranks; ++r)  // every rank sums in the same rank order -> identical results
            for (size_t i = 0; i < count; ++i) sum[i] += g->red_ptr[r][i];
        g->barrier();
        P2P_CUDA_TRY(cudaMemcpyAsync(dev, sum.data(), count * 8, cudaMemcpyHostToDevice, st));
        P2P_CUDA_TRY(cudaStreamSynchronize(st));
        return P2P_OK;
    }
    p2p_status allgather_u64(const unsigned long long *send, unsigned long long *recv, size_t count,
                             cudaStream_t st) override {
        std::vector<unsigned long long> mine(count), all(count * nranks);
        P2P_CUDA_TRY(cudaMemcpyAsync(mine.data(), send, count * 8, cudaMemcpyDeviceToHost, st));
        P2P_CUDA_TRY(cudaStreamSynchronize(st));
        g->red_ptr[rank] = mine.data();
        g->barrier();
        for (int r = 0; r < nranks; ++r) std::memcpy(all.data() + r * count, g->red_ptr[r], count * 8);
        g->barrier();
        P2P_CUDA_TRY(cudaMemcpyAsync(recv, all.data(), count * 8 * nranks, cudaMemcpyHostToDevice, st));
        P2P_CUDA_TRY(cudaStreamSynchronize(st));
        return P2P_OK;
    }
    p2p_status alltoall_counts(const int64_t *send, int64_t *recv, cudaStream_t) override {
        g->cnt_ptr[rank] = send;
        g->barrier();
        for (int r = 0; r < nranks; ++r) recv[r] = g->cnt_ptr[r][rank];
        g->barrier();
        return P2P_OK;
    }
    p2p_status alltoallv(const void *send, const int64_t *soff, const int64_t *scnt, void *recv, const int64_t *roff,
                         const int64_t *rcnt, cudaStream_t st) override {
        P2P_CUDA_TRY(cudaStreamSynchronize(st));  // our send buffer is complete
        g->send_ptr[rank] = send;
        g->soff[rank] = soff;
        g->scnt[rank] = scnt;
        g->barrier();
        for (int r = 0; r < nranks; ++r) {
            if (rcnt[r] <= 0) continue;
            if (g->scnt[r][rank] != rcnt[r]) {
                set_error("loopback alltoallv: count mismatch");
                return P2P_ERR_INVALID_ARGUMENT;
            }
            P2P_CUDA_TRY(cudaMemcpyAsync((char *)recv + roff[r], (const char *)g->send_ptr[r] + g->soff[r][rank],
                                         (size_t)rcnt[r], cudaMemcpyDeviceToDevice, st));
        }
        P2P_CUDA_TRY(cudaStreamSynchronize(st));
        g->barrier();  // peers may reuse their send buffers only after every copy out of them finished
        return P2P_OK;
    }
};
}  // namespace

CommBase *make_nccl_comm(int nranks, int rank, const void *id, p2p_status *st) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    NcclComm *c = new NcclComm();
    c->nranks = nranks;
    c->rank = rank;
    ncclResult_t r = ncclCommInitRank(&c->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
        c->comm = nullptr;
        delete c;
        set_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        *st = P2P_ERR_NCCL;
        return nullptr;
    }
    if (cudaMalloc(&c->dcnt, sizeof(long long) * 2 * nranks) != cudaSuccess) {
        delete c;
        set_error("cannot allocate NCCL count scratch");
        *st = P2P_ERR_OUT_OF_MEMORY;
        return nullptr;
    }
    *st = P2P_OK;
    return c;
}

CommBase *make_loopback_comm(LoopbackGroup *grp, int rank) {
    LoopbackComm *c = new LoopbackComm();
    c->g = grp;
    c->nranks = grp->nranks;
    c->rank = rank;
    return c;
}

}  // namespace p2p

using namespace p2p;

struct p2p_loopback_group {
    LoopbackGroup grp;
    explicit p2p_loopback_group(int n) : grp(n) {}
};

extern "C" {

p2p_status p2p_comm_unique_id(void *id_out) {
    if (!id_out) {
        set_error("id_out is NULL");
        return P2P_ERR_INVALID_ARGUMENT;
    }
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) {
        set_error(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
        return P2P_ERR_NCCL;
    }
    std::memcpy(id_out, &id, sizeof id);
    return P2P_OK;
}

p2p_status p2p_comm_create(int nranks, int rank, const void *id, p2p_comm **out) {
    if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks) {
        set_error("invalid communicator arguments");
        return P2P_ERR_INVALID_ARGUMENT;
    }
    *out = nullptr;
    p2p_status st = P2P_OK;
    CommBase *impl = make_nccl_comm(nranks, rank, id, &st);
    if (!impl) return st;
    p2p_comm *c = new p2p_comm();
    c->impl = impl;
    *out = c;
    return P2P_OK;
}

p2p_status p2p_loopback_group_create(int nranks, p2p_loopback_group **out) {
    if (!out || nranks < 1 || nranks > 64) {
        set_error("invalid loopback group arguments (1 <= nranks <= 64)");
        return P2P_ERR_INVALID_ARGUMENT;
    }
    *out = new p2p_loopback_group(nranks);
    return P2P_OK;
}

void p2p_loopback_group_destroy(p2p_loopback_group *g) { delete g; }

p2p_status p2p_comm_create_loopback(p2p_loopback_group *g, int rank, p2p_comm **out) {
    if (!g || !out || rank < 0 || rank >= g->grp.nranks) {
        set_error("invalid loopback communicator arguments");
        return P2P_ERR_INVALID_ARGUMENT;
    }
    p2p_comm *c = new p2p_comm();
    c->impl = make_loopback_comm(&g->grp, rank);
    *out = c;
    return P2P_OK;
}

void p2p_comm_destroy(p2p_comm *c) {
    if (!c) return;
    delete c->impl;
    delete c;
}

}  // extern "C"
