// comm.hpp -- the collectives the multi-GPU path needs, behind one small interface:
//   allreduce_sum_u64  : the coarse supercell histogram (cost-balanced Morton splitters)
//   allgather_u64      : every rank's route counts (one host read-back per plan build)
//   alltoall_counts    : per-peer element counts before each all-to-all-v (host arrays)
//   alltoallv          : repartition / halo / result return (device buffers, byte counts)
// Two backends: NCCL (one process per GPU, NVLink/NVSwitch; grouped ncclSend/ncclRecv) and an in-process
// loopback group (G emulated ranks = G host threads sharing one device; device-to-device copies + a barrier),
// which lets the whole distributed algorithm run on one GPU and be compared bit for bit with a 1-GPU plan.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <condition_variable>
#include <mutex>
#include <vector>

#include "p2p.h"

namespace p2p {

struct CommBase {
    int nranks = 1, rank = 0;
    virtual ~CommBase() = default;
    // in-place sum over ranks of a device array of u64 (all ranks end with the same values)
    virtual p2p_status allreduce_sum_u64(unsigned long long *dev, size_t count, cudaStream_t st) = 0;
    // recv[r * count + i] = send_i of rank r (device arrays; recv holds nranks * count values)
    virtual p2p_status allgather_u64(const unsigned long long *send, unsigned long long *recv, size_t count,
                                     cudaStream_t st) = 0;
    // send[r] = elements this rank sends to r; recv[r] = elements it receives from r (host arrays, blocking)
    virtual p2p_status alltoall_counts(const int64_t *send, int64_t *recv, cudaStream_t st) = 0;
    // device all-to-all-v of bytes: peer r gets send + soff[r] .. + scnt[r]; we receive rcnt[r] at recv + roff[r]
    virtual p2p_status alltoallv(const void *send, const int64_t *soff, const int64_t *scnt, void *recv,
                                 const int64_t *roff, const int64_t *rcnt, cudaStream_t st) = 0;
    // Peer-memory result return (the a7 + a9 eval fused with the reverse all-to-all-v: the eval epilogue stores every
    // owned target's result straight into its origin rank's receive buffer).  Collective.  begin: this rank's
    // receive buffer holds recv_bytes; my_off[r] = where rank r's results land in it (elements); returns dst[r] =
    // rank r's receive buffer (device address usable here) and dst_off[r] = where MY results land in it
    // (elements), and *recv = my receive buffer.  end: after the eval kernel -- every rank's stores have landed.
    virtual bool has_peer_results() const { return false; }
    virtual p2p_status peer_results_begin(uint64_t, const int64_t *, char **, int64_t *, char **, cudaStream_t) {
        return P2P_ERR_UNSUPPORTED;
    }
    virtual p2p_status peer_results_end(cudaStream_t) { return P2P_ERR_UNSUPPORTED; }
};

// shared state of an in-process loopback group (G emulated ranks, one per host thread)
struct LoopbackGroup {
    int nranks;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long generation = 0;
    std::vector<const void *> send_ptr;
    std::vector<const int64_t *> soff, scnt;
    std::vector<unsigned long long *> red_ptr;
    std::vector<const int64_t *> cnt_ptr;
    explicit LoopbackGroup(int n) : nranks(n), send_ptr(n), soff(n), scnt(n), red_ptr(n), cnt_ptr(n) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const unsigned long long gen = generation;
        if (++arrived == nranks) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

CommBase *make_nccl_comm(int nranks, int rank, const void *id, p2p_status *st);
CommBase *make_loopback_comm(LoopbackGroup *grp, int rank);
CommBase *make_ipc_comm(int nranks, int rank, const char *name, p2p_status *st);

}  // namespace p2p

struct p2p_comm {
    p2p::CommBase *impl = nullptr;
};
