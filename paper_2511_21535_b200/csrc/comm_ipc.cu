// comm_ipc.cu -- a multi-PROCESS communicator over CUDA IPC peer memory (SURVEY §8e "B200-native option":
// peer-mapped device memory instead of NCCL send/recv).  One process per rank, all on one node: several GPUs
// (peer copies over NVLink / NVSwitch) or several processes sharing ONE GPU (which NCCL refuses: one rank per
// device) -- the latter is how the multi-process data path runs on the single B200 the tests can reach.
//
// Rendezvous: a POSIX shared-memory segment named by the caller (a unique token rank 0 draws and the caller
// broadcasts, e.g. over a torch.distributed gloo group) holds a process-shared barrier, every rank's
// cudaIpcMemHandle_t for its device ARENA (cudaMalloc'd, so IPC-exportable; plan buffers come from a
// stream-ordered pool and are not), the all-to-all counts and the published send offsets.
//
// Collectives (same semantics as the NCCL / loopback backends, comm.hpp):
//   alltoallv       : the sender stages its whole send buffer into its own arena (one device copy at HBM speed),
//                     host barrier, every receiver pulls its blocks straight out of the peers' arenas (peer
//                     device pointers from cudaIpcOpenMemHandle: UVA copies, NVLink between GPUs), barrier
//                     (the arenas may be rewritten only after every pull finished).  Arenas grow on demand; a
//                     rank that grows re-publishes its handle and the peers re-open it after the next barrier.
//   allreduce / allgather of u64: the same staging, then a local copy of every rank's array and (reduce) one
//                     kernel summing them in rank order -- identical bits on every rank.
//   alltoall_counts : host arrays through the segment.
// Host synchronisation points are the same as the NCCL path's (the plan build's single read-back) plus one
// stream sync per collective; this backend trades NCCL's in-stream progress for running anywhere CUDA IPC does.
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "comm.hpp"
#include "plan.hpp"

namespace p2p {

namespace {
constexpr int IPC_MAX_RANKS = 64;
constexpr uint64_t IPC_MAGIC = 0x5032504950433031ull;  // "P2PIPC01"

struct IpcShared {
    std::atomic<uint64_t> magic;       // rank 0 sets it once the segment is initialised
    std::atomic<uint32_t> attached;    // ranks attached (rank 0 unlinks the name when all have)
    std::atomic<uint32_t> bar_count;   // barrier arrivals of the current generation
    std::atomic<uint64_t> bar_gen;     // barrier generation
    int32_t nranks;
    cudaIpcMemHandle_t handle[IPC_MAX_RANKS];   // each rank's arena
    uint64_t arena_bytes[IPC_MAX_RANKS];
    uint64_t arena_gen[IPC_MAX_RANKS];          // bumped when a rank re-allocates its arena
    int64_t counts[IPC_MAX_RANKS][IPC_MAX_RANKS];  // counts[src][dst] (alltoall_counts)
    int64_t soff[IPC_MAX_RANKS][IPC_MAX_RANKS];    // soff[src][dst]: byte offset of src's block for dst (alltoallv)
    int32_t dev[IPC_MAX_RANKS];                    // CUDA device ordinal of every rank (diagnostics)
    int64_t res_off[IPC_MAX_RANKS][IPC_MAX_RANKS]; // res_off[dst][src]: where src's results land in dst's buffer
};

__global__ void k_sum_ranks(const unsigned long long *__restrict__ all, int nranks, size_t count,
                            unsigned long long *__restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        unsigned long long s = 0;
        for (int r = 0; r < nranks; ++r) s += all[(size_t)r * count + i];  // fixed rank order
        out[i] = s;
    }
}

struct IpcComm : CommBase {
    std::string name;
    IpcShared *sh = nullptr;
    char *arena = nullptr;               // own arena (device)
    uint64_t arena_bytes = 0;
    std::vector<char *> peer;            // peer arenas (own arena for r == rank)
    std::vector<uint64_t> peer_gen;
    unsigned long long *scratch = nullptr;  // nranks * count u64 for reduce / gather
    size_t scratch_count = 0;

    ~IpcComm() override {
        for (int r = 0; r < nranks; ++r)
            if (r != rank && peer[r]) cudaIpcCloseMemHandle(peer[r]);
        if (arena) cudaFree(arena);
        if (scratch) cudaFree(scratch);
        if (sh) munmap(sh, sizeof(IpcShared));
    }

    void barrier() {
        const uint64_t gen = sh->bar_gen.load(std::memory_order_acquire);
        if (sh->bar_count.fetch_add(1, std::memory_order_acq_rel) == (uint32_t)nranks - 1) {
            sh->bar_count.store(0, std::memory_order_relaxed);
            sh->bar_gen.fetch_add(1, std::memory_order_acq_rel);
        } else {
            unsigned spins = 0;
            while (sh->bar_gen.load(std::memory_order_acquire) == gen) {
                if (++spins > 64) sched_yield();
            }
        }
    }

    // make sure the own arena holds `bytes` (collective-safe: only republished, peers re-open after a barrier)
    p2p_status reserve(uint64_t bytes) {
        if (bytes <= arena_bytes) return P2P_OK;
        uint64_t nb = std::max<uint64_t>(bytes + bytes / 4, 1ull << 20);
        nb = (nb + (2ull << 20) - 1) & ~((2ull << 20) - 1);
        if (arena) P2P_CUDA_TRY(cudaFree(arena));
        arena = nullptr;
        P2P_CUDA_TRY(cudaMalloc(&arena, nb));
        arena_bytes = nb;
        cudaIpcMemHandle_t h;
        P2P_CUDA_TRY(cudaIpcGetMemHandle(&h, arena));
        sh->handle[rank] = h;
        sh->arena_bytes[rank] = nb;
        std::atomic_thread_fence(std::memory_order_release);
        sh->arena_gen[rank] = sh->arena_gen[rank] + 1;
        peer[rank] = arena;
        peer_gen[rank] = sh->arena_gen[rank];
        return P2P_OK;
    }
    // after a barrier: (re)open every peer arena whose generation changed
    p2p_status refresh_peers() {
        std::atomic_thread_fence(std::memory_order_acquire);
        for (int r = 0; r < nranks; ++r) {
            if (r == rank || sh->arena_gen[r] == peer_gen[r]) continue;
            if (peer[r]) cudaIpcCloseMemHandle(peer[r]);
            peer[r] = nullptr;
            void *p = nullptr;
            cudaError_t e = cudaIpcOpenMemHandle(&p, sh->handle[r], cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                set_error(std::string("cudaIpcOpenMemHandle of rank ") + std::to_string(r) + ": " +
                          cudaGetErrorString(e));
                return P2P_ERR_CUDA;
            }
            peer[r] = (char *)p;
            peer_gen[r] = sh->arena_gen[r];
        }
        return P2P_OK;
    }
    p2p_status reserve_scratch(size_t count) {
        if (count * nranks <= scratch_count) return P2P_OK;
        if (scratch) P2P_CUDA_TRY(cudaFree(scratch));
        scratch = nullptr;
        P2P_CUDA_TRY(cudaMalloc(&scratch, sizeof(unsigned long long) * count * nranks));
        scratch_count = count * nranks;
        return P2P_OK;
    }
    // stage `bytes` of device data into the own arena, then barrier + peer refresh
    p2p_status publish(const void *src, uint64_t bytes, cudaStream_t st) {
        p2p_status s = reserve(bytes);
        if (s != P2P_OK) return s;
        if (bytes) P2P_CUDA_TRY(cudaMemcpyAsync(arena, src, bytes, cudaMemcpyDeviceToDevice, st));
        P2P_CUDA_TRY(cudaStreamSynchronize(st));
        barrier();
        return refresh_peers();
    }

    p2p_status gather_all(const unsigned long long *send, size_t count, cudaStream_t st) {
        p2p_status s = publish(send, count * 8, st);
        if (s != P2P_OK) return s;
        s = reserve_scratch(count);
        if (s != P2P_OK) return s;
        for (int r = 0; r < nranks; ++r)
            if (count)
                P2P_CUDA_TRY(cudaMemcpyAsync(scratch + (size_t)r * count, peer[r], count * 8, cudaMemcpyDefault, st));
        P2P_CUDA_TRY(cudaStreamSynchronize(st));
        barrier();  // every rank finished reading every arena
        return P2P_OK;
    }

    p2p_status allreduce_sum_u64(unsigned long long *dev, size_t count, cudaStream_t st) override {
        p2p_status s = gather_all(dev, count, st);
        if (s != P2P_OK) return s;
        if (count) {
            const unsigned grid = (unsigned)std::min<size_t>((count + 255) / 256, 1184);
            P2P_LAUNCH(k_sum_ranks, grid, 256, 0, st, scratch, nranks, count, dev);
            P2P_CUDA_TRY(cudaGetLastError());
        }
        return P2P_OK;
    }
    p2p_status allgather_u64(const unsigned long long *send, unsigned long long *recv, size_t count,
                             cudaStream_t st) override {
        p2p_status s = gather_all(send, count, st);
        if (s != P2P_OK) return s;
        if (count) P2P_CUDA_TRY(cudaMemcpyAsync(recv, scratch, count * 8 * nranks, cudaMemcpyDeviceToDevice, st));
        return P2P_OK;
    }
    bool has_peer_results() const override { return true; }
    // the receive buffer of the fused result return is the rank's own arena: peers store into it directly
    p2p_status peer_results_begin(uint64_t recv_bytes, const int64_t *my_off, char **dst, int64_t *dst_off,
                                  char **recv, cudaStream_t st) override {
        P2P_CUDA_TRY(cudaStreamSynchronize(st));  // every earlier read of the arena (stream-ordered) is done
        barrier();                                // ... on every rank
        p2p_status s = reserve(recv_bytes);
        if (s != P2P_OK) return s;
        for (int r = 0; r < nranks; ++r) sh->res_off[rank][r] = my_off[r];
        std::atomic_thread_fence(std::memory_order_release);
        barrier();
        s = refresh_peers();
        if (s != P2P_OK) return s;
        std::atomic_thread_fence(std::memory_order_acquire);
        for (int r = 0; r < nranks; ++r) {
            dst[r] = peer[r];
            dst_off[r] = sh->res_off[r][rank];
        }
        *recv = arena;
        return P2P_OK;
    }
    p2p_status peer_results_end(cudaStream_t st) override {
        P2P_CUDA_TRY(cudaStreamSynchronize(st));  // this rank's eval (and its stores into peers) finished
        barrier();                                // ... on every rank: my buffer is complete
        return P2P_OK;
    }
    p2p_status alltoall_counts(const int64_t *send, int64_t *recv, cudaStream_t) override {
        for (int r = 0; r < nranks; ++r) sh->counts[rank][r] = send[r];
        std::atomic_thread_fence(std::memory_order_release);
        barrier();
        std::atomic_thread_fence(std::memory_order_acquire);
        for (int r = 0; r < nranks; ++r) recv[r] = sh->counts[r][rank];
        barrier();
        return P2P_OK;
    }
    p2p_status alltoallv(const void *send, const int64_t *soff, const int64_t *scnt, void *recv, const int64_t *roff,
                         const int64_t *rcnt, cudaStream_t st) override {
        uint64_t total = 0;
        for (int r = 0; r < nranks; ++r) {
            sh->soff[rank][r] = soff[r];
            if (scnt[r] > 0) total = std::max<uint64_t>(total, (uint64_t)(soff[r] + scnt[r]));
        }
        std::atomic_thread_fence(std::memory_order_release);
        p2p_status s = publish(send, total, st);  // includes the barrier: every rank's offsets are visible now
        if (s != P2P_OK) return s;
        std::atomic_thread_fence(std::memory_order_acquire);
        for (int r = 0; r < nranks; ++r) {
            if (rcnt[r] <= 0) continue;
            P2P_CUDA_TRY(cudaMemcpyAsync((char *)recv + roff[r], peer[r] + sh->soff[r][rank], (size_t)rcnt[r],
                                         cudaMemcpyDefault, st));
        }
        P2P_CUDA_TRY(cudaStreamSynchronize(st));
        barrier();  // peers may rewrite their arenas only after every pull finished
        return P2P_OK;
    }
};
}  // namespace

CommBase *make_ipc_comm(int nranks, int rank, const char *name, p2p_status *st) {
    *st = P2P_OK;
    std::string nm = std::string("/") + name;
    int fd = -1;
    if (rank == 0) {
        fd = shm_open(nm.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
        if (fd < 0) {
            set_error("shm_open(" + nm + ") failed: the name exists or /dev/shm is unavailable");
            *st = P2P_ERR_INVALID_ARGUMENT;
            return nullptr;
        }
        if (ftruncate(fd, sizeof(IpcShared)) != 0) {
            close(fd);
            shm_unlink(nm.c_str());
            set_error("ftruncate of the IPC segment failed");
            *st = P2P_ERR_OUT_OF_MEMORY;
            return nullptr;
        }
    } else {
        const auto t0 = std::chrono::steady_clock::now();
        while ((fd = shm_open(nm.c_str(), O_RDWR, 0600)) < 0) {
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120)) {
                set_error("timed out waiting for rank 0's IPC segment " + nm);
                *st = P2P_ERR_INVALID_ARGUMENT;
                return nullptr;
            }
            std::this_thread::sleep_for(std::chrono::milliseconds(2));
        }
        struct stat sb;
        while (fstat(fd, &sb) == 0 && (size_t)sb.st_size < sizeof(IpcShared))
            std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    void *m = mmap(nullptr, sizeof(IpcShared), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) {
        set_error("mmap of the IPC segment failed");
        *st = P2P_ERR_OUT_OF_MEMORY;
        return nullptr;
    }
    IpcShared *sh = (IpcShared *)m;
    if (rank == 0) {
        sh->nranks = nranks;
        sh->magic.store(IPC_MAGIC, std::memory_order_release);
    } else {
        while (sh->magic.load(std::memory_order_acquire) != IPC_MAGIC) std::this_thread::yield();
        if (sh->nranks != nranks) {
            munmap(m, sizeof(IpcShared));
            set_error("IPC communicator: ranks disagree on nranks");
            *st = P2P_ERR_INVALID_ARGUMENT;
            return nullptr;
        }
    }
    IpcComm *c = new IpcComm();
    c->name = nm;
    c->sh = sh;
    c->nranks = nranks;
    c->rank = rank;
    c->peer.assign(nranks, nullptr);
    c->peer_gen.assign(nranks, 0);
    int dev = 0;
    cudaGetDevice(&dev);
    sh->dev[rank] = dev;
    p2p_status s = c->reserve(1ull << 20);
    if (s == P2P_OK) {
        c->barrier();
        s = c->refresh_peers();
    }
    // every rank attached and opened the initial arenas: the name can go (the mapping stays valid)
    if (sh->attached.fetch_add(1) == (uint32_t)nranks - 1) shm_unlink(nm.c_str());
    if (s != P2P_OK) {
        delete c;
        *st = s;
        return nullptr;
    }
    c->barrier();
    return c;
}

}  // namespace p2p

using namespace p2p;

extern "C" p2p_status p2p_comm_create_ipc(int nranks, int rank, const char *name, p2p_comm **out) {
    if (!out || !name || !*name || std::strchr(name, '/') || nranks < 1 || nranks > IPC_MAX_RANKS || rank < 0 ||
        rank >= nranks) {
        set_error("invalid IPC communicator arguments (1 <= nranks <= 64, 0 <= rank < nranks, name without '/')");
        return P2P_ERR_INVALID_ARGUMENT;
    }
    *out = nullptr;
    p2p_status st = P2P_OK;
    CommBase *impl = make_ipc_comm(nranks, rank, name, &st);
    if (!impl) return st;
    p2p_comm *c = new p2p_comm();
    c->impl = impl;
    *out = c;
    return P2P_OK;
}
