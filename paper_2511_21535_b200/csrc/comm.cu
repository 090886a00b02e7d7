// comm.cu -- NCCL communicator owned by libp2p.  Bootstrapped from a 128-byte ncclUniqueId that
// rank 0 produces and the caller broadcasts (e.g. over a torch.distributed process group); NCCL 2.28 from the
// wheel PyTorch itself loads (same soname libnccl.so.2).
#include <nccl.h>

#include <cstring>
#include <string>

#include "plan.hpp"

struct p2p_comm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
};

using namespace p2p;

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
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    p2p_comm *c = new p2p_comm();
    ncclResult_t r = ncclCommInitRank(&c->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
        delete c;
        set_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        return P2P_ERR_NCCL;
    }
    c->nranks = nranks;
    c->rank = rank;
    *out = c;
    return P2P_OK;
}

void p2p_comm_destroy(p2p_comm *c) {
    if (!c) return;
    if (c->comm) ncclCommDestroy(c->comm);
    delete c;
}

}  // extern "C"
