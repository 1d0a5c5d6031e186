// kr_comm.cu — one process per GPU over NCCL (NVLink 5 / NVSwitch) for the two partitions of
// z-slab halo exchange + per-step scalar all-gather (PAR1), and the final
// coefficient all-gather of direction sharding (PAR2). The communicator is created from a
// 128-byte ncclUniqueId that the caller broadcasts (torch.distributed) — no private torch API.
#include <nccl.h>

#include "kr_internal.h"

#define KR_NCCL(call)                                                                                      \
    do {                                                                                                   \
        ncclResult_t r_ = (call);                                                                          \
        if (r_ != ncclSuccess) KR_THROW(KR_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_));     \
    } while (0)

static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");

kr_status kr_comm_unique_id_impl(void* id128) {
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return KR_ENCCL;
    memcpy(id128, &id, sizeof(id));
    return KR_OK;
}

kr_comm* kr_comm_create_impl(const void* id128, int32_t rank, int32_t world, int32_t device) {
    KR_CUDA(cudaSetDevice(device));
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    ncclComm_t c;
    KR_NCCL(ncclCommInitRank(&c, world, id, rank));
    kr_comm* k = new kr_comm;
    k->nccl = c;
    k->rank = rank;
    k->world = world;
    k->device = device;
    return k;
}

void kr_comm_destroy_impl(kr_comm* c) {
    if (!c) return;
    ncclCommDestroy(reinterpret_cast<ncclComm_t>(c->nccl));
    delete c;
}

// In-place all-gather: send = recv + rank * count.
void kr_nccl_allgather(kr_comm* c, const double* send, double* recv, size_t count, cudaStream_t s) {
    KR_NCCL(ncclAllGather(send, recv, count, ncclDouble, reinterpret_cast<ncclComm_t>(c->nccl), s));
}

// Halo exchange of buffer `buf` of this rank's single slab: my first two owned planes go to the lower
// neighbour's upper halo (its planes nz+1, nz+2), my last owned plane to the upper neighbour's lower
// halo (its plane 0). Depths: u_i needs 2 planes above (the w ring at z1 reads z1+1) and 1 below.
void kr_nccl_halo(kr_comm* c, kr_handle* h, int buf, cudaStream_t s) {
    ncclComm_t comm = reinterpret_cast<ncclComm_t>(c->nccl);
    Slab& sl = h->slabs[0];
    const size_t plane = (size_t)h->pitch * h->my;
    kr_halo_op ops[4];
    int32_t n = 0;
    if (krylov_zslab_halo_plan(h->mz, c->world, c->rank, ops, &n) != KR_OK) KR_THROW(KR_EINVAL, "halo plan");
    KR_NCCL(ncclGroupStart());
    for (int i = 0; i < n; ++i) {
        double* p = sl.u[buf] + ops[i].plane * plane;
        if (ops[i].is_send)
            KR_NCCL(ncclSend(p, ops[i].nplanes * plane, ncclDouble, ops[i].peer, comm, s));
        else
            KR_NCCL(ncclRecv(p, ops[i].nplanes * plane, ncclDouble, ops[i].peer, comm, s));
    }
    KR_NCCL(ncclGroupEnd());
}
