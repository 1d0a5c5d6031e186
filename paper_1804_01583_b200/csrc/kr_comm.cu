// kr_comm.cu — one process per GPU over NCCL (NVLink 5 / NVSwitch) for the two partitions of
// z-slab halo exchange + per-step scalar all-gather (PAR1), and the final
// coefficient all-gather of direction sharding (PAR2). The communicator is created from a
// 128-byte ncclUniqueId that the caller broadcasts (torch.distributed) — no private torch API.
#include <nccl.h>

#include <algorithm>

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

kr_comm* kr_comm_create_host_impl(int32_t rank, int32_t world, int32_t device, kr_allgather_fn fn, void* ctx) {
    KR_CUDA(cudaSetDevice(device));
    kr_comm* k = new kr_comm;
    k->nccl = nullptr;
    k->rank = rank;
    k->world = world;
    k->device = device;
    k->host_fn = fn;
    k->host_ctx = ctx;
    return k;
}

void kr_comm_destroy_impl(kr_comm* c) {
    if (!c) return;
    if (c->nccl) ncclCommDestroy(reinterpret_cast<ncclComm_t>(c->nccl));
    if (c->pinned) cudaFreeHost(c->pinned);
    delete c;
}

namespace {
// host transport: pinned staging buffer of at least n doubles (grown by doubling)
double* host_stage(kr_comm* c, size_t n) {
    if (c->pinned_doubles < n) {
        if (c->pinned) KR_CUDA(cudaFreeHost(c->pinned));
        c->pinned = nullptr;
        const size_t cap = std::max<size_t>(n, 2 * c->pinned_doubles);
        KR_CUDA(cudaMallocHost(reinterpret_cast<void**>(&c->pinned), cap * sizeof(double)));
        c->pinned_doubles = cap;
    }
    return c->pinned;
}

// all-gather of `count` doubles per rank through the caller's host function: send (count) -> pinned,
// fn gathers world * count into pinned + count, which the caller of this helper reads
double* host_allgather(kr_comm* c, size_t count) {
    double* st = c->pinned;
    if (c->host_fn(c->host_ctx, st, st + count, count * sizeof(double)) != 0)
        KR_THROW(KR_ENCCL, "host all-gather callback failed");
    return st + count;
}
}  // namespace

// Asynchronous NCCL failures (a peer died, a link error) surface here instead of as a hang later.
void kr_nccl_check(kr_comm* c) {
    if (!c || !c->nccl) return;
    ncclResult_t async = ncclSuccess;
    KR_NCCL(ncclCommGetAsyncError(reinterpret_cast<ncclComm_t>(c->nccl), &async));
    if (async != ncclSuccess) KR_THROW(KR_ENCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(async));
}

// Graph-captured all-gather self test (krylov_comm_selftest): each rank writes rank-tagged values into its slot,
// the all-gather runs inside a captured graph replayed `reps` times, every slot is checked on the host.
__global__ void selftest_fill_kernel(double* v, int rank, int count, int rep) {
    for (int i = threadIdx.x; i < count; i += blockDim.x) v[(size_t)rank * count + i] = 1000.0 * (rank + 1) + i + 0.5 * rep;
}

void kr_comm_selftest_impl(kr_comm* c, cudaStream_t s, int reps, int32_t* ok) {
    const int count = 8;
    double* d = nullptr;
    KR_CUDA(cudaMalloc(&d, sizeof(double) * count * c->world));
    std::vector<double> h((size_t)count * c->world);
    bool good = true;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    try {
        for (int rep = 0; rep < reps; ++rep) {
            selftest_fill_kernel<<<1, 32, 0, s>>>(d, c->rank, count, rep);
            KR_CUDA(cudaGetLastError());
            if (!kr_comm_is_host(c)) {
                if (!ge) {  // the all-gather alone, captured once and replayed (as inside the Krylov graph)
                    KR_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
                    kr_nccl_allgather(c, d + (size_t)c->rank * count, d, count, s);
                    KR_CUDA(cudaStreamEndCapture(s, &g));
                    KR_CUDA(cudaGraphInstantiate(&ge, g, 0));
                }
                KR_CUDA(cudaGraphLaunch(ge, s));
            } else {
                kr_nccl_allgather(c, d + (size_t)c->rank * count, d, count, s);
            }
            KR_CUDA(cudaMemcpyAsync(h.data(), d, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s));
            KR_CUDA(cudaStreamSynchronize(s));
            kr_nccl_check(c);
            for (int r = 0; r < c->world; ++r)
                for (int i = 0; i < count; ++i) good &= h[(size_t)r * count + i] == 1000.0 * (r + 1) + i + 0.5 * rep;
        }
    } catch (...) {
        if (ge) cudaGraphExecDestroy(ge);
        if (g) cudaGraphDestroy(g);
        cudaFree(d);
        throw;
    }
    if (ge) cudaGraphExecDestroy(ge);
    if (g) cudaGraphDestroy(g);
    cudaFree(d);
    *ok = good ? 1 : 0;
}

// In-place all-gather: send = recv + rank * count.
void kr_nccl_allgather(kr_comm* c, const double* send, double* recv, size_t count, cudaStream_t s) {
    if (kr_comm_is_host(c)) {
        double* st = host_stage(c, count * (size_t)(c->world + 1));
        KR_CUDA(cudaMemcpyAsync(st, send, count * sizeof(double), cudaMemcpyDeviceToHost, s));
        KR_CUDA(cudaStreamSynchronize(s));
        const double* g = host_allgather(c, count);
        KR_CUDA(cudaMemcpyAsync(recv, g, count * c->world * sizeof(double), cudaMemcpyHostToDevice, s));
        KR_CUDA(cudaStreamSynchronize(s));  // the staging buffer is reused by the next collective
        return;
    }
    KR_NCCL(ncclAllGather(send, recv, count, ncclDouble, reinterpret_cast<ncclComm_t>(c->nccl), s));
}

// Halo exchange of buffer `buf` of this rank's single slab: my first two owned planes go to the lower
// neighbour's upper halo (its planes nz+1, nz+2), my last owned plane to the upper neighbour's lower
// halo (its plane 0). Depths: u_i needs 2 planes above (the w ring at z1 reads z1+1) and 1 below.
void kr_nccl_halo(kr_comm* c, kr_handle* h, int buf, cudaStream_t s) {
    ncclComm_t comm = reinterpret_cast<ncclComm_t>(c->nccl);
    Slab& sl = h->slabs[0];
    const size_t plane = (size_t)h->pitch * h->my;
    if (kr_comm_is_host(c)) {
        // every rank contributes its first two and its last owned planes (buffer planes 1, 2, nz); the lower
        // neighbour's last plane becomes my plane 0, the upper neighbour's first two my planes nz+1, nz+2
        // (the same exchange as krylov_zslab_halo_plan, as one all-gather)
        const size_t cnt = 3 * plane;
        double* st = host_stage(c, cnt * (size_t)(c->world + 1));
        double* u = sl.u[buf];
        KR_CUDA(cudaMemcpyAsync(st, u + plane, 2 * plane * sizeof(double), cudaMemcpyDeviceToHost, s));
        KR_CUDA(cudaMemcpyAsync(st + 2 * plane, u + sl.nz * plane, plane * sizeof(double), cudaMemcpyDeviceToHost, s));
        KR_CUDA(cudaStreamSynchronize(s));
        const double* g = host_allgather(c, cnt);
        if (c->rank > 0)
            KR_CUDA(cudaMemcpyAsync(u, g + (size_t)(c->rank - 1) * cnt + 2 * plane, plane * sizeof(double),
                                    cudaMemcpyHostToDevice, s));
        if (c->rank < c->world - 1)
            KR_CUDA(cudaMemcpyAsync(u + (sl.nz + 1) * plane, g + (size_t)(c->rank + 1) * cnt, 2 * plane * sizeof(double),
                                    cudaMemcpyHostToDevice, s));
        KR_CUDA(cudaStreamSynchronize(s));
        return;
    }
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

// ------------------------------------------------------------------------------------------------
// Peer-memory (NVLink P2P) halo transport across processes: the z-slab step kernel stores the halo planes
// of u_{i+1} directly into the neighbouring ranks' state buffers (CUDA IPC), so the per-step halo
// messages disappear; the per-step scalar all-gather that follows each step orders those stores before
// any neighbour reads them (system-scope fence at the end of the step kernel).
// ------------------------------------------------------------------------------------------------
namespace {

struct IpcBlob {
    int32_t magic, rank;
    int64_t nz, pitch, my;
    int32_t device, pad;
    cudaIpcMemHandle_t handle;  // of the allocation holding the three state buffers
    int64_t off[3];             // byte offsets of u[0..2] from the allocation base
};
static_assert(sizeof(IpcBlob) <= KR_IPC_BLOB_BYTES, "blob size");
constexpr int32_t kMagic = 0x4b525032;  // "KRP2"
constexpr int kPat = 64;                // test-pattern doubles per halo plane

__device__ __host__ inline double pattern(int src_rank, int plane_tag, int i) {
    return 1000.0 * (src_rank + 1) + 10.0 * plane_tag + 1e-3 * i;
}

// writes the test pattern into the neighbours' halo planes of buffer 0 (tags: 1, 2 = lower neighbour's
// upper halo planes; 0 = upper neighbour's lower halo plane)
__global__ void p2p_write_kernel(double* lo, int64_t lo_off1, double* hi, int64_t plane, int rank) {
    const int i = threadIdx.x;
    if (i >= kPat) return;
    if (lo) {
        lo[lo_off1 + i] = pattern(rank, 1, i);
        lo[lo_off1 + plane + i] = pattern(rank, 2, i);
    }
    if (hi) hi[i] = pattern(rank, 0, i);
    __threadfence_system();
}

__global__ void p2p_check_kernel(double* own, int64_t nz, int64_t plane, int has_lo, int has_hi, int rank, int* ok) {
    const int i = threadIdx.x;
    if (i >= kPat) return;
    bool good = true;
    if (has_lo) {  // my plane 0 was written by rank - 1
        good &= own[i] == pattern(rank - 1, 0, i);
        own[i] = 0.0;
    }
    if (has_hi) {  // my planes nz+1, nz+2 were written by rank + 1
        good &= own[(nz + 1) * plane + i] == pattern(rank + 1, 1, i);
        good &= own[(nz + 2) * plane + i] == pattern(rank + 1, 2, i);
        own[(nz + 1) * plane + i] = 0.0;
        own[(nz + 2) * plane + i] = 0.0;
    }
    if (!good) atomicExch(ok, 0);
}

typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

AddrRangeFn get_addr_range() {
    static AddrRangeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        KR_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) KR_THROW(KR_ECUDA, "cuMemGetAddressRange unavailable");
        fn = reinterpret_cast<AddrRangeFn>(p);
    }
    return fn;
}

}  // namespace

void kr_p2p_blob(kr_handle* h, void* out) {
    if (h->path != PATH_FUSED_LANCZOS || h->slabs.size() != 1)
        KR_THROW(KR_EINVAL, "peer-memory halos need the stencil Lanczos path with one slab per rank");
    const Slab& sl = h->slabs[0];
    CUdeviceptr base = 0;
    size_t sz = 0;
    if (get_addr_range()(&base, &sz, reinterpret_cast<CUdeviceptr>(sl.u[0])) != CUDA_SUCCESS)
        KR_THROW(KR_ECUDA, "cuMemGetAddressRange failed");
    IpcBlob b{};
    b.magic = kMagic;
    b.rank = h->rank;
    b.nz = sl.nz;
    b.pitch = h->pitch;
    b.my = h->my;
    b.device = h->device;
    KR_CUDA(cudaIpcGetMemHandle(&b.handle, reinterpret_cast<void*>(base)));
    kr_dev_mark_exported(reinterpret_cast<void*>(base));
    for (int k = 0; k < 3; ++k) b.off[k] = reinterpret_cast<char*>(sl.u[k]) - reinterpret_cast<char*>(base);
    memset(out, 0, KR_IPC_BLOB_BYTES);
    memcpy(out, &b, sizeof(b));
}

void kr_p2p_close(kr_handle* h) {
    for (int s = 0; s < 2; ++s)
        if (h->p2p_base[s]) {
            cudaIpcCloseMemHandle(h->p2p_base[s]);
            h->p2p_base[s] = nullptr;
        }
    if (!h->slabs.empty())
        for (int k = 0; k < 3; ++k) h->slabs[0].peer_lo[k] = h->slabs[0].peer_hi[k] = nullptr;
}

void kr_p2p_open(kr_handle* h, const void* blobs, int32_t rank, int32_t world) {
    if (h->path != PATH_FUSED_LANCZOS || h->slabs.size() != 1) KR_THROW(KR_EINVAL, "peer-memory halos: one slab per rank");
    if (rank < 0 || rank >= world) KR_THROW(KR_EINVAL, "bad rank / world");
    if (h->comm && (h->comm->rank != rank || h->comm->world != world)) KR_THROW(KR_EINVAL, "rank / world != comm");
    kr_p2p_close(h);
    const char* all = reinterpret_cast<const char*>(blobs);
    auto blob = [&](int r) {
        IpcBlob b;
        memcpy(&b, all + (size_t)r * KR_IPC_BLOB_BYTES, sizeof(b));
        if (b.magic != kMagic) KR_THROW(KR_EINVAL, "bad peer blob");
        if (h->comm && b.rank != r) KR_THROW(KR_EINVAL, "peer blob of another rank");
        if (b.pitch != h->pitch || b.my != h->my) KR_THROW(KR_EINVAL, "peer grid layout differs");
        return b;
    };
    Slab& sl = h->slabs[0];
    h->p2p_rank = rank;
    h->p2p_world = world;
    for (int s = 0; s < 2; ++s) {
        const int peer = s == 0 ? rank - 1 : rank + 1;
        if (peer < 0 || peer >= world) continue;
        const IpcBlob b = blob(peer);
        void* base = nullptr;
        KR_CUDA(cudaIpcOpenMemHandle(&base, b.handle, cudaIpcMemLazyEnablePeerAccess));
        h->p2p_base[s] = base;
        for (int k = 0; k < 3; ++k) {
            double* u = reinterpret_cast<double*>(reinterpret_cast<char*>(base) + b.off[k]);
            (s == 0 ? sl.peer_lo : sl.peer_hi)[k] = u;
        }
        if (s == 0) sl.peer_lo_nz = b.nz;
    }
    const int64_t plane = h->pitch * h->my;
    p2p_write_kernel<<<1, kPat, 0, h->stream>>>(sl.peer_lo[0], (sl.peer_lo_nz + 1) * plane, sl.peer_hi[0], plane, rank);
    KR_CUDA(cudaGetLastError());
    h->launches++;
    KR_CUDA(cudaStreamSynchronize(h->stream));
}

void kr_p2p_verify(kr_handle* h, int32_t* ok) {
    if (h->slabs.size() != 1) KR_THROW(KR_EINVAL, "peer-memory halos: one slab per rank");
    const Slab& sl = h->slabs[0];
    const int64_t plane = h->pitch * h->my;
    int* d_ok = reinterpret_cast<int*>(h->d_scratch + 4);  // d_scratch holds 8 doubles; 0-1 belong to the large route
    const int one = 1;
    KR_CUDA(cudaMemcpyAsync(d_ok, &one, 4, cudaMemcpyHostToDevice, h->stream));
    p2p_check_kernel<<<1, kPat, 0, h->stream>>>(sl.u[0], sl.nz, plane, h->p2p_rank > 0,
                                                h->p2p_rank + 1 < h->p2p_world, h->p2p_rank, d_ok);
    KR_CUDA(cudaGetLastError());
    h->launches++;
    int got = 0;
    KR_CUDA(cudaMemcpyAsync(&got, d_ok, 4, cudaMemcpyDeviceToHost, h->stream));
    KR_CUDA(cudaStreamSynchronize(h->stream));
    *ok = got;
}
