// comm.cpp — a6: the per-step halo exchange of C over NCCL (NVLink 5 / NVSwitch).
//
// libnccl.so.2 is dlopen'ed (the copy PyTorch already loaded when present), so
// single-GPU use has no NCCL dependency.  Halo = R whole z-planes of the padded
// state, contiguous because x is fastest: no packing; the offsets
// come from make_halo_plan (fdirw_api.cu), the same plan fdirw_make_plan reports.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "fdirw_internal.h"

namespace fdirw {

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static Nccl g_nccl;
static bool g_loaded = false;

Nccl* nccl_load(std::string* err)
{
    if (g_loaded) return &g_nccl;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        *err = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
        return nullptr;
    }
    Nccl n;
    n.h = h;
#define LOAD(field, name)                                                  \
    n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name));         \
    if (!n.field) {                                                        \
        *err = std::string("libnccl.so.2 lacks ") + name;                  \
        return nullptr;                                                    \
    }
    LOAD(GetUniqueId, "ncclGetUniqueId");
    LOAD(CommInitRank, "ncclCommInitRank");
    LOAD(CommDestroy, "ncclCommDestroy");
    LOAD(CommAbort, "ncclCommAbort");
    LOAD(Send, "ncclSend");
    LOAD(Recv, "ncclRecv");
    LOAD(GroupStart, "ncclGroupStart");
    LOAD(GroupEnd, "ncclGroupEnd");
    LOAD(AllReduce, "ncclAllReduce");
    LOAD(AllGather, "ncclAllGather");
    LOAD(GetErrorString, "ncclGetErrorString");
#undef LOAD
    g_nccl = n;
    g_loaded = true;
    return &g_nccl;
}

static int check(Nccl* n, ncclResult_t r, const char* what, std::string* err)
{
    if (r == ncclSuccess) return 0;
    *err = std::string(what) + ": " + n->GetErrorString(r);
    return 1;
}

int nccl_unique_id(Nccl* n, void* out128, std::string* err)
{
    ncclUniqueId id;
    if (check(n, n->GetUniqueId(&id), "ncclGetUniqueId", err)) return 1;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
    memcpy(out128, &id, sizeof(id));
    return 0;
}

void* nccl_comm_init(Nccl* n, int world, int rank, const void* id128, std::string* err)
{
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    ncclComm_t comm = nullptr;
    if (check(n, n->CommInitRank(&comm, world, id, rank), "ncclCommInitRank", err)) return nullptr;
    return comm;
}

int nccl_halo(Nccl* n, void* comm, float* cpad, const HaloPlan& h, cudaStream_t s, std::string* err)
{
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    if (check(n, n->GroupStart(), "ncclGroupStart", err)) return 1;
    if (h.peer_lo >= 0) {
        if (check(n, n->Send(cpad + h.send_lo, h.count, ncclFloat32, h.peer_lo, c, s), "ncclSend", err)) return 1;
        if (check(n, n->Recv(cpad + h.recv_lo, h.count, ncclFloat32, h.peer_lo, c, s), "ncclRecv", err)) return 1;
    }
    if (h.peer_hi >= 0) {
        if (check(n, n->Send(cpad + h.send_hi, h.count, ncclFloat32, h.peer_hi, c, s), "ncclSend", err)) return 1;
        if (check(n, n->Recv(cpad + h.recv_hi, h.count, ncclFloat32, h.peer_hi, c, s), "ncclRecv", err)) return 1;
    }
    return check(n, n->GroupEnd(), "ncclGroupEnd", err);
}

int nccl_allreduce_sum_f64(Nccl* n, void* comm, double* buf, cudaStream_t s, std::string* err)
{
    return check(n, n->AllReduce(buf, buf, 1, ncclFloat64, ncclSum, static_cast<ncclComm_t>(comm), s),
                 "ncclAllReduce", err);
}

// N2: every rank's [n_tiles, tile sums...] block, so each rank sums them in global tile order
int nccl_allgather_f64(Nccl* n, void* comm, const double* send, long count, double* recv, cudaStream_t s,
                       std::string* err)
{
    return check(n, n->AllGather(send, recv, (size_t)count, ncclFloat64, static_cast<ncclComm_t>(comm), s),
                 "ncclAllGather", err);
}

void nccl_comm_destroy(Nccl* n, void* comm)
{
    if (n && comm) n->CommDestroy(static_cast<ncclComm_t>(comm));
}

}  // namespace fdirw
