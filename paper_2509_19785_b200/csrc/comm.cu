// comm.cu -- multi-GPU plumbing of libtsnet: NCCL communicators and the two
// collectives of one sharded L-tsNET iteration:
//   * all-reduce (sum) of the spread charge grid W1, Mx, My after step a2,
//   * all-gather of the updated layout Y after the move (grouped broadcasts of
//     each rank's contiguous row slice, since nnz-balanced slices differ in size).
// NCCL is loaded at run time (dlopen "libnccl.so.2"): in a process that already
// imported PyTorch this resolves to the NCCL torch loaded; the library has no
// link-time NCCL dependency, so single-GPU use needs no NCCL at all.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <vector>

#include "common.cuh"

namespace tsnet {

struct NcclApi {
    void* handle = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi* nccl_api() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.handle = h;
            api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
            api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
            api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
            api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
            api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast");
            api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
            api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
            api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
        }
    }
    const bool ok = api.handle && api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce &&
                    api.Broadcast && api.GroupStart && api.GroupEnd && api.GetErrorString;
    return ok ? &api : nullptr;
}

#define TSNET_NCCL(call)                                                                        \
    do {                                                                                        \
        ncclResult_t r_ = (call);                                                               \
        if (r_ != ncclSuccess) {                                                                \
            ::tsnet::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, api->GetErrorString(r_)); \
            return TSNET_E_NCCL;                                                                \
        }                                                                                       \
    } while (0)

// sum of the charge grid (count floats at `grid`) over the ranks, in place
int comm_allreduce_grid(void* comm, float* grid, size_t count, cudaStream_t s) {
    NcclApi* api = nccl_api();
    TSNET_ARG(api != nullptr, "libnccl.so.2 could not be loaded");
    TSNET_NCCL(api->AllReduce(grid, grid, count, ncclFloat32, ncclSum, (ncclComm_t)comm, s));
    return TSNET_OK;
}

// every rank's rows [bounds[r], bounds[r+1]) of Y (n x 2 fp32) to every rank
int comm_allgather_rows(void* comm, float* Y, const int64_t* bounds, int world, cudaStream_t s) {
    NcclApi* api = nccl_api();
    TSNET_ARG(api != nullptr, "libnccl.so.2 could not be loaded");
    TSNET_NCCL(api->GroupStart());
    for (int r = 0; r < world; ++r) {
        const size_t cnt = (size_t)(bounds[r + 1] - bounds[r]) * 2;
        if (cnt == 0) continue;
        float* p = Y + 2 * bounds[r];
        ncclResult_t e = api->Broadcast(p, p, cnt, ncclFloat32, r, (ncclComm_t)comm, s);
        if (e != ncclSuccess) {
            api->GroupEnd();
            set_error("ncclBroadcast: %s", api->GetErrorString(e));
            return TSNET_E_NCCL;
        }
    }
    TSNET_NCCL(api->GroupEnd());
    return TSNET_OK;
}

}  // namespace tsnet

using namespace tsnet;

extern "C" {

int tsnet_comm_unique_id(uint8_t* id_out) {
    TSNET_ARG(id_out != nullptr, "NULL argument");
    NcclApi* api = nccl_api();
    TSNET_ARG(api != nullptr, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    TSNET_NCCL(api->GetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == TSNET_COMM_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id_out, &id, sizeof(id));
    return TSNET_OK;
}

int tsnet_comm_init(const uint8_t* id, int32_t world, int32_t rank, void** comm) {
    TSNET_ARG(id != nullptr && comm != nullptr, "NULL argument");
    TSNET_ARG(world >= 1 && rank >= 0 && rank < world, "rank %d / world %d", rank, world);
    NcclApi* api = nccl_api();
    TSNET_ARG(api != nullptr, "libnccl.so.2 could not be loaded");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    TSNET_NCCL(api->CommInitRank(&c, world, uid, rank));
    *comm = c;
    return TSNET_OK;
}

int tsnet_comm_destroy(void* comm) {
    if (comm == nullptr) return TSNET_OK;
    NcclApi* api = nccl_api();
    TSNET_ARG(api != nullptr, "libnccl.so.2 could not be loaded");
    TSNET_NCCL(api->CommDestroy((ncclComm_t)comm));
    return TSNET_OK;
}

int32_t tsnet_shard_rows(const int64_t* indptr_host, int64_t n, int32_t world, int64_t* bounds) {
    if (!indptr_host || !bounds || n < 0 || world < 1) return -1;
    // contiguous row shards with nnz + rows balanced: cut where the running
    // weight indptr[r] + r crosses multiples of (nnz + n) / world
    const int64_t total = indptr_host[n] - indptr_host[0] + n;
    bounds[0] = 0;
    int64_t r = 0;
    for (int32_t g = 1; g < world; ++g) {
        const int64_t target = (total * g + world - 1) / world;
        while (r < n && (indptr_host[r] - indptr_host[0]) + r < target) ++r;
        bounds[g] = r;
    }
    bounds[world] = n;
    return world;
}

}  // extern "C"
