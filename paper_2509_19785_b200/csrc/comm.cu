// comm.cu -- multi-GPU plumbing of libtsnet: the communicator and the two
// exchanges of one sharded L-tsNET iteration:
//   * the sum of the spread charge grid (W1, Mx, My) over the ranks after step
//     a2 -- a peer-memory all-reduce: each rank publishes its live N x N grid
//     (N = 3 I from the device geometry, so only the cells in use move, whatever
//     the I_max the buffers were sized for) into its exchange buffer, and every
//     rank sums all ranks' buffers with direct loads over NVLink (CUDA IPC
//     mappings), after a device-side flag handshake -- no host round trip, so
//     the iteration stays one CUDA graph;
//   * the all-gather of the updated layout Y after the move.  When the ranks
//     step on the communicator's own replicated layout buffer
//     (tsnet_comm_layout: one IPC-shared n x 2 buffer per rank), the move
//     itself stores each new position into every peer's buffer over NVLink
//     (k_update with a PeerPush, iterate.cu) between two device-side
//     handshakes: a rank writes into a peer's Y only after that peer has
//     finished reading Y for the current iteration (field + SpMV), and starts
//     the next iteration only after every peer's move has landed.  Otherwise
//     each rank's rows are padded to an equal slice (the shards are
//     nnz-balanced, their row counts differ) and gathered with one
//     ncclAllGather through a staging buffer.
// NCCL is loaded at run time (dlopen "libnccl.so.2"): in a process that already
// imported PyTorch this resolves to the NCCL torch loaded; the library has no
// link-time NCCL dependency, so single-GPU use needs no NCCL at all.  Where the
// peers are not all reachable by CUDA peer access (e.g. several ranks on one
// device), the grid falls back to an ncclAllReduce of the whole buffer.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
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
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// libnccl is loaded once per process (a function-local static: thread-safe
// initialisation, C++11).
static NcclApi load_nccl() {
    NcclApi api;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
        api.handle = h;
        api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
        api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
        api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
        api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    }
    return api;
}

static NcclApi* nccl_api() {
    static NcclApi api = load_nccl();
    const bool ok = api.handle && api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce &&
                    api.AllGather && api.GetErrorString;
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

constexpr int kMaxWorld = 64;

// The communicator behind tsnet_comm_init's `void* comm`.
struct Comm {
    ncclComm_t nccl = nullptr;
    int world = 1, rank = 0, dev = 0;
    int64_t cells = 0;          // grid cells per exchange buffer ((3 I_max)^2)
    // own exchange memory (cudaMalloc, IPC-shared): flags (256 B: [0] published
    // iteration, [1] the iteration counter), then two grids of `cells` float4
    // (iteration parity)
    char* xbuf = nullptr;
    size_t xbytes = 0;
    bool p2p = false;           // every peer reachable: peer-memory all-reduce
    std::vector<char*> peer;    // per rank: its exchange buffer as mapped here (own = xbuf)
    // device copies of the per-rank pointers: flags[w], grid0[w], grid1[w]
    unsigned long long** d_flags = nullptr;
    float4** d_grid = nullptr;  // [2][world]
    // replicated layout owned by the communicator (tsnet_comm_layout)
    float2* y = nullptr;        // own buffer, n x 2 fp32 (cudaMalloc, IPC-shared)
    int64_t y_n = -1;
    bool ypush = false;         // every peer's buffer mapped: the move pushes Y
    std::vector<float2*> ypeer; // per rank: its layout buffer as mapped here (own = y)
    float2** d_ypeer = nullptr; // device copy of ypeer
};

static unsigned long long* xflags(char* b) { return reinterpret_cast<unsigned long long*>(b); }
static float4* xgrid(char* b, int parity, int64_t cells) {
    return reinterpret_cast<float4*>(b + 256) + (size_t)parity * (size_t)cells;
}

// ----------------------------------------------------------- peer all-reduce
// 1. publish: this rank's live grid (N x N float4 from the geometry) into its
//    exchange grid of the next iteration's parity.
__global__ void k_x_publish(const Geo* __restrict__ g, const float4* __restrict__ wgrid,
                            const unsigned long long* __restrict__ flags, float4* __restrict__ x0,
                            float4* __restrict__ x1) {
    const int64_t cells = (int64_t)g->N * g->N;
    float4* dst = ((flags[1] + 1) & 1) ? x1 : x0;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < cells; c += (int64_t)gridDim.x * blockDim.x)
        dst[c] = wgrid[c];
}

// 2. signal (one thread, after the publish kernel): the iteration counter goes
//    to t + 1 and flags[0] = t + 1 is released at system scope.
__global__ void k_x_signal(unsigned long long* flags) {
    const unsigned long long t = flags[1] + 1;
    flags[1] = t;
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flags), "l"(t) : "memory");
}

// ld_acquire_sys / st_release_sys: common.cuh

// 3. reduce: wait until every rank published iteration t (this rank's counter),
//    then wgrid = sum over ranks of their exchange grid of parity t & 1, read
//    over NVLink.  Parity reuse is safe: a rank overwrites its parity-p grid at
//    iteration t + 2 only after its reduce of t + 1, which waited for every
//    peer's signal of t + 1, issued after that peer's reduce of t.
__global__ void k_x_reduce(const Geo* __restrict__ g, unsigned long long* const* __restrict__ flags,
                           float4* const* __restrict__ grids, int world, const unsigned long long* own_flags,
                           float4* __restrict__ wgrid) {
    const unsigned long long t = own_flags[1];
    if (threadIdx.x == 0) {
        for (int r = 0; r < world; ++r)
            wait_peer_counter(flags[r], t);
    }
    __syncthreads();
    float4* const* gr = grids + (t & 1) * world;
    const int64_t cells = (int64_t)g->N * g->N;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < cells; c += (int64_t)gridDim.x * blockDim.x) {
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r = 0; r < world; ++r) {
            const float4 v = gr[r][c];
            s.x += v.x;
            s.y += v.y;
            s.z += v.z;
        }
        wgrid[c] = s;
    }
}

// sum of several workspaces' live grids on one device, into each of them
// (tsnet_grids_sum: the same reduction without peers, for callers that run
// several shards on one device and for tests)
struct GridTab {
    float4* p[kMaxWorld];
};
__global__ void k_grids_sum(const Geo* __restrict__ g, GridTab grids, int count) {
    const int64_t cells = (int64_t)g->N * g->N;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < cells; c += (int64_t)gridDim.x * blockDim.x) {
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r = 0; r < count; ++r) {
            const float4 v = grids.p[r][c];
            s.x += v.x;
            s.y += v.y;
            s.z += v.z;
        }
        for (int r = 0; r < count; ++r) grids.p[r][c] = s;
    }
}

// ---------------------------------------------------------- Y push handshake
// Flags of the exchange buffer (u64 words): [0] grid published, [1] grid
// iteration counter (above); [kFRead] = t + 1 once this rank has finished
// reading Y for its iteration t (field + SpMV); [kFMoved] = t + 1 once its
// move of iteration t has been stored into every peer's Y; [kFTicket] the
// move kernel's last-block counter; [kFIter] this rank's completed
// iterations t (local).
// before an iteration: wait until every rank's move of every earlier
// iteration has landed in this rank's Y (lane r polls rank r over NVLink)
__global__ void k_y_enter(unsigned long long* const* __restrict__ flags, int world,
                          const unsigned long long* __restrict__ own) {
    const unsigned long long t = own[kFIter];
    for (int r = threadIdx.x; r < world; r += blockDim.x)
        wait_peer_counter(flags[r] + kFMoved, t);
}

// after the field chain and the SpMV of iteration t: this rank no longer reads Y(t)
__global__ void k_y_read_done(unsigned long long* own) {
    __threadfence_system();
    st_release_sys(own + kFRead, own[kFIter] + 1);
}

PeerPush comm_peer_push(void* comm, int64_t n) {
    PeerPush pp{};
    Comm* c = reinterpret_cast<Comm*>(comm);
    if (c == nullptr || !c->ypush || c->y_n != n) return pp;
    pp.y = c->d_ypeer;
    pp.flags = c->d_flags;
    pp.own = xflags(c->xbuf);
    pp.world = c->world;
    pp.self = c->rank;
    return pp;
}

bool comm_owns_layout(const void* comm, const float* Y, int64_t n) {
    const Comm* c = reinterpret_cast<const Comm*>(comm);
    return c != nullptr && c->ypush && c->y_n == n && reinterpret_cast<const float*>(c->y) == Y;
}

cudaError_t comm_y_enter(void* comm, cudaStream_t s) {
    Comm* c = reinterpret_cast<Comm*>(comm);
    k_y_enter<<<1, 32, 0, s>>>(c->d_flags, c->world, xflags(c->xbuf));
    return cudaGetLastError();
}

cudaError_t comm_y_read_done(void* comm, cudaStream_t s) {
    Comm* c = reinterpret_cast<Comm*>(comm);
    k_y_read_done<<<1, 1, 0, s>>>(xflags(c->xbuf));
    return cudaGetLastError();
}

// sum of the charge grid over the ranks, into `wgrid` (this rank's grid on entry)
int comm_allreduce_grid(void* comm, const Geo* geo, float4* wgrid, size_t count_floats, cudaStream_t s) {
    Comm* c = reinterpret_cast<Comm*>(comm);
    if (c->p2p && (size_t)c->cells * 4 >= count_floats) {
        k_x_publish<<<kNumSMs, 256, 0, s>>>(geo, wgrid, xflags(c->xbuf), xgrid(c->xbuf, 0, c->cells),
                                            xgrid(c->xbuf, 1, c->cells));
        k_x_signal<<<1, 1, 0, s>>>(xflags(c->xbuf));
        k_x_reduce<<<kNumSMs, 256, 0, s>>>(geo, c->d_flags, c->d_grid, c->world, xflags(c->xbuf), wgrid);
        TSNET_CUDA(cudaGetLastError());
        return TSNET_OK;
    }
    NcclApi* api = nccl_api();
    TSNET_ARG(api != nullptr, "libnccl.so.2 could not be loaded");
    TSNET_NCCL(api->AllReduce(wgrid, wgrid, count_floats, ncclFloat32, ncclSum, c->nccl, s));
    return TSNET_OK;
}

// ------------------------------------------------------------ Y all-gather
struct Bounds {
    int64_t b[kMaxWorld + 1];
};

// stage[r slice .. + rows_r) -> Y rows [bounds[r], bounds[r+1]) for r != self
__global__ void k_unstage(const float2* __restrict__ stage, float2* __restrict__ Y, Bounds bd, int world, int self,
                          int64_t slice) {
    for (int r = 0; r < world; ++r) {
        if (r == self) continue;
        const int64_t b0 = bd.b[r], rows = bd.b[r + 1] - b0;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
            Y[b0 + i] = stage[(int64_t)r * slice + i];
    }
}

// every rank's rows [bounds[r], bounds[r+1]) of Y (n x 2 fp32) to every rank:
// own rows -> stage[rank slice], ncclAllGather of equal slices, rows back to Y.
// `stage` holds world * max_r(rows_r) float2.
int comm_allgather_rows(void* comm, float* Y, const int64_t* bounds, int world, float2* stage, size_t stage_cap,
                        cudaStream_t s) {
    Comm* c = reinterpret_cast<Comm*>(comm);
    TSNET_ARG(world == c->world && world <= kMaxWorld, "world %d does not match the communicator (%d)", world, c->world);
    if (world == 1) return TSNET_OK;
    int64_t slice = 0;
    Bounds bd{};
    for (int r = 0; r <= world; ++r) bd.b[r] = bounds[r];
    for (int r = 0; r < world; ++r) slice = std::max<int64_t>(slice, bounds[r + 1] - bounds[r]);
    TSNET_ARG((size_t)(slice * world) <= stage_cap, "all-gather staging too small");
    if (slice == 0) return TSNET_OK;
    NcclApi* api = nccl_api();
    TSNET_ARG(api != nullptr, "libnccl.so.2 could not be loaded");
    float2* Y2 = reinterpret_cast<float2*>(Y);
    const int64_t own = bounds[c->rank + 1] - bounds[c->rank];
    if (own > 0)
        TSNET_CUDA(cudaMemcpyAsync(stage + (size_t)c->rank * slice, Y2 + bounds[c->rank], sizeof(float2) * own,
                                   cudaMemcpyDeviceToDevice, s));
    TSNET_NCCL(api->AllGather(stage + (size_t)c->rank * slice, stage, (size_t)slice * 2, ncclFloat32, c->nccl, s));
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((slice + 255) / 256, (int64_t)kNumSMs * 8));
    k_unstage<<<blocks, 256, 0, s>>>(stage, Y2, bd, world, c->rank, slice);
    TSNET_CUDA(cudaGetLastError());
    return TSNET_OK;
}

static void comm_free(Comm* c) {
    if (!c) return;
    for (int r = 0; r < (int)c->peer.size(); ++r)
        if (c->peer[r] && c->peer[r] != c->xbuf) cudaIpcCloseMemHandle(c->peer[r]);
    for (int r = 0; r < (int)c->ypeer.size(); ++r)
        if (c->ypeer[r] && c->ypeer[r] != c->y) cudaIpcCloseMemHandle(c->ypeer[r]);
    if (c->y) cudaFree(c->y);
    if (c->d_ypeer) cudaFree(c->d_ypeer);
    if (c->xbuf) cudaFree(c->xbuf);
    if (c->d_flags) cudaFree(c->d_flags);
    if (c->d_grid) cudaFree(c->d_grid);
    delete c;
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

int tsnet_comm_init(const uint8_t* id, int32_t world, int32_t rank, int32_t I_max, void** comm) {
    TSNET_ARG(id != nullptr && comm != nullptr, "NULL argument");
    TSNET_ARG(world >= 1 && world <= kMaxWorld && rank >= 0 && rank < world, "rank %d / world %d", rank, world);
    TSNET_ARG(I_max >= 1 && I_max <= TSNET_I_MAX_LIMIT, "I_max %d outside [1, %d]", I_max, TSNET_I_MAX_LIMIT);
    NcclApi* api = nccl_api();
    TSNET_ARG(api != nullptr, "libnccl.so.2 could not be loaded");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    Comm* c = new Comm;
    c->world = world;
    c->rank = rank;
    cudaGetDevice(&c->dev);
    ncclResult_t nr = api->CommInitRank(&c->nccl, world, uid, rank);
    if (nr != ncclSuccess) {
        set_error("ncclCommInitRank: %s", api->GetErrorString(nr));
        delete c;
        return TSNET_E_NCCL;
    }
    // exchange buffer, its IPC handle to every rank (all-gather of the handles)
    c->cells = (int64_t)(3 * I_max) * (3 * I_max);
    c->xbytes = 256 + 2 * sizeof(float4) * (size_t)c->cells;
    cudaError_t e = cudaMalloc(&c->xbuf, c->xbytes);
    if (e == cudaSuccess) e = cudaMemset(c->xbuf, 0, c->xbytes);
    if (e != cudaSuccess) {
        set_error("exchange buffer: %s", cudaGetErrorString(e));
        api->CommDestroy(c->nccl);
        comm_free(c);
        return TSNET_E_CUDA;
    }
    int reach = 1;
    std::vector<cudaIpcMemHandle_t> h(world);
    cudaIpcMemHandle_t mine;
    if (cudaIpcGetMemHandle(&mine, c->xbuf) != cudaSuccess) {
        cudaGetLastError();
        reach = 0;
        std::memset(&mine, 0, sizeof(mine));
    }
    // handles + per-rank device ordinal, gathered over NCCL
    struct Rec {
        cudaIpcMemHandle_t h;
        int dev, reach;
        char pad[64 - 8];
    };
    Rec me{};
    me.h = mine;
    me.dev = c->dev;
    me.reach = reach;
    Rec* d_rec = nullptr;
    std::vector<Rec> recs(world);
    e = cudaMalloc(&d_rec, sizeof(Rec) * world);
    if (e == cudaSuccess) e = cudaMemcpy(d_rec + rank, &me, sizeof(Rec), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        nr = api->AllGather(d_rec + rank, d_rec, sizeof(Rec), ncclUint8, c->nccl, 0);
        if (nr == ncclSuccess) e = cudaMemcpy(recs.data(), d_rec, sizeof(Rec) * world, cudaMemcpyDeviceToHost);
    }
    cudaFree(d_rec);
    if (e != cudaSuccess || nr != ncclSuccess) {
        set_error("handle exchange: %s", e != cudaSuccess ? cudaGetErrorString(e) : api->GetErrorString(nr));
        api->CommDestroy(c->nccl);
        comm_free(c);
        return e != cudaSuccess ? TSNET_E_CUDA : TSNET_E_NCCL;
    }
    // peer mappings when every rank sits on its own device and is reachable
    bool p2p = true;
    for (int r = 0; r < world; ++r) {
        if (!recs[r].reach) p2p = false;
        if (r != rank) {
            int can = 0;
            if (recs[r].dev == c->dev || cudaDeviceCanAccessPeer(&can, c->dev, recs[r].dev) != cudaSuccess || !can)
                p2p = false;
        }
    }
    c->peer.assign(world, nullptr);
    c->peer[rank] = c->xbuf;
    if (p2p) {
        for (int r = 0; r < world && p2p; ++r) {
            if (r == rank) continue;
            void* ptr = nullptr;
            if (cudaIpcOpenMemHandle(&ptr, recs[r].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                cudaGetLastError();
                p2p = false;
            } else {
                c->peer[r] = reinterpret_cast<char*>(ptr);
            }
        }
    }
    c->p2p = p2p;
    if (p2p) {
        std::vector<unsigned long long*> fl(world);
        std::vector<float4*> gr(2 * world);
        for (int r = 0; r < world; ++r) {
            fl[r] = xflags(c->peer[r]);
            gr[r] = xgrid(c->peer[r], 0, c->cells);
            gr[world + r] = xgrid(c->peer[r], 1, c->cells);
        }
        e = cudaMalloc(&c->d_flags, sizeof(void*) * world);
        if (e == cudaSuccess) e = cudaMalloc(&c->d_grid, sizeof(void*) * 2 * world);
        if (e == cudaSuccess) e = cudaMemcpy(c->d_flags, fl.data(), sizeof(void*) * world, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(c->d_grid, gr.data(), sizeof(void*) * 2 * world, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            set_error("peer tables: %s", cudaGetErrorString(e));
            api->CommDestroy(c->nccl);
            comm_free(c);
            return TSNET_E_CUDA;
        }
    }
    *comm = c;
    return TSNET_OK;
}

int tsnet_comm_layout(void* comm, int64_t n, float** Y_out) {
    TSNET_ARG(comm != nullptr && Y_out != nullptr, "NULL argument");
    TSNET_ARG(n >= 1, "n = %lld", (long long)n);
    Comm* c = reinterpret_cast<Comm*>(comm);
    if (c->y != nullptr) {
        TSNET_ARG(c->y_n == n, "the communicator's layout has n = %lld, not %lld", (long long)c->y_n, (long long)n);
        *Y_out = reinterpret_cast<float*>(c->y);
        return TSNET_OK;
    }
    NcclApi* api = nccl_api();
    TSNET_ARG(api != nullptr, "libnccl.so.2 could not be loaded");
    TSNET_CUDA(cudaMalloc(&c->y, sizeof(float2) * (size_t)n));
    c->y_n = n;
    c->ypeer.assign(c->world, nullptr);
    c->ypeer[c->rank] = c->y;
    // IPC handles of every rank's buffer (all-gathered like the exchange buffers)
    struct Rec {
        cudaIpcMemHandle_t h;
        int ok;
        char pad[64 - 4];
    };
    Rec me{};
    me.ok = c->p2p && cudaIpcGetMemHandle(&me.h, c->y) == cudaSuccess;
    cudaGetLastError();
    std::vector<Rec> recs(c->world);
    Rec* d_rec = nullptr;
    cudaError_t e = cudaMalloc(&d_rec, sizeof(Rec) * c->world);
    ncclResult_t nr = ncclSuccess;
    if (e == cudaSuccess) e = cudaMemcpy(d_rec + c->rank, &me, sizeof(Rec), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        nr = api->AllGather(d_rec + c->rank, d_rec, sizeof(Rec), ncclUint8, c->nccl, 0);
        if (nr == ncclSuccess) e = cudaMemcpy(recs.data(), d_rec, sizeof(Rec) * c->world, cudaMemcpyDeviceToHost);
    }
    cudaFree(d_rec);
    if (e != cudaSuccess || nr != ncclSuccess) {
        set_error("layout handle exchange: %s", e != cudaSuccess ? cudaGetErrorString(e) : api->GetErrorString(nr));
        return e != cudaSuccess ? TSNET_E_CUDA : TSNET_E_NCCL;
    }
    bool ok = c->p2p;
    for (int r = 0; r < c->world; ++r) ok = ok && recs[r].ok;
    for (int r = 0; r < c->world && ok; ++r) {
        if (r == c->rank) continue;
        void* ptr = nullptr;
        if (cudaIpcOpenMemHandle(&ptr, recs[r].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            ok = false;
        } else {
            c->ypeer[r] = reinterpret_cast<float2*>(ptr);
        }
    }
    if (ok) {
        e = cudaMalloc(&c->d_ypeer, sizeof(float2*) * c->world);
        if (e == cudaSuccess)
            e = cudaMemcpy(c->d_ypeer, c->ypeer.data(), sizeof(float2*) * c->world, cudaMemcpyHostToDevice);
        TSNET_CUDA(e);
    }
    // every rank decides the same (the records are the same everywhere)
    c->ypush = ok;
    *Y_out = reinterpret_cast<float*>(c->y);
    return TSNET_OK;
}

int tsnet_comm_layout_push(const void* comm) {
    return comm != nullptr && reinterpret_cast<const Comm*>(comm)->ypush ? 1 : 0;
}

int tsnet_comm_layout_sync(void* comm, tsnet_stream_t stream) {
    TSNET_ARG(comm != nullptr, "NULL argument");
    Comm* c = reinterpret_cast<Comm*>(comm);
    if (!c->ypush) return TSNET_OK;
    TSNET_CUDA(comm_y_enter(comm, (cudaStream_t)stream));
    return TSNET_OK;
}

int tsnet_comm_peer_reduce(const void* comm) {
    return comm != nullptr && reinterpret_cast<const Comm*>(comm)->p2p ? 1 : 0;
}

int tsnet_comm_destroy(void* comm) {
    if (comm == nullptr) return TSNET_OK;
    Comm* c = reinterpret_cast<Comm*>(comm);
    NcclApi* api = nccl_api();
    TSNET_ARG(api != nullptr, "libnccl.so.2 could not be loaded");
    cudaDeviceSynchronize();
    ncclResult_t nr = api->CommDestroy(c->nccl);
    comm_free(c);
    if (nr != ncclSuccess) {
        set_error("ncclCommDestroy: %s", api->GetErrorString(nr));
        return TSNET_E_NCCL;
    }
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

int tsnet_grids_sum(int32_t count, void* const* ws_list, size_t ws_bytes, int64_t n, int64_t nnz,
                    const tsnet_grad_params* gp, tsnet_stream_t stream) {
    TSNET_ARG(count >= 1 && count <= kMaxWorld && ws_list != nullptr && gp != nullptr, "bad arguments");
    TSNET_ARG(gp->I_max >= 1 && gp->I_max <= TSNET_I_MAX_LIMIT, "bad I_max");
    GridTab tab{};
    Ws w0{};
    for (int r = 0; r < count; ++r) {
        TSNET_ARG(ws_list[r] != nullptr, "workspace %d is NULL", r);
        Ws w = ws_map(ws_list[r], n, nnz, gp->I_max);
        TSNET_ARG(ws_bytes >= w.bytes, "workspace too small");
        tab.p[r] = w.wgrid;
        if (r == 0) w0 = w;
    }
    cudaStream_t s = (cudaStream_t)stream;
    k_grids_sum<<<kNumSMs, 256, 0, s>>>(w0.geo, tab, count);
    TSNET_CUDA(cudaGetLastError());
    TSNET_CUDA(cudaStreamSynchronize(s));
    return TSNET_OK;
}

}  // extern "C"
