// tsnet.cu -- the C-ABI entry points of libtsnet (declared in include/tsnet.h).
// Argument checking, workspace map, orchestration of the kernels of
// field.cu / iterate.cu / cost.cu / knn.cu on the caller's stream.
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace tsnet {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

size_t build_P_ws_bytes(int64_t n, int k);
int build_P_impl(const tsnet_graph* g, double u, int k, uint64_t seed, tsnet_csr* P, int32_t* knn_idx,
                 int32_t* knn_hop, int32_t* knn_len, double* beta, void* ws, size_t ws_bytes, cudaStream_t s);

static int check_grad_params(const tsnet_grad_params* gp) {
    TSNET_ARG(gp != nullptr, "grad params are NULL");
    TSNET_ARG(gp->interp_P == 3, "interp_P = %d: only 3 interpolation points per interval are implemented",
              gp->interp_P);
    TSNET_ARG(gp->I_min >= 1 && gp->I_min <= gp->I_max && gp->I_max <= TSNET_I_MAX_LIMIT,
              "need 1 <= I_min (%d) <= I_max (%d) <= %d", gp->I_min, gp->I_max, TSNET_I_MAX_LIMIT);
    TSNET_ARG(gp->h_max > 0.f && std::isfinite(gp->h_max), "h_max must be > 0");
    TSNET_ARG(gp->eps > 0.f, "eps must be > 0");
    TSNET_ARG(gp->spread >= TSNET_SPREAD_AUTO && gp->spread <= TSNET_SPREAD_RUNS, "spread = %d: not 0, 1 or 2",
              gp->spread);
    return TSNET_OK;
}

int comm_allreduce_grid(void* comm, const Geo* geo, float4* wgrid, size_t count_floats, cudaStream_t s);
int comm_allgather_rows(void* comm, float* Y, const int64_t* bounds, int world, float2* stage, size_t stage_cap,
                        cudaStream_t s);

static int check_shard(const tsnet_shard* sh, int64_t n) {
    if (sh == nullptr) return TSNET_OK;
    TSNET_ARG(sh->world >= 1 && sh->rank >= 0 && sh->rank < sh->world, "shard rank %d / world %d", sh->rank,
              sh->world);
    TSNET_ARG(0 <= sh->row_begin && sh->row_begin <= sh->row_end && sh->row_end <= n,
              "shard rows [%lld, %lld) outside [0, %lld)", (long long)sh->row_begin, (long long)sh->row_end,
              (long long)n);
    if (sh->bounds) {
        TSNET_ARG(sh->bounds[0] == 0 && sh->bounds[sh->world] == n, "shard bounds must cover [0, n)");
        for (int r = 0; r < sh->world; ++r)
            TSNET_ARG(sh->bounds[r] <= sh->bounds[r + 1], "shard bounds must be non-decreasing");
        TSNET_ARG(sh->bounds[sh->rank] == sh->row_begin && sh->bounds[sh->rank + 1] == sh->row_end,
                  "row_begin/row_end differ from bounds[rank], bounds[rank+1]");
    }
    return TSNET_OK;
}

static bool sharded(const tsnet_shard* sh, int64_t n) {
    return sh != nullptr && (sh->world > 1 || sh->row_begin != 0 || sh->row_end != n);
}

// Calls that communicate need the communicator (world > 1) and a plan.
static int check_comm(const tsnet_shard* sh, const GradArgs& a) {
    if (!sharded(sh, a.n)) return TSNET_OK;
    if (sh->world > 1) TSNET_ARG(sh->comm != nullptr, "world = %d needs shard->comm (tsnet_comm_init)", sh->world);
    return TSNET_OK;
}

static int check_csr(const tsnet_csr* P) {
    TSNET_ARG(P != nullptr, "P is NULL");
    TSNET_ARG(P->n >= 0 && P->nnz >= 0, "P has negative sizes");
    TSNET_ARG(P->n == 0 || P->indptr != nullptr, "P->indptr is NULL");
    TSNET_ARG(P->nnz == 0 || (P->indices != nullptr && P->values != nullptr), "P arrays are NULL");
    return TSNET_OK;
}

// the call's rows [0, n) or the shard's; a plan must have been built for them
static int check_rows(const tsnet_csr* P, const tsnet_shard* sh) {
    const int64_t rb = sh ? sh->row_begin : 0, re = sh ? sh->row_end : P->n;
    TSNET_ARG(0 <= rb && rb <= re && re <= P->n, "rows [%lld, %lld) outside [0, %lld)", (long long)rb, (long long)re,
              (long long)P->n);
    TSNET_ARG(P->plan == nullptr || (P->plan_row_begin == rb && P->plan_row_end == re),
              "the plan of P holds rows [%lld, %lld), the call rows [%lld, %lld)", (long long)P->plan_row_begin,
              (long long)P->plan_row_end, (long long)rb, (long long)re);
    return TSNET_OK;
}

static int prepare(const tsnet_csr* P, const float* Y, const tsnet_grad_params* gp, const tsnet_shard* sh, void* ws,
                   size_t ws_bytes, Ws& w, GradArgs& a) {
    int st;
    if ((st = check_csr(P)) != TSNET_OK) return st;
    if ((st = check_grad_params(gp)) != TSNET_OK) return st;
    if ((st = check_shard(sh, P->n)) != TSNET_OK) return st;
    if ((st = check_rows(P, sh)) != TSNET_OK) return st;
    TSNET_ARG(P->n == 0 || Y != nullptr, "Y is NULL");
    w = ws_map(ws, P->n, P->nnz, gp->I_max);
    TSNET_ARG(ws != nullptr && ws_bytes >= w.bytes, "workspace too small (%zu < %zu bytes)", ws_bytes, w.bytes);
    a.n = P->n;
    a.nnz = P->nnz;
    a.rb = sh ? sh->row_begin : 0;
    a.re = sh ? sh->row_end : P->n;
    a.indptr = P->indptr;
    a.indices = P->indices;
    a.values = P->values;
    a.plan = P->plan;
    a.plan_kind = P->plan ? (P->plan_kind == TSNET_PLAN_SELL ? TSNET_PLAN_SELL : TSNET_PLAN_CB) : 0;
    a.Y = reinterpret_cast<const float2*>(Y);
    a.lambda_kl = gp->lambda_kl;
    a.lambda_c = gp->lambda_c;
    a.lambda_r = gp->lambda_r;
    a.eps = gp->eps;
    a.h_max = gp->h_max;
    a.I_min = gp->I_min;
    a.I_max = gp->I_max;
    a.spread = gp->spread;
    return TSNET_OK;
}

static size_t grid_floats(const Ws& w) { return (size_t)4 * w.N_max * w.N_max; }

// field (with the grid all-reduce when world > 1) + attractive SpMV of the own rows
// A second stream per (host thread, device) for the field phase, which is
// independent of the attractive SpMV until the gather/update: the two chains
// run concurrently (fork/join by events, so the pattern is also captured into
// a CUDA graph as two branches).
constexpr int kHostChunksMax = 16;

struct SideStream {
    int dev = -1;
    // side: the field chain + moves of the pipelined host step (highest
    // priority: its moves gate the downloads); field: the field chain forked
    // beside the SpMV in a device step (normal priority: preempting the SpMV's
    // CTAs cost 1% there, r1cn)
    cudaStream_t side = nullptr, field = nullptr, copy = nullptr, d2h = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr, copied = nullptr, y_in = nullptr, drained = nullptr, zeroed = nullptr;
    cudaEvent_t attr_done[kHostChunksMax] = {}, moved[kHostChunksMax] = {}, state_in[kHostChunksMax] = {};
};

static cudaError_t side_stream(SideStream*& out) {
    static thread_local SideStream ss[16];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    SideStream& x = ss[dev & 15];
    if (x.dev != dev) {
        // side (pipelined host step): the field chain is a row of short
        // dependent kernels; at the highest priority its CTAs go ahead of
        // queued SpMV CTAs, so the first moves start early; field (device
        // step): default priority (the highest cost 1% there, r1cn)
        int lo = 0, hi = 0;
        if ((e = cudaDeviceGetStreamPriorityRange(&lo, &hi)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithPriority(&x.side, cudaStreamNonBlocking, hi)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithPriority(&x.field, cudaStreamNonBlocking, lo)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithFlags(&x.copy, cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithFlags(&x.d2h, cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&x.zeroed, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&x.copied, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&x.y_in, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&x.drained, cudaEventDisableTiming)) != cudaSuccess) return e;
        for (int c = 0; c < kHostChunksMax; ++c) {
            if ((e = cudaEventCreateWithFlags(&x.attr_done[c], cudaEventDisableTiming)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&x.moved[c], cudaEventDisableTiming)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&x.state_in[c], cudaEventDisableTiming)) != cudaSuccess) return e;
        }
        x.dev = dev;
    }
    out = &x;
    return cudaSuccess;
}

static int eval_gradient_parts(const Ws& w, const GradArgs& a, const tsnet_shard* sh, cudaStream_t s) {
    int st;
    if ((st = check_comm(sh, a)) != TSNET_OK) return st;
    const bool multi = sh != nullptr && sh->comm != nullptr;   // collectives (also with a 1-rank comm)
    SideStream* ss = nullptr;
    // the grid chain (field + its all-reduce) runs on the side stream, overlapped
    // with the SpMV (SURVEY §8(e) "chain G"); the Y all-gather stays on `s`
    TSNET_CUDA(side_stream(ss));
    cudaStream_t fs = ss->field;
    TSNET_CUDA(cudaEventRecord(ss->fork, s));
    TSNET_CUDA(cudaStreamWaitEvent(fs, ss->fork, 0));
    // the whole I_max-sized grid is zeroed only for the NCCL fallback, which
    // all-reduces it as one fixed-size buffer; the peer all-reduce moves the live cells
    TSNET_CUDA(launch_field_local(w, a, fs, multi && !tsnet_comm_peer_reduce(sh->comm)));
    if (multi && (st = comm_allreduce_grid(sh->comm, w.geo, w.wgrid, grid_floats(w), fs)) != TSNET_OK)
        return st;
    TSNET_CUDA(launch_field_conv(w, a, fs));
    TSNET_CUDA(launch_spmv(w, a, s));
    TSNET_CUDA(cudaEventRecord(ss->join, fs));
    TSNET_CUDA(cudaStreamWaitEvent(s, ss->join, 0));
    return TSNET_OK;
}

}  // namespace tsnet

using namespace tsnet;

extern "C" {

const char* tsnet_last_error(void) { return g_err; }

int32_t tsnet_resolve_k(int64_t n, double u, int32_t k_req) {
    int64_t k = k_req > 0 ? k_req : (int64_t)std::floor(3.0 * u + 0.5);
    if (k > n - 1) k = n - 1;
    if (k < 0) k = 0;
    return (int32_t)k;
}

size_t tsnet_build_P_workspace_bytes(int64_t n, int32_t k) { return build_P_ws_bytes(n, k); }

int tsnet_build_P(const tsnet_graph* g, double u, int32_t k, uint64_t seed, tsnet_csr* P, int32_t* knn_idx,
                  int32_t* knn_hop, int32_t* knn_len, double* beta, void* ws, size_t ws_bytes, tsnet_stream_t stream) {
    TSNET_ARG(g != nullptr && P != nullptr, "graph or P is NULL");
    TSNET_ARG(g->n >= 0, "negative n");
    TSNET_ARG(u >= 1.0 && std::isfinite(u), "perplexity u = %g must be >= 1", u);
    TSNET_ARG(k >= 0 && k <= 256, "k = %d outside [0, 256] (resolve it with tsnet_resolve_k)", k);
    TSNET_ARG(k <= (g->n > 0 ? g->n - 1 : 0), "k = %d > n - 1", k);
    TSNET_ARG(g->n == 0 || (g->indptr && g->indices), "graph arrays are NULL");
    TSNET_ARG(g->n == 0 || k == 0 || (knn_idx && knn_hop && knn_len), "kNN output arrays are NULL");
    TSNET_ARG(P->indptr != nullptr, "P->indptr is NULL");
    return build_P_impl(g, u, k, seed, P, knn_idx, knn_hop, knn_len, beta, ws, ws_bytes, (cudaStream_t)stream);
}

size_t tsnet_workspace_bytes(int64_t n, int64_t nnz, const tsnet_grad_params* gp, const tsnet_shard*) {
    const int I_max = (gp && gp->I_max >= 1 && gp->I_max <= TSNET_I_MAX_LIMIT) ? gp->I_max : TSNET_I_MAX_LIMIT;
    return ws_map(nullptr, n, nnz, I_max).bytes;
}

int tsnet_attr(const tsnet_csr* P, const float* Y, const tsnet_shard* shard, float* f_attr, tsnet_stream_t stream) {
    int st;
    if ((st = check_csr(P)) != TSNET_OK) return st;
    if ((st = check_rows(P, shard)) != TSNET_OK) return st;
    TSNET_ARG(P->n == 0 || (Y != nullptr && f_attr != nullptr), "Y or f_attr is NULL");
    if (P->n == 0) return TSNET_OK;
    Ws w{};
    w.f_attr = reinterpret_cast<float2*>(f_attr);
    GradArgs a{};
    a.n = P->n;
    a.nnz = P->nnz;
    a.rb = shard ? shard->row_begin : 0;
    a.re = shard ? shard->row_end : P->n;
    a.indptr = P->indptr;
    a.indices = P->indices;
    a.values = P->values;
    a.plan = P->plan;
    a.plan_kind = P->plan ? (P->plan_kind == TSNET_PLAN_SELL ? TSNET_PLAN_SELL : TSNET_PLAN_CB) : 0;
    a.Y = reinterpret_cast<const float2*>(Y);
    TSNET_CUDA(launch_spmv(w, a, (cudaStream_t)stream));
    return TSNET_OK;
}

int tsnet_grad_parts(const tsnet_csr* P, const float* Y, const tsnet_grad_params* gp, const tsnet_shard* shard,
                     float* f_attr, float* f_field, double* Z, void* ws, size_t ws_bytes, tsnet_stream_t stream) {
    Ws w;
    GradArgs a;
    int st = prepare(P, Y, gp, shard, ws, ws_bytes, w, a);
    if (st != TSNET_OK) return st;
    if (a.n == 0) return TSNET_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if ((st = eval_gradient_parts(w, a, shard, s)) != TSNET_OK) return st;
    TSNET_CUDA(launch_grad_out(w, a, nullptr, reinterpret_cast<float2*>(f_field), Z, s));
    if (f_attr)
        TSNET_CUDA(cudaMemcpyAsync(f_attr, w.f_attr, sizeof(float2) * (a.re - a.rb), cudaMemcpyDeviceToDevice, s));
    return TSNET_OK;
}

int tsnet_grad(const tsnet_csr* P, const float* Y, const tsnet_grad_params* gp, const tsnet_shard* shard, float* grad,
               double* Z, void* ws, size_t ws_bytes, tsnet_stream_t stream) {
    Ws w;
    GradArgs a;
    int st = prepare(P, Y, gp, shard, ws, ws_bytes, w, a);
    if (st != TSNET_OK) return st;
    TSNET_ARG(a.n == 0 || grad != nullptr, "grad is NULL");
    if (a.n == 0) return TSNET_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if ((st = eval_gradient_parts(w, a, shard, s)) != TSNET_OK) return st;
    TSNET_CUDA(launch_grad_out(w, a, reinterpret_cast<float2*>(grad), nullptr, Z, s));
    return TSNET_OK;
}

}  // extern "C"

namespace tsnet {
// One iteration; if `before_update` is given, the move waits for it (the host
// path's velocity/gains upload runs concurrently with the field phase + SpMV).
static int step_impl(const tsnet_csr* P, float* Y, float* vel, float* gains, const tsnet_grad_params* gp,
                     const tsnet_step_params* sp, const tsnet_shard* shard, void* ws, size_t ws_bytes,
                     cudaStream_t s, cudaEvent_t before_update) {
    Ws w;
    GradArgs a;
    int st = prepare(P, Y, gp, shard, ws, ws_bytes, w, a);
    if (st != TSNET_OK) return st;
    TSNET_ARG(sp != nullptr, "step params are NULL");
    TSNET_ARG(a.n == 0 || (vel && gains), "vel or gains is NULL");
    TSNET_ARG(!(sp->recenter && sharded(shard, a.n)), "recentring is not supported with shards");
    const bool multi = shard != nullptr && shard->comm != nullptr;
    TSNET_ARG(!multi || shard->bounds != nullptr, "a communicating shard needs shard->bounds to all-gather Y");
    if (a.n == 0) return TSNET_OK;
    // multi-GPU on the communicator's own layout buffers: the move pushes the
    // new positions into every peer's Y (comm.cu), between the handshakes
    const bool push = multi && comm_owns_layout(shard->comm, Y, a.n);
    if (push) TSNET_CUDA(comm_y_enter(shard->comm, s));
    if ((st = eval_gradient_parts(w, a, shard, s)) != TSNET_OK) return st;
    if (push) TSNET_CUDA(comm_y_read_done(shard->comm, s));
    if (before_update) TSNET_CUDA(cudaStreamWaitEvent(s, before_update, 0));
    TSNET_CUDA(launch_update(w, a, reinterpret_cast<float2*>(Y), reinterpret_cast<float2*>(vel),
                             reinterpret_cast<float2*>(gains), *sp, s,
                             push ? comm_peer_push(shard->comm, a.n) : PeerPush{}));
    if (multi && !push)
        return comm_allgather_rows(shard->comm, Y, shard->bounds, shard->world, w.state, 4 * (size_t)a.n, s);
    return TSNET_OK;
}
}  // namespace tsnet

extern "C" {

int tsnet_step(const tsnet_csr* P, float* Y, float* vel, float* gains, const tsnet_grad_params* gp,
               const tsnet_step_params* sp, const tsnet_shard* shard, void* ws, size_t ws_bytes,
               tsnet_stream_t stream) {
    return step_impl(P, Y, vel, gains, gp, sp, shard, ws, ws_bytes, (cudaStream_t)stream, nullptr);
}

int tsnet_field_local(const tsnet_csr* P, const float* Y, const tsnet_grad_params* gp, const tsnet_shard* shard,
                      void* ws, size_t ws_bytes, tsnet_stream_t stream) {
    Ws w;
    GradArgs a;
    int st = prepare(P, Y, gp, shard, ws, ws_bytes, w, a);
    if (st != TSNET_OK) return st;
    if (a.n == 0) return TSNET_OK;
    TSNET_CUDA(launch_field_local(w, a, (cudaStream_t)stream, true));
    return TSNET_OK;
}

int tsnet_ws_grid(int64_t n, int64_t nnz, const tsnet_grad_params* gp, size_t* offset_bytes, size_t* count_floats) {
    TSNET_ARG(offset_bytes != nullptr && count_floats != nullptr, "NULL argument");
    int st;
    if ((st = check_grad_params(gp)) != TSNET_OK) return st;
    Ws w = ws_map(nullptr, n, nnz, gp->I_max);
    *offset_bytes = (size_t)((const char*)w.wgrid - (const char*)nullptr);
    *count_floats = grid_floats(w);
    return TSNET_OK;
}

int tsnet_step_finish(const tsnet_csr* P, float* Y, float* vel, float* gains, const tsnet_grad_params* gp,
                      const tsnet_step_params* sp, const tsnet_shard* shard, void* ws, size_t ws_bytes,
                      tsnet_stream_t stream) {
    Ws w;
    GradArgs a;
    int st = prepare(P, Y, gp, shard, ws, ws_bytes, w, a);
    if (st != TSNET_OK) return st;
    TSNET_ARG(sp != nullptr, "step params are NULL");
    TSNET_ARG(a.n == 0 || (vel && gains), "vel or gains is NULL");
    TSNET_ARG(!(sp->recenter && sharded(shard, a.n)), "recentring is not supported with shards");
    if (a.n == 0) return TSNET_OK;
    cudaStream_t s = (cudaStream_t)stream;
    TSNET_CUDA(launch_field_conv(w, a, s));
    TSNET_CUDA(launch_spmv(w, a, s));
    TSNET_CUDA(launch_update(w, a, reinterpret_cast<float2*>(Y), reinterpret_cast<float2*>(vel),
                             reinterpret_cast<float2*>(gains), *sp, s));
    return TSNET_OK;
}

}  // extern "C"

namespace tsnet {

// Row chunks of the pipelined host step (1 = no pipeline): measured on cfg 4
// with the multi-wave SpMV, e2e 815 / 850 / 851 / 827 / 823 / 770 it/s for
// 2 / 3 / 4 / 5 / 6 / 8 chunks (r1bx).
constexpr int kHostChunks = 4;
static int host_chunks(int64_t n) { return n >= (int64_t)kHostChunks * 16384 ? kHostChunks : 1; }

// Row cut of the pipelined host step: chunk c ends at the first row whose
// indptr reaches nnz * (c + 1) / chunks (equal SpMV work per chunk).  Found by
// binary search over the device indptr with single-entry reads on `s`, once per
// (indptr, n, nnz, chunks) and cached; any cut is correct, the cut only
// balances the pipeline.
static int chunk_rows(const tsnet_csr* P, int chunks, int64_t* cut, int64_t* cut_nnz, cudaStream_t s) {
    struct Entry {
        const void* indptr = nullptr;
        int64_t n = -1, nnz = -1;
        int chunks = 0;
        int64_t cut[kHostChunksMax + 1], cut_nnz[kHostChunksMax + 1];
    };
    static thread_local Entry cache[4];
    static thread_local int next = 0;
    for (auto& e : cache)
        if (e.indptr == P->indptr && e.n == P->n && e.nnz == P->nnz && e.chunks == chunks) {
            std::memcpy(cut, e.cut, sizeof(int64_t) * (chunks + 1));
            std::memcpy(cut_nnz, e.cut_nnz, sizeof(int64_t) * (chunks + 1));
            return TSNET_OK;
        }
    const int64_t n = P->n;
    cut[0] = 0;
    cut[chunks] = n;
    cut_nnz[0] = 0;
    cut_nnz[chunks] = P->nnz;
    for (int c = 1; c < chunks; ++c) {
        const int64_t target = (int64_t)((double)P->nnz * c / chunks);
        int64_t lo = cut[c - 1], hi = n;          // first row r with indptr[r] >= target
        while (lo < hi) {
            const int64_t mid = lo + (hi - lo) / 2;
            int64_t v = 0;
            TSNET_CUDA(cudaMemcpyAsync(&v, P->indptr + mid, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
            TSNET_CUDA(cudaStreamSynchronize(s));
            if (v >= target) hi = mid; else lo = mid + 1;
        }
        cut[c] = std::max(lo, cut[c - 1]);
        TSNET_CUDA(cudaMemcpyAsync(&cut_nnz[c], P->indptr + cut[c], sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        TSNET_CUDA(cudaStreamSynchronize(s));
    }
    Entry& e = cache[next++ & 3];
    e.indptr = P->indptr;
    e.n = P->n;
    e.nnz = P->nnz;
    e.chunks = chunks;
    std::memcpy(e.cut, cut, sizeof(int64_t) * (chunks + 1));
    std::memcpy(e.cut_nnz, cut_nnz, sizeof(int64_t) * (chunks + 1));
    return TSNET_OK;
}

// tsnet_step_host without recentring, shards or a plan: the host transfers of
// the state overlap the attractive SpMV.  Rows are cut into `chunks` chunks.
// Streams: `s` uploads Y, then runs the SpMV of chunk after chunk; `copy`
// uploads vel/gains chunk by chunk after Y; the side stream runs the field chain,
// then the move of each chunk once its SpMV and its vel/gains are in (new
// positions into a second buffer: later chunks' SpMV still gathers the old Y);
// `d2h` downloads each moved chunk.  Same arithmetic as step_impl.
static int step_host_pipelined(const tsnet_csr* P, float* Y_host, float* vel_host, float* gains_host,
                               const tsnet_grad_params* gp, const tsnet_step_params* sp, void* ws, size_t ws_bytes,
                               cudaStream_t s, SideStream* ss, int chunks, float2* state) {
    const int64_t n = P->n;
    float2* dY = state;
    float2* dV = state + n;
    float2* dG = state + 2 * n;
    float2* dYn = state + 3 * n;
    const size_t b = sizeof(float2) * (size_t)n;
    int64_t cut[kHostChunksMax + 1], cut_nnz[kHostChunksMax + 1];
    int st0 = chunk_rows(P, chunks, cut, cut_nnz, s);
    if (st0 != TSNET_OK) return st0;
    auto rows = [&](int c) { return cut[c]; };
    TSNET_CUDA(cudaMemcpyAsync(dY, Y_host, b, cudaMemcpyHostToDevice, s));
    TSNET_CUDA(cudaEventRecord(ss->y_in, s));
    // vel/gains after Y (they share the host link; Y gates everything)
    TSNET_CUDA(cudaStreamWaitEvent(ss->copy, ss->y_in, 0));
    for (int k = 0; k < chunks; ++k) {   // in processing order (last chunk first, below)
        const int c = chunks - 1 - k;
        const size_t o = 2 * (size_t)rows(c), cb = sizeof(float2) * (size_t)(rows(c + 1) - rows(c));
        TSNET_CUDA(cudaMemcpyAsync(dV + rows(c), vel_host + o, cb, cudaMemcpyHostToDevice, ss->copy));
        TSNET_CUDA(cudaMemcpyAsync(dG + rows(c), gains_host + o, cb, cudaMemcpyHostToDevice, ss->copy));
        TSNET_CUDA(cudaEventRecord(ss->state_in[c], ss->copy));
    }
    Ws w;
    GradArgs a;
    int st = prepare(P, reinterpret_cast<float*>(dY), gp, nullptr, ws, ws_bytes, w, a);
    if (st != TSNET_OK) return st;
    cudaStream_t fs = ss->side;
    TSNET_CUDA(cudaStreamWaitEvent(fs, ss->y_in, 0));
    TSNET_CUDA(launch_field_local(w, a, fs, false));
    TSNET_CUDA(launch_field_conv(w, a, fs));
    TSNET_CUDA(cudaMemsetAsync(w.f_attr, 0, b, s));
    // last chunk first: chunks have equal nnz, so the first rows (hubs of a
    // power-law graph) form the chunk with the fewest rows -- processed last,
    // its download is the short tail that nothing overlaps
    for (int k = 0; k < chunks; ++k) {
        const int c = chunks - 1 - k;
        const int64_t r0 = rows(c), r1 = rows(c + 1);
        cudaStream_t sa = s;
        TSNET_CUDA(launch_spmv_rows(w, a, r0, r1, cut_nnz[c + 1] - cut_nnz[c], sa));
        TSNET_CUDA(cudaEventRecord(ss->attr_done[c], sa));
        TSNET_CUDA(cudaStreamWaitEvent(fs, ss->attr_done[c], 0));
        TSNET_CUDA(cudaStreamWaitEvent(fs, ss->state_in[c], 0));
        TSNET_CUDA(launch_update_rows(w, a, r0, r1, dYn, dV, dG, *sp, fs));
        TSNET_CUDA(cudaEventRecord(ss->moved[c], fs));
        TSNET_CUDA(cudaStreamWaitEvent(ss->d2h, ss->moved[c], 0));
        const size_t o = 2 * (size_t)r0, cb = sizeof(float2) * (size_t)(r1 - r0);
        TSNET_CUDA(cudaMemcpyAsync(Y_host + o, dYn + r0, cb, cudaMemcpyDeviceToHost, ss->d2h));
        TSNET_CUDA(cudaMemcpyAsync(vel_host + o, dV + r0, cb, cudaMemcpyDeviceToHost, ss->d2h));
        TSNET_CUDA(cudaMemcpyAsync(gains_host + o, dG + r0, cb, cudaMemcpyDeviceToHost, ss->d2h));
    }
    TSNET_CUDA(cudaEventRecord(ss->drained, ss->d2h));
    TSNET_CUDA(cudaStreamWaitEvent(s, ss->drained, 0));
    TSNET_CUDA(cudaStreamSynchronize(s));
    return TSNET_OK;
}

}  // namespace tsnet

extern "C" {

int tsnet_step_host(const tsnet_csr* P, float* Y_host, float* vel_host, float* gains_host,
                    const tsnet_grad_params* gp, const tsnet_step_params* sp, const tsnet_shard* shard, void* ws,
                    size_t ws_bytes, tsnet_stream_t stream) {
    TSNET_ARG(P != nullptr && gp != nullptr, "P or params NULL");
    Ws w0 = ws_map(ws, P->n, P->nnz, (gp->I_max >= 1 && gp->I_max <= TSNET_I_MAX_LIMIT) ? gp->I_max : 1);
    TSNET_ARG(ws != nullptr && ws_bytes >= w0.bytes, "workspace too small");
    const int64_t n = P->n;
    if (n == 0) return TSNET_OK;
    TSNET_ARG(Y_host && vel_host && gains_host, "host state arrays are NULL");
    cudaStream_t s = (cudaStream_t)stream;
    float2* dY = w0.state;
    float2* dV = w0.state + n;
    float2* dG = w0.state + 2 * n;
    const size_t b = sizeof(float2) * (size_t)n;
    // Y first (the field phase and the SpMV need it); velocity and gains are only
    // read by the move, so they upload on a copy stream under the field + SpMV
    SideStream* ss = nullptr;
    TSNET_CUDA(side_stream(ss));
    TSNET_CUDA(cudaEventRecord(ss->fork, s));                  // after the previous work on s
    const int chunks = host_chunks(n);
    if (chunks > 1 && sp != nullptr && !sp->recenter && P->plan == nullptr && !sharded(shard, n) &&
        (shard == nullptr || shard->comm == nullptr)) {
        TSNET_CUDA(cudaStreamWaitEvent(ss->side, ss->fork, 0));
        TSNET_CUDA(cudaStreamWaitEvent(ss->copy, ss->fork, 0));
        return step_host_pipelined(P, Y_host, vel_host, gains_host, gp, sp, ws, ws_bytes, s, ss, chunks, w0.state);
    }
    TSNET_CUDA(cudaStreamWaitEvent(ss->copy, ss->fork, 0));
    TSNET_CUDA(cudaMemcpyAsync(dY, Y_host, b, cudaMemcpyHostToDevice, s));
    TSNET_CUDA(cudaMemcpyAsync(dV, vel_host, b, cudaMemcpyHostToDevice, ss->copy));
    TSNET_CUDA(cudaMemcpyAsync(dG, gains_host, b, cudaMemcpyHostToDevice, ss->copy));
    TSNET_CUDA(cudaEventRecord(ss->copied, ss->copy));
    int st = step_impl(P, reinterpret_cast<float*>(dY), reinterpret_cast<float*>(dV), reinterpret_cast<float*>(dG),
                       gp, sp, shard, ws, ws_bytes, s, ss->copied);
    if (st != TSNET_OK) return st;
    TSNET_CUDA(cudaMemcpyAsync(Y_host, dY, b, cudaMemcpyDeviceToHost, s));
    TSNET_CUDA(cudaMemcpyAsync(vel_host, dV, b, cudaMemcpyDeviceToHost, s));
    TSNET_CUDA(cudaMemcpyAsync(gains_host, dG, b, cudaMemcpyDeviceToHost, s));
    TSNET_CUDA(cudaStreamSynchronize(s));
    return TSNET_OK;
}

int tsnet_grad_tree(const tsnet_csr* P, const float* Y, const tsnet_grad_params* gp, double theta, int32_t variant,
                    float* grad, double* Z_out, void* ws, size_t ws_bytes, void* tree_ws, size_t tree_ws_bytes,
                    tsnet_stream_t stream) {
    Ws w;
    GradArgs a;
    int st = prepare(P, Y, gp, nullptr, ws, ws_bytes, w, a);
    if (st != TSNET_OK) return st;
    TSNET_ARG(grad != nullptr, "grad is NULL");
    if (a.n == 0) return TSNET_OK;
    return tree_gradient(w, a, theta, variant, reinterpret_cast<float2*>(grad), Z_out, tree_ws, tree_ws_bytes,
                         (cudaStream_t)stream);
}

int tsnet_cost(const tsnet_csr* P, const float* Y, const tsnet_grad_params* gp, int32_t mode, const tsnet_shard* shard,
               double* out3, void* ws, size_t ws_bytes, tsnet_stream_t stream) {
    Ws w;
    GradArgs a;
    int st = prepare(P, Y, gp, shard, ws, ws_bytes, w, a);
    if (st != TSNET_OK) return st;
    TSNET_ARG(mode == 0 || mode == 1, "cost mode must be 0 (exact) or 1 (interpolated)");
    TSNET_ARG(!sharded(shard, a.n), "tsnet_cost is single-GPU only");
    TSNET_ARG(out3 != nullptr, "out3 is NULL");
    cudaStream_t s = (cudaStream_t)stream;
    if (a.n == 0) {
        TSNET_CUDA(cudaMemsetAsync(out3, 0, 3 * sizeof(double), s));
        return TSNET_OK;
    }
    if (mode == 1) {
        TSNET_CUDA(launch_field_phase(w, a, s));
        TSNET_CUDA(launch_entropy_sum(w, a, s));
    }
    TSNET_CUDA(launch_cost(w, a, mode, out3, s));
    return TSNET_OK;
}

int tsnet_read_stats(const void* ws, tsnet_stats* out, tsnet_stream_t stream) {
    TSNET_ARG(ws != nullptr && out != nullptr, "NULL argument");
    Geo g;
    cudaStream_t s = (cudaStream_t)stream;
    TSNET_CUDA(cudaMemcpyAsync(&g, ws, sizeof(Geo), cudaMemcpyDeviceToHost, s));
    TSNET_CUDA(cudaStreamSynchronize(s));
    out->Z = g.Z;
    out->lo_x = g.lo_x;
    out->lo_y = g.lo_y;
    out->S = g.S;
    out->h_b = g.h_b;
    out->I = g.I;
    out->N = g.N;
    out->M = g.M;
    out->nonfinite = g.nonfinite;
    out->spread = g.smode == kSpreadRuns ? TSNET_SPREAD_RUNS : TSNET_SPREAD_SORT;
    out->spread_points = (int64_t)g.spts;
    out->spread_flushes = (int64_t)g.sflush;
    return g.nonfinite ? TSNET_E_NONFINITE : TSNET_OK;
}

}  // extern "C"
