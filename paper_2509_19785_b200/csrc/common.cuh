// common.cuh -- internal helpers of libtsnet (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstddef>

#include "../../include/tsnet.h"

namespace tsnet {

constexpr int kWarp = 32;
constexpr int kNumSMs = 148;     // B200; launch geometry only, never correctness

// ------------------------------------------------------------------ errors
void set_error(const char* fmt, ...);

#define TSNET_CUDA(call)                                                                  \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            ::tsnet::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
            return TSNET_E_CUDA;                                                          \
        }                                                                                 \
    } while (0)

#define TSNET_LAUNCH_CHECK()                                                              \
    do {                                                                                  \
        cudaError_t e_ = cudaGetLastError();                                              \
        if (e_ != cudaSuccess) {                                                          \
            ::tsnet::set_error("%s:%d kernel launch: %s", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            return TSNET_E_CUDA;                                                          \
        }                                                                                 \
    } while (0)

#define TSNET_ARG(cond, ...)                                                              \
    do {                                                                                  \
        if (!(cond)) {                                                                    \
            ::tsnet::set_error(__VA_ARGS__);                                              \
            return TSNET_E_ARG;                                                           \
        }                                                                                 \
    } while (0)

// ------------------------------------------------------- per-iteration geometry
// Lives in the workspace header; written by the bbox kernel's last block,
// read by every later kernel of the iteration (no host round trip).
struct Geo {
    double lo_x, lo_y, S, h_b, delta;  // fp64: box assignment matches the fp64 definition (R16)
    double inv_h;                      // 1 / h_b (move.cuh: box_of)
    double zacc;                       // Parseval accumulator  <W1, K1 * W1> * M^2
    double Z;                          // Z = zacc / M^2 - n
    int I, N, M, nrad;
    unsigned long long plan;           // FFT plan for length M: stage s radix = ((plan >> 2s) & 3) + 2
    int pad0;
    int nonfinite;
    unsigned int ticket;               // last-block-done counter of the bbox kernel
    unsigned bbox[4];                  // ~u(min x), ~u(min y), u(max x), u(max y); 0 = empty (field.cu)
    double sum_x, sum_y;               // centroid accumulation (recenter)
    double eacc;                       // cost mode 1: Parseval accumulator <W1, K_ln * W1> * M^2
    // a1/a2 path of this iteration (field.cu, k_bbox decides): kSpreadSort (box
    // counting sort + spread, which also records the box order `perm`) or
    // kSpreadRuns (one pass over the points in the last recorded box order)
    int smode;
    int sruns;                         // consecutive runs-path iterations so far
    int sskip;                         // sorts still to do before the runs path is tried again
    int sfail;                         // consecutive failed first runs (the backoff doubles)
    long long perm_n;                  // points of the recorded box order (0: none)
    unsigned long long spts;           // runs path: points spread by the last iteration
    unsigned long long sflush;         // runs path: box flushes of the last iteration
};
constexpr int kSpreadSort = 0, kSpreadRuns = 1;

// Ordered float <-> int (monotone), for atomicMin/atomicMax on floats.
__device__ __forceinline__ int f2o(float f) {
    int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float o2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }

// ------------------------------------------------------------ workspace map
struct Ws {
    Geo* geo;
    float2* f_attr;      // n
    float2* f_field;     // n (grad_parts only)
    int* box;            // n   box id of each point
    int* rank;           // n   rank of the point inside its box
    int* perm;           // n   the points in box order (k_box_scatter), visited by k_spread_runs
    int* box_cnt;        // I_max^2 + 1
    int* box_start;      // I_max^2 + 1
    float4* wgrid;       // N_max^2 spread charges (W1, Mx, My, 0), row-major [gy][gx]
    float2* tw;          // M_max twiddles exp(-2 pi i k / M)
    float2* spec;        // 10 * (M_max/2+1) * M_max : forward row spectra, [a][kx][y]
    float2* colout;      // 6 * (M_max/2+1) * N_max  : after column pass, [b][kx][y]
    float4* fgrid;       // I_max^2 box records of kBoxRec float4 (P0, R_x, R_y of the 9 nodes; move.cuh)
    float2* state;       // 4 n : host-facing step staging (Y, vel, gains, next Y)
    float2* ynext;       // n   : new positions of the fused SpMV + move (sliced-ELL plan)
    double* cost;        // scratch for tsnet_cost (4 doubles)
    int64_t n, nnz;
    int I_max, N_max, M_max;
    size_t bytes;
};


inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Computes the map; base == nullptr only sizes it.
inline Ws ws_map(void* base, int64_t n, int64_t nnz, int I_max) {
    Ws w{};
    w.n = n;
    w.nnz = nnz;
    w.I_max = I_max;
    w.N_max = 3 * I_max;
    w.M_max = 6 * I_max;
    const int64_t nb = (int64_t)I_max * I_max + 1;
    const int64_t half = w.M_max / 2 + 1;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off = align_up(off + bytes, 256);
        return (char*)base + o;
    };
    w.geo = (Geo*)take(sizeof(Geo));
    w.f_attr = (float2*)take(sizeof(float2) * n);
    w.f_field = (float2*)take(sizeof(float2) * n);
    w.box = (int*)take(sizeof(int) * n);
    w.rank = (int*)take(sizeof(int) * n);
    w.perm = (int*)take(sizeof(int) * n);
    w.box_cnt = (int*)take(sizeof(int) * nb);
    w.box_start = (int*)take(sizeof(int) * nb);
    w.wgrid = (float4*)take(sizeof(float4) * (size_t)w.N_max * w.N_max);
    w.tw = (float2*)take(sizeof(float2) * w.M_max);
    w.spec = (float2*)take(sizeof(float2) * 10 * half * (size_t)w.M_max);
    w.colout = (float2*)take(sizeof(float2) * 6 * half * (size_t)w.N_max);
    w.fgrid = (float4*)take(sizeof(float4) * (size_t)w.N_max * w.N_max);
    w.state = (float2*)take(sizeof(float2) * 4 * n);
    w.ynext = (float2*)take(sizeof(float2) * n);
    w.cost = (double*)take(sizeof(double) * 8);
    w.bytes = off;
    return w;
}

// ------------------------------------------------------------ launchers
// (defined in the .cu files; all enqueue on `s`, return cudaError_t of launch)
struct GradArgs {
    int64_t n, nnz;       // global vertex count and stored entries of P
    int64_t rb, re;       // rows owned by this call (shard), [0, n) on one GPU
    const int64_t* indptr;
    const int32_t* indices;
    const float* values;
    const void* plan;     // re-laid-out P (attr_cb.cu / attr_sell.cu) or nullptr
    int plan_kind;        // TSNET_PLAN_CB / TSNET_PLAN_SELL (with a plan)
    const float2* Y;
    float lambda_kl, lambda_c, lambda_r, eps, h_max;
    int I_min, I_max;
    int spread;           // tsnet_grad_params.spread: 0 adaptive, 1 box sort, 2 index runs
};

cudaError_t launch_field_phase(const Ws& w, const GradArgs& a, cudaStream_t s);
cudaError_t launch_field_local(const Ws& w, const GradArgs& a, cudaStream_t s, bool zero_all);
cudaError_t launch_field_conv(const Ws& w, const GradArgs& a, cudaStream_t s);
cudaError_t launch_spmv(const Ws& w, const GradArgs& a, cudaStream_t s);
cudaError_t launch_attr_cb(const void* plan, const float2* Y, float2* F, int64_t nl, cudaStream_t s);
cudaError_t launch_attr_sell(const void* plan, const float2* Y, float2* F, int64_t nl, cudaStream_t s);
// step a7 fused into the sliced-ELL SpMV (attr_sell.cu); pointers index the
// plan's rows (row r at r - row_begin)
// Multi-GPU layout push (comm.cu, tsnet_comm_layout): the move stores each
// new position into every peer's replicated Y.  y[r] = rank r's Y buffer as
// mapped here, flags[r] = rank r's exchange flags, own = this rank's flags;
// y == nullptr: no push.
struct PeerPush {
    float2* const* y = nullptr;
    unsigned long long* const* flags = nullptr;
    unsigned long long* own = nullptr;
    int world = 0, self = 0;
};
constexpr int kFRead = 2, kFMoved = 3, kFTicket = 4, kFIter = 5;   // exchange flag words
PeerPush comm_peer_push(void* comm, int64_t n);
bool comm_owns_layout(const void* comm, const float* Y, int64_t n);
cudaError_t comm_y_enter(void* comm, cudaStream_t s);
cudaError_t comm_y_read_done(void* comm, cudaStream_t s);

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Wait until *p >= v (a peer's counter, system scope).  A peer that never
// arrives (its process died) would hang the device forever: after kPeerWaitNs
// the kernel traps instead, so the host sees a CUDA error on its next call.
constexpr unsigned long long kPeerWaitNs = 60ull * 1000000000ull;
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void wait_peer_counter(const unsigned long long* p, unsigned long long v) {
    if (ld_acquire_sys(p) >= v) return;
    const unsigned long long t0 = global_ns();
    while (ld_acquire_sys(p) < v) {
        __nanosleep(64);
        if (global_ns() - t0 > kPeerWaitNs) __trap();
    }
}

struct SellMoveArgs {
    Geo* geo;
    const float4* fgrid;
    const int* box;
    const float2* uv;
    float2* Ynew;
    float2* vel;
    float2* gains;
    float lambda_kl, cn;
    tsnet_step_params sp;
};
cudaError_t launch_grad_out(const Ws& w, const GradArgs& a, float2* grad, float2* f_field, double* Z,
                            cudaStream_t s);
cudaError_t launch_update(const Ws& w, const GradArgs& a, float2* Y, float2* vel, float2* gains,
                          const tsnet_step_params& sp, cudaStream_t s, const PeerPush& push = PeerPush{});
// Row-chunk pieces of the same two steps (rows [r0, r1) inside the call's [rb, re)),
// used by the pipelined host step: the SpMV of a chunk (its rows of w.f_attr
// must be zero before the call; nnz_rows = its stored entries, which size the
// grid), and the move of a chunk
// reading a.Y and writing the new positions to Yout (never a.Y: the other chunks'
// SpMV still gathers the old positions).  No recentring.
cudaError_t launch_spmv_rows(const Ws& w, const GradArgs& a, int64_t r0, int64_t r1, int64_t nnz_rows,
                             cudaStream_t s);
cudaError_t launch_update_rows(const Ws& w, const GradArgs& a, int64_t r0, int64_t r1, float2* Yout, float2* vel,
                               float2* gains, const tsnet_step_params& sp, cudaStream_t s);
cudaError_t launch_cost(const Ws& w, const GradArgs& a, int mode, double* out3, cudaStream_t s);
// quadtree gradient of BH-tsNET (variant 0) / FIt-tsNET (variant 1), tree.cu
int tree_gradient(const Ws& w, const GradArgs& a, double theta, int variant, float2* grad, double* Z_out,
                  void* tws, size_t tws_bytes, cudaStream_t s);
cudaError_t launch_entropy_sum(const Ws& w, const GradArgs& a, cudaStream_t s);

}  // namespace tsnet
