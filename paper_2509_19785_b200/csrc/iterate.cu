// iterate.cu -- the attractive SpMV (a6) and the gather/assemble/update (a7)
// of one L-tsNET iteration.
//
// a6  F_attr,i = sum_{j in row i} p_ij w_ij (X_i - X_j),  w = 1/(1 + r^2)
//     (Eq. 6 first term, "analogous to attraction forces"; the
//     sparse P of C0).  HBM-bound: 8 B per stored entry.
// a7  grad_i = 4 lambda_kl F_attr,i + f_field,i + (lambda_c / n) X_i  with
//     f_field gathered from the convolved grid (field.cu), followed by the
//     momentum/gains move (reading R12).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "move.cuh"
#include "ptx.cuh"

namespace tsnet {

constexpr double kHubFactor = 4.0; // hot-column L1 policy threshold (k_spmv2)

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int ld_stream_i32(const int32_t* a, uint64_t pol) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_stream_f32(const float* a, uint64_t pol) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
    return v;
}

// Largest r in [0, n) with indptr[r] <= e (indptr[0] = 0 <= e < indptr[n]),
// 32-ary search by one warp.
__device__ __forceinline__ int64_t warp_row_of(const int64_t* __restrict__ indptr, int64_t n, int64_t e) {
    const int lane = threadIdx.x & 31;
    int64_t lo = 0, hi = n;
    while (hi - lo > 1) {
        const int64_t step = (hi - lo + 31) / 32;
        const int64_t p = lo + lane * step;
        const bool pred = (p < hi) && (__ldg(indptr + p) <= e);
        const unsigned m = __ballot_sync(0xffffffffu, pred);
        const int L = 31 - __clz(m);
        lo = lo + L * step;
        hi = std::min(lo + step, hi);
    }
    return lo;
}

// Row-wise CSR SpMV with the next row's first batch prefetched while the
// current row is gathered and reduced (so a row's HBM stream overlaps the
// previous row's L2 gathers), U entries per lane per batch, CHUNK entries per
// warp work item.  Rows entirely inside the chunk are stored, the two rows a
// chunk may share with its neighbours use vector atomics (F zeroed first).
template <int U>
__device__ __forceinline__ void spmv2_load(const int32_t* __restrict__ indices, const float* __restrict__ values,
                                           int64_t s0, int64_t s1, int lane, int (&col)[U], float (&val)[U],
                                           int fill, uint64_t pol) {
#pragma unroll
    for (int q = 0; q < U; ++q) {
        const int64_t e = s0 + lane + 32 * q;
        const bool ok = e < s1;
        col[q] = ok ? ld_stream_i32(indices + e, pol) : fill;
        val[q] = ok ? ld_stream_f32(values + e, pol) : 0.f;
    }
}

__device__ __forceinline__ float2 ld_y_keep(const float2* a) {
    float2 v;
    asm volatile("ld.global.nc.L1::evict_last.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(a));
    return v;
}
__device__ __forceinline__ float2 ld_y_pass(const float2* a) {
    float2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(a));
    return v;
}

// HUB: columns below `hub` are kept in L1 (evict_last) and the others bypass
// it, so the hot lines are not flushed by the stream of one-off gathers
// (hub_columns() decides when)
template <int U, bool HUB>
__device__ __forceinline__ void spmv2_acc(const float2* __restrict__ Y, float2 yi, const int (&col)[U],
                                          const float (&val)[U], float& fx, float& fy, int hub) {
    float2 yj[U];
    if (HUB) {
#pragma unroll
        for (int q = 0; q < U; ++q) yj[q] = col[q] < hub ? ld_y_keep(Y + col[q]) : ld_y_pass(Y + col[q]);
    } else {
#pragma unroll
        for (int q = 0; q < U; ++q) yj[q] = __ldg(Y + col[q]);
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
        const float dx = yi.x - yj[q].x, dy = yi.y - yj[q].y;
        float w;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(w) : "f"(fmaf(dx, dx, fmaf(dy, dy, 1.0f))));
        const float pw = val[q] * w;
        fx = fmaf(pw, dx, fx);
        fy = fmaf(pw, dy, fy);
    }
}

// Rows [rb, re): the stored entries indptr[rb] .. indptr[re] are cut into
// chunks; F holds rows rb.. (F[r - rb]).
template <int U, bool HUB>
__global__ void __launch_bounds__(256) k_spmv2(int64_t rb, int64_t re_rows, const int64_t* __restrict__ indptr,
                                               const int32_t* __restrict__ indices, const float* __restrict__ values,
                                               const float2* __restrict__ Y, float2* __restrict__ F, int cpw,
                                               int hub) {
    const int lane = threadIdx.x & 31;
    const int64_t e_begin = __ldg(indptr + rb), e_end = __ldg(indptr + re_rows);
    const int64_t nwarps_total = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // every warp gets exactly cpw chunks (no tail wave): chunk length from the range
    const int64_t CHUNK = std::max<int64_t>(
        1024, (((e_end - e_begin + nwarps_total * cpw - 1) / (nwarps_total * cpw)) + 255) & ~int64_t(255));
    const int64_t nchunks = (e_end - e_begin + CHUNK - 1) / CHUNK;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t pol = policy_evict_first();
    F -= rb;
    for (int64_t c = wid; c < nchunks; c += nw) {
        const int64_t cs = e_begin + c * CHUNK, ce = std::min(cs + CHUNK, e_end);
        // row containing entry cs: largest r in [rb, re) with indptr[r] <= cs
        int64_t r = rb + warp_row_of(indptr + rb, re_rows - rb, cs);
        int64_t rs = cs;                                  // current row segment [rs, re)
        int64_t re = std::min(__ldg(indptr + r + 1), ce);
        int col[U];
        float val[U];
        spmv2_load<U>(indices, values, rs, std::min(re, rs + 32 * U), lane, col, val, (int)r, pol);
        while (true) {
            const bool more = re < ce;                    // a next row starts inside the chunk
            int64_t r2 = r + 1, rs2 = re, re2 = re;
            int col2[U];
            float val2[U];
            if (more) {
                re2 = std::min(__ldg(indptr + r2 + 1), ce);
                spmv2_load<U>(indices, values, rs2, std::min(re2, rs2 + 32 * U), lane, col2, val2, (int)r2, pol);
            }
            const float2 yi = __ldg(Y + r);
            float fx = 0.f, fy = 0.f;
            spmv2_acc<U, HUB>(Y, yi, col, val, fx, fy, hub);
            for (int64_t b = rs + 32 * U; b < re; b += 32 * U) {   // long rows: further batches
                int cb[U];
                float vb[U];
                spmv2_load<U>(indices, values, b, re, lane, cb, vb, (int)r, pol);
                spmv2_acc<U, HUB>(Y, yi, cb, vb, fx, fy, hub);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                fx += __shfl_xor_sync(0xffffffffu, fx, o);
                fy += __shfl_xor_sync(0xffffffffu, fy, o);
            }
            if (lane == 0) {
                // rows starting before the chunk or ending after it are shared
                const bool shared = (rs == cs && __ldg(indptr + r) < cs) || re == ce;
                if (shared) atomicAdd(F + r, make_float2(fx, fy));
                else F[r] = make_float2(fx, fy);
            }
            if (!more) break;
            r = r2;
            rs = rs2;
            re = re2;
#pragma unroll
            for (int q = 0; q < U; ++q) {
                col[q] = col2[q];
                val[q] = val2[q];
            }
        }
    }
}

// Launch configuration of the row-wise kernel: the measured best on B200
// (round-1 sweeps of entries per lane, chunks per warp, CTAs
// per SM, waves and the hot-column candidate set, profiles/r1*).
constexpr int kSpmvU = 4;           // entries per lane per batch
constexpr int kSpmvCtasPerSm = 5;   // 256-thread CTAs per SM
constexpr int kSpmvWaves = 16;      // CTAs = waves x resident: short CTAs balance the power-law rows
                                    // dynamically (cfg 4 kernel 0.83 -> 0.80 ms vs one wave)
constexpr int kSpmvHubCols = 8192;  // hot-column L1 policy candidate (hub_columns() decides per P):
                                    // cfg 4 kernel 0.792 -> 0.769 ms (r1cg)

// Hot-column L1 policy for this P: on when its first `cand` columns (P is
// symmetric: column count = row length) hold >= kHubFactor x their share of
// the stored entries -- a power-law graph numbered by weight (cfg 4: 10% of
// the entries in the first 8192 columns, 12x their share; meshes, block
// models and random numberings stay off).  Decided once per (P, n, nnz) (three
// indptr reads on `s`, cached per thread); never inside a stream capture (then
// off until an eager call).
static int hub_columns(const GradArgs& a, int cand, cudaStream_t s) {
    if (cand <= 0 || cand >= a.n) return 0;
    struct Entry {
        const void* indptr = nullptr;
        int64_t n = -1, nnz = -1;
        int dev = -1, hub = 0;
    };
    static thread_local Entry cache[4];
    static thread_local int next = 0;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    for (const auto& e : cache)
        if (e.indptr == a.indptr && e.n == a.n && e.nnz == a.nnz && e.dev == dev) return e.hub;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return 0;
    int64_t v[3] = {0, 0, 0};
    if (cudaMemcpyAsync(&v[0], a.indptr, sizeof(int64_t), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(&v[1], a.indptr + cand, sizeof(int64_t), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(&v[2], a.indptr + a.n, sizeof(int64_t), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return 0;
    const double share = (double)(v[1] - v[0]) / (double)std::max<int64_t>(1, v[2] - v[0]);
    Entry& e = cache[next++ & 3];
    e.indptr = a.indptr;
    e.n = a.n;
    e.nnz = a.nnz;
    e.dev = dev;
    e.hub = share >= kHubFactor * (double)cand / (double)a.n ? cand : 0;
    return e.hub;
}

// Attributes are set on every launch (cheap; per device, no process-wide flags).
template <bool HUB>
static cudaError_t launch_spmv2_h(const GradArgs& a, float2* F, int cpw, int hub, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(k_spmv2<kSpmvU, HUB>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    if (e != cudaSuccess) return e;
    int resident = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, k_spmv2<kSpmvU, HUB>, 256, 0) != cudaSuccess ||
        resident < 1)
        resident = 1;
    // `waves` x the resident CTAs, each warp `cpw` equal chunks (the hardware
    // scheduler balances the CTAs); small problems: fewer CTAs so that chunks
    // stay >= 1024 entries
    const int64_t want = std::max<int64_t>(1, a.nnz / (1024 * 8 * cpw));
    const int per_sm = std::min(kSpmvCtasPerSm, resident);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)kNumSMs * per_sm * kSpmvWaves));
    k_spmv2<kSpmvU, HUB><<<blocks, 256, 0, s>>>(a.rb, a.re, a.indptr, a.indices, a.values, a.Y, F, cpw, hub);
    return cudaGetLastError();
}

static cudaError_t launch_spmv2(const GradArgs& a, float2* F, int cpw, cudaStream_t s) {
    const int hub = hub_columns(a, kSpmvHubCols, s);
    return hub > 0 ? launch_spmv2_h<true>(a, F, cpw, hub, s) : launch_spmv2_h<false>(a, F, cpw, 0, s);
}

// a6 for the rows [rb, re) of the call into w.f_attr (local rows): the
// plan kernel when P has a plan (column-blocked or sliced ELL), else the
// row-wise CSR kernel.
cudaError_t launch_spmv(const Ws& w, const GradArgs& a, cudaStream_t s) {
    if (a.plan && a.plan_kind == TSNET_PLAN_SELL) return launch_attr_sell(a.plan, a.Y, w.f_attr, a.re - a.rb, s);
    if (a.plan) return launch_attr_cb(a.plan, a.Y, w.f_attr, a.re - a.rb, s);   // rows of the plan's shard
    const int64_t nl = a.re - a.rb;
    cudaError_t e = cudaMemsetAsync(w.f_attr, 0, sizeof(float2) * (size_t)nl, s);
    if (e != cudaSuccess || a.nnz == 0 || nl == 0) return e;
    return launch_spmv2(a, w.f_attr, 1, s);
}

// gather (a7) and the gains/momentum move: move.cuh

// mode 0: write grad; mode 1: write f_field (and F_attr stays in ws)
// n = rows of this call (local); cn = lambda_c / n_global
__global__ void __launch_bounds__(256) k_grad_out(int64_t n, const Geo* __restrict__ gp, const float4* __restrict__ fgrid,
                                                  const float2* __restrict__ Y, const float2* __restrict__ Fa,
                                                  float lambda_kl, float cn, float2* __restrict__ grad,
                                                  float2* __restrict__ f_field) {
    const Geo g = *gp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 y = Y[i];
        int b;
        float2 u;
        box_of(y, g.lo_x, g.lo_y, g.h_b, g.inv_h, g.I, b, u.x, u.y);
        const float2 ff = gather_field(g, fgrid, b, u);
        if (f_field) f_field[i] = ff;
        if (grad) {
            const float2 fa = Fa[i];
            grad[i] = make_float2(fmaf(4.0f * lambda_kl, fa.x, ff.x) + cn * y.x,
                                  fmaf(4.0f * lambda_kl, fa.y, ff.y) + cn * y.y);
        }
    }
}

// n = rows of this call (local; Y, vel, gains point at the first own row); cn = lambda_c / n_global.
// SMEM: the field grid (N^2 float4) fits the launch's dynamic shared memory
// (grid_cap float4) and each CTA stages it first -- the 7 record loads per point
// then cost no L2 requests; else (large grids, I > 42, N > 126) the 112-byte box
// records are read through L1 by a launch without shared memory
// (the whole L1 caches the grid).  Both variants are launched each iteration
// (N is only known on the device); the one that does not apply exits at once.
constexpr int kUpdateThreads = 1024;
constexpr int kUpdateThreadsG = 256;
constexpr int kGridSmemCells = 12800;   // 200 KB of float4
// V points per thread and iteration (their loads in flight together); RECOMPUTE:
// the box and in-box coordinates from the position (as k_box_count) instead of
// reading them back (12 B/point less traffic, some fp64 arithmetic more)
template <int V, bool RECOMPUTE, bool SMEM>
__global__ void __launch_bounds__(SMEM ? kUpdateThreads : kUpdateThreadsG, SMEM ? 1 : 4) k_update(int64_t n, Geo* __restrict__ gp,
                                                              const float4* __restrict__ fgrid,
                                                              const int* __restrict__ box, const float2* __restrict__ uv,
                                                              const float2* Yin, float2* Yout,
                                                              const float2* __restrict__ Fa,
                                                              float2* __restrict__ vel, float2* __restrict__ gains,
                                                              float lambda_kl, float cn, tsnet_step_params sp,
                                                              int grid_cap, PeerPush push, int64_t row0) {
    extern __shared__ float4 fsm[];
    const Geo g = *gp;
    const int cells = g.I * g.I * kBoxRec;     // float4 of the box records (move.cuh)
    if (SMEM != (cells <= grid_cap)) return;   // the other variant handles this grid size
    unsigned long long iter = 0;
    if (push.y) {
        // multi-GPU layout push: store into a peer's Y only once that peer has
        // finished reading Y for this iteration (its field + SpMV)
        iter = push.own[kFIter];
        if (threadIdx.x < push.world)
            wait_peer_counter(push.flags[threadIdx.x] + kFRead, iter + 1);
        __syncthreads();
    }
    const float4* fg = fgrid;
    if (SMEM) {
        // the whole grid (N^2 float4, contiguous) in one TMA bulk copy
        __shared__ __align__(8) uint64_t gbar;
        if (threadIdx.x == 0) {
            mbar_init(&gbar, 1);
            fence_mbar_init();
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t bytes = (uint32_t)(sizeof(float4) * (size_t)cells);
            mbar_arrive_tx(&gbar, bytes);
            bulk_g2s(fsm, fgrid, bytes, &gbar);
        }
        mbar_wait(&gbar, 0);
        fg = fsm;
    }
    double sx = 0.0, sy = 0.0;
    bool bad = false;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += V * stride) {
        int b[V];
        float2 u[V], y[V], fa[V], v[V], gn[V];
#pragma unroll
        for (int q = 0; q < V; ++q) {
            const int64_t i = i0 + q * stride;
            const bool h = i < n;
            if (!RECOMPUTE) {
                b[q] = h ? box[i] : 0;
                u[q] = h ? uv[i] : make_float2(0.5f, 0.5f);
            }
            y[q] = h ? Yin[i] : make_float2(0.f, 0.f);
            fa[q] = h ? Fa[i] : make_float2(0.f, 0.f);
            v[q] = h ? vel[i] : make_float2(0.f, 0.f);
            gn[q] = h ? gains[i] : make_float2(1.f, 1.f);
        }
        if (RECOMPUTE) {
#pragma unroll
            for (int q = 0; q < V; ++q) box_of(y[q], g.lo_x, g.lo_y, g.h_b, g.inv_h, g.I, b[q], u[q].x, u[q].y);
        }
#pragma unroll
        for (int q = 0; q < V; ++q) {
            const int64_t i = i0 + q * stride;
            if (i >= n) break;
            const float2 ff = gather_field<!SMEM>(g, fg, b[q], u[q]);
            const float gx = fmaf(4.0f * lambda_kl, fa[q].x, ff.x) + cn * y[q].x;
            const float gy = fmaf(4.0f * lambda_kl, fa[q].y, ff.y) + cn * y[q].y;
            gains_move(gx, v[q].x, gn[q].x, y[q].x, sp);
            gains_move(gy, v[q].y, gn[q].y, y[q].y, sp);
            bad |= !(isfinite(y[q].x) && isfinite(y[q].y));
            Yout[i] = y[q];
            vel[i] = v[q];
            gains[i] = gn[q];
            if (push.y)
                for (int r = 0; r < push.world; ++r)
                    if (r != push.self) push.y[r][row0 + i] = y[q];   // over NVLink
            if (sp.recenter) {
                sx += y[q].x;
                sy += y[q].y;
            }
        }
    }
    if (sp.recenter) {
        for (int o = 16; o > 0; o >>= 1) {
            sx += __shfl_xor_sync(0xffffffffu, sx, o);
            sy += __shfl_xor_sync(0xffffffffu, sy, o);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(&gp->sum_x, sx);
            atomicAdd(&gp->sum_y, sy);
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&gp->nonfinite, 1);
    if (push.y) {
        // the last block to finish publishes "moved t + 1" at system scope
        // after every block's peer stores (fenced before its ticket)
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned long long tk = atomicAdd(push.own + kFTicket, 1ull);
            if (tk == gridDim.x - 1ull) {
                push.own[kFTicket] = 0ull;
                push.own[kFIter] = iter + 1;
                __threadfence_system();
                st_release_sys(push.own + kFMoved, iter + 1);
            }
        }
    }
}

__global__ void k_recenter(int64_t n, const Geo* __restrict__ gp, float2* __restrict__ Y) {
    const float mx = (float)(gp->sum_x / (double)n), my = (float)(gp->sum_y / (double)n);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float2 y = Y[i];
        Y[i] = make_float2(y.x - mx, y.y - my);
    }
}

static int pts_blocks(int64_t n) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)kNumSMs * 8));
}

static float cn_of(const GradArgs& a) { return (float)((double)a.lambda_c / (double)a.n); }

// grad / f_field: (re - rb) x 2, row q = global row rb + q
cudaError_t launch_grad_out(const Ws& w, const GradArgs& a, float2* grad, float2* f_field, double* Z,
                            cudaStream_t s) {
    const int64_t nl = a.re - a.rb;
    k_grad_out<<<pts_blocks(nl), 256, 0, s>>>(nl, w.geo, w.fgrid, a.Y + a.rb, w.f_attr, a.lambda_kl,
                                              cn_of(a), grad, f_field);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (Z) e = cudaMemcpyAsync(Z, &w.geo->Z, sizeof(double), cudaMemcpyDeviceToDevice, s);
    return e;
}

// The move: 2 points per thread, box and in-box coordinates recomputed from
// the position (the chunk-local spread, k_spread_local, does not store them).
static constexpr auto update_kernel = k_update<2, true, true>;
static constexpr auto update_kernel_g = k_update<2, true, false>;

// Y, vel, gains: full n x 2 arrays; rows [rb, re) are updated
cudaError_t launch_update(const Ws& w, const GradArgs& a, float2* Y, float2* vel, float2* gains,
                          const tsnet_step_params& sp, cudaStream_t s, const PeerPush& push) {
    const int64_t nl = a.re - a.rb;
#ifndef MOVE_SMEM_MAX_CELLS   // probe builds: the largest grid the move stages in shared memory
#define MOVE_SMEM_MAX_CELLS kGridSmemCells
#endif
    const int cap = (int)std::min<int64_t>((int64_t)w.I_max * w.I_max * kBoxRec, MOVE_SMEM_MAX_CELLS);
    const size_t smem = sizeof(float4) * (size_t)cap;
    cudaError_t ea = cudaFuncSetAttribute(update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)(sizeof(float4) * kGridSmemCells));
    if (ea != cudaSuccess) return ea;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((nl + kUpdateThreads - 1) / kUpdateThreads, kNumSMs));
    update_kernel<<<blocks, kUpdateThreads, smem, s>>>(nl, w.geo, w.fgrid, w.box, nullptr, Y + a.rb, Y + a.rb, w.f_attr,
                                                  vel + a.rb, gains + a.rb, a.lambda_kl, cn_of(a), sp, cap, push,
                                                  a.rb);
    const int blocks_g =
        (int)std::max<int64_t>(1, std::min<int64_t>((nl + 2 * kUpdateThreadsG - 1) / (2 * kUpdateThreadsG), kNumSMs * 8));
    update_kernel_g<<<blocks_g, kUpdateThreadsG, 0, s>>>(nl, w.geo, w.fgrid, w.box, nullptr, Y + a.rb, Y + a.rb, w.f_attr,
                                                         vel + a.rb, gains + a.rb, a.lambda_kl, cn_of(a), sp, cap,
                                                         push, a.rb);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || !sp.recenter) return e;
    k_recenter<<<pts_blocks(a.n), 256, 0, s>>>(a.n, w.geo, Y);
    return cudaGetLastError();
}

cudaError_t launch_spmv_rows(const Ws& w, const GradArgs& a, int64_t r0, int64_t r1, int64_t nnz_rows,
                             cudaStream_t s) {
    if (a.plan || r0 < a.rb || r1 > a.re || r0 > r1) return cudaErrorInvalidValue;
    const int64_t nc = r1 - r0;
    float2* F = w.f_attr + (r0 - a.rb);     // zeroed by the caller (rows split across warps add)
    if (a.nnz == 0 || nc == 0) return cudaSuccess;
    GradArgs b = a;
    b.rb = r0;
    b.re = r1;
    b.nnz = std::max<int64_t>(1, nnz_rows);     // sizes the grid
    return launch_spmv2(b, F, 1, s);
}

cudaError_t launch_update_rows(const Ws& w, const GradArgs& a, int64_t r0, int64_t r1, float2* Yout, float2* vel,
                               float2* gains, const tsnet_step_params& sp, cudaStream_t s) {
    if (sp.recenter || r0 < a.rb || r1 > a.re || r0 > r1) return cudaErrorInvalidValue;
    const int64_t nc = r1 - r0, q = r0 - a.rb;
    if (nc == 0) return cudaSuccess;
    // no shared-memory grid here: this move runs beside the SpMV of the next
    // chunk, whose CTAs run with the whole L1 carveout (a 200 KB shared-memory
    // CTA would wait for an idle SM); the field nodes are read through L1/L2
    const int blocks =
        (int)std::max<int64_t>(1, std::min<int64_t>((nc + 2 * kUpdateThreadsG - 1) / (2 * kUpdateThreadsG), kNumSMs * 8));
    update_kernel_g<<<blocks, kUpdateThreadsG, 0, s>>>(nc, w.geo, w.fgrid, w.box + q, nullptr, a.Y + r0, Yout + r0,
                                               w.f_attr + q, vel + r0, gains + r0, a.lambda_kl, cn_of(a), sp, 0,
                                               PeerPush{}, 0);
    return cudaGetLastError();
}

}  // namespace tsnet
