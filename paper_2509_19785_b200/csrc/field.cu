// field.cu -- the FFT-accelerated interpolation phase of one L-tsNET iteration
// (FIt-SNE interpolation; Alg. 3 l.397-400 and l.403,
// PAPER.md:397-403; entropy kernel K_e = 1/(eps + r^2)).
//
// Steps, all device-driven (no host round trip):
//   a0 k_bbox                 bounding box -> grid geometry (I, h_b, N = 3I, M = 6I, FFT plan)
//   a1 k_box_count/k_box_scan/k_box_scatter  counting sort of the points by box into
//                             the box order `perm` (the scan zeroes the box counters for
//                             the next iteration); run only on the sort path
//   a2 k_spread_runs          box-local charges W1 and local moments M_x, M_y over the
//                             points in box order (register runs, 9 vector reds per run);
//                             also writes the twiddles of length M
//   a3/a4 k_row_fwd, k_col, k_row_inv   kernel tabulation + 2-D FFT convolution
//                             (rows -> columns with products -> inverse rows)
//   a5 Z by Parseval inside k_col (fp64 accumulation)
// Output: fgrid = one 112-byte record per box, box-major (box (gx / 3, gy / 3)
// at (gy / 3) I + gx / 3; node k = 3 (gy % 3) + gx % 3 holds P0, R_x = Qx - s_a h P0
// and R_y = Qy - s_c h P0 at floats k, 9 + k, 18 + k: move.cuh), with the combined kernel
//   C = alpha K2 + beta K_e,  alpha = -4 lambda_kl / Z,  beta = -lambda_r / n^2,
//   P0 = C * W1,  Qx = (D_x C) * W1 + C * M_x,  Qy = (D_y C) * W1 + C * M_y,
// so that for a point in box (bx, by) with in-box coordinates (u_x, u_y):
//   f_field = sum_{a,b} L_a(u_x) L_b(u_y) [ (X - t_ab) P0 + Q ]
//           = -4 lambda_kl F_rep + lambda_r g_ent   (local-moment form).
#include "common.cuh"
#include "fft.cuh"
#include "move.cuh"

namespace tsnet {

// Lagrange basis on the nodes s_t = (t + 1/2)/3 of one interval.
__device__ __forceinline__ void lagrange3(float u, float (&L)[3]) {
    const float s0 = 1.0f / 6.0f, s1 = 0.5f, s2 = 5.0f / 6.0f;
    L[0] = 4.5f * (u - s1) * (u - s2);
    L[1] = -9.0f * (u - s0) * (u - s2);
    L[2] = 4.5f * (u - s0) * (u - s1);
}

__device__ __forceinline__ bool is5smooth(int m) {
    while (m % 2 == 0) m /= 2;
    while (m % 3 == 0) m /= 3;
    while (m % 5 == 0) m /= 5;
    return m == 1;
}

// Bounding-box accumulators whose all-zero state means "empty", so a zeroed
// workspace needs no initialisation kernel: max as the monotone unsigned key
// u(x), min as ~u(x); both reduced with atomicMax.
__device__ __forceinline__ unsigned bb_key(float x) { return (unsigned)f2o(x) ^ 0x80000000u; }
__device__ __forceinline__ float bb_val(unsigned u) { return o2f((int)(u ^ 0x80000000u)); }

// The field chain's kernels are launched with programmatic stream serialization
// (FIELD_PDL, on; 0 = plain launches, the probe baseline): a kernel's CTAs may become resident while its
// predecessor still runs; each waits here for the predecessor to complete (and
// its writes to be visible) before it touches memory, then lets its own
// successor's CTAs in.  Every kernel of the chain calls it first, also on the
// paths that exit at once, so completion stays transitive along the chain.
#ifndef FIELD_PDL
#define FIELD_PDL 1
#endif
__device__ __forceinline__ void chain_wait() {
#if FIELD_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
template <typename... KArgs, typename... Args>
static cudaError_t launch_chain(void (*k)(KArgs...), int grid, int block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = FIELD_PDL ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, KArgs(args)...);
}

// a0: bounding box of Y and, in the last block, the grid geometry (R9).
constexpr int kBBoxPts = 8;
#ifndef RUNS_RESORT       // probe builds (scripts/tile_variants.sh SRC=field): the re-sort threshold
#define RUNS_RESORT 16
#endif
constexpr int kRunsResort = RUNS_RESORT;   // adaptive spread: re-sort when flushes * this > points
constexpr int kRunsBackoff = 8;            // sorts before retrying the runs after a failed first run (doubling)
//
// The CTAs also zero the charge grid cells the previous iteration used
// ([0, N_prev^2), N_prev read before the last block sets the new geometry;
// every reader of that grid has run).  No kernel writes beyond the live cells
// of its iteration and a fresh workspace is zero, so the whole grid is zero
// when the spread starts, whatever N this iteration takes.  The last block also
// picks the a1/a2 path (kSpreadSort / kSpreadRuns) from the request `spread`
// (tsnet_grad_params.spread) and, when adaptive, from the previous
// iteration's measure (k_box_count / k_spread_runs).
__global__ void __launch_bounds__(256) k_bbox(const float2* __restrict__ Y, int64_t n, Geo* g, float h_max,
                                              int I_min, int I_max, float4* __restrict__ wgrid, int spread) {
    {
        const int64_t prev = (int64_t)g->N * g->N;
        for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < prev; c += (int64_t)gridDim.x * blockDim.x)
            wgrid[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    bool bad = false;
    // kBBoxPts points per thread and sweep, their loads in flight together (a
    // grid of 4 CTAs per SM: 4 same-address atomics per CTA below)
    const int64_t sweep = (int64_t)gridDim.x * blockDim.x * kBBoxPts;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x * kBBoxPts + threadIdx.x; i0 < n; i0 += sweep) {
        float2 y[kBBoxPts];
#pragma unroll
        for (int j = 0; j < kBBoxPts; ++j) {
            const int64_t i = i0 + (int64_t)j * blockDim.x;
            y[j] = i < n ? __ldg(Y + i) : make_float2(NAN, NAN);
        }
#pragma unroll
        for (int j = 0; j < kBBoxPts; ++j) {
            if (i0 + (int64_t)j * blockDim.x >= n) break;
            bad |= !(isfinite(y[j].x) && isfinite(y[j].y));
            mnx = fminf(mnx, y[j].x);
            mny = fminf(mny, y[j].y);
            mxx = fmaxf(mxx, y[j].x);
            mxy = fmaxf(mxy, y[j].y);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        mnx = fminf(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
        mny = fminf(mny, __shfl_xor_sync(0xffffffffu, mny, o));
        mxx = fmaxf(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
        mxy = fmaxf(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
    }
    bad = __any_sync(0xffffffffu, bad);
    __shared__ float s[4][8];
    __shared__ int sbad;
    __shared__ bool last;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (threadIdx.x == 0) sbad = 0;
    __syncthreads();
    if (l == 0) {
        s[0][w] = mnx; s[1][w] = mny; s[2][w] = mxx; s[3][w] = mxy;
        if (bad) atomicOr(&sbad, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
            mnx = fminf(mnx, s[0][k]); mny = fminf(mny, s[1][k]);
            mxx = fmaxf(mxx, s[2][k]); mxy = fmaxf(mxy, s[3][k]);
        }
        if (n > 0) {
            atomicMax(&g->bbox[0], ~bb_key(mnx));
            atomicMax(&g->bbox[1], ~bb_key(mny));
            atomicMax(&g->bbox[2], bb_key(mxx));
            atomicMax(&g->bbox[3], bb_key(mxy));
        }
        if (sbad) atomicOr(&g->nonfinite, 1);
        __threadfence();
        unsigned int t = atomicAdd(&g->ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    // ---- geometry (fp64, identical to the oracle's definition) ----
    volatile unsigned* bb = g->bbox;
    double lo_x = (double)bb_val(~bb[0]), lo_y = (double)bb_val(~bb[1]);
    double hi_x = (double)bb_val(bb[2]), hi_y = (double)bb_val(bb[3]);
    // reset the per-iteration accumulators for the next call (this block runs
    // after every other block's atomics; zacc / sums are accumulated later)
    bb[0] = 0u;
    bb[1] = 0u;
    bb[2] = 0u;
    bb[3] = 0u;
    g->ticket = 0u;
    g->zacc = 0.0;
    g->sum_x = 0.0;
    g->sum_y = 0.0;
    {
        int mode;
        if (spread == TSNET_SPREAD_SORT) {
            mode = kSpreadSort;
        } else if (spread == TSNET_SPREAD_RUNS) {
            mode = kSpreadRuns;
        } else if (g->smode == kSpreadRuns) {   // re-sort once a run averages < kRunsResort points
            mode = g->sflush * (unsigned long long)kRunsResort > g->spts ? kSpreadSort : kSpreadRuns;
            // the order was already too stale one iteration after a sort (the
            // layout moves fast): sort for the next kRunsBackoff iterations,
            // twice as many after each further failed first run (up to 8x)
            if (mode == kSpreadSort && g->sruns <= 1) {
                g->sfail = min(g->sfail + 1, 4);
                g->sskip = kRunsBackoff << (g->sfail - 1);
            } else if (mode == kSpreadRuns) {
                g->sfail = 0;
            }
        } else if (g->sskip > 0) {
            --g->sskip;
            mode = kSpreadSort;
        } else {                                // a fresh box order: runs
            mode = g->perm_n > 0 ? kSpreadRuns : kSpreadSort;
        }
        g->sruns = mode == kSpreadRuns ? g->sruns + 1 : 0;
        g->smode = mode;
        g->spts = 0ull;
        g->sflush = 0ull;
    }
    double S = fmax(hi_x - lo_x, hi_y - lo_y);
    if (!(S >= 1e-12)) S = 1e-12;            // also catches NaN (non-finite layouts)
    if (!isfinite(S) || !isfinite(lo_x) || !isfinite(lo_y)) {
        g->nonfinite = 1;
        S = 1.0; lo_x = 0.0; lo_y = 0.0;
    }
    double q = ceil(S / (double)h_max);
    double qc = fmin(fmax(q, (double)I_min), (double)I_max);
    int I = (int)qc;
    int Iu = I;
    while (!is5smooth(Iu)) ++Iu;
    if (Iu > I_max) {
        Iu = I_max;
        while (!is5smooth(Iu)) --Iu;
    }
    I = Iu;
    g->lo_x = lo_x;
    g->lo_y = lo_y;
    g->S = S;
    g->I = I;
    g->h_b = S / (double)I;
    g->delta = g->h_b / 3.0;
    g->inv_h = 1.0 / g->h_b;
    g->N = 3 * I;
    g->M = 6 * I;
    int m = 6 * I, nr = 0;
    unsigned long long plan = 0ull;
    const int rads[4] = {4, 2, 3, 5};
    for (int q = 0; q < 4; ++q)
        while (m % rads[q] == 0) {
            plan |= (unsigned long long)(rads[q] - 2) << (2 * nr++);
            m /= rads[q];
        }
    g->plan = plan;
    g->nrad = nr;
}

// a1: box of every point (fp64 arithmetic, R16) and its rank inside the box.
// Each CTA takes kBoxChunk consecutive points (kBoxPts per thread, loads of
// all of them in flight together).  When the I^2 box counters fit in shared
// memory (kBoxSmem), the CTA counts its chunk there (shared atomics, native
// on sm_100), reserves one range per non-empty box with a single global
// atomicAdd, and adds that offset to the local ranks it kept in registers --
// so a layout packed into a few boxes (stage A: 1e6 points in <= 400 boxes)
// does not serialise on global atomics, and box/rank are written once.
// Otherwise (many boxes, little contention) global atomics per point.  The
// order of points inside a box is not deterministic (neither is the fp32
// spread that follows).
constexpr int kBoxSmem = 4096;     // counters (16 KB): I <= 64
constexpr int kBoxPts = 8;         // points per thread
constexpr int kBoxChunk = 256 * kBoxPts;

// box_of (the box of a point and its in-box coordinates): move.cuh

// The CTAs also zero the live charge grid (N^2 cells; every reader of the
// previous iteration's grid has run) and write the twiddles of length M (what
// a separate preparation kernel did); the box counters were zeroed by the
// previous k_box_scan (or are zero in a fresh workspace).
__device__ __forceinline__ void write_twiddles(const Geo* __restrict__ g, float2* __restrict__ tw) {
    const int M = g->M;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < M; k += gridDim.x * blockDim.x) {
        double sn, cs;
        sincospi(-2.0 * (double)k / (double)M, &sn, &cs);
        tw[k] = make_float2((float)cs, (float)sn);
    }
}

// Sort path only (exits at once on the runs path).  The CTAs also write the
// box counters were zeroed by the previous k_box_scan (or are zero in a fresh
// workspace).
__global__ void __launch_bounds__(256, 4) k_box_count(const float2* __restrict__ Y, int64_t n, Geo* __restrict__ g,
                                                   int* __restrict__ box_cnt, int* __restrict__ box,
                                                   int* __restrict__ rank) {
    chain_wait();
    __shared__ int hist[kBoxSmem];
    if (g->smode != kSpreadSort) return;
    const double lo_x = g->lo_x, lo_y = g->lo_y, h_b = g->h_b, inv_h = g->inv_h;
    const int I = g->I;
    const int nb = I * I;
    const bool local = nb <= kBoxSmem;
    const int64_t c0 = (int64_t)blockIdx.x * kBoxChunk + threadIdx.x;
    if (local) {
        for (int q = threadIdx.x; q < nb; q += blockDim.x) hist[q] = 0;
        __syncthreads();
    }
    int* cnt = local ? hist : box_cnt;
    float2 y[kBoxPts];
#pragma unroll
    for (int j = 0; j < kBoxPts; ++j) {
        const int64_t i = c0 + (int64_t)j * 256;
        y[j] = i < n ? Y[i] : make_float2(0.f, 0.f);
    }
    int bj[kBoxPts], rj[kBoxPts];
#pragma unroll
    for (int j = 0; j < kBoxPts; ++j) {
        const int64_t i = c0 + (int64_t)j * 256;
        bj[j] = -1;
        rj[j] = 0;
        if (i < n) {
            float ux, uy;
            box_of(y[j], lo_x, lo_y, h_b, inv_h, I, bj[j], ux, uy);
            rj[j] = atomicAdd(&cnt[bj[j]], 1);
        }
    }
    if (local) {
        __syncthreads();
        for (int q = threadIdx.x; q < nb; q += blockDim.x) {
            const int c = hist[q];
            if (c) hist[q] = atomicAdd(&box_cnt[q], c);   // this CTA's range inside box q
        }
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < kBoxPts; ++j) {
        const int64_t i = c0 + (int64_t)j * 256;
        if (i < n) {
            box[i] = bj[j];
            rank[i] = rj[j] + (local ? hist[bj[j]] : 0);
        }
    }
}

// a1: exclusive scan of box counts -> box_start.  Single CTA of 1024 threads.
__global__ void __launch_bounds__(1024) k_box_scan(Geo* g, int* __restrict__ box_cnt, int* __restrict__ box_start,
                                                   int64_t n) {
    chain_wait();
    if (g->smode != kSpreadSort) return;
    const int nb = g->I * g->I;
    const int T = blockDim.x;
    const int per = (nb + T - 1) / T;
    const int b0 = threadIdx.x * per, b1 = min(nb, b0 + per);
    int cs = 0;
    for (int b = b0; b < b1; ++b) cs += box_cnt[b];
    __shared__ int sc[1024];
    sc[threadIdx.x] = cs;
    __syncthreads();
    for (int o = 1; o < T; o <<= 1) {            // Hillis-Steele inclusive scan
        const int a = threadIdx.x >= o ? sc[threadIdx.x - o] : 0;
        __syncthreads();
        sc[threadIdx.x] += a;
        __syncthreads();
    }
    int run = sc[threadIdx.x] - cs;
    for (int b = b0; b < b1; ++b) {
        const int c = box_cnt[b];
        box_cnt[b] = 0;                                // zero for the next iteration's count
        box_start[b] = run;
        run += c;
    }
    if (threadIdx.x == T - 1) box_start[nb] = (int)n;
}

// the box order of the points: perm[box_start[b] + rank] = i.  4 points per
// thread and iteration: their loads, then the box_start gathers, then the
// stores, each in flight together
__global__ void __launch_bounds__(256) k_box_scatter(Geo* __restrict__ g, int64_t n, const int* __restrict__ box,
                                                     const int* __restrict__ rank, const int* __restrict__ box_start,
                                                     int* __restrict__ perm) {
    chain_wait();
    constexpr int V = 4;
    if (g->smode != kSpreadSort) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) g->perm_n = n;   // the box order of these n points
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += V * stride) {
        int b[V], r[V], st[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int64_t i = i0 + v * stride;
            b[v] = i < n ? box[i] : 0;
            r[v] = i < n ? rank[i] : 0;
        }
#pragma unroll
        for (int v = 0; v < V; ++v) st[v] = __ldg(box_start + b[v]);
#pragma unroll
        for (int v = 0; v < V; ++v)
            if (i0 + v * stride < n) perm[st[v] + r[v]] = (int)(i0 + v * stride);
    }
}

__device__ __forceinline__ void red_add_v4(float4* addr, float a, float b, float c) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(0.0f)
                 : "memory");
}

// a1 + a2 in one pass over the points in the box order the last sort recorded
// (perm; the index order when there is none): the points have moved little
// since, so most consecutive points of that order still share a box.  Any
// order gives the same sums; the order only decides how often a run breaks.
// Every iteration: on the sort path right after the sort (a fresh order: a run
// only ends where the box does), on the runs path over an order a few
// iterations old.
// A warp takes chunks of 32 kRunPts consecutive positions of the order, lane l
// the kRunPts positions from l kRunPts on.  A lane sums the charges of its points in 27
// registers (9 nodes x (W1, M_x, M_y)) while the box stays the
// same, and adds them to the grid (9 red.global.add.v4) when the box changes;
// at the end of the chunk the lanes' last runs are summed across lanes by a
// segmented warp scan keyed on the box (a run continuing into the next lane's
// points joins it), and the last lane of each segment adds the sum.  The same
// sums as the box sort, in another fp32 order.  The CTAs also
// write the twiddles; per CTA the box flushes are counted for the next
// iteration's path choice (k_bbox).
#ifndef RUNS_PTS
#define RUNS_PTS 8
#endif
constexpr int kRunPts = RUNS_PTS;
__device__ __forceinline__ void runs_flush(float4* __restrict__ wgrid, int b, int I, int N, float h_b,
                                           const float (&acc)[27]) {
    const int bx = b % I, by = b / I;
#pragma unroll
    for (int t = 0; t < 9; ++t) {
        const int gx = 3 * bx + t % 3, gy = 3 * by + t / 3;
        red_add_v4(&wgrid[(int64_t)gy * N + gx], acc[3 * t], acc[3 * t + 1] * h_b, acc[3 * t + 2] * h_b);
    }
}

// the charges of one point on the 9 nodes of its box b
__device__ __forceinline__ void runs_point(float4* __restrict__ wgrid, int b, int I, int N, float h_b, float ux,
                                           float uy) {
    const float dx[3] = {1.0f / 6.0f - ux, 0.5f - ux, 5.0f / 6.0f - ux};
    const float dy[3] = {1.0f / 6.0f - uy, 0.5f - uy, 5.0f / 6.0f - uy};
    const float Lx[3] = {4.5f * dx[1] * dx[2], -9.0f * dx[0] * dx[2], 4.5f * dx[0] * dx[1]};
    const float Ly[3] = {4.5f * dy[1] * dy[2], -9.0f * dy[0] * dy[2], 4.5f * dy[0] * dy[1]};
    const int bx = b % I, by = b / I;
#pragma unroll
    for (int bb = 0; bb < 3; ++bb)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float w = Lx[a] * Ly[bb];
            red_add_v4(&wgrid[(int64_t)(3 * by + bb) * N + 3 * bx + a], w, w * dx[a] * h_b, w * dy[bb] * h_b);
        }
}

constexpr int kStrayCap = 2048;   // per CTA (16 B each)

#ifndef RUNS_MINB
#define RUNS_MINB 3
#endif
#ifndef RUNS_PIPE         // probe builds: the next chunk's order entries / positions loaded under this chunk's work
#define RUNS_PIPE 0
#endif
// the order entries (or indices) of a lane's kRunPts positions from base
__device__ __forceinline__ void runs_idx(const int* __restrict__ perm, bool ordered, int64_t base, int64_t n,
                                         int (&idx)[kRunPts]) {
    if (ordered) {
#pragma unroll
        for (int v = 0; v < kRunPts; ++v) idx[v] = __ldg(perm + min(base + v, n - 1));
    } else {
#pragma unroll
        for (int v = 0; v < kRunPts; ++v) idx[v] = (int)min(base + v, n - 1);
    }
}
__global__ void __launch_bounds__(256, RUNS_MINB) k_spread_runs(const float2* __restrict__ Y, int64_t n, Geo* __restrict__ g,
                                                     const int* __restrict__ perm, float4* __restrict__ wgrid,
                                                     float2* __restrict__ tw) {
    chain_wait();
    __shared__ unsigned s_flush;
    __shared__ int s_nstray;
    __shared__ int4 s_stray[kStrayCap];    // (box, u_x, u_y) of points outside their lane's run
    const bool ordered = g->perm_n == n;
    write_twiddles(g, tw);
    if (threadIdx.x == 0) {
        s_flush = 0u;
        s_nstray = 0;
    }
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) g->spts = (unsigned long long)n;
    const double lo_x = g->lo_x, lo_y = g->lo_y, h_b = g->h_b, inv_h = g->inv_h;
    const int I = g->I, N = g->N;
    const float h_bf = (float)h_b;
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    unsigned flushes = 0u;
    const int64_t cfirst = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
#if RUNS_PIPE
    float2 y[kRunPts];
    if (cfirst * (32 * kRunPts) < n) {
        int idx[kRunPts];
        runs_idx(perm, ordered, cfirst * (32 * kRunPts) + (int64_t)lane * kRunPts, n, idx);
#pragma unroll
        for (int v = 0; v < kRunPts; ++v) y[v] = __ldg(Y + idx[v]);
    }
#endif
    for (int64_t c = cfirst; c * (32 * kRunPts) < n; c += warps) {
        const int64_t base = c * (32 * kRunPts) + (int64_t)lane * kRunPts;
#if RUNS_PIPE
        // the next chunk's order entries now (they land under this chunk's
        // accumulation), its positions after the accumulation (under the reduction)
        const int64_t c1 = c + warps;
        const bool more = c1 * (32 * kRunPts) < n;
        int idx1[kRunPts];
        if (more) runs_idx(perm, ordered, c1 * (32 * kRunPts) + (int64_t)lane * kRunPts, n, idx1);
#else
        // all kRunPts order entries, then all kRunPts gathers, in flight together
        // (branch-free: positions past n read the last point and are masked below)
        int idx[kRunPts];
        runs_idx(perm, ordered, base, n, idx);
        float2 y[kRunPts];
#pragma unroll
        for (int v = 0; v < kRunPts; ++v) y[v] = __ldg(Y + idx[v]);
#endif
        float acc[27];
#pragma unroll
        for (int q = 0; q < 27; ++q) acc[q] = 0.f;
        int cur = -1;
#pragma unroll
        for (int v = 0; v < kRunPts; ++v) {
            if (base + v < n) {
                int b;
                float ux, uy;
                box_of(y[v], lo_x, lo_y, h_b, inv_h, I, b, ux, uy);
                if (cur < 0) cur = b;          // the lane's run: the box of its first point
                bool stray = b != cur;
                if (stray) {
                    // a point outside the run (it crossed a box boundary since
                    // the sort, or the order moves on to the next box): kept for
                    // the CTA's stray pass below, so the warp does not diverge
                    // into a flush here
                    ++flushes;
                    const int slot = atomicAdd(&s_nstray, 1);
                    if (slot < kStrayCap) s_stray[slot] = make_int4(b, __float_as_int(ux), __float_as_int(uy), 0);
                    else runs_point(wgrid, b, I, N, h_bf, ux, uy);
                    ux = 0.5f;                 // contributes nothing to the run below
                    uy = 0.5f;
                }
                const float keep = stray ? 0.f : 1.f;
                // offsets to the 3 nodes per axis, Lagrange weights from them
                const float dx0 = 1.0f / 6.0f - ux, dx1 = 0.5f - ux, dx2 = 5.0f / 6.0f - ux;
                const float dy0 = 1.0f / 6.0f - uy, dy1 = 0.5f - uy, dy2 = 5.0f / 6.0f - uy;
                const float Lx[3] = {4.5f * dx1 * dx2, -9.0f * dx0 * dx2, 4.5f * dx0 * dx1};
                const float Ly[3] = {4.5f * dy1 * dy2, -9.0f * dy0 * dy2, 4.5f * dy0 * dy1};
                const float dx[3] = {dx0, dx1, dx2}, dy[3] = {dy0, dy1, dy2};
#pragma unroll
                for (int bb = 0; bb < 3; ++bb)
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const float w = Lx[a] * (Ly[bb] * keep);
                        const int q = 3 * (3 * bb + a);
                        acc[q] += w;
                        acc[q + 1] = fmaf(w, dx[a], acc[q + 1]);
                        acc[q + 2] = fmaf(w, dy[bb], acc[q + 2]);
                    }
            }
        }
#if RUNS_PIPE
        if (more) {
#pragma unroll
            for (int v = 0; v < kRunPts; ++v) y[v] = __ldg(Y + idx1[v]);
        }
#endif
        __syncwarp();
        // segmented inclusive scan over the lanes, segments = equal boxes
        // (lanes without points: key -1 - lane, a segment of their own)
        const int key = cur >= 0 ? cur : -1 - lane;
        const int kp = __shfl_up_sync(full, key, 1);
        const int kn = __shfl_down_sync(full, key, 1);
        if (__all_sync(full, kp == key || lane == 0)) {
            // one segment (the common case): butterfly sums, lane t adds node t
#pragma unroll
            for (int q = 0; q < 27; ++q)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(full, acc[q], o);
            if (cur >= 0 && lane < 9) {
                float a0 = 0.f, a1 = 0.f, a2 = 0.f;
#pragma unroll
                for (int t = 0; t < 9; ++t)
                    if (t == lane) {
                        a0 = acc[3 * t];
                        a1 = acc[3 * t + 1];
                        a2 = acc[3 * t + 2];
                    }
                const int bx = cur % I, by = cur / I;
                red_add_v4(&wgrid[(int64_t)(3 * by + lane / 3) * N + 3 * bx + lane % 3], a0, a1 * h_bf, a2 * h_bf);
                if (lane == 0) ++flushes;
            }
        } else {
            bool head = lane == 0 || kp != key;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const bool uh = __shfl_up_sync(full, head, o);
#pragma unroll
                for (int q = 0; q < 27; ++q) {
                    const float u = __shfl_up_sync(full, acc[q], o);
                    if (lane >= o && !head) acc[q] += u;
                }
                if (lane >= o) head = head || uh;
            }
            if (cur >= 0 && (lane == 31 || kn != key)) {
                runs_flush(wgrid, cur, I, N, h_bf, acc);
                ++flushes;
            }
        }
    }
    flushes = __reduce_add_sync(full, flushes);
    if (lane == 0 && flushes) atomicAdd(&s_flush, flushes);
    __syncthreads();
    // the strays, one per thread
    const int ns = min(s_nstray, kStrayCap);
    for (int t = threadIdx.x; t < ns; t += blockDim.x) {
        const int4 e = s_stray[t];
        runs_point(wgrid, e.x, I, N, h_bf, __int_as_float(e.y), __int_as_float(e.z));
    }
    if (threadIdx.x == 0 && s_flush) atomicAdd(&g->sflush, (unsigned long long)s_flush);
}

// ---------------------------------------------------------------- FFT passes
constexpr int kRowThreads = 512;
constexpr int kInvThreads = 256;
constexpr int kColThreads = 512;
constexpr int kMfast = 1536;   // M = 6 I <= 1536 (I <= 256): every pass keeps all its transforms in shared memory
// Shared memory of each pass, in float2, for grids up to M_max: the fast
// layout for M <= kMfast, else one transform (plus twiddles and scratch) at a
// time, 3 M floats2 (M = 6144 at I = 1024: 147 KB).  The passes read the cap
// and pick the batch size from the run-time M.
static int smem_cap_row(int M_max) { return std::max(11 * std::min(M_max, kMfast), 3 * M_max); }
static int smem_cap_col(int M_max) { return std::max(17 * std::min(M_max, kMfast), 3 * M_max); }
static int smem_cap_inv(int M_max) { return std::max(5 * std::min(M_max, kMfast), 3 * M_max); }
// transforms per batch for a pass needing tw (M) + buf (B M) + scratch (B M)
__device__ __forceinline__ int fft_batch(int cap, int M, int want) {
    return max(1, min(want, (cap / M - 1) / 2));
}
// spectra layout: array a, column kx, row y  ->  spec[(a * half_max + kx) * M_max + y]

// a3 + first half of a4: per row y of the M x M circulant grid, build the 10
// real arrays (3 charges, 7 kernel tables), FFT them along x in 5 packed
// complex transforms (in batches that fit the shared memory), unpack to half
// spectra and store transposed.
//   arrays: 0 W1, 1 Mx, 2 My, 3 K1, 4 K2, 5 Ke, 6 DxK2, 7 DxKe, 8 DyK2, 9 DyKe
__global__ void __launch_bounds__(kRowThreads, 1) k_row_fwd(const Geo* __restrict__ gp, const float4* __restrict__ wgrid,
                                                         const float2* __restrict__ twg, float2* __restrict__ spec,
                                                         int M_max, float eps, int cap) {
    chain_wait();
    extern __shared__ float2 sm[];
    const int M = gp->M, N = gp->N, half = M / 2 + 1, nrad = gp->nrad;
    const int B = fft_batch(cap, M, 5);
    float2* tw = sm;                      // M
    float2* buf = sm + M;                 // B M
    float2* scr = buf + B * M;            // B M
    const unsigned long long plan = gp->plan;
    const int half_max = M_max / 2 + 1;
    const double dlt = gp->delta;
    for (int k = threadIdx.x; k < M; k += blockDim.x) tw[k] = twg[k];
    // Rows y < N only (M = 2N): the charges are zero in rows y >= N, and the
    // kernel tables there are those of row M - y mirrored in dy -- even (K1,
    // K2, K_e, D_x K2, D_x K_e: the same row spectrum) or odd (D_y K2, D_y K_e:
    // negated) -- so the spectra of rows N+1 .. M-1 are written from rows
    // M-y without their FFTs; row N (|dy| = N) is zero.
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < 10 * half; t += gridDim.x * blockDim.x)
        spec[((int64_t)(t / half) * half_max + t % half) * M_max + N] = make_float2(0.f, 0.f);
    for (int y = blockIdx.x; y < N; y += gridDim.x) {
        const int dy = y;
        const bool ky = true;                        // |dy| <= N - 1
        for (int p0 = 0; p0 < 5; p0 += B) {
            const int nb = min(B, 5 - p0);
            for (int x = threadIdx.x; x < M; x += blockDim.x) {
                const int dx = (x <= M / 2) ? x : x - M;
                float4 wv = make_float4(0.f, 0.f, 0.f, 0.f);
                if (y < N && x < N) wv = wgrid[(int64_t)y * N + x];
                float k1 = 0.f, k2 = 0.f, ke = 0.f, dxk2 = 0.f, dxke = 0.f, dyk2 = 0.f, dyke = 0.f;
                if (ky && dx < N && -dx < N) {
                    const double ox = dx * dlt, oy = dy * dlt;
                    const double r2 = ox * ox + oy * oy;
                    const double K1 = 1.0 / (1.0 + r2), K2 = K1 * K1, Ke = 1.0 / ((double)eps + r2);
                    k1 = (float)K1; k2 = (float)K2; ke = (float)Ke;
                    dxk2 = (float)(ox * K2); dxke = (float)(ox * Ke);
                    dyk2 = (float)(oy * K2); dyke = (float)(oy * Ke);
                }
                const float2 pk[5] = {make_float2(wv.x, wv.y), make_float2(wv.z, k1), make_float2(k2, ke),
                                      make_float2(dxk2, dxke), make_float2(dyk2, dyke)};
                for (int q = 0; q < nb; ++q) buf[q * M + x] = pk[p0 + q];
            }
            __syncthreads();
            fft_block(buf, scr, M, nb, M, plan, nrad, tw, false);
            // unpack z = A + iB:  A_k = (Z_k + conj Z_{M-k}) / 2,  B_k = -i (Z_k - conj Z_{M-k}) / 2
            for (int t = threadIdx.x; t < nb * half; t += blockDim.x) {
                const int q = t / half, k = t - q * half, p = p0 + q;
                const float2 Zk = buf[q * M + k];
                const float2 Zm = cconj(buf[q * M + (k == 0 ? 0 : M - k)]);
                const float2 A = make_float2(0.5f * (Zk.x + Zm.x), 0.5f * (Zk.y + Zm.y));
                const float2 D = make_float2(0.5f * (Zk.x - Zm.x), 0.5f * (Zk.y - Zm.y));
                const float2 Bv = mul_mi(D);
                spec[((int64_t)(2 * p) * half_max + k) * M_max + y] = A;
                spec[((int64_t)(2 * p + 1) * half_max + k) * M_max + y] = Bv;
                if (y > 0) {
                    // row M - y: arrays 0-2 (charges) zero, 3-7 even, 8-9 odd in dy
                    const int a0 = 2 * p, a1 = 2 * p + 1;
                    const float s0 = a0 <= 2 ? 0.f : (a0 >= 8 ? -1.f : 1.f);
                    const float s1 = a1 <= 2 ? 0.f : (a1 >= 8 ? -1.f : 1.f);
                    spec[((int64_t)a0 * half_max + k) * M_max + (M - y)] = make_float2(s0 * A.x, s0 * A.y);
                    spec[((int64_t)a1 * half_max + k) * M_max + (M - y)] = make_float2(s1 * Bv.x, s1 * Bv.y);
                }
            }
            __syncthreads();
        }
    }
}

// Kernel-charge products of one frequency k (10 spectra in, 6 out) and the
// Parseval term of Z:
//   A0 = K2 W1, Ax = DxK2 W1 + K2 Mx, Ay = DyK2 W1 + K2 My   (alpha part)
//   B0 = Ke W1, Bx = DxKe W1 + Ke Mx, By = DyKe W1 + Ke My   (beta part)
__device__ __forceinline__ double col_products(const float2 (&v)[10], float2 (&o)[6]) {
    const float2 W1 = v[0], Mx = v[1], My = v[2], K1 = v[3], K2 = v[4], Ke = v[5];
    const float2 DxK2 = v[6], DxKe = v[7], DyK2 = v[8], DyKe = v[9];
    o[0] = cmul(K2, W1);
    o[1] = cadd(cmul(DxK2, W1), cmul(K2, Mx));
    o[2] = cadd(cmul(DyK2, W1), cmul(K2, My));
    o[3] = cmul(Ke, W1);
    o[4] = cadd(cmul(DxKe, W1), cmul(Ke, Mx));
    o[5] = cadd(cmul(DyKe, W1), cmul(Ke, My));
    return (double)K1.x * ((double)W1.x * W1.x + (double)W1.y * W1.y);
}

// Second half of a4 + a5: per column kx, forward FFT along y of the 10
// arrays, Parseval partial of Z, the kernel-charge products, inverse FFT of
// the 6 products along y; rows y < N are stored.  M <= kMfast: all 16
// transforms of a column in shared memory; larger M: the column's spectra are
// transformed in place in `spec` a batch at a time, multiplied there, and the
// products transformed back a batch at a time.
__global__ void __launch_bounds__(kColThreads, 1) k_col(Geo* __restrict__ gp, float2* __restrict__ spec,
                                                        const float2* __restrict__ twg, float2* __restrict__ colout,
                                                        int M_max, int N_max, int cap) {
    chain_wait();
    extern __shared__ float2 sm[];
    __shared__ double zred[kColThreads / 32];
    const int M = gp->M, N = gp->N, half = M / 2 + 1, nrad = gp->nrad;
    const unsigned long long plan = gp->plan;
    const int half_max = M_max / 2 + 1;
    float2* tw = sm;                      // M
    for (int k = threadIdx.x; k < M; k += blockDim.x) tw[k] = twg[k];
    double zpart = 0.0;
    const bool fast = 17 * M <= cap;
    for (int kx = blockIdx.x; kx < half; kx += gridDim.x) {
        auto col = [&](int a) { return spec + ((int64_t)a * half_max + kx) * M_max; };
        if (fast) {
            float2* buf = sm + M;             // 10 M
            float2* scr = buf + 10 * M;       // 6 M
            for (int t = threadIdx.x; t < 10 * M; t += blockDim.x) {
                const int a = t / M, y = t - a * M;
                buf[t] = col(a)[y];
            }
            __syncthreads();
            fft_block(buf, scr, M, 5, M, plan, nrad, tw, false);
            fft_block(buf + 5 * M, scr, M, 5, M, plan, nrad, tw, false);
            const double wt = (kx == 0 || 2 * kx == M) ? 1.0 : 2.0;
            for (int k = threadIdx.x; k < M; k += blockDim.x) {
                float2 v[10], o[6];
#pragma unroll
                for (int a = 0; a < 10; ++a) v[a] = buf[a * M + k];
                zpart += wt * col_products(v, o);
#pragma unroll
                for (int b = 0; b < 6; ++b) buf[b * M + k] = o[b];
            }
            __syncthreads();
            fft_block(buf, scr, M, 6, M, plan, nrad, tw, true);
            for (int t = threadIdx.x; t < 6 * N; t += blockDim.x) {
                const int b = t / N, y = t - b * N;
                colout[((int64_t)b * half_max + kx) * N_max + y] = buf[b * M + y];
            }
            __syncthreads();
        } else {
            const int B = fft_batch(cap, M, 10);
            float2* buf = sm + M;             // B M
            float2* scr = buf + B * M;        // B M
            for (int a0 = 0; a0 < 10; a0 += B) {          // forward, in place in spec
                const int nb = min(B, 10 - a0);
                for (int t = threadIdx.x; t < nb * M; t += blockDim.x) {
                    const int q = t / M, y = t - q * M;
                    buf[t] = col(a0 + q)[y];
                }
                __syncthreads();
                fft_block(buf, scr, M, nb, M, plan, nrad, tw, false);
                for (int t = threadIdx.x; t < nb * M; t += blockDim.x) {
                    const int q = t / M, y = t - q * M;
                    col(a0 + q)[y] = buf[t];
                }
                __syncthreads();
            }
            const double wt = (kx == 0 || 2 * kx == M) ? 1.0 : 2.0;
            for (int k = threadIdx.x; k < M; k += blockDim.x) {   // products, in place (arrays 0-5)
                float2 v[10], o[6];
#pragma unroll
                for (int a = 0; a < 10; ++a) v[a] = col(a)[k];
                zpart += wt * col_products(v, o);
#pragma unroll
                for (int b = 0; b < 6; ++b) col(b)[k] = o[b];
            }
            __syncthreads();
            for (int b0 = 0; b0 < 6; b0 += B) {           // inverse, rows y < N out
                const int nb = min(B, 6 - b0);
                for (int t = threadIdx.x; t < nb * M; t += blockDim.x) {
                    const int q = t / M, y = t - q * M;
                    buf[t] = col(b0 + q)[y];
                }
                __syncthreads();
                fft_block(buf, scr, M, nb, M, plan, nrad, tw, true);
                for (int t = threadIdx.x; t < nb * N; t += blockDim.x) {
                    const int q = t / N, y = t - q * N;
                    colout[((int64_t)(b0 + q) * half_max + kx) * N_max + y] = buf[q * M + y];
                }
                __syncthreads();
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) zpart += __shfl_xor_sync(0xffffffffu, zpart, o);
    if ((threadIdx.x & 31) == 0) zred[threadIdx.x >> 5] = zpart;
    __syncthreads();
    if (threadIdx.x == 0) {
        double z = 0.0;
        for (int k = 0; k < kColThreads / 32; ++k) z += zred[k];
        atomicAdd(&gp->zacc, z);
    }
}

// Last part of a4: per row y < N, combine with alpha/beta (Z is complete now),
// inverse FFT along x (P0 + i Qx packed, Qy alone; one at a time when the two
// do not fit), scale 1/M^2, keep x < N.
__global__ void __launch_bounds__(kInvThreads) k_row_inv(Geo* __restrict__ gp, const float2* __restrict__ colout,
                                                         const float2* __restrict__ twg, float4* __restrict__ fgrid,
                                                         int M_max, int N_max, int64_t n, float lambda_kl,
                                                         float lambda_r, int cap) {
    chain_wait();
    extern __shared__ float2 sm[];
    const int M = gp->M, N = gp->N, nrad = gp->nrad, I = gp->I;
    const int B = fft_batch(cap, M, 2);
    float2* tw = sm;
    float2* buf = sm + M;                 // B M
    float2* scr = buf + B * M;            // B M
    const unsigned long long plan = gp->plan;
    const int half_max = M_max / 2 + 1;
    const double M2 = (double)M * (double)M;
    const double Z = gp->zacc / M2 - (double)n;
    // n < 2: there are no pairs, the repulsion sum and Z are both empty (alpha = 0)
    const float alpha = (n >= 2 && Z > 0.0) ? (float)(-4.0 * (double)lambda_kl / Z) : 0.0f;
    const float beta = (float)(-(double)lambda_r / ((double)n * (double)n));
    if (blockIdx.x == 0 && threadIdx.x == 0) gp->Z = Z;
    const float sc = (float)(1.0 / M2);
    const float hb = (float)gp->h_b;
    for (int k = threadIdx.x; k < M; k += blockDim.x) tw[k] = twg[k];
    for (int y = blockIdx.x; y < N; y += gridDim.x) {
        for (int t0 = 0; t0 < 2; t0 += B) {               // transform 0: P0 + i Qx, 1: Qy
            const int nb = min(B, 2 - t0);
            for (int k = threadIdx.x; k < M; k += blockDim.x) {
                const bool lo = (k <= M / 2);
                const int kk = lo ? k : M - k;
                float2 c[6];
#pragma unroll
                for (int b = 0; b < 6; ++b) {
                    c[b] = colout[((int64_t)b * half_max + kk) * N_max + y];
                    if (!lo) c[b] = cconj(c[b]);
                }
                const float2 C0 = make_float2(alpha * c[0].x + beta * c[3].x, alpha * c[0].y + beta * c[3].y);
                const float2 Cx = make_float2(alpha * c[1].x + beta * c[4].x, alpha * c[1].y + beta * c[4].y);
                const float2 Cy = make_float2(alpha * c[2].x + beta * c[5].x, alpha * c[2].y + beta * c[5].y);
                const float2 tr[2] = {cadd(C0, mul_pi(Cx)), Cy};
                for (int q = 0; q < nb; ++q) buf[q * M + k] = tr[t0 + q];
            }
            __syncthreads();
            fft_block(buf, scr, M, nb, M, plan, nrad, tw, true);
            for (int x = threadIdx.x; x < N; x += blockDim.x) {
                // box record (kBoxRec float4 = 112 B per box, box-major): node
                // k = 3 (y % 3) + x % 3 of box (x / 3, y / 3) puts P0 at float k,
                // R_x = Q_x - s_a h P0 at 9 + k and R_y = Q_y - s_c h P0 at 18 + k
                float* f = reinterpret_cast<float*>(fgrid + ((int64_t)(y / 3) * I + x / 3) * kBoxRec);
                const int k = (y % 3) * 3 + x % 3;
                const float sh_x = node_s(x % 3) * hb, sh_y = node_s(y % 3) * hb;
                for (int q = 0; q < nb; ++q) {
                    const float2 a = buf[q * M + x];
                    if (t0 + q == 0) {
                        const float p0 = a.x * sc;
                        f[k] = p0;
                        f[9 + k] = fmaf(-sh_x, p0, a.y * sc);
                    } else {
                        // P0: this pass's transform 0, else the value this thread stored in the first pass
                        const float p0 = nb == 2 ? buf[x].x * sc : f[k];
                        f[18 + k] = fmaf(-sh_y, p0, a.x * sc);
                        if (k == 0) f[27] = 0.f;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------- interpolated entropy sum (cost)
// sum_{i != j} ln(eps + r_ij^2) ~ <W1, K_ln * W1> - n ln(eps) with the same
// spread W1 and the kernel table K_ln = ln(eps + d^2) on node offsets
// (tsnet_cost mode 1; the smooth log kernel is interpolated like K1 for Z).
// Row pass: per row y of the M x M circulant, FFT of (W1 + i K_ln) along x,
// half spectra of both stored transposed; column pass: FFT along y and the
// Parseval sum (K_ln is even, its spectrum real) into g->eacc (fp64).
__global__ void __launch_bounds__(kInvThreads) k_ent_row(const Geo* __restrict__ gp, const float4* __restrict__ wgrid,
                                                         const float2* __restrict__ twg, float2* __restrict__ spec,
                                                         int M_max, float eps) {
    extern __shared__ float2 sm[];
    const int M = gp->M, N = gp->N, half = M / 2 + 1, nrad = gp->nrad;
    float2* tw = sm;                     // M
    float2* buf = sm + M;                // M
    float2* scr = buf + M;               // M
    const unsigned long long plan = gp->plan;
    const int half_max = M_max / 2 + 1;
    const double dlt = gp->delta;
    for (int k = threadIdx.x; k < M; k += blockDim.x) tw[k] = twg[k];
    for (int y = blockIdx.x; y < M; y += gridDim.x) {
        const int dy = (y <= M / 2) ? y : y - M;
        const bool ky = (dy < N) && (-dy < N);
        for (int x = threadIdx.x; x < M; x += blockDim.x) {
            const int dx = (x <= M / 2) ? x : x - M;
            const float w1 = (y < N && x < N) ? wgrid[(int64_t)y * N + x].x : 0.f;
            float kl = 0.f;
            if (ky && dx < N && -dx < N) {
                const double ox = dx * dlt, oy = dy * dlt;
                kl = (float)log((double)eps + ox * ox + oy * oy);
            }
            buf[x] = make_float2(w1, kl);
        }
        __syncthreads();
        fft_block(buf, scr, M, 1, M, plan, nrad, tw, false);
        for (int k = threadIdx.x; k < half; k += blockDim.x) {
            const float2 Zk = buf[k];
            const float2 Zm = cconj(buf[k == 0 ? 0 : M - k]);
            spec[((int64_t)0 * half_max + k) * M_max + y] = make_float2(0.5f * (Zk.x + Zm.x), 0.5f * (Zk.y + Zm.y));
            spec[((int64_t)1 * half_max + k) * M_max + y] = mul_mi(make_float2(0.5f * (Zk.x - Zm.x), 0.5f * (Zk.y - Zm.y)));
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kInvThreads) k_ent_col(Geo* __restrict__ gp, float2* __restrict__ spec,
                                                         const float2* __restrict__ twg, int M_max, int cap) {
    extern __shared__ float2 sm[];
    __shared__ double red[kInvThreads / 32];
    const int M = gp->M, half = M / 2 + 1, nrad = gp->nrad;
    const int B = fft_batch(cap, M, 2);
    float2* tw = sm;
    float2* buf = sm + M;                // B M
    float2* scr = buf + B * M;           // B M
    const unsigned long long plan = gp->plan;
    const int half_max = M_max / 2 + 1;
    for (int k = threadIdx.x; k < M; k += blockDim.x) tw[k] = twg[k];
    double part = 0.0;
    for (int kx = blockIdx.x; kx < half; kx += gridDim.x) {
        auto col = [&](int a) { return spec + ((int64_t)a * half_max + kx) * M_max; };
        if (B >= 2) {
            for (int t = threadIdx.x; t < 2 * M; t += blockDim.x) {
                const int a = t / M, y = t - a * M;
                buf[t] = col(a)[y];
            }
            __syncthreads();
            fft_block(buf, scr, M, 2, M, plan, nrad, tw, false);
        } else {
            // one transform at a time: W1 in place in spec, then K_ln in shared memory
            for (int y = threadIdx.x; y < M; y += blockDim.x) buf[y] = col(0)[y];
            __syncthreads();
            fft_block(buf, scr, M, 1, M, plan, nrad, tw, false);
            for (int y = threadIdx.x; y < M; y += blockDim.x) col(0)[y] = buf[y];
            __syncthreads();
            for (int y = threadIdx.x; y < M; y += blockDim.x) buf[y] = col(1)[y];
            __syncthreads();
            fft_block(buf, scr, M, 1, M, plan, nrad, tw, false);
        }
        const double wt = (kx == 0 || 2 * kx == M) ? 1.0 : 2.0;
        for (int k = threadIdx.x; k < M; k += blockDim.x) {
            const float2 W = B >= 2 ? buf[k] : col(0)[k];
            const float2 K = B >= 2 ? buf[M + k] : buf[k];
            part += wt * (double)K.x * ((double)W.x * W.x + (double)W.y * W.y);
        }
        __syncthreads();
    }
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        double z = 0.0;
        for (int k = 0; k < kInvThreads / 32; ++k) z += red[k];
        atomicAdd(&gp->eacc, z);
    }
}

__global__ void k_ent_zero(Geo* g) { g->eacc = 0.0; }

size_t field_smem_row(int M_max) { return sizeof(float2) * (size_t)smem_cap_row(M_max); }
size_t field_smem_col(int M_max) { return sizeof(float2) * (size_t)smem_cap_col(M_max); }
size_t field_smem_inv(int M_max) { return sizeof(float2) * (size_t)smem_cap_inv(M_max); }

cudaError_t field_set_attrs(int M_max) {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_row_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)field_smem_row(M_max))) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(k_col, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)field_smem_col(M_max))) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(k_row_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)field_smem_inv(M_max))) != cudaSuccess) return e;
    return cudaSuccess;
}

// a0-a2 for the rows [rb, re) this call owns: geometry from the bounding box of
// the FULL layout Y (replicated on every rank, so every rank derives the same
// grid without a collective), then box sort + spread of the own rows only.
// On one GPU rb = 0, re = n.  With `zero_all`, the whole I_max-sized grid is
// zeroed (it is all-reduced as one fixed-size buffer across ranks).
cudaError_t launch_field_local(const Ws& w, const GradArgs& a, cudaStream_t s, bool zero_all) {
    cudaError_t e;
    if ((e = field_set_attrs(w.M_max)) != cudaSuccess) return e;
    const int64_t n = a.n, nl = a.re - a.rb;
    const int pb = (int)std::max<int64_t>(1, std::min<int64_t>((n + 256 * kBBoxPts - 1) / (256 * kBBoxPts),
                                                                  (int64_t)kNumSMs * 4));
    const int pbl = (int)std::max<int64_t>(1, std::min<int64_t>((nl + 255) / 256, (int64_t)kNumSMs * 8));
    k_bbox<<<pb, 256, 0, s>>>(a.Y, n, w.geo, a.h_max, a.I_min, a.I_max, w.wgrid, a.spread);
    if (zero_all && (e = cudaMemsetAsync(w.wgrid, 0, sizeof(float4) * (size_t)w.N_max * w.N_max, s)) != cudaSuccess)
        return e;
    const float2* Yl = a.Y + a.rb;
    // the sort's kernels are launched every iteration (the path is only known
    // on the device, and the iteration is one CUDA graph) and exit at once on
    // the runs path
    const int cb = (int)std::max<int64_t>(kNumSMs, (nl + kBoxChunk - 1) / kBoxChunk);
    if ((e = launch_chain(k_box_count, cb, 256, 0, s, Yl, nl, w.geo, w.box_cnt, w.box, w.rank)) != cudaSuccess) return e;
    if ((e = launch_chain(k_box_scan, 1, 1024, 0, s, w.geo, w.box_cnt, w.box_start, nl)) != cudaSuccess) return e;
    if ((e = launch_chain(k_box_scatter, pbl, 256, 0, s, w.geo, nl, w.box, w.rank, w.box_start, w.perm)) != cudaSuccess) return e;
    const int rbk = (int)std::max<int64_t>(1, std::min<int64_t>((nl + 8 * 32 * kRunPts - 1) / (8 * 32 * kRunPts),
                                                                  (int64_t)kNumSMs * RUNS_MINB));
    if ((e = launch_chain(k_spread_runs, rbk, 256, 0, s, Yl, nl, w.geo, w.perm, w.wgrid, w.tw)) != cudaSuccess) return e;
    return cudaGetLastError();
}

// a3-a5 from the (all-reduced) charge grid: kernel tabulation, FFT
// convolution, Z by Parseval (global n), combined fields.  Replicated.
cudaError_t launch_field_conv(const Ws& w, const GradArgs& a, cudaStream_t s) {
    cudaError_t e;
    if ((e = field_set_attrs(w.M_max)) != cudaSuccess) return e;
    if ((e = launch_chain(k_row_fwd, kNumSMs * 2, kRowThreads, field_smem_row(w.M_max), s, w.geo, w.wgrid, w.tw, w.spec,
                          w.M_max, a.eps, smem_cap_row(w.M_max))) != cudaSuccess)
        return e;
    if ((e = launch_chain(k_col, kNumSMs, kColThreads, field_smem_col(w.M_max), s, w.geo, w.spec, w.tw, w.colout, w.M_max,
                          w.N_max, smem_cap_col(w.M_max))) != cudaSuccess)
        return e;
    if ((e = launch_chain(k_row_inv, kNumSMs * 2, kInvThreads, field_smem_inv(w.M_max), s, w.geo, w.colout, w.tw, w.fgrid,
                          w.M_max, w.N_max, a.n, a.lambda_kl, a.lambda_r, smem_cap_inv(w.M_max))) != cudaSuccess)
        return e;
    return cudaGetLastError();
}

// sum_{i != j} ln(eps + r^2) * M^2 + n ln(eps) M^2 into g->eacc, after launch_field_local
cudaError_t launch_entropy_sum(const Ws& w, const GradArgs& a, cudaStream_t s) {
    cudaError_t e;
    const int capc = std::max(5 * std::min(w.M_max, kMfast), 3 * w.M_max);
    const size_t smr = sizeof(float2) * (size_t)w.M_max * 3, smc = sizeof(float2) * (size_t)capc;
    if ((e = cudaFuncSetAttribute(k_ent_row, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smr)) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(k_ent_col, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smc)) != cudaSuccess)
        return e;
    k_ent_zero<<<1, 1, 0, s>>>(w.geo);
    k_ent_row<<<kNumSMs * 2, kInvThreads, smr, s>>>(w.geo, w.wgrid, w.tw, w.spec, w.M_max, a.eps);
    k_ent_col<<<kNumSMs, kInvThreads, smc, s>>>(w.geo, w.spec, w.tw, w.M_max, capc);
    return cudaGetLastError();
}

cudaError_t launch_field_phase(const Ws& w, const GradArgs& a, cudaStream_t s) {
    cudaError_t e = launch_field_local(w, a, s, false);
    if (e != cudaSuccess) return e;
    return launch_field_conv(w, a, s);
}

}  // namespace tsnet
