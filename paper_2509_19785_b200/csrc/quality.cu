// quality.cu -- drawing-quality metrics of §4.3 (NEXT-4): neighbourhood
// preservation (r = 2) and the optimally scaled aggregated
// stress (SPEC stress), readings R25-R26:
//   NP  mean over v of |N_G ∩ N_D| / |N_G ∪ N_D|; N_G(v, r) = vertices within
//       r hops (v excluded), N_D = the |N_G| closest others in the drawing by
//       fp64 squared distance of the fp32 coordinates (dx*dx + dy*dy, no fused
//       ops), ties by smaller id; an empty N_G scores 1;
//   ST  r_ij = |X_i - X_j| / d(i, j) over ordered pairs of a connected graph,
//       ST = (N - (sum r)^2 / sum r^2) / N, N = n (n - 1)  (= 1/N sum (1 - s* r)^2
//       with the optimal scale s* = sum r / sum r^2).
// Evaluation of small drawings (n <= kQualityMaxN), not the iteration: a CTA
// per vertex.  NP: hop neighbourhood by bitmap BFS to depth r, all fp64
// squared distances in shared memory, the |N_G|-th smallest (distance, id) by
// bisection on the 64-bit key, then the intersection count.  ST: a CTA per
// source, bitmap-frontier BFS with uint16 distances in shared memory, fp64
// sums of r and r^2.
//
// Also the stand-alone move (tsnet_move): the gains/momentum update of a7 for
// a gradient computed elsewhere (the quadtree variants).
#include <cmath>

#include "common.cuh"
#include "move.cuh"
#include "tsnet.h"

namespace tsnet {

constexpr int kQualityMaxN = 24576;
constexpr int kQualityThreads = 512;

__device__ __forceinline__ double qsq(float2 a, float2 b) {
    const double dx = (double)a.x - (double)b.x, dy = (double)a.y - (double)b.y;
    return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

__device__ __forceinline__ int block_sum_int(int x, int* red) {
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    int s = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s += red[q];
    __syncthreads();
    return s;
}

// bitmap BFS from v to depth r: visited bitmap (v included) in `vis`
__device__ void bfs_bitmap(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, int n, int v,
                           int r, unsigned* vis, unsigned* cur, unsigned* nxt) {
    const int W = (n + 31) / 32;
    for (int q = threadIdx.x; q < W; q += blockDim.x) {
        vis[q] = 0u;
        cur[q] = 0u;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        vis[v >> 5] |= 1u << (v & 31);
        cur[v >> 5] |= 1u << (v & 31);
    }
    __syncthreads();
    for (int lev = 0; lev < r; ++lev) {
        for (int q = threadIdx.x; q < W; q += blockDim.x) nxt[q] = 0u;
        __syncthreads();
        // a warp per frontier vertex
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int q = warp; q < W; q += nw) {
            unsigned bits = cur[q];
            while (bits) {
                const int b = __ffs(bits) - 1;
                bits &= bits - 1;
                const int u = q * 32 + b;
                for (int64_t e = indptr[u] + lane; e < indptr[u + 1]; e += 32) {
                    const int w = indices[e];
                    if (!(vis[w >> 5] & (1u << (w & 31)))) atomicOr(&nxt[w >> 5], 1u << (w & 31));
                }
            }
        }
        __syncthreads();
        for (int q = threadIdx.x; q < W; q += blockDim.x) {
            const unsigned f = nxt[q] & ~vis[q];
            cur[q] = f;
            vis[q] |= f;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kQualityThreads) k_quality_np(const int64_t* __restrict__ indptr,
                                                                const int32_t* __restrict__ indices, int n,
                                                                const float2* __restrict__ Y, int r,
                                                                double* __restrict__ out) {
    extern __shared__ unsigned long long qsm[];
    unsigned long long* key = qsm;                                   // n fp64 bit patterns
    const int W = (n + 31) / 32;
    unsigned* vis = reinterpret_cast<unsigned*>(qsm + n);
    unsigned* cur = vis + W;
    unsigned* nxt = cur + W;
    __shared__ int red[32];
    for (int v = blockIdx.x; v < n; v += gridDim.x) {
        bfs_bitmap(indptr, indices, n, v, r, vis, cur, nxt);
        int k = 0;
        for (int q = threadIdx.x; q < W; q += blockDim.x) k += __popc(vis[q]);
        k = block_sum_int(k, red) - 1;                               // v excluded
        if (k == 0) {
            if (threadIdx.x == 0) atomicAdd(out, 1.0);
            continue;
        }
        const float2 yv = Y[v];
        for (int w = threadIdx.x; w < n; w += blockDim.x)
            key[w] = w == v ? ~0ull : (unsigned long long)__double_as_longlong(qsq(yv, Y[w]));
        __syncthreads();
        // T = the k-th smallest key among w != v (keys of non-negative doubles order as integers)
        unsigned long long lo = 0ull, hi = ~0ull;                    // count(<= hi) >= k
        while (lo < hi) {
            const unsigned long long mid = lo + (hi - lo) / 2;
            int c = 0;
            for (int w = threadIdx.x; w < n; w += blockDim.x) c += key[w] <= mid;
            c = block_sum_int(c, red);
            if (c >= k) hi = mid; else lo = mid + 1;
        }
        const unsigned long long T = lo;
        int less = 0;
        for (int w = threadIdx.x; w < n; w += blockDim.x) less += key[w] < T;
        less = block_sum_int(less, red);
        const int m = k - less;                                      // tied vertices taken, smallest ids first
        // id threshold: the m-th smallest id among key == T
        int ilo = 0, ihi = n - 1;
        while (ilo < ihi) {
            const int mid = (ilo + ihi) / 2;
            int c = 0;
            for (int w = threadIdx.x; w <= mid; w += blockDim.x) c += key[w] == T;
            c = block_sum_int(c, red);
            if (c >= m) ihi = mid; else ilo = mid + 1;
        }
        const int idmax = ilo;
        int inter = 0;
        for (int w = threadIdx.x; w < n; w += blockDim.x) {
            const bool g = w != v && (vis[w >> 5] & (1u << (w & 31)));
            const bool d = key[w] < T || (key[w] == T && w <= idmax);
            inter += g && d;
        }
        inter = block_sum_int(inter, red);
        if (threadIdx.x == 0) atomicAdd(out, (double)inter / (double)(2 * k - inter));
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kQualityThreads) k_quality_stress(const int64_t* __restrict__ indptr,
                                                                    const int32_t* __restrict__ indices, int n,
                                                                    const float2* __restrict__ Y,
                                                                    double* __restrict__ sums) {
    extern __shared__ unsigned qsm2[];
    const int W = (n + 31) / 32;
    unsigned* vis = qsm2;
    unsigned* cur = vis + W;
    unsigned* nxt = cur + W;
    unsigned short* dist = reinterpret_cast<unsigned short*>(nxt + W);
    __shared__ int red[32];
    for (int s = blockIdx.x; s < n; s += gridDim.x) {
        for (int q = threadIdx.x; q < W; q += blockDim.x) {
            vis[q] = 0u;
            cur[q] = 0u;
        }
        for (int w = threadIdx.x; w < n; w += blockDim.x) dist[w] = 0xFFFF;
        __syncthreads();
        if (threadIdx.x == 0) {
            vis[s >> 5] |= 1u << (s & 31);
            cur[s >> 5] |= 1u << (s & 31);
            dist[s] = 0;
        }
        __syncthreads();
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int lev = 0;; ++lev) {
            for (int q = threadIdx.x; q < W; q += blockDim.x) nxt[q] = 0u;
            __syncthreads();
            for (int q = warp; q < W; q += nw) {
                unsigned bits = cur[q];
                while (bits) {
                    const int b = __ffs(bits) - 1;
                    bits &= bits - 1;
                    const int u = q * 32 + b;
                    for (int64_t e = indptr[u] + lane; e < indptr[u + 1]; e += 32) {
                        const int w = indices[e];
                        if (!(vis[w >> 5] & (1u << (w & 31)))) atomicOr(&nxt[w >> 5], 1u << (w & 31));
                    }
                }
            }
            __syncthreads();
            int any = 0;
            for (int q = threadIdx.x; q < W; q += blockDim.x) {
                const unsigned f = nxt[q] & ~vis[q];
                cur[q] = f;
                vis[q] |= f;
                any |= f != 0u;
                unsigned bits = f;
                while (bits) {
                    const int b = __ffs(bits) - 1;
                    bits &= bits - 1;
                    dist[q * 32 + b] = (unsigned short)(lev + 1);
                }
            }
            any = block_sum_int(any, red);
            if (!any) break;
        }
        double s1 = 0.0, s2 = 0.0, miss = 0.0;
        const float2 ys = Y[s];
        for (int w = threadIdx.x; w < n; w += blockDim.x) {
            if (w == s) continue;
            if (dist[w] == 0xFFFF) {
                miss += 1.0;
                continue;
            }
            const double rr = sqrt(qsq(ys, Y[w])) / (double)dist[w];
            s1 += rr;
            s2 += rr * rr;
        }
        for (int o = 16; o > 0; o >>= 1) {
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
            s2 += __shfl_xor_sync(0xffffffffu, s2, o);
            miss += __shfl_xor_sync(0xffffffffu, miss, o);
        }
        if (lane == 0) {
            atomicAdd(&sums[0], s1);
            atomicAdd(&sums[1], s2);
            atomicAdd(&sums[2], miss);
        }
        __syncthreads();
    }
}

__global__ void k_quality_final(const double* __restrict__ np_sum, const double* __restrict__ sums, int n,
                                double* __restrict__ out2) {
    const double N = (double)n * (double)(n - 1);
    out2[0] = np_sum[0] / (double)n;
    out2[1] = sums[2] > 0.0 ? NAN : (N - sums[0] * sums[0] / sums[1]) / N;   // disconnected: undefined
}

__global__ void k_move(int64_t n, float2* __restrict__ Y, float2* __restrict__ vel, float2* __restrict__ gains,
                       const float2* __restrict__ grad, tsnet_step_params sp) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float2 y = Y[i], v = vel[i], gn = gains[i];
        const float2 g = grad[i];
        gains_move(g.x, v.x, gn.x, y.x, sp);
        gains_move(g.y, v.y, gn.y, y.y, sp);
        Y[i] = y;
        vel[i] = v;
        gains[i] = gn;
    }
}

}  // namespace tsnet

using namespace tsnet;

extern "C" {

size_t tsnet_quality_workspace_bytes(int64_t n) { return n < 0 ? 0 : 256; }

int tsnet_quality(const tsnet_graph* g, const float* Y, int32_t r, double* out2, void* ws, size_t ws_bytes,
                  tsnet_stream_t stream) {
    TSNET_ARG(g != nullptr && Y != nullptr && out2 != nullptr, "NULL argument");
    const int64_t n = g->n;
    TSNET_ARG(n >= 2 && n <= kQualityMaxN, "n = %lld must be in [2, %d]", (long long)n, kQualityMaxN);
    TSNET_ARG(g->indptr && g->indices, "graph arrays are NULL");
    TSNET_ARG(r >= 1 && r <= 64, "r = %d must be in [1, 64]", r);
    TSNET_ARG(ws != nullptr && ws_bytes >= 256, "workspace too small (%zu < 256 bytes)", ws_bytes);
    cudaStream_t s = (cudaStream_t)stream;
    double* acc = reinterpret_cast<double*>(ws);     // np sum, sum r, sum r^2, missing pairs
    TSNET_CUDA(cudaMemsetAsync(acc, 0, sizeof(double) * 4, s));
    const int W = (int)((n + 31) / 32);
    const size_t smem_np = sizeof(unsigned long long) * (size_t)n + sizeof(unsigned) * 3 * (size_t)W;
    const size_t smem_st = sizeof(unsigned) * 3 * (size_t)W + sizeof(unsigned short) * (size_t)n;
    TSNET_CUDA(cudaFuncSetAttribute(k_quality_np, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_np));
    TSNET_CUDA(cudaFuncSetAttribute(k_quality_stress, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_st));
    const int blocks = (int)std::min<int64_t>(n, (int64_t)kNumSMs * 2);
    const float2* Y2 = reinterpret_cast<const float2*>(Y);
    k_quality_np<<<blocks, kQualityThreads, smem_np, s>>>(g->indptr, g->indices, (int)n, Y2, r, acc);
    TSNET_LAUNCH_CHECK();
    k_quality_stress<<<blocks, kQualityThreads, smem_st, s>>>(g->indptr, g->indices, (int)n, Y2, acc + 1);
    TSNET_LAUNCH_CHECK();
    k_quality_final<<<1, 1, 0, s>>>(acc, acc + 1, (int)n, out2);
    TSNET_LAUNCH_CHECK();
    return TSNET_OK;
}

int tsnet_move(float* Y, float* vel, float* gains, const float* grad, int64_t n, const tsnet_step_params* sp,
               tsnet_stream_t stream) {
    TSNET_ARG(sp != nullptr && n >= 0, "bad arguments");
    if (n == 0) return TSNET_OK;
    TSNET_ARG(Y && vel && gains && grad, "NULL array");
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)kNumSMs * 8));
    k_move<<<blocks, 256, 0, (cudaStream_t)stream>>>(n, reinterpret_cast<float2*>(Y), reinterpret_cast<float2*>(vel),
                                                     reinterpret_cast<float2*>(gains),
                                                     reinterpret_cast<const float2*>(grad), *sp);
    TSNET_LAUNCH_CHECK();
    return TSNET_OK;
}

}  // extern "C"
