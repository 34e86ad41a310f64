// pmds.cu -- Pivot MDS initial layout (Alg. 3 line 2; tsNET* =
// tsNET with a PMDS initialisation).  Set-up, outside the
// iteration loop, like C0.  Readings R20-R22:
//   pivots   farthest-first: first = splitmix64(seed) mod n, each next pivot
//            maximises the hop distance to the chosen set, ties -> smallest
//            id; unreachable vertices count as distance n;
//   embed    D2 = hop^2 (n x p); C = -1/2 (D2 - row means - column means +
//            grand mean); top-2 eigenvectors of G = C^T C by power iteration
//            (splitmix64 start vectors, <= 1000 iterations, |v' - v| < 1e-10;
//            the second deflated and re-orthogonalised), each flipped so its
//            largest-magnitude entry is positive; Y = C [v1 v2]; a second
//            eigenvalue <= 1e-12 of the first gives a zero second coordinate.
//
// GPU pieces: level-synchronous BFS per pivot (warp per frontier vertex,
// CAS on the distance, warp-aggregated queue appends) writing the hop column
// directly; one pass per pivot folds the column into the running minimum and
// finds the next pivot with a packed (distance, ~id) atomicMax; exact integer
// row/column sums of D2; G = C^T C by 32 x 32 fp64 tiles over row chunks (C
// formed on the fly from the hops, same operation order as the definition);
// power iteration in one CTA; Y by a thread per vertex.
#include <cmath>
#include <vector>

#include "common.cuh"
#include "tsnet.h"

namespace tsnet {

constexpr int kPmdsMaxPivots = 1024;

struct PmdsWs {
    int32_t* hops;           // p x n, pivot-major
    int32_t* mind;           // n
    int32_t* front[2];       // n each
    int32_t* qsize;          // 4
    unsigned long long* key; // 1
    int64_t* rowsum;         // n   : sum_k hop^2 (exact)
    int64_t* colsum;         // p
    double* cmean;           // p   : column means of D2
    double* G;               // p x p
    double* V;               // 2 p
    double* lam;             // 2
    size_t bytes;
};

static PmdsWs pmds_ws_map(void* base, int64_t n, int p) {
    PmdsWs w{};
    size_t off = 0;
    auto take = [&](size_t b) {
        void* q = (char*)base + off;
        off = (off + b + 255) / 256 * 256;
        return q;
    };
    w.hops = (int32_t*)take(sizeof(int32_t) * (size_t)p * (size_t)n);
    w.mind = (int32_t*)take(sizeof(int32_t) * (size_t)n);
    w.front[0] = (int32_t*)take(sizeof(int32_t) * (size_t)n);
    w.front[1] = (int32_t*)take(sizeof(int32_t) * (size_t)n);
    w.qsize = (int32_t*)take(sizeof(int32_t) * 4);
    w.key = (unsigned long long*)take(sizeof(unsigned long long));
    w.rowsum = (int64_t*)take(sizeof(int64_t) * (size_t)n);
    w.colsum = (int64_t*)take(sizeof(int64_t) * (size_t)p);
    w.cmean = (double*)take(sizeof(double) * (size_t)p);
    w.G = (double*)take(sizeof(double) * (size_t)p * p);
    w.V = (double*)take(sizeof(double) * 2 * (size_t)p);
    w.lam = (double*)take(sizeof(double) * 2);
    w.bytes = off;
    return w;
}

static uint64_t splitmix64_host(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// one BFS level: warp per frontier vertex
__global__ void k_bfs_level(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                            const int32_t* __restrict__ frontier, int fsize, int32_t* __restrict__ next,
                            int32_t* __restrict__ next_size, int32_t* __restrict__ dist, int level) {
    const int lane = threadIdx.x & 31;
    for (int64_t f = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; f < fsize;
         f += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int v = frontier[f];
        const int64_t a = indptr[v], b = indptr[v + 1];
        for (int64_t e0 = a; e0 < b; e0 += 32) {
            const int64_t e = e0 + lane;
            bool won = false;
            int u = 0;
            if (e < b) {
                u = indices[e];
                won = dist[u] < 0 && atomicCAS(&dist[u], -1, level + 1) == -1;
            }
            const unsigned m = __ballot_sync(0xffffffffu, won);
            if (m) {
                int base = 0;
                if (lane == 0) base = atomicAdd(next_size, __popc(m));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (won) next[base + __popc(m & ((1u << lane) - 1u))] = u;
            }
        }
    }
}

// unreachable -> n (R21); running minimum; next pivot = argmax (ties -> smallest id)
__global__ void k_pmds_fold(int32_t* __restrict__ col, int32_t* __restrict__ mind, int64_t n, int first,
                            unsigned long long* __restrict__ key) {
    unsigned long long best = 0ull;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        int d = col[v];
        if (d < 0) {
            d = (int)n;
            col[v] = d;
        }
        const int m = first ? d : min(mind[v], d);
        mind[v] = m;
        const unsigned long long k = ((unsigned long long)(unsigned)m << 32) | (0xFFFFFFFFu - (unsigned)v);
        best = k > best ? k : best;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
        best = t > best ? t : best;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(key, best);
}

// exact integer sums of D2 = hop^2: per row (over pivots) and per pivot (over rows)
__global__ void k_pmds_rowsum(const int32_t* __restrict__ hops, int64_t n, int p, int64_t* __restrict__ rowsum) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t s = 0;
        for (int k = 0; k < p; ++k) {
            const int64_t h = hops[(int64_t)k * n + i];
            s += h * h;
        }
        rowsum[i] = s;
    }
}

__global__ void k_pmds_colsum(const int32_t* __restrict__ hops, int64_t n, int64_t* __restrict__ colsum) {
    const int k = blockIdx.y;
    int64_t s = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t h = hops[(int64_t)k * n + i];
        s += h * h;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd((unsigned long long*)&colsum[k], (unsigned long long)s);
}

// C[i, k] = -1/2 (((D2 - row mean) - column mean) + grand mean): the order of the definition
__device__ __forceinline__ double pmds_c(int32_t h, double rm, double cm, double gm) {
    const double d2 = (double)h * (double)h;
    return -0.5 * (((d2 - rm) - cm) + gm);
}

struct PmdsMeans {
    const int64_t* rowsum;   // row mean = rowsum / p (a division, as the definition)
    double p, gm;
};

// G = C^T C: CTA = one 32 x 32 tile (kb <= lb) over a chunk of rows; fp64
// partial sums added atomically; the lower triangle is mirrored afterwards
__global__ void __launch_bounds__(256) k_pmds_gram(const int32_t* __restrict__ hops, int64_t n, int p, PmdsMeans mm,
                                                   const double* __restrict__ cmean, int64_t rows_per_cta,
                                                   double* __restrict__ G) {
    __shared__ double A[32][33], B[32][33];
    // tile (kb, lb) with kb <= lb from blockIdx.y
    const int nt = (p + 31) / 32;
    int t = blockIdx.y, kb = 0;
    while (t >= nt - kb) {
        t -= nt - kb;
        ++kb;
    }
    const int lb = kb + t;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;   // 16 x 16 threads, 2 x 2 entries each
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    const int64_t i0 = blockIdx.x * rows_per_cta, i1 = (n < i0 + rows_per_cta) ? n : i0 + rows_per_cta;
    for (int64_t r0 = i0; r0 < i1; r0 += 32) {
        // load 32 rows x 32 pivot columns of C for the k and l tiles
        for (int q = threadIdx.x; q < 32 * 32; q += blockDim.x) {
            const int rr = q >> 5, cc = q & 31;     // consecutive threads: consecutive rows (coalesced hops)
            const int64_t i = r0 + cc;
            const int kk = kb * 32 + rr, ll = lb * 32 + rr;
            double a = 0.0, b = 0.0;
            if (i < i1) {
                const double rm = (double)mm.rowsum[i] / mm.p;
                if (kk < p) a = pmds_c(hops[(int64_t)kk * n + i], rm, cmean[kk], mm.gm);
                if (ll < p) b = pmds_c(hops[(int64_t)ll * n + i], rm, cmean[ll], mm.gm);
            }
            A[cc][rr] = a;
            B[cc][rr] = b;
        }
        __syncthreads();
#pragma unroll 8
        for (int r = 0; r < 32; ++r) {
            const double a0 = A[r][ty], a1 = A[r][ty + 16];
            const double b0 = B[r][tx], b1 = B[r][tx + 16];
            acc[0][0] = fma(a0, b0, acc[0][0]);
            acc[0][1] = fma(a0, b1, acc[0][1]);
            acc[1][0] = fma(a1, b0, acc[1][0]);
            acc[1][1] = fma(a1, b1, acc[1][1]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const int k = kb * 32 + ty + 16 * u, l = lb * 32 + tx + 16 * v;
            if (k < p && l < p && (kb < lb || k <= l)) atomicAdd(&G[(int64_t)k * p + l], acc[u][v]);
        }
}

__global__ void k_pmds_mirror(double* G, int p) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < p * p; q += gridDim.x * blockDim.x) {
        const int k = q / p, l = q % p;
        if (k > l) G[q] = G[(int64_t)l * p + k];
    }
}

__device__ double pmds_block_sum(double x, double* red) {
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    double s = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s += red[q];
    return s;
}

__device__ __forceinline__ double pmds_u(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return (double)(z >> 11) * 0x1.0p-53;
}

// power iteration for the top-2 eigenpairs of G (one CTA, thread per pivot)
__global__ void __launch_bounds__(1024) k_pmds_power(const double* __restrict__ G, int p, uint64_t seed, double* V,
                                                     double* lam) {
    __shared__ double v[kPmdsMaxPivots], w[kPmdsMaxPivots], v1[kPmdsMaxPivots];
    __shared__ double red[32];
    __shared__ int s_arg;
    const int k = threadIdx.x;
    double l1 = 0.0;
    for (int which = 1; which <= 2; ++which) {
        if (which == 2 && p < 2) {                 // one pivot: rank 1 (R22)
            if (k < p) V[p + k] = 0.0;
            if (k == 0) lam[1] = 0.0;
            break;
        }
        if (k < p) v[k] = pmds_u(seed ^ (uint64_t)(2 * k + which)) - 0.5;
        __syncthreads();
        if (which == 2) {                          // start orthogonal to v1
            const double d = pmds_block_sum(k < p ? v[k] * v1[k] : 0.0, red);
            if (k < p) v[k] -= d * v1[k];
        }
        __syncthreads();
        double nv = sqrt(pmds_block_sum(k < p ? v[k] * v[k] : 0.0, red));
        if (k < p) v[k] /= nv;
        __syncthreads();
        double l = 0.0;
        for (int it = 0; it < 1000; ++it) {
            double x = 0.0;
            if (k < p) {
                for (int j = 0; j < p; ++j) x = fma(G[(int64_t)k * p + j], v[j], x);
            }
            if (which == 2) {                      // G2 = G - l1 v1 v1^T
                const double d = pmds_block_sum(k < p ? v1[k] * v[k] : 0.0, red);
                if (k < p) x -= l1 * d * v1[k];
                const double e = pmds_block_sum(k < p ? x * v1[k] : 0.0, red);
                if (k < p) x -= e * v1[k];
            }
            l = sqrt(pmds_block_sum(k < p ? x * x : 0.0, red));
            if (l == 0.0) break;
            const double xn = k < p ? x / l : 0.0;
            const double dd = sqrt(pmds_block_sum(k < p ? (xn - v[k]) * (xn - v[k]) : 0.0, red));
            __syncthreads();
            if (k < p) v[k] = xn;
            __syncthreads();
            if (dd < 1e-10) break;
        }
        // orientation: largest |entry| (first on ties) positive
        if (k == 0) {
            int arg = 0;
            double best = -1.0;
            for (int j = 0; j < p; ++j)
                if (fabs(v[j]) > best) {
                    best = fabs(v[j]);
                    arg = j;
                }
            s_arg = arg;
        }
        __syncthreads();
        const double sgn = v[s_arg] < 0.0 ? -1.0 : 1.0;
        bool zero = false;
        if (which == 1) {
            l1 = l;
        } else {
            zero = l <= 1e-12 * l1;
        }
        if (k < p) {
            const double val = zero ? 0.0 : sgn * v[k];
            V[(int64_t)(which - 1) * p + k] = val;
            if (which == 1) v1[k] = val;
        }
        if (k == 0) lam[which - 1] = l;
        __syncthreads();
    }
}

__global__ void k_pmds_embed(const int32_t* __restrict__ hops, int64_t n, int p, PmdsMeans mm,
                             const double* __restrict__ cmean, const double* __restrict__ V, float* __restrict__ Y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double rm = (double)mm.rowsum[i] / mm.p;
        double y0 = 0.0, y1 = 0.0;
        for (int k = 0; k < p; ++k) {
            const double c = pmds_c(hops[(int64_t)k * n + i], rm, cmean[k], mm.gm);
            y0 = fma(c, V[k], y0);
            y1 = fma(c, V[p + k], y1);
        }
        Y[2 * i] = (float)y0;
        Y[2 * i + 1] = (float)y1;
    }
}

}  // namespace tsnet

using namespace tsnet;

extern "C" {

size_t tsnet_pmds_workspace_bytes(int64_t n, int32_t pivots) {
    if (n < 0 || pivots < 1) return 0;
    return pmds_ws_map(nullptr, n, pivots).bytes;
}

int tsnet_pmds(const tsnet_graph* g, int32_t p, uint64_t seed, float* Y, int32_t* pivots_out, int32_t* hops_out,
               double* eig_out, void* ws, size_t ws_bytes, tsnet_stream_t stream) {
    TSNET_ARG(g != nullptr && Y != nullptr, "graph or Y is NULL");
    const int64_t n = g->n;
    TSNET_ARG(n >= 1 && n < ((int64_t)1 << 31) - 1, "n = %lld must be in [1, 2^31 - 1)", (long long)n);
    TSNET_ARG(g->indptr && (g->indices || n == 1), "graph arrays are NULL");
    TSNET_ARG(p >= 1 && p <= n && p <= kPmdsMaxPivots, "pivots = %d must be in [1, min(n, %d)]", p, kPmdsMaxPivots);
    const PmdsWs w = pmds_ws_map(ws, n, p);
    TSNET_ARG(ws != nullptr && ws_bytes >= w.bytes, "workspace too small (%zu < %zu bytes)", ws_bytes, w.bytes);
    cudaStream_t s = (cudaStream_t)stream;
    const int pb = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)kNumSMs * 8));
    std::vector<int32_t> piv(p);
    int src = (int)(splitmix64_host(seed) % (uint64_t)n);
    for (int k = 0; k < p; ++k) {
        piv[k] = src;
        int32_t* col = w.hops + (int64_t)k * n;
        TSNET_CUDA(cudaMemsetAsync(col, 0xFF, sizeof(int32_t) * (size_t)n, s));
        const int32_t zero = 0;
        TSNET_CUDA(cudaMemcpyAsync(col + src, &zero, sizeof(int32_t), cudaMemcpyHostToDevice, s));
        TSNET_CUDA(cudaMemcpyAsync(w.front[0], &src, sizeof(int32_t), cudaMemcpyHostToDevice, s));
        int fsize = 1, cur = 0, level = 0;
        while (fsize > 0) {
            TSNET_CUDA(cudaMemsetAsync(w.qsize, 0, sizeof(int32_t), s));
            const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)fsize * 32 + 255) / 256,
                                                                        (int64_t)kNumSMs * 8));
            k_bfs_level<<<blocks, 256, 0, s>>>(g->indptr, g->indices, w.front[cur], fsize, w.front[cur ^ 1], w.qsize,
                                               col, level);
            TSNET_LAUNCH_CHECK();
            TSNET_CUDA(cudaMemcpyAsync(&fsize, w.qsize, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            TSNET_CUDA(cudaStreamSynchronize(s));
            cur ^= 1;
            ++level;
        }
        TSNET_CUDA(cudaMemsetAsync(w.key, 0, sizeof(unsigned long long), s));
        k_pmds_fold<<<pb, 256, 0, s>>>(col, w.mind, n, k == 0, w.key);
        TSNET_LAUNCH_CHECK();
        if (k + 1 < p) {
            unsigned long long key = 0;
            TSNET_CUDA(cudaMemcpyAsync(&key, w.key, sizeof(key), cudaMemcpyDeviceToHost, s));
            TSNET_CUDA(cudaStreamSynchronize(s));
            src = (int)(0xFFFFFFFFu - (unsigned)(key & 0xFFFFFFFFull));
        }
    }
    // exact sums of D2, means (same roundings as dividing the exact sums)
    k_pmds_rowsum<<<pb, 256, 0, s>>>(w.hops, n, p, w.rowsum);
    TSNET_LAUNCH_CHECK();
    TSNET_CUDA(cudaMemsetAsync(w.colsum, 0, sizeof(int64_t) * (size_t)p, s));
    k_pmds_colsum<<<dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 64)), (unsigned)p), 256, 0,
                    s>>>(w.hops, n, w.colsum);
    TSNET_LAUNCH_CHECK();
    std::vector<int64_t> cs(p);
    TSNET_CUDA(cudaMemcpyAsync(cs.data(), w.colsum, sizeof(int64_t) * (size_t)p, cudaMemcpyDeviceToHost, s));
    TSNET_CUDA(cudaStreamSynchronize(s));
    // means = exact integer sums divided once, as the definition (numpy's
    // pairwise fp64 sums of these integers are exact too)
    int64_t tot = 0;
    std::vector<double> cm(p);
    for (int k = 0; k < p; ++k) {
        tot += cs[k];
        cm[k] = (double)cs[k] / (double)n;
    }
    const PmdsMeans mm{w.rowsum, (double)p, (double)tot / ((double)n * (double)p)};
    TSNET_CUDA(cudaMemcpyAsync(w.cmean, cm.data(), sizeof(double) * (size_t)p, cudaMemcpyHostToDevice, s));
    // G = C^T C over row chunks, upper-triangle tiles
    TSNET_CUDA(cudaMemsetAsync(w.G, 0, sizeof(double) * (size_t)p * p, s));
    const int nt = (p + 31) / 32, ntiles = nt * (nt + 1) / 2;
    const int64_t chunks =
        std::max<int64_t>(1, std::min<int64_t>((n + 4095) / 4096, ((int64_t)kNumSMs * 8 + ntiles - 1) / ntiles));
    const int64_t rows_per = ((n + chunks - 1) / chunks + 31) / 32 * 32;
    k_pmds_gram<<<dim3((unsigned)((n + rows_per - 1) / rows_per), (unsigned)ntiles), 256, 0, s>>>(
        w.hops, n, p, mm, w.cmean, rows_per, w.G);
    TSNET_LAUNCH_CHECK();
    k_pmds_mirror<<<64, 256, 0, s>>>(w.G, p);
    TSNET_LAUNCH_CHECK();
    k_pmds_power<<<1, 1024, 0, s>>>(w.G, p, seed, w.V, w.lam);
    TSNET_LAUNCH_CHECK();
    k_pmds_embed<<<pb, 256, 0, s>>>(w.hops, n, p, mm, w.cmean, w.V, Y);
    TSNET_LAUNCH_CHECK();
    if (pivots_out)
        TSNET_CUDA(cudaMemcpyAsync(pivots_out, piv.data(), sizeof(int32_t) * (size_t)p, cudaMemcpyHostToDevice, s));
    if (hops_out)
        TSNET_CUDA(cudaMemcpyAsync(hops_out, w.hops, sizeof(int32_t) * (size_t)p * (size_t)n, cudaMemcpyDeviceToDevice,
                                   s));
    if (eig_out) TSNET_CUDA(cudaMemcpyAsync(eig_out, w.lam, sizeof(double) * 2, cudaMemcpyDeviceToDevice, s));
    TSNET_CUDA(cudaStreamSynchronize(s));   // host vectors above are sources of async copies
    return TSNET_OK;
}

}  // extern "C"
