// knn.cu -- C0 on the GPU: partial-BFS kNN, perplexity calibration and
// symmetrisation of P (Alg. 3 l.385-394; Eq. 2-3,
// PAPER.md:101-115; partial BFS §3.1).
//
//  k_knn    one warp per source v.  Level-synchronous BFS with two per-warp
//           shared-memory hash sets (visited, current level).  Pass A counts
//           the distinct vertices of the next level and stops as soon as the
//           count exceeds k - taken; if it fits, the whole level is taken.
//           Otherwise pass B streams the level once more and keeps the
//           k - taken smallest (SplitMix64(seed ^ (v<<32 | w)), w) -- the
//           reproducible reading R4 of "ties are broken randomly".
//  k_calib  one thread per row: beta by bisection on H(beta) = ln u over the
//           hop-distance runs of the row (R6, R7).
//  symmetrise: emit (i,j,p_j|i) and (j,i,p_j|i), radix-sort by i*n+j (CUB),
//           add equal keys, divide by 2n (fp64), drop zeros, write CSR.
#include <cub/cub.cuh>

#include <algorithm>

#include "common.cuh"

namespace tsnet {

constexpr int kKnnMax = 256;      // largest supported k
constexpr int kHash = 1024;       // per-warp hash set slots (power of two)
constexpr int kKnnWarps = 4;      // warps per CTA

struct KnnWarpSmem {
    int vis[kHash];
    int lvl[kHash];
    int tl_w[kKnnMax];
    int tl_h[kKnnMax];
    unsigned long long tk[kKnnMax];
    int tw[kKnnMax];
};

__device__ __forceinline__ uint64_t splitmix64_dev(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ unsigned hslot(int w) { return ((unsigned)w * 0x9E3779B1u) >> (32 - 10); }

__device__ __forceinline__ bool hset_insert(int* tab, int w) {
    unsigned h = hslot(w);
    while (true) {
        const int old = atomicCAS(&tab[h], -1, w);
        if (old == -1) return true;
        if (old == w) return false;
        h = (h + 1) & (kHash - 1);
    }
}

__device__ __forceinline__ bool hset_contains(const volatile int* tab, int w) {
    unsigned h = hslot(w);
    while (true) {
        const int x = tab[h];
        if (x == w) return true;
        if (x == -1) return false;
        h = (h + 1) & (kHash - 1);
    }
}

__device__ __forceinline__ bool key_less(unsigned long long ka, int wa, unsigned long long kb, int wb) {
    return ka < kb || (ka == kb && wa < wb);
}

// warp argmax of (tk, tw) over [0, s): returns position (all lanes)
__device__ __forceinline__ int warp_argmax(const KnnWarpSmem& S, int s, unsigned long long& mk, int& mw) {
    const int lane = threadIdx.x & 31;
    unsigned long long bk = 0;
    int bw = -1, bp = -1;
    for (int t = lane; t < s; t += 32) {
        const unsigned long long kk = S.tk[t];
        const int ww = S.tw[t];
        if (bp < 0 || key_less(bk, bw, kk, ww)) { bk = kk; bw = ww; bp = t; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long ok = __shfl_xor_sync(0xffffffffu, bk, o);
        const int ow = __shfl_xor_sync(0xffffffffu, bw, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp, o);
        if (op >= 0 && (bp < 0 || key_less(bk, bw, ok, ow))) { bk = ok; bw = ow; bp = op; }
    }
    mk = bk;
    mw = bw;
    return bp;
}

__global__ void __launch_bounds__(32 * kKnnWarps) k_knn(int64_t n, const int64_t* __restrict__ indptr,
                                                        const int32_t* __restrict__ indices, int k, uint64_t seed,
                                                        int32_t* __restrict__ knn_idx, int32_t* __restrict__ knn_hop,
                                                        int32_t* __restrict__ knn_len,
                                                        unsigned long long* __restrict__ total_len) {
    extern __shared__ KnnWarpSmem smw[];
    KnnWarpSmem& S = smw[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const unsigned FULL = 0xffffffffu;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long my_total = 0;
    for (int64_t v = wid; v < n; v += nw) {
        for (int i = lane; i < kHash; i += 32) S.vis[i] = -1;
        __syncwarp();
        if (lane == 0) hset_insert(S.vis, (int)v);
        __syncwarp();
        int taken = 0, fbeg = 0, fend = 0, d = 0;
        bool first = true;
        while (taken < k) {
            ++d;
            const int cap = k - taken;
            // ---- pass A: count distinct new vertices of level d (stop past cap)
            for (int i = lane; i < kHash; i += 32) S.lvl[i] = -1;
            __syncwarp();
            int cnt = 0;
            bool overflow = false;
            const int nf = first ? 1 : fend - fbeg;
            for (int fi = 0; fi < nf && !overflow; ++fi) {
                const int f = first ? (int)v : S.tl_w[fbeg + fi];
                const int64_t e0 = __ldg(indptr + f), e1 = __ldg(indptr + f + 1);
                for (int64_t e = e0; e < e1; e += 32) {
                    bool ins = false;
                    if (e + lane < e1) {
                        const int w = __ldg(indices + e + lane);
                        if (!hset_contains(S.vis, w)) ins = hset_insert(S.lvl, w);
                    }
                    cnt += __popc(__ballot_sync(FULL, ins));
                    if (cnt > cap) { overflow = true; break; }
                }
            }
            __syncwarp();
            if (cnt == 0) break;                       // component exhausted
            if (!overflow) {
                // take the whole level
                const int old = taken;
                for (int base = 0; base < kHash; base += 32) {
                    const int x = S.lvl[base + lane];
                    const bool has = x != -1;
                    const unsigned m = __ballot_sync(FULL, has);
                    if (has) {
                        const int pos = taken + __popc(m & lt_mask);
                        S.tl_w[pos] = x;
                        S.tl_h[pos] = d;
                    }
                    taken += __popc(m);
                }
                __syncwarp();
                for (int t = old + lane; t < taken; t += 32) hset_insert(S.vis, S.tl_w[t]);
                __syncwarp();
                fbeg = old;
                fend = taken;
                first = false;
                continue;
            }
            // ---- pass B: the cap smallest (key, w) of level d
            int s = 0, maxpos = -1, maxw = -1;
            unsigned long long maxk = 0;
            for (int fi = 0; fi < nf; ++fi) {
                const int f = first ? (int)v : S.tl_w[fbeg + fi];
                const int64_t e0 = __ldg(indptr + f), e1 = __ldg(indptr + f + 1);
                for (int64_t e = e0; e < e1; e += 32) {
                    int w = -1;
                    unsigned long long key = 0;
                    bool cand = false;
                    if (e + lane < e1) {
                        w = __ldg(indices + e + lane);
                        if (!hset_contains(S.vis, w)) {
                            key = splitmix64_dev(seed ^ (((unsigned long long)v << 32) | (unsigned)w));
                            cand = (s < cap) || key_less(key, w, maxk, maxw);
                        }
                    }
                    unsigned m = __ballot_sync(FULL, cand);
                    while (m) {
                        const int l = __ffs(m) - 1;
                        m &= m - 1;
                        const unsigned long long kk = __shfl_sync(FULL, key, l);
                        const int ww = __shfl_sync(FULL, w, l);
                        if (s == cap && !key_less(kk, ww, maxk, maxw)) continue;
                        bool dup = false;
                        for (int t = lane; t < s; t += 32) dup |= (S.tw[t] == ww);
                        if (__any_sync(FULL, dup)) continue;
                        const int slot = (s < cap) ? s : maxpos;
                        if (lane == 0) {
                            S.tk[slot] = kk;
                            S.tw[slot] = ww;
                        }
                        __syncwarp();
                        if (s < cap) ++s;
                        if (s == cap) maxpos = warp_argmax(S, s, maxk, maxw);
                        __syncwarp();
                    }
                }
            }
            for (int t = lane; t < s; t += 32) {
                S.tl_w[taken + t] = S.tw[t];
                S.tl_h[taken + t] = d;
            }
            taken += s;
            __syncwarp();
            break;
        }
        // ---- sort the row by (hop, w) (rank sort) and write it out
        int32_t* oi = knn_idx + v * (int64_t)k;
        int32_t* oh = knn_hop + v * (int64_t)k;
        for (int t = lane; t < taken; t += 32) {
            const int h = S.tl_h[t], w = S.tl_w[t];
            int r = 0;
            for (int q = 0; q < taken; ++q) {
                const int hq = S.tl_h[q], wq = S.tl_w[q];
                r += (hq < h) || (hq == h && wq < w);
            }
            oi[r] = w;
            oh[r] = h;
        }
        for (int t = taken + lane; t < k; t += 32) {
            oi[t] = -1;
            oh[t] = -1;
        }
        if (lane == 0) knn_len[v] = taken;
        my_total += (unsigned long long)taken;
        __syncwarp();
    }
    if (lane == 0 && my_total) atomicAdd(total_len, my_total);
}

// Entropy (nats) H(beta) = ln S + beta sum_j D_j e_j / S, summed over the runs
// of equal hop distance of the (sorted) row (Eq. 3).
__device__ double row_entropy_runs(const int32_t* hop, int len, int dmin, double beta) {
    double S = 0.0, SD = 0.0;
    for (int t = 0; t < len;) {
        const int h = hop[t];
        int c = 1;
        while (t + c < len && hop[t + c] == h) ++c;
        const double D = (double)h * h - (double)dmin * dmin;
        const double e = exp(-beta * D);
        S += c * e;
        SD += c * D * e;
        t += c;
    }
    return log(S) + beta * SD / S;
}

__global__ void __launch_bounds__(256) k_calib(int64_t n, int k, double u, const int32_t* __restrict__ knn_hop,
                                               const int32_t* __restrict__ knn_len, double* __restrict__ p_cond,
                                               double* __restrict__ beta_out, unsigned long long* __restrict__ unreach) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int len = knn_len[v];
        const int32_t* hop = knn_hop + v * (int64_t)k;
        double* p = p_cond + v * (int64_t)k;
        double beta = 0.0;
        if (len > 0) {
            const int dmin = hop[0];             // rows are sorted by hop
            int cmin = 1;
            while (cmin < len && hop[cmin] == dmin) ++cmin;
            if ((double)len <= u) {
                for (int t = 0; t < len; ++t) p[t] = 1.0 / (double)len;
            } else if ((double)cmin >= u) {
                beta = INFINITY;
                for (int t = 0; t < len; ++t) p[t] = (hop[t] == dmin) ? 1.0 / (double)cmin : 0.0;
                atomicAdd(unreach, 1ull);
            } else {
                const double Hs = log(u);
                double lo = 0.0, hi = INFINITY;
                beta = 1.0;
                for (int it = 0; it < 200; ++it) {
                    const double diff = row_entropy_runs(hop, len, dmin, beta) - Hs;
                    if (fabs(diff) <= 1e-13) break;
                    if (diff > 0) {
                        lo = beta;
                        beta = isinf(hi) ? 2.0 * beta : 0.5 * (lo + hi);
                    } else {
                        hi = beta;
                        beta = 0.5 * (lo + hi);
                    }
                    if (!isinf(hi) && nextafter(nextafter(lo, INFINITY), INFINITY) >= hi) break;
                }
                double S = 0.0;
                for (int t = 0; t < len;) {
                    const int h = hop[t];
                    int c = 1;
                    while (t + c < len && hop[t + c] == h) ++c;
                    S += c * exp(-beta * ((double)h * h - (double)dmin * dmin));
                    t += c;
                }
                for (int t = 0; t < len; ++t) p[t] = exp(-beta * ((double)hop[t] * hop[t] - (double)dmin * dmin)) / S;
            }
        }
        if (beta_out) beta_out[v] = beta;
    }
}

__global__ void k_sym_emit(int64_t n, int k, const int32_t* __restrict__ knn_idx, const int32_t* __restrict__ knn_len,
                           const double* __restrict__ p_cond, unsigned long long* __restrict__ keys,
                           double* __restrict__ vals) {
    const unsigned long long sentinel = (unsigned long long)n * (unsigned long long)n;
    const int64_t tot = n * (int64_t)k;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < tot; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = q / k;
        const int t = (int)(q - v * k);
        if (t < knn_len[v]) {
            const unsigned long long w = (unsigned long long)knn_idx[q];
            const double p = p_cond[q];
            keys[2 * q] = (unsigned long long)v * n + w;
            keys[2 * q + 1] = w * n + (unsigned long long)v;
            vals[2 * q] = p;
            vals[2 * q + 1] = p;
        } else {
            keys[2 * q] = sentinel;
            keys[2 * q + 1] = sentinel;
            vals[2 * q] = 0.0;
            vals[2 * q + 1] = 0.0;
        }
    }
}

// heads of equal-key runs: p_ij = (p_j|i + p_i|j) / (2n) (Eq. 2)
__global__ void k_sym_flag(int64_t n, int64_t L, const unsigned long long* __restrict__ keys,
                           const double* __restrict__ vals, double* __restrict__ psum, int* __restrict__ flag) {
    const unsigned long long sentinel = (unsigned long long)n * (unsigned long long)n;
    const double two_n = 2.0 * (double)n;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < L; s += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = keys[s];
        int f = 0;
        double pij = 0.0;
        if (key < sentinel && (s == 0 || keys[s - 1] != key)) {
            double sum = vals[s];
            if (s + 1 < L && keys[s + 1] == key) sum += vals[s + 1];
            pij = sum / two_n;
            f = (pij != 0.0);
        }
        flag[s] = f;
        psum[s] = pij;
    }
}

__global__ void k_sym_write(int64_t n, int64_t L, const unsigned long long* __restrict__ keys,
                            const double* __restrict__ psum, const int* __restrict__ flag, const int* __restrict__ pos,
                            int32_t* __restrict__ indices, float* __restrict__ values, int* __restrict__ rows) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < L; s += (int64_t)gridDim.x * blockDim.x) {
        if (!flag[s]) continue;
        const int e = pos[s];
        const unsigned long long key = keys[s];
        indices[e] = (int32_t)(key % (unsigned long long)n);
        values[e] = (float)psum[s];
        rows[e] = (int)(key / (unsigned long long)n);
    }
}

__global__ void k_sym_indptr(int64_t n, int64_t nnz, const int* __restrict__ rows, int64_t* __restrict__ indptr) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x) {
        const int r = rows[e];
        const int rp = (e == 0) ? -1 : rows[e - 1];
        for (int rr = rp + 1; rr <= r; ++rr) indptr[rr] = e;
        if (e == nnz - 1)
            for (int64_t rr = r + 1; rr <= n; ++rr) indptr[rr] = nnz;
    }
}

// ----------------------------------------------------------------- host side
struct BuildWs {
    double* p_cond;
    unsigned long long* keys_a;
    unsigned long long* keys_b;
    double* vals_a;
    double* vals_b;
    int* flag;
    int* pos;
    int* rows;
    unsigned long long* counters;   // [0] total kNN entries, [1] unreachable rows
    void* cub_tmp;
    size_t cub_bytes;
    size_t bytes;
};

static size_t cub_tmp_bytes(int64_t L) {
    size_t a = 0, b = 0;
    cub::DoubleBuffer<unsigned long long> dk(nullptr, nullptr);
    cub::DoubleBuffer<double> dv(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, a, dk, dv, (int)L, 0, 64);
    cub::DeviceScan::ExclusiveSum(nullptr, b, (int*)nullptr, (int*)nullptr, (int)L);
    return std::max(a, b);
}

static BuildWs build_ws_map(void* base, int64_t n, int k) {
    BuildWs w{};
    const int64_t nk = n * (int64_t)k, L = 2 * nk;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off = align_up(off + bytes, 256);
        return (char*)base + o;
    };
    w.p_cond = (double*)take(sizeof(double) * nk);
    w.keys_a = (unsigned long long*)take(8 * L);
    w.keys_b = (unsigned long long*)take(8 * L);
    w.vals_a = (double*)take(8 * L);
    w.vals_b = (double*)take(8 * L);
    w.flag = (int*)take(4 * L);
    w.pos = (int*)take(4 * L);
    w.rows = (int*)take(4 * L);
    w.counters = (unsigned long long*)take(64);
    w.cub_bytes = cub_tmp_bytes(L > 0 ? L : 1);
    w.cub_tmp = take(w.cub_bytes);
    w.bytes = off;
    return w;
}

size_t build_P_ws_bytes(int64_t n, int k) { return build_ws_map(nullptr, n, k).bytes; }

int build_P_impl(const tsnet_graph* g, double u, int k, uint64_t seed, tsnet_csr* P, int32_t* knn_idx,
                 int32_t* knn_hop, int32_t* knn_len, double* beta, void* ws, size_t ws_bytes, cudaStream_t s) {
    const int64_t n = g->n;
    BuildWs w = build_ws_map(ws, n, k);
    TSNET_ARG(ws_bytes >= w.bytes, "tsnet_build_P: workspace too small (%zu < %zu)", ws_bytes, w.bytes);
    const int64_t L = 2 * n * (int64_t)k;
    TSNET_ARG(L < (int64_t)0x7FFFFFFF, "tsnet_build_P: 2 n k = %lld exceeds the int32 scan range", (long long)L);
    TSNET_CUDA(cudaMemsetAsync(w.counters, 0, 64, s));
    const size_t smem = sizeof(KnnWarpSmem) * kKnnWarps;
    TSNET_CUDA(cudaFuncSetAttribute(k_knn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (n > 0) {
        const int blocks = (int)std::min<int64_t>((n + kKnnWarps - 1) / kKnnWarps, (int64_t)kNumSMs * 16);
        k_knn<<<blocks, 32 * kKnnWarps, smem, s>>>(n, g->indptr, g->indices, k, seed, knn_idx, knn_hop, knn_len,
                                                   w.counters);
        TSNET_LAUNCH_CHECK();
        const int cb = (int)std::min<int64_t>((n + 255) / 256, (int64_t)kNumSMs * 8);
        k_calib<<<cb, 256, 0, s>>>(n, k, u, knn_hop, knn_len, w.p_cond, beta, w.counters + 1);
        TSNET_LAUNCH_CHECK();
    }
    int64_t nnz = 0;
    unsigned long long cnt[2] = {0, 0};
    if (L > 0) {
        const int eb = (int)std::min<int64_t>((n * (int64_t)k + 255) / 256, (int64_t)kNumSMs * 16);
        k_sym_emit<<<eb, 256, 0, s>>>(n, k, knn_idx, knn_len, w.p_cond, w.keys_a, w.vals_a);
        TSNET_LAUNCH_CHECK();
        const unsigned long long maxkey = (unsigned long long)n * (unsigned long long)n;
        int end_bit = 64 - __builtin_clzll(maxkey | 1ull);
        cub::DoubleBuffer<unsigned long long> dk(w.keys_a, w.keys_b);
        cub::DoubleBuffer<double> dv(w.vals_a, w.vals_b);
        size_t tb = w.cub_bytes;
        TSNET_CUDA(cub::DeviceRadixSort::SortPairs(w.cub_tmp, tb, dk, dv, (int)L, 0, end_bit, s));
        unsigned long long* ks = dk.Current();
        double* vs = dv.Current();
        double* psum = dv.Alternate();
        const int fb = (int)std::min<int64_t>((L + 255) / 256, (int64_t)kNumSMs * 16);
        k_sym_flag<<<fb, 256, 0, s>>>(n, L, ks, vs, psum, w.flag);
        TSNET_LAUNCH_CHECK();
        tb = w.cub_bytes;
        TSNET_CUDA(cub::DeviceScan::ExclusiveSum(w.cub_tmp, tb, w.flag, w.pos, (int)L, s));
        int last[2];
        TSNET_CUDA(cudaMemcpyAsync(&last[0], w.pos + (L - 1), sizeof(int), cudaMemcpyDeviceToHost, s));
        TSNET_CUDA(cudaMemcpyAsync(&last[1], w.flag + (L - 1), sizeof(int), cudaMemcpyDeviceToHost, s));
        TSNET_CUDA(cudaMemcpyAsync(cnt, w.counters, sizeof(cnt), cudaMemcpyDeviceToHost, s));
        TSNET_CUDA(cudaStreamSynchronize(s));
        nnz = (int64_t)last[0] + last[1];
        if (nnz > P->capacity) {
            P->nnz = nnz;
            set_error("tsnet_build_P: P capacity %lld < required nnz %lld", (long long)P->capacity, (long long)nnz);
            return TSNET_E_CAPACITY;
        }
        k_sym_write<<<fb, 256, 0, s>>>(n, L, ks, psum, w.flag, w.pos, P->indices, P->values, w.rows);
        TSNET_LAUNCH_CHECK();
    }
    TSNET_CUDA(cudaMemsetAsync(P->indptr, 0, sizeof(int64_t) * (size_t)(n + 1), s));
    if (nnz > 0) {
        const int ib = (int)std::min<int64_t>((nnz + 255) / 256, (int64_t)kNumSMs * 16);
        k_sym_indptr<<<ib, 256, 0, s>>>(n, nnz, w.rows, P->indptr);
        TSNET_LAUNCH_CHECK();
    }
    TSNET_CUDA(cudaStreamSynchronize(s));
    P->nnz = nnz;
    P->n = n;
    return cnt[1] > 0 ? TSNET_W_PERPLEXITY : TSNET_OK;
}

}  // namespace tsnet
