// attr_cb.cu -- column-blocked attractive SpMV (step a6, Eq. 6 first term,
// PAPER.md:162): F_attr,i = sum_{j in row i} p_ij w_ij (X_i - X_j).
//
// Why a second layout of P: on the power-law graph of config 4
// the CSR kernel (iterate.cu k_spmv) is bound by the L1TEX->L2 request path,
// not by HBM -- every Y[j] gather is its own 32-B sector request (ncu r1a:
// 2.75e8 L2 read sectors per launch against 5.2e7 for the CSR stream, 23% of
// DRAM peak).  Here Y is read from shared memory instead:
//
//   * rows are cut into T tasks (contiguous row ranges, nnz-balanced, at most
//     kCbRowsMax rows), one persistent CTA per SM walks its tasks;
//   * columns are cut into blocks of kCbCols points; a task's entries are
//     stored block by block ("segments"), each entry 8 bytes:
//       word0 = (row - task_row0) << 16 | (col - block_col0),  word1 = p_ij (fp32 bits),
//     rows ascending inside a segment, segments padded to an even length;
//   * a producer warp streams the Y slice of each non-empty block into a
//     double-buffered shared-memory tile with cp.async.bulk (TMA bulk copy,
//     mbarrier completion) while the consumer warps stream the segment's
//     entries from HBM (coalesced 16-B loads, L2 evict-first), gather Y_j from
//     shared memory, and reduce runs of equal rows with a warp segmented scan
//     into a per-task shared-memory accumulator F_s (fp32 shared atomics at run
//     ends only);
//   * at the end of a task F_s is written to F with plain stores (no global
//     atomics, no memset of F).
// HBM bytes per launch: 8 per stored entry (+ padding) + 8 per (task, block)
// segment offset + 8 per row written; Y slices come from L2.
#include <algorithm>
#include <cstring>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"

namespace tsnet {

constexpr int kCbCols = 8192;       // points per column block (2 x 64 KB shared tiles)
constexpr int kCbRowsMax = 11264;   // rows per task (88 KB shared accumulator)
constexpr int kCbWarps = 16;        // consumer warps per CTA (+1 producer warp)
constexpr int kCbThreads = (kCbWarps + 1) * 32;
constexpr uint32_t kCbSentinel = 0xFFFFu;
constexpr uint64_t kCbMagic = 0x4243544e53545354ull;  // "TSTSNTCB"

struct CbHeader {
    uint64_t magic;
    int64_t n, row_begin, row_end, nnz, entries;
    int32_t T, NB, C, rows_max;
    int64_t off_row0, off_rows, off_seg, off_entries, bytes;
};

static size_t cb_align(size_t x) { return (x + 255) / 256 * 256; }

static CbHeader cb_layout(int64_t n, int64_t rb, int64_t re, int64_t nnz, int32_t T) {
    CbHeader h{};
    h.magic = kCbMagic;
    h.n = n;
    h.row_begin = rb;
    h.row_end = re;
    h.nnz = nnz;
    h.T = T;
    h.C = kCbCols;
    h.NB = (int32_t)((n + kCbCols - 1) / kCbCols);
    h.rows_max = kCbRowsMax;
    const int64_t nseg = (int64_t)T * h.NB;
    h.entries = nnz + nseg;   // upper bound with padding
    size_t off = cb_align(sizeof(CbHeader));
    h.off_row0 = (int64_t)off;
    off = cb_align(off + sizeof(int64_t) * (size_t)T);
    h.off_rows = (int64_t)off;
    off = cb_align(off + sizeof(int32_t) * (size_t)T);
    h.off_seg = (int64_t)off;
    off = cb_align(off + sizeof(int64_t) * (size_t)(nseg + 1));
    h.off_entries = (int64_t)off;
    off = cb_align(off + sizeof(uint2) * (size_t)h.entries);
    h.bytes = (int64_t)off;
    return h;
}

// Host partition of rows [rb, re) into tasks: T = 148 w (w = 1, 2, ...) tasks,
// nnz-balanced (greedy cut at multiples of nnz/T) with at most rows_max rows.
// ipr[q] = indptr[rb + q], q = 0 .. re - rb.
static int32_t cb_partition(const int64_t* ipr, int64_t rb, int64_t re, int32_t rows_max, int32_t base,
                            std::vector<int64_t>& row0, std::vector<int32_t>& rows) {
    const int64_t nr = re - rb;
    const int64_t nnz = ipr[nr] - ipr[0];
    if (nr <= 0) {
        row0.assign(1, rb);
        rows.assign(1, 0);
        return 1;
    }
    for (int32_t w = 1; w < (1 << 20); ++w) {
        const int64_t T = (int64_t)base * w;
        row0.clear();
        rows.clear();
        int64_t r = rb;
        bool ok = true;
        for (int64_t t = 0; t < T && ok; ++t) {
            const int64_t target = ipr[0] + (nnz * (t + 1) + T - 1) / T;
            int64_t r1 = r;
            // extend while the next row's start is below the target and the cap allows
            while (r1 < re && ipr[r1 - rb] < target && r1 - r < rows_max) ++r1;
            if (t == T - 1 && r1 < re) ok = false;
            row0.push_back(r);
            rows.push_back((int32_t)(r1 - r));
            r = r1;
        }
        if (ok && r == re) return (int32_t)T;
    }
    return -1;
}

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ uint64_t cb_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint4 ld_stream_v4(const uint4* a, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ------------------------------------------------------------------ kernel
// Run-end update of the shared accumulator.  Inside one block segment a row is
// shared between warps only at the two ends of a warp's share (keys kf, kl):
// those go through atomicAdd (a CAS loop on shared fp32, rare); every other row
// of the share is owned by this warp for the block, so a plain read-modify-write
// suffices (flush keys within one sweep are distinct; sweeps of a warp are
// ordered by __syncwarp; blocks are separated by a consumer barrier).
__device__ __forceinline__ void cb_flush(float* Fs, uint32_t k, float x, float y, uint32_t kf, uint32_t kl) {
    if (k == kf || k == kl) {
        atomicAdd(Fs + 2 * k, x);
        atomicAdd(Fs + 2 * k + 1, y);
    } else {
        float2* f = reinterpret_cast<float2*>(Fs) + k;
        float2 v = *f;
        v.x += x;
        v.y += y;
        *f = v;
    }
}

// One entry: contribution p w (X_i - X_j) with w = 1 / (1 + r^2).
__device__ __forceinline__ void cb_term(uint32_t word, uint32_t vbits, const float2* __restrict__ Ys,
                                        const float2* __restrict__ Yrow, uint32_t& key, float& fx, float& fy) {
    key = word >> 16;
    if (key == kCbSentinel) {
        fx = 0.f;
        fy = 0.f;
        return;
    }
    const float2 yj = Ys[word & 0xFFFFu];
    const float2 yi = __ldg(Yrow + key);
    const float dx = yi.x - yj.x, dy = yi.y - yj.y;
    const float w = __frcp_rn(1.0f + dx * dx + dy * dy);
    const float pw = __uint_as_float(vbits) * w;
    fx = pw * dx;
    fy = pw * dy;
}

// Process one sweep: lane holds entries 4 lane .. 4 lane + 3 of 128 consecutive
// entries (keys non-decreasing across the sweep; masked entries carry the
// sentinel key and sit at the end).
__device__ __forceinline__ void cb_sweep(uint4 a, uint4 b, const float2* __restrict__ Ys,
                                         const float2* __restrict__ Yrow, float* Fs, int lane, uint32_t kf,
                                         uint32_t kl) {
    uint32_t k[4];
    float fx[4], fy[4];
    cb_term(a.x, a.y, Ys, Yrow, k[0], fx[0], fy[0]);
    cb_term(a.z, a.w, Ys, Yrow, k[1], fx[1], fy[1]);
    cb_term(b.x, b.y, Ys, Yrow, k[2], fx[2], fy[2]);
    cb_term(b.z, b.w, Ys, Yrow, k[3], fx[3], fy[3]);
    // runs inside the lane: head (first run, if the lane has >= 2 runs), middles, tail
    uint32_t hk = kCbSentinel, tk = k[0];
    float hx = 0.f, hy = 0.f, tx = fx[0], ty = fy[0];
    bool open_first = true;
#pragma unroll
    for (int q = 1; q < 4; ++q) {
        if (k[q] == tk) {
            tx += fx[q];
            ty += fy[q];
        } else {
            if (open_first) {
                hk = tk;
                hx = tx;
                hy = ty;
                open_first = false;
            } else if (tk != kCbSentinel) {
                cb_flush(Fs, tk, tx, ty, kf, kl);
            }
            tk = k[q];
            tx = fx[q];
            ty = fy[q];
        }
    }
    // segmented inclusive scan of the tails over lanes (keys sorted => runs contiguous)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t uk = __shfl_up_sync(0xffffffffu, tk, o);
        const float ux = __shfl_up_sync(0xffffffffu, tx, o);
        const float uy = __shfl_up_sync(0xffffffffu, ty, o);
        if (lane >= o && uk == tk) {
            tx += ux;
            ty += uy;
        }
    }
    const uint32_t nk = __shfl_down_sync(0xffffffffu, tk, 1);
    const uint32_t pk = __shfl_up_sync(0xffffffffu, tk, 1);
    const bool last = (lane == 31) || (nk != tk);
    // a head run continues the previous lane's tail run, or stands alone
    const bool give = (hk != kCbSentinel) && lane > 0 && hk == pk;
    if (hk != kCbSentinel && !give) cb_flush(Fs, hk, hx, hy, kf, kl);
    const float gx = __shfl_down_sync(0xffffffffu, give ? hx : 0.f, 1);
    const float gy = __shfl_down_sync(0xffffffffu, give ? hy : 0.f, 1);
    if (last && tk != kCbSentinel) {
        const bool got = (lane < 31);
        cb_flush(Fs, tk, tx + (got ? gx : 0.f), ty + (got ? gy : 0.f), kf, kl);
    }
}

__global__ void __launch_bounds__(kCbThreads, 1) k_attr_cb(const uint8_t* __restrict__ plan, const float2* __restrict__ Y,
                                                           float2* __restrict__ F, int y_aligned) {
    extern __shared__ __align__(128) uint8_t cb_smem[];
    float2* Ys0 = reinterpret_cast<float2*>(cb_smem);
    float2* Ys1 = Ys0 + kCbCols;
    float* Fs = reinterpret_cast<float*>(Ys1 + kCbCols);
    uint64_t* bars = reinterpret_cast<uint64_t*>(Fs + 2 * kCbRowsMax);   // full[2], empty[2]
    const CbHeader* h = reinterpret_cast<const CbHeader*>(plan);
    const int T = h->T, NB = h->NB;
    const int64_t n = h->n, rb = h->row_begin;
    const int64_t* row0s = reinterpret_cast<const int64_t*>(plan + h->off_row0);
    const int32_t* rowss = reinterpret_cast<const int32_t*>(plan + h->off_rows);
    const int64_t* seg = reinterpret_cast<const int64_t*>(plan + h->off_seg);
    const uint4* ent = reinterpret_cast<const uint4*>(plan + h->off_entries);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], kCbWarps);
        mbar_init(&bars[3], kCbWarps);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kCbWarps) {
        // ---------------- producer: Y slices of the non-empty blocks, in order
        uint32_t k = 0;
        for (int t = blockIdx.x; t < T; t += gridDim.x) {
            const int64_t* sg = seg + (int64_t)t * NB;
            for (int J = 0; J < NB; ++J) {
                if (sg[J] == sg[J + 1]) continue;
                const int b = k & 1;
                float2* dst = b ? Ys1 : Ys0;
                if (k >= 2) mbar_wait(&bars[2 + b], ((k >> 1) - 1) & 1);
                const int64_t lo = (int64_t)J * kCbCols;
                const int cnt = (int)std::min<int64_t>(kCbCols, n - lo);
                if (y_aligned) {
                    const int even = cnt & ~1;
                    if (lane == 0) {
                        if (cnt & 1) dst[cnt - 1] = Y[lo + cnt - 1];
                        mbar_arrive_tx(&bars[b], (uint32_t)(even * sizeof(float2)));
                        if (even) bulk_g2s(dst, Y + lo, (uint32_t)(even * sizeof(float2)), &bars[b]);
                    }
                } else {
                    for (int q = lane; q < cnt; q += 32) dst[q] = Y[lo + q];
                    __threadfence_block();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bars[b]);
                }
                __syncwarp();
                ++k;
            }
        }
        return;
    }

    // ---------------- consumers
    const uint64_t pol = cb_policy_evict_first();
    const int nthr = kCbWarps * 32;
    uint32_t k = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
        const int64_t row0 = row0s[t];
        const int rows = rowss[t];
        const float2* Yrow = Y + row0;
        for (int q = threadIdx.x; q < 2 * rows; q += nthr) Fs[q] = 0.f;
        named_bar(1, nthr);
        const int64_t* sg = seg + (int64_t)t * NB;
        for (int J = 0; J < NB; ++J) {
            const int64_t s0 = sg[J], s1 = sg[J + 1];
            if (s0 == s1) continue;
            const int b = k & 1;
            const float2* Ys = b ? Ys1 : Ys0;
            // this warp's share of the segment, in pairs of entries (16 B)
            const int64_t p0 = s0 >> 1, np = (s1 - s0) >> 1;
            const int64_t per = (np + kCbWarps - 1) / kCbWarps;
            const int64_t w0 = p0 + std::min<int64_t>(np, per * warp), w1 = p0 + std::min<int64_t>(np, per * (warp + 1));
            const uint4 pad = make_uint4(kCbSentinel << 16, 0u, kCbSentinel << 16, 0u);
            int64_t p = w0;
            uint4 a = pad, c = pad;
            if (p + 2 * lane < w1) a = ld_stream_v4(ent + p + 2 * lane, pol);
            if (p + 2 * lane + 1 < w1) c = ld_stream_v4(ent + p + 2 * lane + 1, pol);
            // keys of the share's first and last entries (rows possibly shared with neighbours)
            uint32_t kf = kCbSentinel, kl = kCbSentinel;
            if (w0 < w1) {
                kf = __shfl_sync(0xffffffffu, a.x, 0) >> 16;
                kl = __ldg(reinterpret_cast<const uint32_t*>(ent + w1 - 1) + 2) >> 16;
            }
            mbar_wait(&bars[b], (k >> 1) & 1);
            for (; p < w1; p += 64) {
                uint4 a2 = pad, c2 = pad;
                const int64_t pn = p + 64;
                if (pn + 2 * lane < w1) a2 = ld_stream_v4(ent + pn + 2 * lane, pol);
                if (pn + 2 * lane + 1 < w1) c2 = ld_stream_v4(ent + pn + 2 * lane + 1, pol);
                cb_sweep(a, c, Ys, Yrow, Fs, lane, kf, kl);
                __syncwarp();
                a = a2;
                c = c2;
            }
            if (lane == 0) mbar_arrive(&bars[2 + b]);
            ++k;
            named_bar(1, nthr);   // rows owned by one warp in this block may be shared in the next
        }
        named_bar(1, nthr);
        float2* Fo = F + (row0 - rb);
        const float2* Fs2 = reinterpret_cast<const float2*>(Fs);
        for (int q = threadIdx.x; q < rows; q += nthr) Fo[q] = Fs2[q];
        named_bar(1, nthr);
    }
}

size_t cb_smem_bytes() { return sizeof(float2) * 2 * kCbCols + sizeof(float) * 2 * kCbRowsMax + 4 * sizeof(uint64_t); }

static int num_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = kNumSMs;
    }
    return sms;
}

cudaError_t launch_attr_cb(const void* plan, const float2* Y, float2* F, cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_attr_cb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cb_smem_bytes());
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int aligned = ((uintptr_t)Y % 16) == 0;
    k_attr_cb<<<num_sms(), kCbThreads, cb_smem_bytes(), s>>>(reinterpret_cast<const uint8_t*>(plan), Y, F, aligned);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ plan build
// Sort keys: (task, block) of every entry of the shard; payload: the packed
// 8-byte entry.  A stable LSD radix sort keeps the CSR (row, col) order inside
// each segment.
__global__ void k_cb_row_task(const int64_t* row0, const int32_t* rows, int T, int64_t rb, int32_t* row_task) {
    for (int t = blockIdx.x; t < T; t += gridDim.x)
        for (int q = threadIdx.x; q < rows[t]; q += blockDim.x) row_task[row0[t] - rb + q] = t;
}

__global__ void k_cb_keys(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                          const float* __restrict__ values, int64_t rb, int64_t re, const int64_t* __restrict__ row0,
                          const int32_t* __restrict__ row_task, int NB, uint32_t* __restrict__ keys,
                          unsigned long long* __restrict__ vals) {
    const int lane = threadIdx.x & 31;
    const int64_t e0 = indptr[rb];
    for (int64_t r = rb + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); r < re;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int t = row_task[r - rb];
        const uint32_t lr = (uint32_t)(r - row0[t]);
        for (int64_t e = indptr[r] + lane; e < indptr[r + 1]; e += 32) {
            const int32_t c = indices[e];
            const int J = c / kCbCols;
            keys[e - e0] = (uint32_t)t * (uint32_t)NB + (uint32_t)J;
            const uint32_t word = (lr << 16) | (uint32_t)(c - J * kCbCols);
            vals[e - e0] = ((unsigned long long)__float_as_uint(values[e]) << 32) | word;
        }
    }
}

// segment start / end positions in the sorted order (empty segments stay 0, 0)
__global__ void k_cb_bounds(const uint32_t* __restrict__ keys, int64_t m, int64_t* __restrict__ sstart,
                            int64_t* __restrict__ send) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = keys[q];
        if (q == 0 || keys[q - 1] != k) sstart[k] = q;
        if (q == m - 1 || keys[q + 1] != k) send[k] = q + 1;
    }
}

// send -> padded (even) segment length, in place
__global__ void k_cb_pad(const int64_t* __restrict__ sstart, int64_t* __restrict__ slen, int64_t nseg) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nseg; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t L = slen[q] - sstart[q];
        slen[q] = L + (L & 1);
    }
}

__global__ void k_cb_fill(const uint32_t* __restrict__ keys, const unsigned long long* __restrict__ vals, int64_t m,
                          const int64_t* __restrict__ sstart, const int64_t* __restrict__ seg, uint2* __restrict__ ent) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = keys[q];
        const unsigned long long v = vals[q];
        const int64_t pos = seg[k] + (q - sstart[k]);
        ent[pos] = make_uint2((uint32_t)v, (uint32_t)(v >> 32));
        // odd segment: duplicate the last entry's key with p = 0 (keeps rows sorted)
        const bool lastq = (q == m - 1) || keys[q + 1] != k;
        if (lastq && pos + 1 < seg[k + 1]) ent[pos + 1] = make_uint2((uint32_t)v, 0u);
    }
}

struct CbWs {
    int32_t* row_task;
    uint32_t *keys_a, *keys_b;
    unsigned long long *vals_a, *vals_b;
    int64_t *sstart, *slen;
    void* cub_tmp;
    size_t cub_bytes, bytes;
};

static CbWs cb_ws_map(void* base, int64_t nr, int64_t m, int64_t nseg) {
    CbWs w{};
    size_t cb = 0, cs = 0;
    cub::DoubleBuffer<uint32_t> dk(nullptr, nullptr);
    cub::DoubleBuffer<unsigned long long> dv(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, cb, dk, dv, (int64_t)std::max<int64_t>(m, 1), 0, 32);
    cub::DeviceScan::ExclusiveSum(nullptr, cs, (int64_t*)nullptr, (int64_t*)nullptr, (int64_t)(nseg + 1));
    w.cub_bytes = std::max(cb, cs);
    size_t off = 0;
    auto take = [&](size_t b) {
        size_t o = off;
        off = cb_align(off + b);
        return (char*)base + o;
    };
    w.row_task = (int32_t*)take(sizeof(int32_t) * std::max<int64_t>(nr, 1));
    w.keys_a = (uint32_t*)take(sizeof(uint32_t) * std::max<int64_t>(m, 1));
    w.keys_b = (uint32_t*)take(sizeof(uint32_t) * std::max<int64_t>(m, 1));
    w.vals_a = (unsigned long long*)take(sizeof(unsigned long long) * std::max<int64_t>(m, 1));
    w.vals_b = (unsigned long long*)take(sizeof(unsigned long long) * std::max<int64_t>(m, 1));
    w.sstart = (int64_t*)take(sizeof(int64_t) * (nseg + 1));
    w.slen = (int64_t*)take(sizeof(int64_t) * (nseg + 1));
    w.cub_tmp = take(w.cub_bytes);
    w.bytes = off;
    return w;
}

static int cb_rows(const tsnet_csr* P, const tsnet_shard* sh, int64_t& rb, int64_t& re) {
    rb = 0;
    re = P->n;
    if (sh) {
        rb = sh->row_begin;
        re = sh->row_end;
    }
    TSNET_ARG(0 <= rb && rb <= re && re <= P->n, "shard rows [%lld, %lld) outside [0, %lld)", (long long)rb,
              (long long)re, (long long)P->n);
    TSNET_ARG(P->n < (int64_t)1 << 31, "n >= 2^31 is not supported");
    return TSNET_OK;
}

static int cb_host_partition(const tsnet_csr* P, int64_t rb, int64_t re, cudaStream_t s, std::vector<int64_t>& row0,
                             std::vector<int32_t>& rows, int64_t& nnz_s) {
    std::vector<int64_t> ip(re - rb + 1);
    TSNET_CUDA(cudaMemcpyAsync(ip.data(), P->indptr + rb, sizeof(int64_t) * ip.size(), cudaMemcpyDeviceToHost, s));
    TSNET_CUDA(cudaStreamSynchronize(s));
    nnz_s = ip.back() - ip.front();
    TSNET_ARG(nnz_s < ((int64_t)1 << 31), "a plan holds < 2^31 entries per shard (got %lld)", (long long)nnz_s);
    const int32_t T = cb_partition(ip.data(), rb, re, kCbRowsMax, num_sms(), row0, rows);
    TSNET_ARG(T > 0, "row partition failed");
    return TSNET_OK;
}

}  // namespace tsnet

using namespace tsnet;

extern "C" {

int32_t tsnet_plan_partition(const int64_t* indptr_host, int64_t row_begin, int64_t row_end, int32_t rows_max,
                             int32_t base_tasks, int32_t max_tasks, int64_t* task_row0, int32_t* task_rows) {
    if (!indptr_host || row_begin < 0 || row_end < row_begin || rows_max < 1 || base_tasks < 1) return -1;
    std::vector<int64_t> row0;
    std::vector<int32_t> rows;
    const int32_t T = cb_partition(indptr_host + row_begin, row_begin, row_end, rows_max, base_tasks, row0, rows);
    if (T < 0 || T > max_tasks) return -1;
    std::memcpy(task_row0, row0.data(), sizeof(int64_t) * T);
    std::memcpy(task_rows, rows.data(), sizeof(int32_t) * T);
    return T;
}

int tsnet_plan_query(const tsnet_csr* P, const tsnet_shard* shard, size_t* plan_bytes, size_t* ws_bytes,
                     tsnet_stream_t stream) {
    TSNET_ARG(P != nullptr && plan_bytes != nullptr && ws_bytes != nullptr, "NULL argument");
    TSNET_ARG(P->n >= 0 && P->nnz >= 0 && (P->n == 0 || P->indptr), "invalid P");
    int64_t rb, re;
    int st = cb_rows(P, shard, rb, re);
    if (st != TSNET_OK) return st;
    std::vector<int64_t> row0;
    std::vector<int32_t> rows;
    int64_t m = 0;
    if (P->n == 0) {
        row0.assign(1, 0);
        rows.assign(1, 0);
    } else if ((st = cb_host_partition(P, rb, re, (cudaStream_t)stream, row0, rows, m)) != TSNET_OK) {
        return st;
    }
    const CbHeader h = cb_layout(P->n, rb, re, m, (int32_t)row0.size());
    *plan_bytes = (size_t)h.bytes;
    *ws_bytes = cb_ws_map(nullptr, re - rb, m, (int64_t)h.T * h.NB).bytes;
    return TSNET_OK;
}

int tsnet_plan_build(const tsnet_csr* P, const tsnet_shard* shard, void* plan, size_t plan_bytes, void* ws,
                     size_t ws_bytes, tsnet_stream_t stream) {
    TSNET_ARG(P != nullptr && plan != nullptr, "NULL argument");
    TSNET_ARG(((uintptr_t)plan % 256) == 0, "plan buffer must be 256-byte aligned");
    TSNET_ARG(P->n >= 0 && P->nnz >= 0 && (P->n == 0 || P->indptr), "invalid P");
    TSNET_ARG(P->nnz == 0 || (P->indices && P->values), "P arrays are NULL");
    cudaStream_t s = (cudaStream_t)stream;
    int64_t rb, re;
    int st = cb_rows(P, shard, rb, re);
    if (st != TSNET_OK) return st;
    std::vector<int64_t> row0;
    std::vector<int32_t> rows;
    int64_t m = 0;
    if (P->n == 0) {
        row0.assign(1, 0);
        rows.assign(1, 0);
    } else if ((st = cb_host_partition(P, rb, re, s, row0, rows, m)) != TSNET_OK) {
        return st;
    }
    CbHeader h = cb_layout(P->n, rb, re, m, (int32_t)row0.size());
    TSNET_ARG(plan_bytes >= (size_t)h.bytes, "plan buffer too small (%zu < %lld bytes)", plan_bytes, (long long)h.bytes);
    const int64_t nseg = (int64_t)h.T * h.NB;
    TSNET_ARG((uint64_t)nseg < ((uint64_t)1 << 32), "too many (task, block) segments");
    CbWs w = cb_ws_map(ws, re - rb, m, nseg);
    TSNET_ARG(ws != nullptr && ws_bytes >= w.bytes, "plan workspace too small (%zu < %zu bytes)", ws_bytes, w.bytes);
    uint8_t* pb = reinterpret_cast<uint8_t*>(plan);
    int64_t* d_row0 = reinterpret_cast<int64_t*>(pb + h.off_row0);
    int32_t* d_rows = reinterpret_cast<int32_t*>(pb + h.off_rows);
    int64_t* d_seg = reinterpret_cast<int64_t*>(pb + h.off_seg);
    uint2* d_ent = reinterpret_cast<uint2*>(pb + h.off_entries);
    TSNET_CUDA(cudaMemcpyAsync(d_row0, row0.data(), sizeof(int64_t) * h.T, cudaMemcpyHostToDevice, s));
    TSNET_CUDA(cudaMemcpyAsync(d_rows, rows.data(), sizeof(int32_t) * h.T, cudaMemcpyHostToDevice, s));
    TSNET_CUDA(cudaMemsetAsync(w.slen, 0, sizeof(int64_t) * (nseg + 1), s));
    TSNET_CUDA(cudaMemsetAsync(w.sstart, 0, sizeof(int64_t) * (nseg + 1), s));
    if (m > 0) {
        k_cb_row_task<<<std::min<int>(h.T, 4096), 256, 0, s>>>(d_row0, d_rows, h.T, rb, w.row_task);
        TSNET_LAUNCH_CHECK();
        k_cb_keys<<<num_sms() * 8, 256, 0, s>>>(P->indptr, P->indices, P->values, rb, re, d_row0, w.row_task, h.NB,
                                                w.keys_a, w.vals_a);
        TSNET_LAUNCH_CHECK();
        int end_bit = 1;
        while (end_bit < 32 && ((uint64_t)1 << end_bit) < (uint64_t)nseg) ++end_bit;
        cub::DoubleBuffer<uint32_t> dk(w.keys_a, w.keys_b);
        cub::DoubleBuffer<unsigned long long> dv(w.vals_a, w.vals_b);
        size_t tb = w.cub_bytes;
        TSNET_CUDA(cub::DeviceRadixSort::SortPairs(w.cub_tmp, tb, dk, dv, m, 0, end_bit, s));
        k_cb_bounds<<<num_sms() * 8, 256, 0, s>>>(dk.Current(), m, w.sstart, w.slen);
        TSNET_LAUNCH_CHECK();
        k_cb_pad<<<num_sms() * 4, 256, 0, s>>>(w.sstart, w.slen, nseg);
        TSNET_LAUNCH_CHECK();
        tb = w.cub_bytes;
        TSNET_CUDA(cub::DeviceScan::ExclusiveSum(w.cub_tmp, tb, w.slen, d_seg, nseg + 1, s));
        k_cb_fill<<<num_sms() * 8, 256, 0, s>>>(dk.Current(), dv.Current(), m, w.sstart, d_seg, d_ent);
        TSNET_LAUNCH_CHECK();
    } else {
        TSNET_CUDA(cudaMemsetAsync(d_seg, 0, sizeof(int64_t) * (nseg + 1), s));
    }
    int64_t total = 0;
    TSNET_CUDA(cudaMemcpyAsync(&total, d_seg + nseg, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TSNET_CUDA(cudaStreamSynchronize(s));
    h.entries = total;
    TSNET_CUDA(cudaMemcpyAsync(pb, &h, sizeof(CbHeader), cudaMemcpyHostToDevice, s));
    TSNET_CUDA(cudaStreamSynchronize(s));
    return TSNET_OK;
}

}  // extern "C"
