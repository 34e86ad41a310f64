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
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"

namespace tsnet {

constexpr int kCbCols = 8192;       // points per column block (2 x 64 KB shared tiles)
constexpr int kCbRowsMax = 11264;   // rows per task (88 KB shared accumulator)
constexpr int kCbWarpsDefault = 24;   // consumer warps per CTA (+1 producer warp); env TSNET_CB_WARPS
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
// balanced on nnz + rows (greedy cut at multiples of (nnz + rows)/T) with at
// most rows_max rows each.
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
    // enough tasks for the row cap, whatever the nnz balance asks
    const int64_t wmax = 2 + (nr + (int64_t)rows_max * base - 1) / ((int64_t)rows_max * base);
    for (int64_t w = 1; w <= wmax; ++w) {
        const int64_t T = (int64_t)base * w;
        row0.clear();
        rows.clear();
        int64_t r = rb;
        for (int64_t t = 0; t < T; ++t) {
            // balance nnz + rows (empty rows weigh 1); the last task takes every
            // remaining row (trailing empty rows included)
            const int64_t target = (t == T - 1) ? INT64_MAX : ((nnz + nr) * (t + 1) + T - 1) / T;
            int64_t r1 = r;
            // extend while the weight before the next row is below the target and the cap allows
            while (r1 < re && (ipr[r1 - rb] - ipr[0]) + (r1 - rb) < target && r1 - r < rows_max) ++r1;
            row0.push_back(r);
            rows.push_back((int32_t)(r1 - r));
            r = r1;
        }
        if (r == re && T <= INT32_MAX) return (int32_t)T;
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
// One entry: contribution p w (X_i - X_j) with w = 1 / (1 + r^2).  Padding
// entries (p = 0) contribute exactly 0.  rcp.approx: 1 + r^2 >= 1, relative
// error <= 2^-22, far below the fp32 summation error of a row.
__device__ __forceinline__ float2 cb_term(float2 yi, float2 yj, float p) {
    const float dx = yi.x - yj.x, dy = yi.y - yj.y;
    float w;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(w) : "f"(fmaf(dx, dx, fmaf(dy, dy, 1.0f))));
    const float pw = p * w;
    return make_float2(pw * dx, pw * dy);
}

__device__ __forceinline__ void fs_add(float2* Fs, uint32_t k, float x, float y) {
    float2 v = Fs[k];
    v.x += x;
    v.y += y;
    Fs[k] = v;
}

// Run-end update of F_s.  Inside one block segment a row is shared between
// warps only at the two ends of a warp's share (keys kf, kl): those runs go to
// the warp's private slots edge[0..1] and are folded into F_s with shared
// atomics once per share; every other row of the share is owned by this warp
// for the block -> plain read-modify-write (one emit per key per sweep; sweeps
// of a warp are ordered by __syncwarp; blocks are separated by a barrier).
__device__ __forceinline__ void cb_emit(bool on, uint32_t k, float x, float y, float2* Fs, float2* edge, uint32_t kf,
                                        uint32_t kl) {
    float2* dst = (k == kf) ? edge : ((k == kl) ? edge + 1 : Fs + k);
    if (on) {
        float2 v = *dst;
        v.x += x;
        v.y += y;
        *dst = v;
    }
}

// One sweep: lane holds entries 4 lane .. 4 lane + 3 of 128 consecutive entries
// of the segment (keys = local rows, non-decreasing; masked entries carry the
// sentinel key and p = 0 and sit at the end).
// Y_i of the lane's four entries (issued one sweep ahead; one load per
// distinct row of the lane, sentinel keys read row 0 and are multiplied by p = 0)
struct CbYi {
    float2 y[4];
};
__device__ __forceinline__ CbYi cb_yi(uint4 a, uint4 b, const float2* __restrict__ Yrow) {
    const uint32_t k0 = a.x >> 16, k1 = a.z >> 16, k2 = b.x >> 16, k3 = b.z >> 16;
    CbYi r;
    r.y[0] = __ldg(Yrow + (k0 == kCbSentinel ? 0u : k0));
    r.y[1] = (k1 == k0) ? r.y[0] : __ldg(Yrow + (k1 == kCbSentinel ? 0u : k1));
    r.y[2] = (k2 == k1) ? r.y[1] : __ldg(Yrow + (k2 == kCbSentinel ? 0u : k2));
    r.y[3] = (k3 == k2) ? r.y[2] : __ldg(Yrow + (k3 == kCbSentinel ? 0u : k3));
    return r;
}

__device__ __forceinline__ void cb_sweep(uint4 a, uint4 b, const CbYi& yi, const float2* __restrict__ Ys,
                                         float2* Fs, int lane, float2* edge, uint32_t kf, uint32_t kl) {
    const uint32_t wd[4] = {a.x, a.z, b.x, b.z};
    const float pv[4] = {__uint_as_float(a.y), __uint_as_float(a.w), __uint_as_float(b.y), __uint_as_float(b.w)};
    uint32_t k[4];
    float2 yj[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        k[q] = wd[q] >> 16;
        yj[q] = Ys[wd[q] & 0xFFFFu];
    }
    const bool mid1 = k[1] != k[0] && k[1] != k[3], mid2 = k[2] != k[0] && k[2] != k[3];
    float2 f[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) f[q] = cb_term(yi.y[q], yj[q], pv[q]);
    // lane runs: tail (key k3), head (key k0 if != k3), middles (rare)
    const uint32_t tk = k[3];
    float tx = f[3].x, ty = f[3].y;
    float hx = 0.f, hy = 0.f;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const bool t = k[q] == tk, h = k[q] == k[0];
        tx += t ? f[q].x : 0.f;
        ty += t ? f[q].y : 0.f;
        hx += (h && !t) ? f[q].x : 0.f;
        hy += (h && !t) ? f[q].y : 0.f;
    }
    const bool has_head = k[0] != tk;
    // middle runs: keys k1 / k2 different from both ends (a row with <= 2 entries
    // inside this lane); they are complete here
    if (__any_sync(0xffffffffu, mid1 || mid2)) {
        float m1x = 0.f, m1y = 0.f, m2x = 0.f, m2y = 0.f;
        if (mid1) {
            m1x = f[1].x;
            m1y = f[1].y;
            if (k[2] == k[1]) {
                m1x += f[2].x;
                m1y += f[2].y;
            }
        }
        const bool m2 = mid2 && k[2] != k[1];
        if (m2) {
            m2x = f[2].x;
            m2y = f[2].y;
        }
        cb_emit(mid1, k[1], m1x, m1y, Fs, edge, kf, kl);
        cb_emit(m2, k[2], m2x, m2y, Fs, edge, kf, kl);
    }
    // join the lane runs across lanes.  Usually a run spans at most two lanes
    // (the tail of lane l continues as the head of lane l+1): one hand-down.  When
    // some run covers a whole lane (rows with many entries in this block), a
    // segmented inclusive scan of the tails does the general case.
    const uint32_t pk = __shfl_up_sync(0xffffffffu, tk, 1);
    const uint32_t nk = __shfl_down_sync(0xffffffffu, tk, 1);
    float sx = tx, sy = ty;
    const bool through = lane > 0 && !has_head && tk == pk;   // whole lane continues the previous run
    if (__any_sync(0xffffffffu, through)) {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t uk = __shfl_up_sync(0xffffffffu, tk, o);
            const float ux = __shfl_up_sync(0xffffffffu, sx, o);
            const float uy = __shfl_up_sync(0xffffffffu, sy, o);
            const bool add = lane >= o && uk == tk;
            sx += add ? ux : 0.f;
            sy += add ? uy : 0.f;
        }
    }
    const bool last = (lane == 31) || (nk != tk);
    // a head run continues the previous lane's tail run (hand it down), or stands alone
    const bool give = has_head && lane > 0 && k[0] == pk;
    const float gx = __shfl_down_sync(0xffffffffu, give ? hx : 0.f, 1);
    const float gy = __shfl_down_sync(0xffffffffu, give ? hy : 0.f, 1);
    const bool gv = lane < 31;
    cb_emit(has_head && !give && k[0] != kCbSentinel, k[0], hx, hy, Fs, edge, kf, kl);
    // without the scan, a tail that continues into the next lane is not "last"
    // there, so only run ends emit: sum = own tail (+ scanned prefix) + next head
    cb_emit(last && tk != kCbSentinel, tk, sx + (gv ? gx : 0.f), sy + (gv ? gy : 0.f), Fs, edge, kf, kl);
}

template <int kCbWarps>
__global__ void __launch_bounds__((kCbWarps + 1) * 32, 1) k_attr_cb(const uint8_t* __restrict__ plan, const float2* __restrict__ Y,
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
    float2* F2s = reinterpret_cast<float2*>(Fs);
    float2* edge = reinterpret_cast<float2*>(bars + 4) + 2 * warp;   // this warp's two boundary slots
    if (lane < 2) edge[lane] = make_float2(0.f, 0.f);
    __syncwarp();
    uint32_t k = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
        const int64_t row0 = row0s[t];
        const int rows = rowss[t];
        const float2* Yrow = Y + row0;
        for (int q = threadIdx.x; q < 2 * rows; q += nthr) Fs[q] = 0.f;
        named_bar(1, nthr);
        const int64_t* sg = seg + (int64_t)t * NB;
        const uint4 pad = make_uint4(kCbSentinel << 16, 0u, kCbSentinel << 16, 0u);
        const int l2 = 2 * lane;
        // this warp's share of block J's segment, in pairs of entries (16 B), and the
        // keys of its first and last entries (rows possibly shared with neighbours)
        // kf / kl come back as the raw words; the >> 16 happens after the Ys wait so
        // the loads' latency hides behind the barrier instead of stalling here
        auto share = [&](int J, const uint4*& sp, int& npw, uint32_t& kf, uint32_t& kl) {
            const int64_t s0 = sg[J], s1 = sg[J + 1];
            const int np = (int)((s1 - s0) >> 1);
            const int per = (np + kCbWarps - 1) / kCbWarps;
            const int q0 = min(np, per * warp);
            npw = min(np, per * (warp + 1)) - q0;
            sp = ent + (s0 >> 1) + q0;
            kf = kl = kCbSentinel << 16;
            if (npw > 0) {
                kf = __ldg(reinterpret_cast<const uint32_t*>(sp));
                kl = __ldg(reinterpret_cast<const uint32_t*>(sp + npw - 1) + 2);
            }
        };
        auto next_block = [&](int J) {
            while (J < NB && sg[J] == sg[J + 1]) ++J;
            return J;
        };
        // prologue of the first block; later blocks are prefetched during the previous one
        int J = next_block(0);
        const uint4* sp = ent;
        int npw = 0;
        uint32_t kfw = kCbSentinel << 16, klw = kCbSentinel << 16;   // raw first / last words of the share
        uint4 a0 = pad, c0 = pad, a1 = pad, c1 = pad;
        if (J < NB) {
            share(J, sp, npw, kfw, klw);
            if (l2 < npw) a0 = ld_stream_v4(sp + l2, pol);
            if (l2 + 1 < npw) c0 = ld_stream_v4(sp + l2 + 1, pol);
            if (l2 + 64 < npw) a1 = ld_stream_v4(sp + l2 + 64, pol);
            if (l2 + 65 < npw) c1 = ld_stream_v4(sp + l2 + 65, pol);
        }
        while (J < NB) {
            const int b = k & 1;
            const float2* Ys = b ? Ys1 : Ys0;
            mbar_wait(&bars[b], (k >> 1) & 1);
            const uint32_t kf = kfw >> 16, kl = klw >> 16;
            CbYi y0 = cb_yi(a0, c0, Yrow);
            const int nsw = (npw + 63) >> 6;
#pragma unroll 1
            for (int sw = 0; sw < nsw; ++sw) {
                const int o = (sw + 2) * 64 + l2;
                const uint4 a2 = o < npw ? ld_stream_v4(sp + o, pol) : pad;
                const uint4 c2 = o + 1 < npw ? ld_stream_v4(sp + o + 1, pol) : pad;
                const CbYi y1 = cb_yi(a1, c1, Yrow);   // rows of the next sweep, one sweep ahead
                cb_sweep(a0, c0, y0, Ys, F2s, lane, edge, kf, kl);
                __syncwarp();
                a0 = a1;
                c0 = c1;
                a1 = a2;
                c1 = c2;
                y0 = y1;
            }
            if (lane == 0) mbar_arrive(&bars[2 + b]);
            if (lane < 4) {   // fold the two boundary rows: one shared atomic per lane
                const uint32_t ke = (lane < 2) ? kf : kl;
                const bool ok = ke != kCbSentinel && (lane < 2 || kl != kf);
                float* e = reinterpret_cast<float*>(edge) + lane;
                if (ok) atomicAdd(Fs + 2 * ke + (lane & 1), *e);
                *e = 0.f;
            }
            __syncwarp();
            ++k;
            // prefetch the next block's first two sweeps before the barrier
            J = next_block(J + 1);
            a0 = c0 = a1 = c1 = pad;
            if (J < NB) {
                share(J, sp, npw, kfw, klw);
                if (l2 < npw) a0 = ld_stream_v4(sp + l2, pol);
                if (l2 + 1 < npw) c0 = ld_stream_v4(sp + l2 + 1, pol);
                if (l2 + 64 < npw) a1 = ld_stream_v4(sp + l2 + 64, pol);
                if (l2 + 65 < npw) c1 = ld_stream_v4(sp + l2 + 65, pol);
            }
            named_bar(1, nthr);   // rows owned by one warp in this block may be shared in the next
        }
        named_bar(1, nthr);
        float2* Fo = F + (row0 - rb);
        const float2* Fs2 = reinterpret_cast<const float2*>(Fs);
        for (int q = threadIdx.x; q < rows; q += nthr) Fo[q] = Fs2[q];
        named_bar(1, nthr);
    }
}

constexpr int kCbWarpsMax = 31;
size_t cb_smem_bytes() {
    return sizeof(float2) * 2 * kCbCols + sizeof(float) * 2 * kCbRowsMax + 4 * sizeof(uint64_t) +
           sizeof(float2) * 2 * kCbWarpsMax;
}

static int num_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = kNumSMs;
    }
    return sms;
}

template <int W>
static cudaError_t launch_cb_w(const void* plan, const float2* Y, float2* F, cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_attr_cb<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)cb_smem_bytes());
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int aligned = ((uintptr_t)Y % 16) == 0;
    k_attr_cb<W><<<num_sms(), (W + 1) * 32, cb_smem_bytes(), s>>>(reinterpret_cast<const uint8_t*>(plan), Y, F,
                                                                  aligned);
    return cudaGetLastError();
}

static int cb_warps() {
    static int w = 0;
    if (w == 0) {
        const char* e = getenv("TSNET_CB_WARPS");
        w = e ? atoi(e) : kCbWarpsDefault;
        if (w != 8 && w != 12 && w != 16 && w != 24) w = kCbWarpsDefault;
    }
    return w;
}

cudaError_t launch_attr_cb(const void* plan, const float2* Y, float2* F, cudaStream_t s) {
    switch (cb_warps()) {
        case 8: return launch_cb_w<8>(plan, Y, F, s);
        case 12: return launch_cb_w<12>(plan, Y, F, s);
        case 16: return launch_cb_w<16>(plan, Y, F, s);
        default: return launch_cb_w<24>(plan, Y, F, s);
    }
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
