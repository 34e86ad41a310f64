// attr_cb.cu -- column-blocked attractive SpMV (step a6, Eq. 6 first term,
// PAPER.md:162): F_attr,i = sum_{j in row i} p_ij w_ij (X_i - X_j).
//
// Why a second layout of P: on the power-law graph of config 4
// every CSR kernel is bound by the L2 request rate of the random Y[j] gathers
// (one 32-B sector request per stored entry; ncu: l1tex2xbar request cycles
// ~80%, DRAM ~25%).  Here Y is read from shared memory instead:
//
//   * columns are cut into blocks of kCbCols points; a producer warp streams
//     the Y slice of each block into a double-buffered shared tile with
//     cp.async.bulk (TMA bulk copy, mbarrier completion);
//   * rows are cut into mini-tasks: runs of consecutive rows (at most kCbRows
//     rows, balanced nnz + rows), except that a long row (> cap entries) is
//     split into K mini-tasks of one "piece" each -- piece k takes the k-th
//     K-th of the row's entries inside EVERY block, so hub rows spread evenly
//     over warps and blocks; kCbW mini-tasks form a group, processed by one
//     CTA, one mini-task per consumer warp;
//   * a warp accumulates its mini-task's rows in its own slice of shared
//     memory (F_s), so nothing is shared between warps: no atomics and no
//     barriers in the hot loop -- warps only meet at the Y-tile pipeline;
//   * per (group, block, warp) the entries are a contiguous segment of 8-byte
//     words ((row - mini-task row0) << 16 | col - block_col0, p_ij fp32 bits),
//     rows ascending, padded to an even length; a warp streams its segment in
//     sweeps of 128 entries (16-byte loads, two sweeps ahead, L2 evict-first),
//     gathers Y_j from the tile and Y_i (one sweep ahead) from L2, reduces runs
//     of equal rows in registers (hand-down between lanes, segmented scan when
//     a run covers whole lanes) and adds run sums into F_s;
//   * at the end of a group each warp writes its rows of F (plain stores; the
//     pieces of split rows add with vector atomics into F, zeroed before).
// HBM bytes per launch: 8 per stored entry (+ padding) + 8 per (group, block,
// warp) segment offset + 8 per row of F; Y tiles come from L2.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"
#include "ptx.cuh"

namespace tsnet {

constexpr int kCbCols = 8192;       // points per column block (2 x 64 KB shared tiles)
constexpr int kCbW = 16;            // consumer warps per CTA = mini-tasks per group (+1 producer warp)
constexpr int kCbRows = 704;        // rows per mini-task (16 x 704 x 8 B = 88 KB of F_s)
constexpr uint32_t kCbSentinel = 0xFFFFu;
constexpr uint64_t kCbMagic = 0x3456434e53545354ull;  // "TSTSNCV4"

struct CbHeader {
    uint64_t magic;
    int64_t n, row_begin, row_end, nnz, entries;
    int32_t G, NB, C, W, rows_max, pad;
    int64_t off_seg, off_mt, off_entries, bytes;
};

static size_t cb_align(size_t x) { return (x + 255) / 256 * 256; }

static CbHeader cb_layout(int64_t n, int64_t rb, int64_t re, int64_t nnz, int32_t G) {
    CbHeader h{};
    h.magic = kCbMagic;
    h.n = n;
    h.row_begin = rb;
    h.row_end = re;
    h.nnz = nnz;
    h.G = G;
    h.C = kCbCols;
    h.W = kCbW;
    h.rows_max = kCbRows;
    h.NB = (int32_t)((n + kCbCols - 1) / kCbCols);
    const int64_t nseg = (int64_t)G * h.NB * kCbW;
    h.entries = nnz + nseg;   // upper bound with padding
    size_t off = cb_align(sizeof(CbHeader));
    h.off_seg = (int64_t)off;
    off = cb_align(off + sizeof(int64_t) * (size_t)(nseg + 1));
    h.off_mt = (int64_t)off;
    off = cb_align(off + sizeof(int2) * (size_t)((int64_t)G * kCbW));
    h.off_entries = (int64_t)off;
    off = cb_align(off + sizeof(uint2) * (size_t)h.entries);
    h.bytes = (int64_t)off;
    return h;
}

// Host cut (pure).  ipr[q] = indptr[rb + q], q = 0 .. nr.  A row of L > cap
// entries (cap = max(256, nnz / (base W) / 2)) is split into K = ceil(L / cap)
// one-piece mini-tasks; the other rows form runs of consecutive rows (<=
// rows_max each) with boundaries at multiples of their mean weight (entries +
// rows); T = W G mini-tasks in row order, G = base k for the smallest k that
// fits, padded with empty mini-tasks.  Output:
//   row_mt[q]: first mini-task of row q; row_K[q]: its pieces (1 = not split);
//   mt_r0[t]: first row of mini-task t; mt_info[t]: its rows (>= 0), or -1 for
//   a piece.  Returns G, or -1.
static int32_t cb_partition(const int64_t* ipr, int64_t nr, int32_t W, int32_t rows_max, int32_t base,
                            std::vector<int32_t>& row_mt, std::vector<int32_t>& row_K, std::vector<int32_t>& mt_r0,
                            std::vector<int32_t>& mt_info) {
    const int64_t nnz = ipr[nr] - ipr[0];
    const int64_t cap = std::max<int64_t>(256, nnz / ((int64_t)base * W) / 2);
    row_mt.assign(nr, 0);
    row_K.assign(nr, 1);
    int64_t pieces = 0, nsplit = 0;
    double wrows = 0.0;
    for (int64_t q = 0; q < nr; ++q) {
        const int64_t L = ipr[q + 1] - ipr[q];
        if (L > cap) {
            row_K[q] = (int32_t)((L + cap - 1) / cap);
            pieces += row_K[q];
            ++nsplit;
        } else {
            wrows += (double)L + 1.0;
        }
    }
    const int64_t kmax = 2 + (nr + (int64_t)rows_max * W * base - 1) / ((int64_t)rows_max * W * base) +
                         (pieces + nsplit + (int64_t)W * base - 1) / ((int64_t)W * base);
    for (int64_t k = 1; k <= kmax; ++k) {
        const int64_t G = (int64_t)base * k, T = G * W;
        if (G > INT32_MAX / W) break;
        const int64_t T_rows = T - pieces - nsplit;   // a split may close a run early: reserve one each
        if (T_rows < 1) continue;
        const double target = wrows / (double)T_rows;
        mt_r0.clear();
        mt_info.clear();
        double acc = 0.0;
        int64_t open = -1, runs = 0;   // index of the open run in mt_*
        for (int64_t q = 0; q < nr; ++q) {
            const int64_t L = ipr[q + 1] - ipr[q];
            if (row_K[q] > 1) {
                open = -1;
                row_mt[q] = (int32_t)mt_r0.size();
                for (int32_t p = 0; p < row_K[q]; ++p) {
                    mt_r0.push_back((int32_t)q);
                    mt_info.push_back(-1);
                }
                continue;
            }
            // close the open run at multiples of the target, or when full
            if (open >= 0 && (mt_info[open] >= rows_max || acc >= target * (double)runs)) open = -1;
            if (open < 0) {
                open = (int64_t)mt_r0.size();
                mt_r0.push_back((int32_t)q);
                mt_info.push_back(0);
                ++runs;
            }
            mt_info[open] += 1;
            row_mt[q] = (int32_t)open;
            acc += (double)L + 1.0;
        }
        if ((int64_t)mt_r0.size() > T) continue;
        while ((int64_t)mt_r0.size() < T) {   // empty mini-tasks
            mt_r0.push_back(0);
            mt_info.push_back(0);
        }
        return (int32_t)G;
    }
    return -1;
}

// PTX helpers (mbarrier, bulk copy): ptx.cuh

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

// Y_i of the lane's four entries (issued one sweep ahead): row = row0 + key
// (a piece mini-task has the single row row0: key 0);
// sentinel keys read row0 and are multiplied by p = 0.
struct CbYi {
    float2 y[4];
};
__device__ __forceinline__ CbYi cb_yi(uint4 a, uint4 b, const float2* __restrict__ Yr0) {
    // four independent loads (repeated rows hit L1): selecting between a loaded
    // value and another load would make the issue wait for the first one
    const uint32_t k[4] = {a.x >> 16, a.z >> 16, b.x >> 16, b.z >> 16};
    CbYi r;
#pragma unroll
    for (int q = 0; q < 4; ++q) r.y[q] = __ldg(Yr0 + (k[q] == kCbSentinel ? 0u : k[q]));
    return r;
}

__device__ __forceinline__ void fs_add(float2* Fs, uint32_t k, float x, float y) {
    float2 v = Fs[k];
    v.x += x;
    v.y += y;
    Fs[k] = v;
}

// One sweep: lane holds entries 4 lane .. 4 lane + 3 of 128 consecutive entries
// of the warp's segment (keys = local rows, non-decreasing; masked entries
// carry the sentinel key and p = 0 and sit at the end).  Run sums are added to
// the warp's own F_s slice (one add per key per sweep; sweeps of a warp are
// ordered by __syncwarp).
__device__ __forceinline__ void cb_sweep(uint4 a, uint4 b, const CbYi& yi, const float2* __restrict__ Ys,
                                         float2* Fs, int lane) {
    const uint32_t wd[4] = {a.x, a.z, b.x, b.z};
    const float pv[4] = {__uint_as_float(a.y), __uint_as_float(a.w), __uint_as_float(b.y), __uint_as_float(b.w)};
    uint32_t k[4];
    float2 yj[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        k[q] = wd[q] >> 16;
        yj[q] = Ys[wd[q] & 0xFFFFu];
    }
    float2 f[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) f[q] = cb_term(yi.y[q], yj[q], pv[q]);
    // lane runs: head (key k0, if != k3), middles (keys strictly between), tail (key k3)
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
    const bool mid1 = k[1] != k[0] && k[1] != tk;
    const bool mid2 = k[2] != k[0] && k[2] != tk && k[2] != k[1];
    if (mid1) fs_add(Fs, k[1], f[1].x + (k[2] == k[1] ? f[2].x : 0.f), f[1].y + (k[2] == k[1] ? f[2].y : 0.f));
    if (mid2) fs_add(Fs, k[2], f[2].x, f[2].y);
    // join runs across lanes: a tail continuing as the next lane's head is handed
    // down; a run covering whole lanes needs the segmented scan
    const uint32_t pk = __shfl_up_sync(0xffffffffu, tk, 1);
    const uint32_t nk = __shfl_down_sync(0xffffffffu, tk, 1);
    float sx = tx, sy = ty;
    const bool through = lane > 0 && !has_head && tk == pk;
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
    const bool give = has_head && lane > 0 && k[0] == pk;
    const float gx = __shfl_down_sync(0xffffffffu, give ? hx : 0.f, 1);
    const float gy = __shfl_down_sync(0xffffffffu, give ? hy : 0.f, 1);
    if (has_head && !give) fs_add(Fs, k[0], hx, hy);
    if (last && tk != kCbSentinel) fs_add(Fs, tk, sx + (lane < 31 ? gx : 0.f), sy + (lane < 31 ? gy : 0.f));
}

__global__ void __launch_bounds__((kCbW + 1) * 32, 1) k_attr_cb(const uint8_t* __restrict__ plan,
                                                                const float2* __restrict__ Y,
                                                                float2* __restrict__ F, int y_aligned) {
    extern __shared__ __align__(128) uint8_t cb_smem[];
    float2* Ys0 = reinterpret_cast<float2*>(cb_smem);
    float2* Ys1 = Ys0 + kCbCols;
    float2* Fs_all = Ys1 + kCbCols;
    uint64_t* bars = reinterpret_cast<uint64_t*>(Fs_all + kCbW * kCbRows);   // full[2], empty[2]
    const CbHeader* h = reinterpret_cast<const CbHeader*>(plan);
    const int G = h->G, NB = h->NB;
    const int64_t n = h->n, rb = h->row_begin;
    const int64_t* seg = reinterpret_cast<const int64_t*>(plan + h->off_seg);
    const int2* mt_desc = reinterpret_cast<const int2*>(plan + h->off_mt);   // (row0 - rb, rows | -1 piece)
    const uint4* ent = reinterpret_cast<const uint4*>(plan + h->off_entries);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        mbar_init(&bars[2], kCbW);
        mbar_init(&bars[3], kCbW);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // blocks any mini-task of group g needs: the group's block-J segments are contiguous
    auto group_block_used = [&](const int64_t* og, int J) { return og[(int64_t)J * kCbW] < og[(int64_t)(J + 1) * kCbW]; };

    if (warp == kCbW) {
        // ---------------- producer: Y slices of the blocks the group uses, in order
        uint32_t k = 0;
        for (int g = blockIdx.x; g < G; g += gridDim.x) {
            const int64_t* og = seg + (int64_t)g * NB * kCbW;
            for (int J = 0; J < NB; ++J) {
                if (!group_block_used(og, J)) continue;
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

    // ---------------- consumer warp: mini-task g * W + warp of every group g
    const uint64_t pol = cb_policy_evict_first();
    float2* Fs = Fs_all + warp * kCbRows;
    const uint4 pad = make_uint4(kCbSentinel << 16, 0u, kCbSentinel << 16, 0u);
    const int l2 = 2 * lane;
    uint32_t k = 0;
    for (int g = blockIdx.x; g < G; g += gridDim.x) {
        const int2 md = mt_desc[(int64_t)g * kCbW + warp];
        const bool piece = md.y < 0;
        const int nu = piece ? 1 : md.y;
        const float2* Yr0 = Y + rb + md.x;
        for (int q = lane; q < nu; q += 32) Fs[q] = make_float2(0.f, 0.f);
        __syncwarp();
        const int64_t* og = seg + (int64_t)g * NB * kCbW;
        auto next_block = [&](int J) {
            while (J < NB && !group_block_used(og, J)) ++J;
            return J;
        };
        auto my_seg = [&](int J, const uint4*& sp, int& np) {
            const int64_t s0 = og[(int64_t)J * kCbW + warp], s1 = og[(int64_t)J * kCbW + warp + 1];
            sp = ent + (s0 >> 1);
            np = (int)((s1 - s0) >> 1);
        };
        // Software pipeline over sweeps with four register sets rotated by
        // unrolling (no register moves: a move of a value still in flight would
        // wait for it): entries are loaded three sweeps ahead, Y_i one sweep
        // ahead (two sweeps after its entries were issued).
        struct Set {
            uint4 a, c;
            CbYi y;
        };
        Set S0, S1, S2, S3;
        const uint4* sp = ent;
        int np = 0;
        auto load_e = [&](int sw, Set& S) {
            const int o = sw * 64 + l2;
            S.a = o < np ? ld_stream_v4(sp + o, pol) : pad;
            S.c = o + 1 < np ? ld_stream_v4(sp + o + 1, pol) : pad;
        };
        auto load_y = [&](Set& S) { S.y = cb_yi(S.a, S.c, Yr0); };
        int J = next_block(0);
        if (J < NB) {
            my_seg(J, sp, np);
            load_e(0, S0);
            load_e(1, S1);
            load_e(2, S2);
        }
        while (J < NB) {
            const int b = k & 1;
            const float2* Ys = b ? Ys1 : Ys0;
            const int nsw = (np + 63) >> 6;
            if (nsw > 0) load_y(S0);
            mbar_wait(&bars[b], (k >> 1) & 1);
#pragma unroll 1
            for (int sw = 0; sw < nsw; sw += 4) {
                load_e(sw + 3, S3);
                if (sw + 1 < nsw) load_y(S1);
                cb_sweep(S0.a, S0.c, S0.y, Ys, Fs, lane);
                __syncwarp();
                if (sw + 1 >= nsw) break;
                load_e(sw + 4, S0);
                if (sw + 2 < nsw) load_y(S2);
                cb_sweep(S1.a, S1.c, S1.y, Ys, Fs, lane);
                __syncwarp();
                if (sw + 2 >= nsw) break;
                load_e(sw + 5, S1);
                if (sw + 3 < nsw) load_y(S3);
                cb_sweep(S2.a, S2.c, S2.y, Ys, Fs, lane);
                __syncwarp();
                if (sw + 3 >= nsw) break;
                load_e(sw + 6, S2);
                if (sw + 4 < nsw) load_y(S0);
                cb_sweep(S3.a, S3.c, S3.y, Ys, Fs, lane);
                __syncwarp();
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars[2 + b]);
            ++k;
            // prefetch this warp's segment of the next block the group uses
            J = next_block(J + 1);
            if (J < NB) {
                my_seg(J, sp, np);
                load_e(0, S0);
                load_e(1, S1);
                load_e(2, S2);
            }
        }
        __syncwarp();
        // rows of F: whole rows stored, pieces of split rows added (F zeroed before)
        if (piece) {
            if (lane == 0) atomicAdd(F + md.x, Fs[0]);
        } else {
            for (int q = lane; q < nu; q += 32) F[md.x + q] = Fs[q];
        }
        __syncwarp();
    }
}

size_t cb_smem_bytes() {
    return sizeof(float2) * (2 * kCbCols + kCbW * kCbRows) + 4 * sizeof(uint64_t);
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

// F: rows [row_begin, row_end) of the plan's shard (nl = row_end - row_begin)
cudaError_t launch_attr_cb(const void* plan, const float2* Y, float2* F, int64_t nl, cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_attr_cb, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)cb_smem_bytes());
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    cudaError_t e = cudaMemsetAsync(F, 0, sizeof(float2) * (size_t)nl, s);   // split rows accumulate
    if (e != cudaSuccess) return e;
    const int aligned = ((uintptr_t)Y % 16) == 0;
    k_attr_cb<<<num_sms(), (kCbW + 1) * 32, cb_smem_bytes(), s>>>(reinterpret_cast<const uint8_t*>(plan), Y, F,
                                                                  aligned);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ plan build
// Sort keys: (group, block, warp) of every entry of the shard; payload: the
// packed 8-byte entry.  A stable LSD radix sort keeps the CSR (row, col)
// order, i.e. rows ascending, inside each segment.
__global__ void k_cb_keys(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                          const float* __restrict__ values, int64_t rb, int64_t re, const int32_t* __restrict__ row_mt,
                          const int32_t* __restrict__ row_K, const int2* __restrict__ mt_desc, int NB,
                          uint32_t* __restrict__ keys, unsigned long long* __restrict__ vals) {
    const int lane = threadIdx.x & 31;
    const int64_t e0 = indptr[rb];
    for (int64_t r = rb + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); r < re;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t a = indptr[r], z = indptr[r + 1];
        const int32_t mt0 = row_mt[r - rb];
        const int K = row_K[r - rb];
        for (int64_t e = a + lane; e < z; e += 32) {
            const int32_t c = indices[e];
            const int J = c / kCbCols;
            int32_t mt = mt0;
            uint32_t lr = 0;
            if (K > 1) {
                // the row's entries inside block J: [lo, x) (columns ascending); piece by rank
                int64_t lo = a, hi = z, x = a, y = z;
                while (lo < hi) { const int64_t m = (lo + hi) >> 1; if (indices[m] < J * kCbCols) lo = m + 1; else hi = m; }
                while (x < y) { const int64_t m = (x + y) >> 1; if (indices[m] < (J + 1) * kCbCols) x = m + 1; else y = m; }
                mt += (int32_t)(((e - lo) * K) / (x - lo));
            } else {
                lr = (uint32_t)(r - rb - mt_desc[mt].x);
            }
            const uint32_t g = (uint32_t)(mt / kCbW), w = (uint32_t)(mt % kCbW);
            keys[e - e0] = (g * (uint32_t)NB + (uint32_t)J) * (uint32_t)kCbW + w;
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
    int32_t *row_mt, *row_K;
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
    w.row_mt = (int32_t*)take(sizeof(int32_t) * std::max<int64_t>(nr, 1));
    w.row_K = (int32_t*)take(sizeof(int32_t) * std::max<int64_t>(nr, 1));
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

struct CbCut {
    std::vector<int32_t> row_mt, row_K, mt_r0, mt_info;
    int32_t G = 0;
    int64_t nnz_s = 0;
};

static int cb_host_cut(const tsnet_csr* P, int64_t rb, int64_t re, cudaStream_t s, CbCut& cut) {
    std::vector<int64_t> ip(re - rb + 1, 0);
    if (P->n > 0) {
        TSNET_CUDA(cudaMemcpyAsync(ip.data(), P->indptr + rb, sizeof(int64_t) * ip.size(), cudaMemcpyDeviceToHost, s));
        TSNET_CUDA(cudaStreamSynchronize(s));
    }
    cut.nnz_s = ip.back() - ip.front();
    TSNET_ARG(cut.nnz_s < ((int64_t)1 << 31), "a plan holds < 2^31 entries per shard (got %lld)", (long long)cut.nnz_s);
    cut.G = cb_partition(ip.data(), re - rb, kCbW, kCbRows, num_sms(), cut.row_mt, cut.row_K, cut.mt_r0, cut.mt_info);
    TSNET_ARG(cut.G > 0, "row partition failed");
    return TSNET_OK;
}

}  // namespace tsnet

using namespace tsnet;

extern "C" {

int32_t tsnet_plan_partition(const int64_t* indptr_host, int64_t row_begin, int64_t row_end, int32_t warps,
                             int32_t rows_max, int32_t base_groups, int64_t max_minitasks, int32_t* row_mt,
                             int32_t* row_K, int32_t* mt_r0, int32_t* mt_info) {
    if (!indptr_host || !row_mt || !row_K || !mt_r0 || !mt_info || row_begin < 0 || row_end < row_begin ||
        warps < 1 || rows_max < 1 || base_groups < 1)
        return -1;
    std::vector<int32_t> a, b, c, d;
    const int32_t G = cb_partition(indptr_host + row_begin, row_end - row_begin, warps, rows_max, base_groups, a, b, c, d);
    if (G < 0 || (int64_t)G * warps > max_minitasks) return -1;
    std::memcpy(row_mt, a.data(), sizeof(int32_t) * a.size());
    std::memcpy(row_K, b.data(), sizeof(int32_t) * b.size());
    std::memcpy(mt_r0, c.data(), sizeof(int32_t) * c.size());
    std::memcpy(mt_info, d.data(), sizeof(int32_t) * d.size());
    return G;
}

int tsnet_plan_query(const tsnet_csr* P, const tsnet_shard* shard, size_t* plan_bytes, size_t* ws_bytes,
                     tsnet_stream_t stream) {
    TSNET_ARG(P != nullptr && plan_bytes != nullptr && ws_bytes != nullptr, "NULL argument");
    TSNET_ARG(P->n >= 0 && P->nnz >= 0 && (P->n == 0 || P->indptr), "invalid P");
    int64_t rb, re;
    int st = cb_rows(P, shard, rb, re);
    if (st != TSNET_OK) return st;
    CbCut cut;
    if ((st = cb_host_cut(P, rb, re, (cudaStream_t)stream, cut)) != TSNET_OK) return st;
    const CbHeader h = cb_layout(P->n, rb, re, cut.nnz_s, cut.G);
    *plan_bytes = (size_t)h.bytes;
    *ws_bytes = cb_ws_map(nullptr, re - rb, cut.nnz_s, (int64_t)h.G * h.NB * kCbW).bytes;
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
    CbCut cut;
    if ((st = cb_host_cut(P, rb, re, s, cut)) != TSNET_OK) return st;
    CbHeader h = cb_layout(P->n, rb, re, cut.nnz_s, cut.G);
    TSNET_ARG(plan_bytes >= (size_t)h.bytes, "plan buffer too small (%zu < %lld bytes)", plan_bytes, (long long)h.bytes);
    const int64_t nseg = (int64_t)h.G * h.NB * kCbW;
    TSNET_ARG((uint64_t)nseg < ((uint64_t)1 << 32), "too many (group, block, warp) segments");
    const int64_t nr = re - rb, T = (int64_t)h.G * kCbW;
    CbWs w = cb_ws_map(ws, nr, cut.nnz_s, nseg);
    TSNET_ARG(ws != nullptr && ws_bytes >= w.bytes, "plan workspace too small (%zu < %zu bytes)", ws_bytes, w.bytes);
    std::vector<int2> desc(T);
    for (int64_t t = 0; t < T; ++t) desc[t] = make_int2(cut.mt_r0[t], cut.mt_info[t]);
    uint8_t* pb = reinterpret_cast<uint8_t*>(plan);
    int64_t* d_seg = reinterpret_cast<int64_t*>(pb + h.off_seg);
    int2* d_mt = reinterpret_cast<int2*>(pb + h.off_mt);
    uint2* d_ent = reinterpret_cast<uint2*>(pb + h.off_entries);
    TSNET_CUDA(cudaMemcpyAsync(d_mt, desc.data(), sizeof(int2) * T, cudaMemcpyHostToDevice, s));
    if (nr > 0) {
        TSNET_CUDA(cudaMemcpyAsync(w.row_mt, cut.row_mt.data(), sizeof(int32_t) * nr, cudaMemcpyHostToDevice, s));
        TSNET_CUDA(cudaMemcpyAsync(w.row_K, cut.row_K.data(), sizeof(int32_t) * nr, cudaMemcpyHostToDevice, s));
    }
    TSNET_CUDA(cudaMemsetAsync(w.slen, 0, sizeof(int64_t) * (nseg + 1), s));
    TSNET_CUDA(cudaMemsetAsync(w.sstart, 0, sizeof(int64_t) * (nseg + 1), s));
    const int64_t m = cut.nnz_s;
    if (m > 0) {
        k_cb_keys<<<num_sms() * 8, 256, 0, s>>>(P->indptr, P->indices, P->values, rb, re, w.row_mt, w.row_K, d_mt,
                                                h.NB, w.keys_a, w.vals_a);
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
