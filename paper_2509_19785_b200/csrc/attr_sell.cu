// attr_sell.cu -- sliced-ELL attractive SpMV (step a6, Eq. 6 first term,
// PAPER.md:162): F_attr,i = sum_{j in row i} p_ij w_ij (X_i - X_j),
// w_ij = 1 / (1 + |X_i - X_j|^2).
//
// Why a third layout of P: on a mesh (config 5) the CSR
// kernel, one warp per row, gathers Y_j for 32 consecutive entries of ONE row;
// those columns lie on ~11 different 128-byte lines (the row's ball spans
// x-, y- and z-neighbours), so the kernel is bound by L1 wavefronts (ncu:
// l1tex 84%) at ~52% of HBM.  Here a lane owns a row and a warp a slice of 32
// consecutive rows; at step k every lane reads the k-th entry of its row.  On
// a mesh the k-th neighbours of consecutive vertices are themselves mostly
// consecutive, so the 32 gathers of a step touch ~5 lines, and the entry loads
// are fully coalesced (32 x 8 bytes).  No warp reduction, no atomics: each
// lane writes its own F_i.
//
// Layout (one plan = rows [row_begin, row_end) of P):
//   slice s = rows row_begin + 32 s .. + 31; K_s = its longest row;
//   slot (s, k, lane) at base[s] + 32 k + lane, base = exclusive scan of 32 K_s;
//   slot = (col, p_ij fp32 bits) as a uint2; slots past a row's end hold
//   (its own row, +0.0f) and add exactly 0 (X_i - X_i = 0, p = 0).
// On a power-law graph (config 4) slices pad heavily (a hub in a slice) and
// the gathers stay random: tsnet_sell_query reports the slots per entry so a
// caller can keep the CSR kernel there.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "move.cuh"
#include "ptx.cuh"
#include "tsnet.h"

namespace tsnet {

constexpr uint64_t kSellMagic = 0x4c4c455354534e54ull;   // "TNSTSELL"

struct SellHeader {
    uint64_t magic;
    int64_t n, row_begin, row_end, nnz, slices, slots;
    int64_t off_base, off_slots, bytes;
};

static size_t sell_align(size_t x) { return (x + 255) / 256 * 256; }

__device__ __forceinline__ uint64_t sell_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint2 sell_ld_stream(const uint2* a, uint64_t pol) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y)
                 : "l"(a), "l"(pol));
    return v;
}

static SellHeader sell_layout(int64_t n, int64_t rb, int64_t re, int64_t nnz, int64_t slots) {
    SellHeader h{};
    h.magic = kSellMagic;
    h.n = n;
    h.row_begin = rb;
    h.row_end = re;
    h.nnz = nnz;
    h.slices = (re - rb + 31) / 32;
    h.slots = slots;
    size_t off = sell_align(sizeof(SellHeader));
    h.off_base = (int64_t)off;
    off = sell_align(off + sizeof(int64_t) * (size_t)(h.slices + 1));
    h.off_slots = (int64_t)off;
    off = sell_align(off + sizeof(uint2) * (size_t)slots);
    h.bytes = (int64_t)off;
    return h;
}

__device__ __forceinline__ void sell_acc(const float2* __restrict__ Y, float2 yi, uint2 e, float& fx, float& fy) {
    const float2 yj = __ldg(Y + (int)e.x);
    const float dx = yi.x - yj.x, dy = yi.y - yj.y;
    const float w = __frcp_rn(fmaf(dx, dx, fmaf(dy, dy, 1.0f)));
    const float pw = __uint_as_float(e.y) * w;
    fx = fmaf(pw, dx, fx);
    fy = fmaf(pw, dy, fy);
}

// One warp per slice (grid-stride).  The entry stream is prefetched NS - 1
// register sets of U steps ahead (HBM latency), the sets rotate by unrolling
// (no copies of in-flight loads), and the Y_j gathers of set j + 1 are
// issued before set j is computed (two gather sets in flight per warp).
// NS even (the unrolled body covers NS sets; gather sets alternate).
//
// MOVE: step a7 fused into the epilogue -- each lane, holding its row's
// F_attr,i in registers, gathers the field at its point, forms the gradient
// and moves the point (gains/momentum), writing the new position to m.Ynew
// (never Y: other warps still gather the old positions) and vel/gains in
// place.  Same arithmetic as k_update.
template <int U, int NS, bool MOVE, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) k_attr_sell_g(const uint8_t* __restrict__ plan,
                                                           const float2* __restrict__ Y, float2* __restrict__ F,
                                                           SellMoveArgs m) {
    static_assert(NS % 2 == 0, "NS must be even");
    const SellHeader* h = reinterpret_cast<const SellHeader*>(plan);
    const int64_t rb = h->row_begin, re = h->row_end, S = h->slices;
    const int64_t* __restrict__ base = reinterpret_cast<const int64_t*>(plan + h->off_base);
    const uint2* __restrict__ slots = reinterpret_cast<const uint2*>(plan + h->off_slots);
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t pol = sell_policy_evict_first();
    for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; s < S; s += nw) {
        const int64_t b0 = __ldg(base + s), K = (__ldg(base + s + 1) - b0) >> 5;
        const int64_t r = rb + s * 32 + lane;
        const bool live = r < re;
        const float2 yi = live ? __ldg(Y + r) : make_float2(0.f, 0.f);
        const uint2* p = slots + b0 + lane;
        float fx = 0.f, fy = 0.f;
        uint2 E[NS][U];
        float2 G[2][U];
#pragma unroll
        for (int j = 0; j < NS - 1; ++j)
#pragma unroll
            for (int q = 0; q < U; ++q)
                E[j][q] = j * U + q < K ? sell_ld_stream(p + 32 * (j * U + q), pol) : make_uint2(0u, 0u);
#pragma unroll
        for (int q = 0; q < U; ++q) G[0][q] = __ldg(Y + (int)E[0][q].x);
        for (int64_t k = 0; k < K; k += NS * U) {
#pragma unroll
            for (int j = 0; j < NS; ++j) {
                const int jl = (j + NS - 1) % NS;
                const int64_t kl = k + (int64_t)(j + NS - 1) * U;
#pragma unroll
                for (int q = 0; q < U; ++q)
                    E[jl][q] = kl + q < K ? sell_ld_stream(p + 32 * (kl + q), pol) : make_uint2(0u, 0u);
                const int jn = (j + 1) % NS;
#pragma unroll
                for (int q = 0; q < U; ++q) G[(j + 1) & 1][q] = __ldg(Y + (int)E[jn][q].x);
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    const float dx = yi.x - G[j & 1][q].x, dy = yi.y - G[j & 1][q].y;
                    const float w = __frcp_rn(fmaf(dx, dx, fmaf(dy, dy, 1.0f)));
                    const float pw = __uint_as_float(E[j][q].y) * w;
                    fx = fmaf(pw, dx, fx);
                    fy = fmaf(pw, dy, fy);
                }
            }
        }
        if constexpr (MOVE) {
            bool bad = false;
            if (live) {
                const int64_t q = r - rb;
                const Geo g = *m.geo;
                const float2 ff = gather_field(g, m.fgrid, m.box[q], m.uv[q]);
                float2 y = yi, v = m.vel[q], gn = m.gains[q];
                const float gx = fmaf(4.0f * m.lambda_kl, fx, ff.x) + m.cn * y.x;
                const float gy = fmaf(4.0f * m.lambda_kl, fy, ff.y) + m.cn * y.y;
                gains_move(gx, v.x, gn.x, y.x, m.sp);
                gains_move(gy, v.y, gn.y, y.y, m.sp);
                bad = !(isfinite(y.x) && isfinite(y.y));
                m.Ynew[q] = y;
                m.vel[q] = v;
                m.gains[q] = gn;
            }
            if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&m.geo->nonfinite, 1);
        } else {
            if (live) F[r - rb] = make_float2(fx, fy);
        }
    }
}

// Kernel shape (measured on config 5, kernel alone, B200; CSR kernel 1.22 ms,
// round-1 sweep r1cq): U = 4 steps per set, NS = 4 sets, 4 CTAs per SM
// promised to ptxas: 0.751 ms (64 registers, 87% of the measured HBM peak);
// g4,4 with 3 / 1 CTAs per SM 0.771 / 0.996 ms (94 registers), g4,2 0.816,
// g2,4 0.879, g1,8 1.537; entries pipelined without the gather pipeline
// 0.921-0.943; TMA-staged entries 1.01-1.47 (the ring's shared memory takes
// L1 capacity from the Y_j gathers, which hit L1 on a mesh).
static constexpr auto sell_kernel = k_attr_sell_g<4, 4, false, 4>;

static int resident_of(const void* k) {
    int r = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, k, 256, 0) != cudaSuccess || r < 1) r = 1;
    return r;
}

// F: rows [row_begin, row_end) of the plan's shard (nl = row_end - row_begin)
cudaError_t launch_attr_sell(const void* plan, const float2* Y, float2* F, int64_t nl, cudaStream_t s) {
    if (nl == 0) return cudaSuccess;
    const int64_t slices = (nl + 31) / 32;
    const int blocks = (int)std::max<int64_t>(
        1, std::min<int64_t>((slices + 7) / 8, (int64_t)kNumSMs * resident_of((const void*)sell_kernel)));
    sell_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const uint8_t*>(plan), Y, F, SellMoveArgs{});
    return cudaGetLastError();
}

// ------------------------------------------------------------------ plan build
// one warp per slice: lane = row; every slot of the slice written once
__global__ void k_sell_fill(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                            const float* __restrict__ values, int64_t rb, int64_t re, int64_t S,
                            const int64_t* __restrict__ base, uint2* __restrict__ slots) {
    const int lane = threadIdx.x & 31;
    for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; s < S;
         s += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t r = rb + s * 32 + lane;
        const int64_t b0 = base[s], K = (base[s + 1] - b0) >> 5;
        const int64_t a = r < re ? indptr[r] : 0, L = r < re ? indptr[r + 1] - a : 0;
        const uint32_t self = (uint32_t)(r < re ? r : rb);
        for (int64_t k = 0; k < K; ++k)
            slots[b0 + 32 * k + lane] = k < L ? make_uint2((uint32_t)indices[a + k], __float_as_uint(values[a + k]))
                                              : make_uint2(self, 0u);
    }
}

static int sell_rows(const tsnet_csr* P, const tsnet_shard* sh, int64_t& rb, int64_t& re) {
    rb = 0;
    re = P->n;
    if (sh) {
        TSNET_ARG(sh->row_begin >= 0 && sh->row_begin <= sh->row_end && sh->row_end <= P->n, "bad shard rows");
        rb = sh->row_begin;
        re = sh->row_end;
    }
    TSNET_ARG(P->n < ((int64_t)1 << 31), "a sliced-ELL plan needs n < 2^31");
    return TSNET_OK;
}

// Slot offsets base[0..S] of the slices (host; reads indptr[rb..re], blocking).
static int sell_base(const tsnet_csr* P, int64_t rb, int64_t re, cudaStream_t s, std::vector<int64_t>& base,
                     int64_t& nnz_s) {
    const int64_t nr = re - rb, S = (nr + 31) / 32;
    std::vector<int64_t> ip((size_t)nr + 1, 0);
    if (nr > 0) {
        TSNET_CUDA(cudaMemcpyAsync(ip.data(), P->indptr + rb, sizeof(int64_t) * (size_t)(nr + 1),
                                   cudaMemcpyDeviceToHost, s));
        TSNET_CUDA(cudaStreamSynchronize(s));
    }
    base.assign((size_t)S + 1, 0);
    for (int64_t q = 0; q < S; ++q) {
        int64_t K = 0;
        for (int64_t r = 32 * q; r < std::min(nr, 32 * q + 32); ++r) K = std::max(K, ip[r + 1] - ip[r]);
        base[q + 1] = base[q] + 32 * K;
    }
    nnz_s = ip[nr] - ip[0];
    return TSNET_OK;
}

}  // namespace tsnet

using namespace tsnet;

extern "C" {

int tsnet_sell_query(const tsnet_csr* P, const tsnet_shard* shard, size_t* plan_bytes, double* slots_per_nnz,
                     tsnet_stream_t stream) {
    TSNET_ARG(P != nullptr && plan_bytes != nullptr, "NULL argument");
    TSNET_ARG(P->n >= 0 && P->nnz >= 0 && (P->n == 0 || P->indptr), "invalid P");
    int64_t rb, re, nnz_s = 0;
    int st = sell_rows(P, shard, rb, re);
    if (st != TSNET_OK) return st;
    std::vector<int64_t> base;
    if ((st = sell_base(P, rb, re, (cudaStream_t)stream, base, nnz_s)) != TSNET_OK) return st;
    *plan_bytes = (size_t)sell_layout(P->n, rb, re, nnz_s, base.back()).bytes;
    if (slots_per_nnz) *slots_per_nnz = nnz_s > 0 ? (double)base.back() / (double)nnz_s : 1.0;
    return TSNET_OK;
}

int tsnet_sell_build(const tsnet_csr* P, const tsnet_shard* shard, void* plan, size_t plan_bytes,
                     tsnet_stream_t stream) {
    TSNET_ARG(P != nullptr && plan != nullptr, "NULL argument");
    TSNET_ARG(((uintptr_t)plan % 256) == 0, "plan buffer must be 256-byte aligned");
    TSNET_ARG(P->n >= 0 && P->nnz >= 0 && (P->n == 0 || P->indptr), "invalid P");
    TSNET_ARG(P->nnz == 0 || (P->indices && P->values), "P arrays are NULL");
    cudaStream_t s = (cudaStream_t)stream;
    int64_t rb, re, nnz_s = 0;
    int st = sell_rows(P, shard, rb, re);
    if (st != TSNET_OK) return st;
    std::vector<int64_t> base;
    if ((st = sell_base(P, rb, re, s, base, nnz_s)) != TSNET_OK) return st;
    const SellHeader h = sell_layout(P->n, rb, re, nnz_s, base.back());
    TSNET_ARG(plan_bytes >= (size_t)h.bytes, "plan buffer too small (%zu < %lld bytes)", plan_bytes,
              (long long)h.bytes);
    uint8_t* pb = reinterpret_cast<uint8_t*>(plan);
    int64_t* d_base = reinterpret_cast<int64_t*>(pb + h.off_base);
    TSNET_CUDA(cudaMemcpyAsync(pb, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    TSNET_CUDA(cudaMemcpyAsync(d_base, base.data(), sizeof(int64_t) * base.size(), cudaMemcpyHostToDevice, s));
    if (h.slices > 0 && h.slots > 0) {
        k_sell_fill<<<kNumSMs * 8, 256, 0, s>>>(P->indptr, P->indices, P->values, rb, re, h.slices, d_base,
                                                reinterpret_cast<uint2*>(pb + h.off_slots));
        TSNET_LAUNCH_CHECK();
    }
    TSNET_CUDA(cudaStreamSynchronize(s));   // the host copies of h and base are stack/heap memory
    return TSNET_OK;
}

}  // extern "C"
