// attr_cb.cu -- column-blocked attractive SpMV (step a6, Eq. 6 first term,
// PAPER.md:162): F_attr,i = sum_{j in row i} p_ij w_ij (X_i - X_j).
//
// Why a second layout of P: on the power-law graph of config 4
// every row-wise CSR kernel is bound by the L1->L2 request path of the random
// Y[j] gathers (one 32-B sector request per stored entry; ncu: l1tex2xbar
// request cycles 88 %, DRAM 33 %; a measured ceiling of ~1 gather per
// SM-cycle).  Here every Y[j] comes from shared memory (~4 gathers per
// SM-cycle) and nothing per entry leaves the SM except the 8-byte entry
// stream itself:
//
//   * panels: the rows of P (or of a shard) are dealt to P panels, 148 k of
//     them, by longest-processing-time on (entries + 8) with at most kTR rows
//     each, so every CTA gets the same work whatever the degree distribution
//     (hub rows go first, short rows fill the gaps); inside a panel the rows
//     keep ascending order and get a local index < kTR;
//   * column blocks of kTB points: one CTA per panel sweeps all blocks; a
//     producer warp streams Y[block] into a kTS-stage shared ring with
//     cp.async.bulk (TMA bulk copy, mbarrier completion) and prefetches the
//     tile's entries into L2 (cp.async.bulk.prefetch.L2), kTS - 1 blocks
//     ahead of the consumers;
//   * per (panel, block) tile the entries are sorted by (local row, column)
//     and cut into kTW warp segments of equal size, each boundary moved to
//     the nearest row boundary (within kSnap entries; a longer run is split
//     and its row marked shared, "hub"), so every warp does the same work in
//     every block whatever the row lengths (hub rows of 1e5 entries included);
//     the warps meet at one named barrier per block (rows change owners
//     between blocks);
//   * a warp segment is cut into 32 equal contiguous chunks, one per lane;
//     slot (step k, lane l) = k-th entry of chunk l, so a warp's step is one
//     coalesced 256-B load, and the segment is padded to whole steps (< 32
//     slots) with (0, p = 0) slots that add exactly 0;
//   * a lane accumulates its run of equal rows in registers and adds it to
//     the row's accumulator in shared memory when the run ends inside its
//     chunk (FLUSH bit; the lane that sees a run end is unique).  A run that
//     continues past the chunk's end is carried out: after the tile the
//     carries are summed per row across lanes (segmented warp scan, merge-path
//     style) and added by one lane, after the row's own flush in program
//     order; only the few shared rows use atomics (shared-memory float
//     atomics are CAS loops on sm_100);
// HBM bytes per launch: 8 per slot (stored entries + < 512 pads per tile) +
// 4 per tile + 12 per row (row list, Y_i, F_i); Y blocks come from L2
// (P x 8 n bytes of L2 reads).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <queue>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"
#include "ptx.cuh"

namespace tsnet {

#ifndef TILE_TB
#define TILE_TB 8000
#endif
#ifndef TILE_TR
#define TILE_TR 6464
#endif
constexpr int kTB = TILE_TB;         // points per column block
constexpr int kTS = 2;               // Y ring stages (2 x 62.5 KB, double buffer)
#ifndef TILE_PREF
#define TILE_PREF 1
#endif
constexpr int kTPre = TILE_PREF;     // blocks of entries prefetched into L2 ahead of the producer
// probe builds only (scripts/tile_variants.sh): the slot-load cache policy
#ifndef TILE_LDPOL
#define TILE_LDPOL 0
#endif
#ifndef TILE_DIAG   // timing diagnostics only (wrong results): 1 no F read-modify-write, 2 Y_j from one address,
                    // 3/4 cycle counters, 5 no per-block barrier
#define TILE_DIAG 0
#endif
constexpr int kTW = 15;           // consumer warps per CTA (+1 producer warp: 16 warps, <= 128 registers)
constexpr int kTL = kTW * 32;        // consumer threads
constexpr int kTR = TILE_TR;         // max rows per panel (16 B of shared memory each; a multiple of 16
                                     // for the row-slot swizzle)
constexpr int kTRbits = 13;          // local row bits of the plan-build sort keys
constexpr unsigned long long kLocalMask = (1ull << kTRbits) - 1;
constexpr int bits_for(int x) { return x <= 1 ? 0 : 1 + bits_for((x + 1) / 2); }
constexpr int kColBits = bits_for(kTB);   // column in block
constexpr int kSlotBits = bits_for(kTR);  // row slot
static_assert(kTR % 16 == 0 && kTR <= (1 << kTRbits), "rows per panel");
static_assert(kColBits + kSlotBits <= 26, "slot word: 3 + column + row-slot bits + 3 flags <= 32");
// slot word: column in block * 8 (bits 0 .. 3 + kColBits: the byte offset of
// Y_j in the ring stage) | row slot << (3 + kColBits) (the row-slot field
// shifted right by kColBits is the byte offset of Y_i and F_i) | HUB (bit 29:
// the row is shared between warps; its flushes are atomic) | NEWROW (bit 30: a
// run starts here) | FLUSH (bit 31: a run ends here).  Real entries have p > 0
// (C0 drops exact zeros); pads are (0, p = 0).
constexpr uint32_t kColMask = ((1u << kColBits) - 1u) << 3;
constexpr uint32_t kRowMask = ((1u << kSlotBits) - 1u) << 3;
constexpr uint32_t kHub = 1u << 29, kNewRow = 1u << 30, kFlush = 1u << 31;
constexpr int kRowShift = kColBits;  // (word >> kRowShift) & kRowMask = row slot * 8
// Shared memory: Y_i[kTR] at 0, F_i[kTR] at kFsOff, a dummy float2 (lanes with
// nothing to read there all read it: one broadcast address), the Y ring, the
// mbarriers.  Row slot = swizzled local row (tile_slot): the rows a warp's
// lanes touch at one step are spaced by about a run per chunk, so plain
// indices would put them in a few banks.
constexpr uint32_t kFsOff = kTR * 8u, kDummyOff = 2u * kTR * 8u, kRingOff = 2u * kTR * 8u + 16u;
__host__ __device__ __forceinline__ uint32_t tile_slot(uint32_t r) { return r ^ ((r >> 4) & 15u); }
// Panel p sweeps the column blocks rot, rot + 1, .., NB - 1, 0, .., rot - 1 with
// rot = (p mod G) NB / G: the panels that run at the same time (one per CTA)
// read different Y blocks, so the L2 is not hit by every SM for the same block.
__host__ __device__ __forceinline__ int tile_rot(int p, int G, int NB) {
    return (int)(((int64_t)(p % G) * NB) / G);
}
constexpr uint64_t kTileMagic = 0x3754534e53545354ull;   // "TSTSNST7"

struct TileHeader {
    uint64_t magic;
    int64_t n, row_begin, row_end, nnz;
    int32_t P, NB, R_max, G;            // G: the CTAs the sweep rotations are spread over
    int64_t steps;                      // total warp steps (slots / 32)
    int64_t off_wtab, off_rowoff, off_rows, off_slots, bytes;
};

static int num_sms() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = kNumSMs;
    return sms;
}

static size_t t_align(size_t x) { return (x + 255) / 256 * 256; }

static TileHeader tile_layout(int64_t n, int64_t rb, int64_t re, int64_t nnz, int32_t P, int32_t R_max,
                              int64_t steps) {
    TileHeader h{};
    h.magic = kTileMagic;
    h.n = n;
    h.row_begin = rb;
    h.row_end = re;
    h.nnz = nnz;
    h.P = P;
    h.NB = (int32_t)std::max<int64_t>(1, (n + kTB - 1) / kTB);
    h.R_max = R_max;
    h.G = std::max(1, num_sms());
    h.steps = steps;
    size_t off = t_align(sizeof(TileHeader));
    h.off_wtab = (int64_t)off;
    off = t_align(off + sizeof(int2) * ((size_t)P * kTW * h.NB));
    h.off_rowoff = (int64_t)off;
    off = t_align(off + sizeof(int32_t) * ((size_t)P + 1));
    h.off_rows = (int64_t)off;
    off = t_align(off + sizeof(int32_t) * (size_t)std::max<int64_t>(re - rb, 1));
    h.off_slots = (int64_t)off;
    off = t_align(off + sizeof(uint2) * 32 * (size_t)steps);
    h.bytes = (int64_t)off;
    return h;
}

// Host cut (pure).  ipr[q] = indptr[rb + q], q = 0 .. nr.  Panels:
// P = G ceil(nr / (G R_cap)) (at most nr, at least 1), rows dealt by LPT on
// weight (entries + 8, plus the hub penalty of tile_row_weight below): rows in decreasing entries (ties: smaller row), each to
// the panel with the least weight so far (ties: smaller panel) among those
// with < R_cap rows.  Inside a panel rows are in ascending order.  Outputs:
// row_panel[q], row_local[q], panel_off[P + 1] (exclusive scan of the panel
// sizes), panel_rows[panel_off[p] + l] = the row q with local index l.
// Returns P, or -1.
// Rows with >= TILE_HUB_MIN entries weigh TILE_HUB_PM per mille more in the
// deal: a hub row's runs are split between warps in every block (shared rows,
// atomic flushes), so its panel ran ~3 % longer than the others at equal
// entries (cfg 4: the 7 panels holding the 74k-200k-entry rows were the 7
// slowest CTAs, 946k vs 918k cycles mean); measured on cfg 4, the kernel takes
// 0.4946 ms without the penalty, 0.4848-0.4861 ms for thresholds 8k-64k and
// 400-900 per mille (profiles/r2s4gh_tile_hub_weight_cfg4.jsonl).
#ifndef TILE_HUB_MIN
#define TILE_HUB_MIN 32768
#endif
#ifndef TILE_HUB_PM
#define TILE_HUB_PM 600
#endif
static inline int64_t tile_row_weight(int64_t e) {
    return e + 8 + ((TILE_HUB_MIN > 0 && e >= TILE_HUB_MIN) ? e * TILE_HUB_PM / 1000 : 0);
}
static int32_t tile_partition(const int64_t* ipr, int64_t nr, int32_t G, int32_t R_cap, std::vector<int32_t>& row_panel,
                              std::vector<int32_t>& row_local, std::vector<int32_t>& panel_off,
                              std::vector<int32_t>& panel_rows) {
    if (nr < 0 || G < 1 || R_cap < 1 || nr >= ((int64_t)1 << 31)) return -1;
    int64_t P64 = (int64_t)G * ((nr + (int64_t)G * R_cap - 1) / ((int64_t)G * R_cap));
    P64 = std::max<int64_t>(1, std::min<int64_t>(P64, std::max<int64_t>(nr, 1)));
    if (P64 >= ((int64_t)1 << 31)) return -1;
    const int32_t P = (int32_t)P64;
    row_panel.assign(nr, 0);
    row_local.assign(nr, 0);
    panel_off.assign(P + 1, 0);
    panel_rows.assign(nr, 0);
    std::vector<int64_t> order(nr);
    for (int64_t q = 0; q < nr; ++q) order[q] = q;
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        return (ipr[a + 1] - ipr[a]) > (ipr[b + 1] - ipr[b]);
    });
    using Item = std::pair<int64_t, int32_t>;   // (weight, panel): min-heap
    std::priority_queue<Item, std::vector<Item>, std::greater<Item>> heap;
    for (int32_t p = 0; p < P; ++p) heap.push({0, p});
    std::vector<int32_t> cnt(P, 0);
    for (int64_t t = 0; t < nr; ++t) {
        if (heap.empty()) return -1;
        const int64_t q = order[t];
        Item it = heap.top();
        heap.pop();
        row_panel[q] = it.second;
        ++cnt[it.second];
        if (cnt[it.second] < R_cap) heap.push({it.first + tile_row_weight(ipr[q + 1] - ipr[q]), it.second});
    }
    for (int32_t p = 0; p < P; ++p) panel_off[p + 1] = panel_off[p] + cnt[p];
    std::vector<int32_t> fill(panel_off.begin(), panel_off.end() - 1);
    for (int64_t q = 0; q < nr; ++q) {
        const int32_t p = row_panel[q];
        row_local[q] = fill[p] - panel_off[p];
        panel_rows[fill[p]++] = (int32_t)q;
    }
    return P;
}

// ------------------------------------------------------------------ kernel
__device__ __forceinline__ uint2 ld_slot(const uint2* a) {
    uint2 v;
#if TILE_LDPOL == 0
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(a));
#elif TILE_LDPOL == 1
    asm volatile("ld.global.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(a));
#elif TILE_LDPOL == 3
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(a));
#else
    asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(a));
#endif
    return v;
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_consumers() { asm volatile("bar.sync 1, %0;" ::"n"(kTL) : "memory"); }

struct TileSet {
    uint2 s[4];
};

// Four consecutive steps of this lane from `at` (`left` steps remain in the
// tile; steps past it are pad slots: no load).
__device__ __forceinline__ void load4(TileSet& S, const uint2* at, int left) {
#pragma unroll
    for (int q = 0; q < 4; ++q) S.s[q] = (q < left) ? ld_slot(at + q * 32) : make_uint2(0u, 0u);
}

__device__ __forceinline__ float2 lds2(const char* base, uint32_t off) {
    return *reinterpret_cast<const float2*>(base + off);
}
// a predicated 64-bit shared load (v kept where p is false).  Lanes that are
// off take no part in the access: a warp's active lanes are served together
// when they fit one wavefront, and an unused lane reading a common dummy
// address instead costs a wavefront more (measured,
// scripts/probes/lds_bank_probe{2,3,4}.cu).  volatile: kept in program order
// with the block barriers (rows of F change owners between blocks).
__device__ __forceinline__ void lds2_if(float2& v, uint32_t sbase, uint32_t off, bool p) {
    asm volatile(
        "{\n.reg .pred q;\nsetp.ne.u32 q, %2, 0;\n@q ld.shared.v2.f32 {%0, %1}, [%3];\n}"
        : "+f"(v.x), "+f"(v.y)
        : "r"((uint32_t)p), "r"(sbase + off));
}


// NQ consecutive entries of this lane: contribution p w (X_i - X_j), w = 1 /
// (1 + r^2) (rcp.approx: 1 + r^2 >= 1, relative error <= 2^-22); pad slots
// (word 0, p = 0) add exactly 0.  Y_i is read when a run starts (NEWROW) and
// kept in registers; a run's sum goes to its row when it ends here (FLUSH).
// All loads of the NQ entries are issued first; Y_i and F_i loads are
// predicated on NEWROW / FLUSH (lanes that are off add no bank conflicts).
// The flush values are formed in registers and the (distinct: a row is one run
// of a lane) rows read-modified-written together.  lastw = the slot word of the
// lane's last real entry (a real word is never 0: the first entry of a run
// carries NEWROW, later ones a column > 0).
template <int NQ>
__device__ __forceinline__ void tileq(const TileSet& S, const char* sm, uint32_t ysoff, float2& yi, float& ax,
                                      float& ay, uint32_t& lastw) {
    const uint32_t sb = smem_u32(sm);
    float2 yj[NQ], yl[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const uint32_t w = S.s[q].x;
        const uint32_t ro = (w >> kRowShift) & kRowMask;
#if TILE_DIAG == 2
        yj[q] = lds2(sm, ysoff);
#else
        yj[q] = lds2(sm, ysoff + (w & kColMask));
#endif
        yl[q] = make_float2(0.f, 0.f);
        lds2_if(yl[q], sb, ro, w & kNewRow);
    }
    float fx[NQ], fy[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const uint32_t w = S.s[q].x;
        const float p = __uint_as_float(S.s[q].y);
        if (w & kNewRow) yi = yl[q];
        const float dx = yi.x - yj[q].x, dy = yi.y - yj[q].y;
        float rw;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rw) : "f"(fmaf(dx, dx, fmaf(dy, dy, 1.0f))));
        const float pw = p * rw;
        ax = fmaf(pw, dx, ax);
        ay = fmaf(pw, dy, ay);
        const bool fl = (int)w < 0;
        fx[q] = ax;
        fy[q] = ay;
        ax = fl ? 0.f : ax;
        ay = fl ? 0.f : ay;
        lastw = w ? w : lastw;
    }
#if TILE_DIAG == 1
    if (fx[0] == 1.2345f) *reinterpret_cast<float2*>(const_cast<char*>(sm) + kFsOff) = make_float2(fx[NQ - 1], fy[NQ - 1]);
#else
    // plain read-modify-write: rows owned by this lane in this block
    float2 v[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const uint32_t w = S.s[q].x;
        v[q] = make_float2(0.f, 0.f);
        lds2_if(v[q], sb, kFsOff + ((w >> kRowShift) & kRowMask), (w & (kFlush | kHub)) == kFlush);
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q)
        if ((S.s[q].x & (kFlush | kHub)) == kFlush)
            *reinterpret_cast<float2*>(const_cast<char*>(sm) + kFsOff + ((S.s[q].x >> kRowShift) & kRowMask)) =
                make_float2(v[q].x + fx[q], v[q].y + fy[q]);
    // shared (hub) rows: atomic adds (rare: runs split between warps)
    bool hf = false;
#pragma unroll
    for (int q = 0; q < NQ; ++q) hf |= (S.s[q].x & (kFlush | kHub)) == (kFlush | kHub);
    if (__any_sync(0xffffffffu, hf)) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
            if ((S.s[q].x & (kFlush | kHub)) == (kFlush | kHub)) {
                float* f = reinterpret_cast<float*>(const_cast<char*>(sm) + kFsOff + ((S.s[q].x >> kRowShift) & kRowMask));
                atomicAdd(f, fx[q]);
                atomicAdd(f + 1, fy[q]);
            }
    }
#endif
}

// the last r = 1..3 steps of a tile (set S, statically indexed)
__device__ __forceinline__ void tile_tail(const TileSet& S, int r, const char* sm, uint32_t ysoff, float2& yi,
                                          float& ax, float& ay, uint32_t& lastw) {
    if (r == 3) tileq<3>(S, sm, ysoff, yi, ax, ay, lastw);
    else if (r == 2) tileq<2>(S, sm, ysoff, yi, ax, ay, lastw);
    else tileq<1>(S, sm, ysoff, yi, ax, ay, lastw);
}

// a carry-out sum into its row: plain for rows owned by this warp in this
// block, atomic for shared (hub) rows
__device__ __forceinline__ void carry_add(char* Fs, int kc, float ax, float ay, uint32_t hub) {
    float2* f = reinterpret_cast<float2*>(Fs + kc);
    if (hub) {
        atomicAdd(&f->x, ax);
        atomicAdd(&f->y, ay);
    } else {
        const float2 v = *f;
        *f = make_float2(v.x + ax, v.y + ay);
    }
}

// After a tile: carry-outs (ax, ay) of runs that continue into the next lane's
// chunk (cv), keyed by row kc.  Sum them per row over consecutive lanes (a
// run's lanes are consecutive: rows are sorted; every lane a run passes through
// carries, so a row forms exactly one group) and add each sum once, by the last
// lane of its group.  The row's own flush (by the lane where the run ends, in
// this warp for an unshared row) happened earlier in program order; a shared
// (hub) row, whose run continues into another warp, only ever gets atomic adds.
__device__ __forceinline__ void tile_carry(float ax, float ay, uint32_t lastw, char* Fs, int lane) {
    const unsigned full = 0xffffffffu;
    const int kc = (int)((lastw >> kRowShift) & kRowMask);
    const bool nz = lastw != 0 && (int)lastw >= 0;   // a real last entry whose run does not end here
    const int kp = __shfl_up_sync(full, nz ? kc : -1, 1);
    if (__any_sync(full, nz && lane > 0 && kp == kc)) {
        // runs carried over more than one lane boundary: segmented inclusive
        // scan with head flags (a lane without a carry is its own segment)
        const int key = nz ? kc : -1 - lane;
        bool head = lane == 0 || kp != key;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float ux = __shfl_up_sync(full, ax, o), uy = __shfl_up_sync(full, ay, o);
            const bool uh = __shfl_up_sync(full, head, o);
            if (lane >= o) {
                if (!head) {
                    ax += ux;
                    ay += uy;
                }
                head = head || uh;
            }
        }
        const int kn = __shfl_down_sync(full, key, 1);
        if (nz && (lane == 31 || kn != key)) carry_add(Fs, kc, ax, ay, lastw & kHub);
    } else if (nz) {
        carry_add(Fs, kc, ax, ay, lastw & kHub);
    }
}

__device__ __forceinline__ int2 ld_tab(const int2* __restrict__ t, int J, int NB) {
    return J < NB ? __ldg(t + J) : make_int2(0, 0);
}
__device__ __forceinline__ bool mbar_try_wait_hint(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(20000u)
        : "memory");
    return ok != 0;
}

__global__ void __launch_bounds__((kTW + 1) * 32, 1) k_attr_tile(const uint8_t* __restrict__ plan,
                                                                 const float2* __restrict__ Y, float2* __restrict__ F,
                                                                 int y_aligned) {
    extern __shared__ __align__(128) uint8_t t_smem[];
    const TileHeader* h = reinterpret_cast<const TileHeader*>(plan);
    const int P = h->P, NB = h->NB;
    float2* Yi = reinterpret_cast<float2*>(t_smem);                   // kTR (swizzled row slots)
    float2* Fs = reinterpret_cast<float2*>(t_smem + kFsOff);          // kTR
    float2* ring = reinterpret_cast<float2*>(t_smem + kRingOff);      // kTS x kTB
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + kTS * kTB);   // full[kTS], empty[kTS]
    const int64_t n = h->n, rb = h->row_begin;
    const int2* wtab = reinterpret_cast<const int2*>(plan + h->off_wtab);   // [(p kTW + w) NB + J] = (step, K)
    const int32_t* roff = reinterpret_cast<const int32_t*>(plan + h->off_rowoff);
    const int32_t* rows = reinterpret_cast<const int32_t*>(plan + h->off_rows);
    const uint2* slots = reinterpret_cast<const uint2*>(plan + h->off_slots);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTS; ++s) {
            mbar_init(&bars[s], 1);
            mbar_init(&bars[kTS + s], 1);
        }
        *reinterpret_cast<float2*>(t_smem + kDummyOff) = make_float2(0.f, 0.f);
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kTW) {
        // ---------------- producer: Y of every block, in order, for each panel;
        // the entries of block J + kTPre (all warps' tiles: one contiguous
        // range) are prefetched into L2 before the ring wait for block J
        uint32_t k = 0;
        const unsigned full = 0xffffffffu;
        for (int p = blockIdx.x; p < P; p += gridDim.x) {
            // The panel sweeps the column blocks from block rot (tile_rot): sweep
            // position J is block jm(J).  wtab is in sweep order.  First step of
            // the block at sweep position J (warp 0's tile) in lane J - B0 of bv / bn.
            const int rot = tile_rot(p, h->G, NB);
            auto jm = [&](int J) { return J + rot < NB ? J + rot : J + rot - NB; };
            const int2* w0 = wtab + (int64_t)p * kTW * NB;
            const int2 lastt = w0[(int64_t)(kTW - 1) * NB + (NB - 1 - rot)];   // block NB - 1
            const int pend = lastt.x + lastt.y;                               // the panel's end step
            auto start_of = [&](int J) { return J < NB ? __ldg(&w0[J].x) : pend; };
            int bv = start_of(min(lane, NB)), bn = start_of(min(32 + lane, NB));
            int B0 = 0;
            auto block_start = [&](int J) {     // warp-uniform, J in [B0, B0 + 64)
                const int v = (J - B0 < 32) ? bv : bn;
                return __shfl_sync(full, v, (J - B0) & 31);
            };
            auto prefetch_block = [&](int J) {  // the entries of the block at sweep position J
                if (J >= NB) return;
                const int s0 = block_start(J);
                const int s1n = block_start(J + 1);   // the next sweep position's start (block jm(J) + 1)
                const int s1 = jm(J) == NB - 1 ? pend : (J + 1 < NB ? s1n : __ldg(&w0[0].x));
                if (lane == 0 && s1 > s0) prefetch_l2(slots + (size_t)s0 * 32, (uint32_t)(s1 - s0) * 32u * 8u);
            };
            for (int J = 0; J < NB; ++J) {
                if (J + kTPre + 1 - B0 >= 64) {   // keep sweep positions [B0, B0 + 64) in bv / bn
                    B0 += 32;
                    bv = bn;
                    bn = start_of(min(B0 + 32 + lane, NB));
                }
                if (kTPre >= 0) {
                    if (J == 0)
                        for (int q = 0; q < kTPre; ++q) prefetch_block(q);
                    prefetch_block(J + kTPre);
                }
                const int b = (int)(k % kTS);
                float2* dst = ring + b * kTB;
                if (k >= (uint32_t)kTS) mbar_wait(&bars[kTS + b], ((k / kTS) - 1) & 1);
                const int64_t lo = (int64_t)jm(J) * kTB;
                const int cnt = (int)std::min<int64_t>(kTB, n - lo);
                if (y_aligned) {
                    const int even = cnt & ~1;
                    if (lane == 0) {
                        if (cnt & 1) dst[cnt - 1] = Y[lo + cnt - 1];
#if TILE_DIAG == 6      // timing probe (wrong results): half of every Y block
                        const int ev = (even / 2) & ~1;
#elif TILE_DIAG == 7    // timing probe (wrong results): no Y block loads
                        const int ev = 0;
#else
                        const int ev = even;
#endif
                        mbar_arrive_tx(&bars[b], (uint32_t)(ev * sizeof(float2)));
                        if (ev) bulk_g2s(dst, Y + lo, (uint32_t)(ev * sizeof(float2)), &bars[b]);
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

    // ---------------- consumer warp `warp`: its tile of every block, lane = chunk
#if TILE_DIAG >= 3
    const long long t_start = clock64();
    long long t_wait = 0, t_bar = 0;
#endif
    const char* sm = reinterpret_cast<const char*>(t_smem);
    const unsigned full = 0xffffffffu;
    uint32_t k = 0;
    for (int p = blockIdx.x; p < P; p += gridDim.x) {
        const int r0 = roff[p], R = roff[p + 1] - r0;
        for (int r = threadIdx.x; r < R; r += kTL) {
            const uint32_t q = tile_slot((uint32_t)r);
            Yi[q] = Y[rb + (rows[r0 + r] & 0x7FFFFFFF)];
            Fs[q] = make_float2(0.f, 0.f);
        }
        bar_consumers();
        // this warp's (first step, steps) of blocks J0 .. J0 + 31 in tv (lane J - J0),
        // of the next 32 blocks in tn
        const int2* wt = wtab + ((int64_t)p * kTW + warp) * NB;
        int2 tv = ld_tab(wt, lane, NB), tn = ld_tab(wt, 32 + lane, NB);
        auto tile_of = [&](int J, int J0) {   // (first step, K) of block J >= J0 (warp-uniform)
            const int2 src = (J - J0 < 32) ? tv : tn;
            return make_int2(__shfl_sync(full, src.x, (J - J0) & 31), __shfl_sync(full, src.y, (J - J0) & 31));
        };
        int2 cur = tile_of(0, 0);
        TileSet A, B, C, D, E;
        const uint2* at = slots + (size_t)cur.x * 32 + lane;
        load4(A, at, cur.y);
        load4(B, at + 128, cur.y - 4);
        int J0 = 0;
        for (int J = 0; J < NB; ++J) {
            if (J - J0 == 32) {              // next 32 blocks
                J0 += 32;
                tv = tn;
                tn = ld_tab(wt, J0 + 32 + lane, NB);
            }
            const int K = cur.y;
            const int2 nxt = (J + 1 < NB) ? tile_of(J + 1, J0) : make_int2(0, 0);
            // the next tile's first two groups, a whole tile ahead of their use
            const uint2* atn = slots + (size_t)nxt.x * 32 + lane;
            load4(D, atn, nxt.y);
            load4(E, atn + 128, nxt.y - 4);
            const int b = (int)(k % kTS);
            const uint32_t ysoff = kRingOff + (uint32_t)b * (kTB * 8u);
#if TILE_DIAG >= 3
            const long long tw0 = clock64();
#endif
            while (!mbar_try_wait_hint(&bars[b], (k / kTS) & 1)) {
            }
#if TILE_DIAG >= 3
            t_wait += clock64() - tw0;
#endif
            if (K > 0) {
                float ax = 0.f, ay = 0.f;
                float2 yi = make_float2(0.f, 0.f);
                uint32_t lastw = 0;
                // three register sets rotated by unrolling, loads two groups ahead;
                // the last 1-3 steps of the tile run exactly (no pad steps computed)
                const uint2* ld = at + 256;          // step 8
#pragma unroll 1
                for (int left = K;;) {
                    load4(C, ld, left - 8);
                    if (left < 4) { tile_tail(A, left, sm, ysoff, yi, ax, ay, lastw); break; }
                    tileq<4>(A, sm, ysoff, yi, ax, ay, lastw);
                    left -= 4;
                    ld += 128;
                    if (left <= 0) break;
                    load4(A, ld, left - 8);
                    if (left < 4) { tile_tail(B, left, sm, ysoff, yi, ax, ay, lastw); break; }
                    tileq<4>(B, sm, ysoff, yi, ax, ay, lastw);
                    left -= 4;
                    ld += 128;
                    if (left <= 0) break;
                    load4(B, ld, left - 8);
                    if (left < 4) { tile_tail(C, left, sm, ysoff, yi, ax, ay, lastw); break; }
                    tileq<4>(C, sm, ysoff, yi, ax, ay, lastw);
                    left -= 4;
                    ld += 128;
                    if (left <= 0) break;
                }
                tile_carry(ax, ay, lastw, const_cast<char*>(sm) + kFsOff, lane);
            }
            cur = nxt;
            at = atn;
            A = D;
            B = E;
            // all warps done with block J: its ring stage is free, and no row is
            // read-modified-written by two warps (rows change owners between blocks)
#if TILE_DIAG == 4
            const long long tb0 = clock64();
            bar_consumers();
            t_bar += clock64() - tb0;
#elif TILE_DIAG == 5
            // timing probe (wrong results): no block barrier
#else
            bar_consumers();
#endif
            if (threadIdx.x == 0) mbar_arrive(&bars[kTS + b]);
            ++k;
        }
        bar_consumers();
        // rows of F: plain stores; a piece of a row split over several panels (bit 31) adds
        for (int r = threadIdx.x; r < R; r += kTL) {
            const int32_t q = rows[r0 + r];
            const float2 f = Fs[tile_slot((uint32_t)r)];
#if TILE_DIAG >= 3
            if (f.x == 1.2345f) F[q & 0x7FFFFFFF] = f;   // timing probes: F holds the counters
#else
            if (q >= 0) F[q] = f;
            else atomicAdd(F + (q & 0x7FFFFFFF), f);
#endif
        }
        bar_consumers();              // the next panel reuses Yi / Fs
    }
#if TILE_DIAG == 3
    // timing probe: per (CTA, warp) total cycles and cycles waiting for Y (results overwritten)
    if (lane == 0) F[blockIdx.x * kTW + warp] = make_float2((float)(clock64() - t_start), (float)t_wait);
#elif TILE_DIAG == 4
    // timing probe: per (CTA, warp) total cycles, cycles waiting for Y, cycles at the block barrier
    if (lane == 0) {
        F[2 * (blockIdx.x * kTW + warp)] = make_float2((float)(clock64() - t_start), (float)t_wait);
        F[2 * (blockIdx.x * kTW + warp) + 1] = make_float2((float)t_bar, 0.f);
    }
#endif
}

static size_t tile_smem_bytes(int) {
    return kRingOff + sizeof(float2) * (size_t)kTS * kTB + 2 * kTS * sizeof(uint64_t);
}

// F: rows [row_begin, row_end) of the plan's shard (nl = row_end - row_begin).
// No host read of the plan (the launch is captured in CUDA graphs): the shared
// memory is sized for kTR rows per panel and the grid is one CTA per SM; the
// kernel reads P and the panel sizes from the plan header.
cudaError_t launch_attr_cb(const void* plan, const float2* Y, float2* F, int64_t nl, cudaStream_t s) {
    if (nl == 0) return cudaSuccess;
    const size_t smem = tile_smem_bytes(kTR);
    cudaError_t e = cudaFuncSetAttribute(k_attr_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int aligned = ((uintptr_t)Y % 16) == 0;
    k_attr_tile<<<num_sms(), (kTW + 1) * 32, smem, s>>>(reinterpret_cast<const uint8_t*>(plan), Y, F, aligned);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ plan build
// Sort key of an entry: ((panel NB + block) << kTRbits) | local row; value:
// the shard-local entry index.  A stable LSD radix sort of entries in CSR order
// keeps columns ascending inside a (block tile, row) run.
__global__ void k_tile_keys(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, int64_t rb,
                            int64_t re, const int32_t* __restrict__ row_panel, const int32_t* __restrict__ row_local,
                            int NB, unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals) {
    const int lane = threadIdx.x & 31;
    const int64_t e0 = indptr[rb];
    for (int64_t r = rb + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); r < re;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t a = indptr[r], z = indptr[r + 1];
        const unsigned long long pk = (unsigned long long)row_panel[r - rb] * (unsigned long long)NB;
        const unsigned long long lr = (unsigned long long)row_local[r - rb];
        for (int64_t e = a + lane; e < z; e += 32) {
            const unsigned long long J = (unsigned long long)(indices[e] / kTB);
            keys[e - e0] = ((pk + J) << kTRbits) | lr;
            vals[e - e0] = (uint32_t)(e - e0);
        }
    }
}

// block-tile start / end positions in the sorted order (empty tiles stay 0, 0)
__global__ void k_tile_bounds(const unsigned long long* __restrict__ keys, int64_t m, int64_t* __restrict__ tstart,
                              int64_t* __restrict__ tend) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long t = keys[q] >> kTRbits;
        if (q == 0 || (keys[q - 1] >> kTRbits) != t) tstart[t] = q;
        if (q == m - 1 || (keys[q + 1] >> kTRbits) != t) tend[t] = q + 1;
    }
}

constexpr int kSnap = 48;   // a warp boundary moves to a run boundary within this many entries

// Per block tile (p, J): the row-sorted entries cut into kTW warp segments of
// equal size, each boundary moved to the nearest run (row) boundary within
// kSnap entries; a run longer than that is split between warps and its row
// marked shared (hub: every flush of the row, in any block, is atomic).
// seg[t (kTW + 1) + w] = first index of warp w's segment (seg[.. + kTW] = E);
// steps[t kTW + w] = ceil(E_w / 32).
__global__ void k_tile_segment(const unsigned long long* __restrict__ keys, const int64_t* __restrict__ tstart,
                               const int64_t* __restrict__ tend, int64_t ntb, int NB,
                               const int32_t* __restrict__ panel_off, int32_t* __restrict__ seg,
                               int64_t* __restrict__ steps, int32_t* __restrict__ hub) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntb; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s0 = tstart[t], E = tend[t] - s0;
        int32_t* sg = seg + t * (kTW + 1);
        sg[0] = 0;
        int64_t prev = 0;
        for (int w = 1; w < kTW; ++w) {
            const int64_t ideal = std::max<int64_t>(prev, E * w / kTW);
            int64_t cut = -1;
            for (int d = 0; d <= kSnap && cut < 0; ++d) {      // nearest q with a row change before q
                const int64_t qa = ideal - d, qb = ideal + d;
                if (qa >= prev && qa > 0 && qa < E && keys[s0 + qa - 1] != keys[s0 + qa]) cut = qa;
                else if (qb < E && qb > 0 && qb >= prev && keys[s0 + qb - 1] != keys[s0 + qb]) cut = qb;
            }
            if (ideal <= 0 || ideal >= E) cut = std::min<int64_t>(std::max<int64_t>(ideal, prev), E);
            if (cut < 0) {                                       // inside a long run: split it, shared row
                cut = ideal;
                const unsigned long long key = keys[s0 + cut];
                const int64_t p = (int64_t)((key >> kTRbits) / (unsigned long long)NB);
                atomicOr(&hub[panel_off[p] + (int32_t)(key & kLocalMask)], 1);
            }
            sg[w] = (int32_t)cut;
            prev = cut;
        }
        sg[kTW] = (int32_t)E;
        for (int w = 0; w < kTW; ++w) steps[t * kTW + w] = ((int64_t)sg[w + 1] - sg[w] + 31) / 32;
    }
}

// per-warp tile table in sweep order: wtab[(p kTW + w) NB + J] = (first step,
// steps) of the warp tile (p, jm, w), jm = (J + tile_rot(p)) mod NB: toff[u],
// toff[u + 1] - toff[u], u = (p NB + jm) kTW + w
__global__ void k_tile_wtab(const int64_t* __restrict__ toff, int64_t P, int64_t NB, int G, int2* __restrict__ wtab) {
    const int64_t m = P * NB * kTW;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t J = q % NB, pw = q / NB, w = pw % kTW, p = pw / kTW;
        const int64_t rot = tile_rot((int)p, G, (int)NB), jm = J + rot < NB ? J + rot : J + rot - NB;
        const int64_t u = (p * NB + jm) * kTW + w;
        wtab[q] = make_int2((int32_t)toff[u], (int32_t)(toff[u + 1] - toff[u]));
    }
}

// Bank byte of sorted position q: Y_j bank pair (column mod 16) | Y_i / F_i
// bank pair of the row slot << 4 (8-byte words: 16 bank pairs).
__global__ void k_tile_banks(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ vals, int64_t m,
                             const int32_t* __restrict__ indices, int64_t e0, uint8_t* __restrict__ cb) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t col = (uint32_t)(indices[(int64_t)vals[q] + e0] % kTB);
        const uint32_t sl = tile_slot((uint32_t)(keys[q] & kLocalMask));
        cb[q] = (uint8_t)((col & 15u) | ((sl & 15u) << 4));
    }
}

constexpr int kSchedMaxK = 512;    // chunks longer than this keep the row-sorted order
constexpr int kSchedW = kSchedMaxK / 64;
#ifndef SCHED_WY    // probe builds: weights of the Y_j and the Y_i / F_i bank counts
#define SCHED_WY 1
#endif
#ifndef SCHED_WR
#define SCHED_WR 2
#endif

// A lane's chunk as a set of entries not yet placed (bit i: chunk index i).
struct ChunkSet {
    unsigned long long w[kSchedW];
    __device__ bool has(int i) const { return (w[i >> 6] >> (i & 63)) & 1ull; }
    __device__ void take(int i) { w[i >> 6] &= ~(1ull << (i & 63)); }
    __device__ int count(int lo, int hi) const {     // entries left in [lo, hi)
        int c = 0;
        for (int q = lo >> 6; q <= (hi - 1) >> 6 && lo < hi; ++q) {
            unsigned long long m = w[q];
            if (q == lo >> 6) m &= ~0ull << (lo & 63);
            if (q == (hi - 1) >> 6 && (hi & 63)) m &= (1ull << (hi & 63)) - 1;
            c += __popcll(m);
        }
        return c;
    }
};

// Per warp tile (one thread): the order in which each lane walks its chunk.
// Any order keeps the arithmetic of a chunk (each row's entries form one run,
// a run's entries are summed in registers) as long as a run's entries stay
// consecutive and the run carried into the next chunk (if any) comes last.
// Within those rules a greedy pass picks, step by step, an entry for every
// lane whose shared-memory banks (Y_j, and Y_i / F_i where a run starts / ends)
// are least used so far by the lanes of the same half-warp at that step (a
// 64-bit shared access is served per half-warp: scripts/probes/) -- random
// gathers otherwise pile up ~3 deep per bank pair.  The most constrained lanes
// choose first: those with one entry to choose from, then those inside a run,
// then those starting a run.  Output per sorted position: step << 5 | lane |
// NEWROW << 30 | FLUSH << 31.
__global__ void k_tile_schedule(const unsigned long long* __restrict__ keys, const uint8_t* __restrict__ cb,
                                const int64_t* __restrict__ tstart, const int64_t* __restrict__ tend,
                                const int32_t* __restrict__ seg, const int64_t* __restrict__ toff, int64_t ntiles,
                                uint32_t* __restrict__ sched) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < ntiles; u += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = u / kTW, w = u % kTW;
        const int32_t* sg = seg + t * (kTW + 1);
        const int64_t base = tstart[t] + sg[w], tile_end = tend[t];
        const int64_t E = sg[w + 1] - sg[w];
        const int64_t K = toff[u + 1] - toff[u];
        if (E == 0) continue;
        auto key = [&](int64_t i) { return keys[base + i]; };
        // does the entry after segment index i (in tile order) continue its row?
        auto cont = [&](int64_t i) { return base + i + 1 < tile_end && keys[base + i + 1] == keys[base + i]; };
        if (K > kSchedMaxK) {    // row-sorted order (flags as in the sorted list)
            for (int64_t i = 0; i < E; ++i) {
                const int64_t l = i / K, k = i - l * K;
                const bool newrow = k == 0 || key(i - 1) != key(i);
                sched[base + i] = (uint32_t)(k << 5) | (uint32_t)l | (newrow ? kNewRow : 0u) | (cont(i) ? 0u : kFlush);
            }
            continue;
        }
        ChunkSet left[32];
        int16_t rs[32], re[32], tail[32], nleft[32];
        for (int l = 0; l < 32; ++l) {
            const int64_t a = l * K, b = std::min<int64_t>(a + K, E);
            const int n = a < b ? (int)(b - a) : 0;
            for (int q = 0; q < kSchedW; ++q) {
                const int lo = q * 64;
                left[l].w[q] = n <= lo ? 0ull : (n - lo >= 64 ? ~0ull : ((1ull << (n - lo)) - 1));
            }
            nleft[l] = (int16_t)n;
            rs[l] = re[l] = -1;
            tail[l] = -1;
            if (n > 0 && cont(b - 1)) {    // the chunk's last run goes on past it: it must come last
                int64_t st = b - 1;
                while (st > a && key(st - 1) == key(b - 1)) --st;
                tail[l] = (int16_t)(st - a);
            }
        }
        for (int64_t k = 0; k < K; ++k) {
            uint8_t hy[2][16], hr[2][16];
            for (int q = 0; q < 16; ++q) hy[0][q] = hy[1][q] = hr[0][q] = hr[1][q] = 0;
            // class of each lane at this step: 0 one choice, 1 inside a run, 2 a new run, 3 done
            uint8_t cls[32];
            for (int l = 0; l < 32; ++l) {
                if (nleft[l] == 0) { cls[l] = 3; continue; }
                const bool inrun = rs[l] >= 0 && left[l].count(rs[l], re[l]) > 0;
                const int choices = inrun ? left[l].count(rs[l], re[l]) : nleft[l];
                cls[l] = choices == 1 ? 0 : (inrun ? 1 : 2);
            }
            for (int c = 0; c < 3; ++c)
                for (int l = 0; l < 32; ++l) {
                    if (cls[l] != c) continue;
                    const int64_t a = l * K;
                    const int n = (int)(std::min<int64_t>(a + K, E) - a);
                    const int h = l >> 4;
                    int pick = -1;
                    bool newrow = false;
                    if (rs[l] >= 0 && left[l].count(rs[l], re[l]) > 0) {
                        int best = 1 << 30;
                        for (int i = rs[l]; i < re[l]; ++i) {
                            if (!left[l].has(i)) continue;
                            const int cst = hy[h][cb[base + a + i] & 15];
                            if (cst < best) { best = cst; pick = i; }
                        }
                    } else {
                        // a new run: any remaining entry; the tail run only when nothing else is left
                        const bool only_tail = tail[l] >= 0 && left[l].count(0, tail[l]) == 0;
                        const int hi = (tail[l] >= 0 && !only_tail) ? tail[l] : n;
                        int best = 1 << 30;
                        for (int i = 0; i < hi; ++i) {
                            if (!left[l].has(i)) continue;
                            const uint8_t bb = cb[base + a + i];
                            const bool single = (i == 0 || key(a + i - 1) != key(a + i)) &&
                                                (i == n - 1 || key(a + i + 1) != key(a + i));
                            const int cst = SCHED_WY * hy[h][bb & 15] + SCHED_WR * hr[h][bb >> 4] * (single ? 2 : 1);
                            if (cst < best) { best = cst; pick = i; }
                        }
                        int st = pick, en = pick + 1;
                        while (st > 0 && key(a + st - 1) == key(a + pick)) --st;
                        while (en < n && key(a + en) == key(a + pick)) ++en;
                        rs[l] = (int16_t)st;
                        re[l] = (int16_t)en;
                        newrow = true;
                    }
                    left[l].take(pick);
                    --nleft[l];
                    const uint8_t bb = cb[base + a + pick];
                    hy[h][bb & 15]++;
                    if (newrow) hr[h][bb >> 4]++;
                    bool flush = false;
                    if (left[l].count(rs[l], re[l]) == 0) {
                        // the run's part in this chunk is done: it ends here unless it goes on past the chunk
                        flush = !(re[l] == n && cont(a + n - 1));
                        if (flush) hr[h][bb >> 4]++;
                        rs[l] = re[l] = -1;
                    }
                    sched[base + a + pick] = (uint32_t)(k << 5) | (uint32_t)l | (newrow ? kNewRow : 0u) | (flush ? kFlush : 0u);
                }
        }
    }
}

// Slot of sorted position q: block tile t, index i in the tile, warp w (its
// segment holds i), index iw in the segment, chunk (lane) l = iw / K, step
// k = iw - l K with K = the segment's steps.  FLUSH: the row's run ends at
// this entry (the next entry of the tile is another row, or the tile ends);
// at a chunk end a run that continues is carried out instead (tile_carry).
// NEWROW: the first entry of a chunk or of a run.  HUB: the row is shared.
__global__ void k_tile_fill(const unsigned long long* __restrict__ keys, const uint32_t* __restrict__ vals, int64_t m,
                            const uint32_t* __restrict__ sched, const int64_t* __restrict__ toff,
                            const int32_t* __restrict__ seg, const int64_t* __restrict__ tstart, int NB,
                            const int32_t* __restrict__ panel_off, const int32_t* __restrict__ hub,
                            const int32_t* __restrict__ indices, const float* __restrict__ values, int64_t e0,
                            uint2* __restrict__ slots) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = keys[q];
        const unsigned long long t = key >> kTRbits;
        const int64_t i = q - tstart[t];
        const int32_t* sg = seg + t * (kTW + 1);
        int w = 0;
        while (w + 1 < kTW && sg[w + 1] <= i) ++w;
        const int64_t u = (int64_t)t * kTW + w;
        const uint32_t sc = sched[q];
        const int64_t l = sc & 31u, kk = (sc & ~(kNewRow | kFlush)) >> 5;
        const int64_t e = (int64_t)vals[q] + e0;
        const uint32_t col = (uint32_t)(indices[e] % kTB);
        const uint32_t lr = (uint32_t)(key & kLocalMask);
        const int64_t p = (int64_t)(t / (unsigned long long)NB);
        uint32_t word = (col << 3) | (tile_slot(lr) << (3 + kColBits)) | (sc & (kNewRow | kFlush));
        if (hub[panel_off[p] + (int32_t)lr]) word |= kHub;
        slots[(size_t)(toff[u] + kk) * 32 + l] = make_uint2(word, __float_as_uint(values[e]));
    }
}

struct TileWs {
    int32_t *row_panel, *row_local, *seg, *hub, *panel_off;
    unsigned long long *keys_a, *keys_b;
    uint32_t *vals_a, *vals_b;
    int64_t *tstart, *tend, *steps, *toff;
    uint8_t* cb;
    uint32_t* sched;
    void* cub_tmp;
    size_t cub_bytes, bytes;
};

// ntb block tiles (P NB), ntiles = ntb kTW warp tiles
static TileWs tile_ws_map(void* base, int64_t nr, int64_t m, int64_t ntb, int64_t P) {
    const int64_t ntiles = ntb * kTW;
    TileWs w{};
    size_t cb = 0, cs = 0;
    cub::DoubleBuffer<unsigned long long> dk(nullptr, nullptr);
    cub::DoubleBuffer<uint32_t> dv(nullptr, nullptr);
    cub::DeviceRadixSort::SortPairs(nullptr, cb, dk, dv, (int64_t)std::max<int64_t>(m, 1), 0, 64);
    cub::DeviceScan::ExclusiveSum(nullptr, cs, (int64_t*)nullptr, (int64_t*)nullptr, (int64_t)(ntiles + 1));
    w.cub_bytes = std::max(cb, cs);
    size_t off = 0;
    auto take = [&](size_t b) {
        size_t o = off;
        off = t_align(off + b);
        return (char*)base + o;
    };
    w.row_panel = (int32_t*)take(sizeof(int32_t) * std::max<int64_t>(nr, 1));
    w.row_local = (int32_t*)take(sizeof(int32_t) * std::max<int64_t>(nr, 1));
    w.seg = (int32_t*)take(sizeof(int32_t) * (size_t)(ntb * (kTW + 1)));
    w.hub = (int32_t*)take(sizeof(int32_t) * std::max<int64_t>(nr, 1));
    w.panel_off = (int32_t*)take(sizeof(int32_t) * (size_t)(P + 1));
    w.keys_a = (unsigned long long*)take(sizeof(unsigned long long) * std::max<int64_t>(m, 1));
    w.keys_b = (unsigned long long*)take(sizeof(unsigned long long) * std::max<int64_t>(m, 1));
    w.vals_a = (uint32_t*)take(sizeof(uint32_t) * std::max<int64_t>(m, 1));
    w.vals_b = (uint32_t*)take(sizeof(uint32_t) * std::max<int64_t>(m, 1));
    w.tstart = (int64_t*)take(sizeof(int64_t) * (ntb + 1));
    w.tend = (int64_t*)take(sizeof(int64_t) * (ntb + 1));
    w.steps = (int64_t*)take(sizeof(int64_t) * (ntiles + 1));
    w.toff = (int64_t*)take(sizeof(int64_t) * (ntiles + 1));
    w.cb = (uint8_t*)take(sizeof(uint8_t) * std::max<int64_t>(m, 1));
    w.sched = (uint32_t*)take(sizeof(uint32_t) * std::max<int64_t>(m, 1));
    w.cub_tmp = take(w.cub_bytes);
    w.bytes = off;
    return w;
}

static int tile_rows(const tsnet_csr* P, const tsnet_shard* sh, int64_t& rb, int64_t& re) {
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

struct TileCut {
    std::vector<int32_t> row_panel, row_local, panel_off, panel_rows;
    std::vector<int64_t> ip;
    int32_t P = 0, R_max = 0;
    int64_t nnz_s = 0;
};

static int tile_host_cut(const tsnet_csr* P, int64_t rb, int64_t re, cudaStream_t s, TileCut& cut) {
    cut.ip.assign(re - rb + 1, 0);
    if (P->n > 0) {
        TSNET_CUDA(cudaMemcpyAsync(cut.ip.data(), P->indptr + rb, sizeof(int64_t) * cut.ip.size(),
                                   cudaMemcpyDeviceToHost, s));
        TSNET_CUDA(cudaStreamSynchronize(s));
    }
    cut.nnz_s = cut.ip.back() - cut.ip.front();
    TSNET_ARG(cut.nnz_s < ((int64_t)1 << 32), "a plan holds < 2^32 entries per shard (got %lld)", (long long)cut.nnz_s);
    cut.P = tile_partition(cut.ip.data(), re - rb, num_sms(), kTR, cut.row_panel, cut.row_local, cut.panel_off,
                           cut.panel_rows);
    TSNET_ARG(cut.P > 0, "row partition failed");
    cut.R_max = 0;
    for (int32_t p = 0; p < cut.P; ++p) cut.R_max = std::max(cut.R_max, cut.panel_off[p + 1] - cut.panel_off[p]);
    return TSNET_OK;
}

}  // namespace tsnet

using namespace tsnet;

extern "C" {

int32_t tsnet_plan_partition(const int64_t* indptr_host, int64_t row_begin, int64_t row_end, int32_t groups,
                             int32_t rows_cap, int32_t* row_panel, int32_t* row_local, int32_t* panel_off,
                             int32_t* panel_rows, int64_t max_panels) {
    if (!indptr_host || !row_panel || !row_local || !panel_off || !panel_rows || row_begin < 0 ||
        row_end < row_begin || groups < 1 || rows_cap < 1)
        return -1;
    std::vector<int32_t> a, b, c, d;
    const int32_t P = tile_partition(indptr_host + row_begin, row_end - row_begin, groups, rows_cap, a, b, c, d);
    if (P < 0 || (int64_t)P > max_panels) return -1;
    std::memcpy(row_panel, a.data(), sizeof(int32_t) * a.size());
    std::memcpy(row_local, b.data(), sizeof(int32_t) * b.size());
    std::memcpy(panel_off, c.data(), sizeof(int32_t) * c.size());
    std::memcpy(panel_rows, d.data(), sizeof(int32_t) * d.size());
    return P;
}

int tsnet_plan_query(const tsnet_csr* P, const tsnet_shard* shard, size_t* plan_bytes, size_t* ws_bytes,
                     tsnet_stream_t stream) {
    TSNET_ARG(P != nullptr && plan_bytes != nullptr && ws_bytes != nullptr, "NULL argument");
    TSNET_ARG(P->n >= 0 && P->nnz >= 0 && (P->n == 0 || P->indptr), "invalid P");
    int64_t rb, re;
    int st = tile_rows(P, shard, rb, re);
    if (st != TSNET_OK) return st;
    TileCut cut;
    if ((st = tile_host_cut(P, rb, re, (cudaStream_t)stream, cut)) != TSNET_OK) return st;
    // upper bound of the steps: every non-empty warp tile pads < one step
    const int64_t NB = std::max<int64_t>(1, (P->n + kTB - 1) / kTB);
    const int64_t ntb = (int64_t)cut.P * NB, ntiles = ntb * kTW;
    const int64_t steps_max = (cut.nnz_s + 31) / 32 + std::min<int64_t>(ntiles, cut.nnz_s);
    const TileHeader h = tile_layout(P->n, rb, re, cut.nnz_s, cut.P, cut.R_max, steps_max);
    *plan_bytes = (size_t)h.bytes;
    *ws_bytes = tile_ws_map(nullptr, re - rb, cut.nnz_s, ntb, cut.P).bytes;
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
    int st = tile_rows(P, shard, rb, re);
    if (st != TSNET_OK) return st;
    TileCut cut;
    if ((st = tile_host_cut(P, rb, re, s, cut)) != TSNET_OK) return st;
    const int64_t nr = re - rb, m = cut.nnz_s;
    const int64_t NB = std::max<int64_t>(1, (P->n + kTB - 1) / kTB);
    const int64_t ntb = (int64_t)cut.P * NB, ntiles = ntb * kTW;
    TSNET_ARG(ntb < ((int64_t)1 << (64 - kTRbits - 1)), "too many tiles");
    TileWs w = tile_ws_map(ws, nr, m, ntb, cut.P);
    TSNET_ARG(ws != nullptr && ws_bytes >= w.bytes, "plan workspace too small (%zu < %zu bytes)", ws_bytes, w.bytes);
    if (nr > 0) {
        TSNET_CUDA(cudaMemcpyAsync(w.row_panel, cut.row_panel.data(), sizeof(int32_t) * nr, cudaMemcpyHostToDevice, s));
        TSNET_CUDA(cudaMemcpyAsync(w.row_local, cut.row_local.data(), sizeof(int32_t) * nr, cudaMemcpyHostToDevice, s));
    }
    TSNET_CUDA(cudaMemcpyAsync(w.panel_off, cut.panel_off.data(), sizeof(int32_t) * (cut.P + 1), cudaMemcpyHostToDevice,
                               s));
    TSNET_CUDA(cudaMemsetAsync(w.hub, 0, sizeof(int32_t) * std::max<int64_t>(nr, 1), s));
    TSNET_CUDA(cudaMemsetAsync(w.tstart, 0, sizeof(int64_t) * (ntb + 1), s));
    TSNET_CUDA(cudaMemsetAsync(w.tend, 0, sizeof(int64_t) * (ntb + 1), s));
    TSNET_CUDA(cudaMemsetAsync(w.steps, 0, sizeof(int64_t) * (ntiles + 1), s));
    int end_bit = kTRbits;
    while (end_bit < 64 && ((uint64_t)1 << (end_bit - kTRbits)) < (uint64_t)ntb) ++end_bit;
    cub::DoubleBuffer<unsigned long long> dk(w.keys_a, w.keys_b);
    cub::DoubleBuffer<uint32_t> dv(w.vals_a, w.vals_b);
    if (m > 0) {
        k_tile_keys<<<num_sms() * 8, 256, 0, s>>>(P->indptr, P->indices, rb, re, w.row_panel, w.row_local, (int)NB,
                                                  w.keys_a, w.vals_a);
        TSNET_LAUNCH_CHECK();
        size_t tb = w.cub_bytes;
        TSNET_CUDA(cub::DeviceRadixSort::SortPairs(w.cub_tmp, tb, dk, dv, m, 0, end_bit, s));
        k_tile_bounds<<<num_sms() * 8, 256, 0, s>>>(dk.Current(), m, w.tstart, w.tend);
        TSNET_LAUNCH_CHECK();
    }
    k_tile_segment<<<std::max<int64_t>(1, std::min<int64_t>((ntb + 255) / 256, num_sms() * 8)), 256, 0, s>>>(
        dk.Current(), w.tstart, w.tend, ntb, (int)NB, w.panel_off, w.seg, w.steps, w.hub);
    TSNET_LAUNCH_CHECK();
    size_t tb = w.cub_bytes;
    TSNET_CUDA(cub::DeviceScan::ExclusiveSum(w.cub_tmp, tb, w.steps, w.toff, ntiles + 1, s));
    int64_t steps = 0;
    TSNET_CUDA(cudaMemcpyAsync(&steps, w.toff + ntiles, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TSNET_CUDA(cudaStreamSynchronize(s));
    TSNET_ARG(steps < ((int64_t)1 << 31), "plan too large (%lld steps)", (long long)steps);
    TileHeader h = tile_layout(P->n, rb, re, m, cut.P, cut.R_max, steps);
    TSNET_ARG(plan_bytes >= (size_t)h.bytes, "plan buffer too small (%zu < %lld bytes)", plan_bytes, (long long)h.bytes);
    uint8_t* pb = reinterpret_cast<uint8_t*>(plan);
    uint2* d_slots = reinterpret_cast<uint2*>(pb + h.off_slots);
    k_tile_wtab<<<num_sms() * 4, 256, 0, s>>>(w.toff, cut.P, NB, h.G, reinterpret_cast<int2*>(pb + h.off_wtab));
    TSNET_LAUNCH_CHECK();
    TSNET_CUDA(cudaMemcpyAsync(pb + h.off_rowoff, cut.panel_off.data(), sizeof(int32_t) * (cut.P + 1),
                               cudaMemcpyHostToDevice, s));
    if (nr > 0)
        TSNET_CUDA(cudaMemcpyAsync(pb + h.off_rows, cut.panel_rows.data(), sizeof(int32_t) * nr,
                                   cudaMemcpyHostToDevice, s));
    if (steps > 0) TSNET_CUDA(cudaMemsetAsync(d_slots, 0, sizeof(uint2) * 32 * (size_t)steps, s));
    if (m > 0) {
        k_tile_banks<<<num_sms() * 8, 256, 0, s>>>(dk.Current(), dv.Current(), m, P->indices, cut.ip.front(), w.cb);
        TSNET_LAUNCH_CHECK();
        k_tile_schedule<<<(int)std::max<int64_t>(1, std::min<int64_t>((ntiles + 127) / 128, (int64_t)num_sms() * 16)),
                          128, 0, s>>>(dk.Current(), w.cb, w.tstart, w.tend, w.seg, w.toff, ntiles, w.sched);
        TSNET_LAUNCH_CHECK();
        k_tile_fill<<<num_sms() * 8, 256, 0, s>>>(dk.Current(), dv.Current(), m, w.sched, w.toff, w.seg, w.tstart,
                                                  (int)NB, w.panel_off, w.hub, P->indices, P->values, cut.ip.front(),
                                                  d_slots);
        TSNET_LAUNCH_CHECK();
    }
    TSNET_CUDA(cudaMemcpyAsync(pb, &h, sizeof(TileHeader), cudaMemcpyHostToDevice, s));
    TSNET_CUDA(cudaStreamSynchronize(s));
    return TSNET_OK;
}

}  // extern "C"
