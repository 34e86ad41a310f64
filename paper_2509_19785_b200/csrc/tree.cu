// tree.cu -- quadtree (Barnes-Hut) gradient of BH-tsNET and FIt-tsNET (NEXT-3).
//
// BH-tsNET: a quadtree on the drawing; per point
// a depth-first search from the root where a node that can be used as a
// summary stands for its points at their centre of mass;
// the KL repulsion (Eq. 6 second term, with Z summed the same way) and the
// entropy gradient of Eq. 7 (R2/R3) are accumulated over the
// summaries.  FIt-tsNET takes the repulsion from the
// interpolation grid and only the entropy from the quadtree.  Readings R23-R24
// (DESIGN.md), the same as the test oracle O9:
//   tree    root = square [lo, lo + S]^2 of the bounding box; depth-16 cells
//           ix = floor((x - lo_x) / S * 2^16) (fp64), Morton code = ix bits
//           even, iy bits odd; a node at level l = a maximal run of the
//           Morton-sorted points (stable) sharing the top 2l bits, side
//           S / 2^l, centre of mass from fp64 prefix sums of the sorted
//           coordinates;
//   summary side^2 < theta^2 |X_i - com|^2 (fp64) for nodes of > 1 point;
//           one-point nodes are exact pairs (skip i); a level-16 node that is
//           not a summary is taken point by point.
//
// GPU layout: Morton codes + CUB radix sort (stable), CUB scans of the sorted
// coordinates, per level a start flag + exclusive scan (node index of every
// run start) and the compacted run starts, so that the children of node
// (l, k) are the level-(l+1) nodes scan_{l+1}[start] .. scan_{l+1}[end].  The
// walk is a thread per point in Morton order (neighbouring threads take
// similar paths), with a local-memory stack, fp64 accumulation.
#include <cmath>

#include <cub/cub.cuh>

#include "common.cuh"
#include "tsnet.h"

namespace tsnet {

constexpr int kTreeDepth = 16;
constexpr int kTreeLevels = kTreeDepth + 1;
constexpr int kTreeStack = 64;

struct TreeHdr {
    double lo_x, lo_y, S;
    double Z;
    unsigned bb[4];          // encoded min x, min y, max x, max y
};

struct TreeWs {
    TreeHdr* hdr;
    uint32_t* code_in;
    int32_t* idx_in;
    uint32_t* code;          // sorted
    int32_t* perm;           // sorted position -> point
    double* Px;              // n + 1 prefix sums of the sorted x (P[0] = 0)
    double* Py;
    double* xs;              // n sorted x, then y (scan inputs)
    int32_t* flag;           // n + 1
    int32_t* scan;           // kTreeLevels x (n + 1)
    int32_t* starts;         // kTreeLevels x (n + 1)
    double2* R;              // n : repulsion sums (by point)
    double2* E;              // n : entropy sums (by point)
    void* cub_tmp;
    size_t cub_bytes, bytes;
};

static size_t tree_cub_bytes(int64_t n) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (uint32_t*)nullptr, (uint32_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, (int)n, 0, 32);
    cub::DeviceScan::InclusiveSum(nullptr, b, (double*)nullptr, (double*)nullptr, (int)n);
    cub::DeviceScan::ExclusiveSum(nullptr, c, (int32_t*)nullptr, (int32_t*)nullptr, (int)(n + 1));
    return std::max(a, std::max(b, c));
}

static TreeWs tree_ws_map(void* base, int64_t n) {
    TreeWs w{};
    size_t off = 0;
    auto take = [&](size_t b) {
        void* q = (char*)base + off;
        off = (off + b + 255) / 256 * 256;
        return q;
    };
    w.hdr = (TreeHdr*)take(sizeof(TreeHdr));
    w.code_in = (uint32_t*)take(sizeof(uint32_t) * (size_t)n);
    w.idx_in = (int32_t*)take(sizeof(int32_t) * (size_t)n);
    w.code = (uint32_t*)take(sizeof(uint32_t) * (size_t)n);
    w.perm = (int32_t*)take(sizeof(int32_t) * (size_t)n);
    w.Px = (double*)take(sizeof(double) * (size_t)(n + 1));
    w.Py = (double*)take(sizeof(double) * (size_t)(n + 1));
    w.xs = (double*)take(sizeof(double) * 2 * (size_t)n);
    w.flag = (int32_t*)take(sizeof(int32_t) * (size_t)(n + 1));
    w.scan = (int32_t*)take(sizeof(int32_t) * (size_t)(n + 1) * kTreeLevels);
    w.starts = (int32_t*)take(sizeof(int32_t) * (size_t)(n + 1) * kTreeLevels);
    w.R = (double2*)take(sizeof(double2) * (size_t)n);
    w.E = (double2*)take(sizeof(double2) * (size_t)n);
    w.cub_bytes = tree_cub_bytes(std::max<int64_t>(n, 1));
    w.cub_tmp = take(w.cub_bytes);
    w.bytes = off;
    return w;
}

// order-preserving unsigned keys of floats (0 = empty: max of ~key for minima)
__device__ __forceinline__ unsigned tkey(float x) {
    const unsigned u = __float_as_uint(x);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float tval(unsigned k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

__global__ void k_tree_bbox(const float2* __restrict__ Y, int64_t n, TreeHdr* h) {
    unsigned mnx = 0u, mny = 0u, mxx = 0u, mxy = 0u;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 y = Y[i];
        mnx = max(mnx, ~tkey(y.x));
        mny = max(mny, ~tkey(y.y));
        mxx = max(mxx, tkey(y.x));
        mxy = max(mxy, tkey(y.y));
    }
    for (int o = 16; o > 0; o >>= 1) {
        mnx = max(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
        mny = max(mny, __shfl_xor_sync(0xffffffffu, mny, o));
        mxx = max(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
        mxy = max(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&h->bb[0], mnx);
        atomicMax(&h->bb[1], mny);
        atomicMax(&h->bb[2], mxx);
        atomicMax(&h->bb[3], mxy);
    }
}

__global__ void k_tree_geom(TreeHdr* h) {
    const double lo_x = (double)tval(~h->bb[0]), lo_y = (double)tval(~h->bb[1]);
    const double hi_x = (double)tval(h->bb[2]), hi_y = (double)tval(h->bb[3]);
    double S = fmax(hi_x - lo_x, hi_y - lo_y);
    if (!(S > 0.0)) S = 1.0;
    h->lo_x = lo_x;
    h->lo_y = lo_y;
    h->S = S;
    h->Z = 0.0;
}

__device__ __forceinline__ uint32_t spread_bits(uint32_t v) {   // 16 bits -> even positions
    v &= 0xFFFFu;
    v = (v | (v << 8)) & 0x00FF00FFu;
    v = (v | (v << 4)) & 0x0F0F0F0Fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}

__global__ void k_tree_codes(const float2* __restrict__ Y, int64_t n, const TreeHdr* __restrict__ h,
                             uint32_t* __restrict__ code, int32_t* __restrict__ idx) {
    const double lo_x = h->lo_x, lo_y = h->lo_y, S = h->S;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 y = Y[i];
        double cx = floor(((double)y.x - lo_x) / S * 65536.0), cy = floor(((double)y.y - lo_y) / S * 65536.0);
        cx = fmin(fmax(cx, 0.0), 65535.0);
        cy = fmin(fmax(cy, 0.0), 65535.0);
        code[i] = spread_bits((uint32_t)cx) | (spread_bits((uint32_t)cy) << 1);
        idx[i] = (int32_t)i;
    }
}

__global__ void k_tree_gather(const float2* __restrict__ Y, const int32_t* __restrict__ perm, int64_t n,
                              double* __restrict__ xs) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const float2 y = Y[perm[t]];
        xs[t] = (double)y.x;
        xs[n + t] = (double)y.y;
    }
}

__global__ void k_tree_flags(const uint32_t* __restrict__ code, int64_t n, int shift, int32_t* __restrict__ flag) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s <= n; s += (int64_t)gridDim.x * blockDim.x) {
        int f = 0;
        if (s < n) f = (s == 0) || ((code[s] >> shift) != (code[s - 1] >> shift));
        flag[s] = f;
    }
}

__global__ void k_tree_starts(const int32_t* __restrict__ flag, const int32_t* __restrict__ scan, int64_t n,
                              int32_t* __restrict__ starts) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s <= n; s += (int64_t)gridDim.x * blockDim.x) {
        if (s == n) starts[scan[n]] = (int32_t)n;
        else if (flag[s]) starts[scan[s]] = (int32_t)s;
    }
}

struct TreeView {
    const int32_t* perm;
    const double* Px;
    const double* Py;
    const int32_t* scan;     // level l at scan + l (n + 1)
    const int32_t* starts;   // level l at starts + l (n + 1)
    int64_t n;
};

// per point (thread per Morton-sorted position): Z part, R_i, E_i
__global__ void __launch_bounds__(256) k_tree_walk(const float2* __restrict__ Y, TreeView tv, TreeHdr* h,
                                                   double theta, double eps, double2* __restrict__ R,
                                                   double2* __restrict__ E) {
    const int64_t n = tv.n;
    const int64_t ld = n + 1;
    const double S = h->S, th2 = theta * theta;
    double zsum = 0.0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int i = tv.perm[t];
        const float2 yi = Y[i];
        const double xi = (double)yi.x, yv = (double)yi.y;
        double z = 0.0, rx = 0.0, ry = 0.0, ex = 0.0, ey = 0.0;
        auto pair = [&](double px, double py, double cnt) {
            const double dx = xi - px, dy = yv - py;
            const double r2 = dx * dx + dy * dy;
            const double w = 1.0 / (1.0 + r2);
            z += cnt * w;
            rx += cnt * w * w * dx;
            ry += cnt * w * w * dy;
            const double ke = cnt / (eps + r2);
            ex += ke * dx;
            ey += ke * dy;
        };
        int stack[kTreeStack];
        int sp = 0;
        stack[sp++] = 0;                                  // (level 0, node 0)
        while (sp > 0) {
            const int code = stack[--sp];
            const int lev = code & 31, k = code >> 5;
            const int s = tv.starts[lev * ld + k], e = tv.starts[lev * ld + k + 1];
            const int cnt = e - s;
            if (cnt == 1) {
                const int j = tv.perm[s];
                if (j != i) {
                    const float2 yj = Y[j];
                    pair((double)yj.x, (double)yj.y, 1.0);
                }
                continue;
            }
            const double cx = (tv.Px[e] - tv.Px[s]) / cnt, cy = (tv.Py[e] - tv.Py[s]) / cnt;
            const double dx = xi - cx, dy = yv - cy;
            const double side = ldexp(S, -lev);
            if (side * side < th2 * (dx * dx + dy * dy)) {
                pair(cx, cy, (double)cnt);
            } else if (lev == kTreeDepth) {
                for (int q = s; q < e; ++q) {
                    const int j = tv.perm[q];
                    if (j != i) {
                        const float2 yj = Y[j];
                        pair((double)yj.x, (double)yj.y, 1.0);
                    }
                }
            } else {
                const int j0 = tv.scan[(lev + 1) * ld + s], j1 = tv.scan[(lev + 1) * ld + e];
                for (int j = j1 - 1; j >= j0 && sp < kTreeStack; --j) stack[sp++] = (j << 5) | (lev + 1);
            }
        }
        R[i] = make_double2(rx, ry);
        E[i] = make_double2(ex, ey);
        zsum += z;
    }
    for (int o = 16; o > 0; o >>= 1) zsum += __shfl_xor_sync(0xffffffffu, zsum, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&h->Z, zsum);
}

// BH-tsNET: g = 4 lkl (F_attr - R / Z) + (lc / n) X - (lr / n^2) E
__global__ void k_tree_grad_bh(int64_t n, const float2* __restrict__ Y, const float2* __restrict__ Fa,
                               const double2* __restrict__ R, const double2* __restrict__ E,
                               const TreeHdr* __restrict__ h, double lkl, double lc, double lr, float2* __restrict__ g) {
    const double Z = h->Z, nn = (double)n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 y = Y[i], fa = Fa[i];
        const double2 r = R[i], e = E[i];
        g[i] = make_float2((float)(4.0 * lkl * ((double)fa.x - r.x / Z) + (lc / nn) * (double)y.x - (lr / (nn * nn)) * e.x),
                           (float)(4.0 * lkl * ((double)fa.y - r.y / Z) + (lc / nn) * (double)y.y - (lr / (nn * nn)) * e.y));
    }
}

// FIt-tsNET: g (interpolated, lr = 0) -= (lr / n^2) E
__global__ void k_tree_grad_fit(int64_t n, const double2* __restrict__ E, double lr, float2* __restrict__ g) {
    const double nn = (double)n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 v = g[i];
        const double2 e = E[i];
        g[i] = make_float2((float)((double)v.x - (lr / (nn * nn)) * e.x), (float)((double)v.y - (lr / (nn * nn)) * e.y));
    }
}

static int tree_blocks(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)kNumSMs * 8)); }

// build the quadtree of Y and walk it: h->Z, R, E
cudaError_t tree_sums(const float2* Y, int64_t n, double theta, double eps, void* tws, cudaStream_t s) {
    TreeWs w = tree_ws_map(tws, n);
    cudaError_t e;
    const int nb = tree_blocks(n);
    if ((e = cudaMemsetAsync(w.hdr, 0, sizeof(TreeHdr), s)) != cudaSuccess) return e;
    k_tree_bbox<<<nb, 256, 0, s>>>(Y, n, w.hdr);
    k_tree_geom<<<1, 1, 0, s>>>(w.hdr);
    k_tree_codes<<<nb, 256, 0, s>>>(Y, n, w.hdr, w.code_in, w.idx_in);
    size_t tb = w.cub_bytes;
    if ((e = cub::DeviceRadixSort::SortPairs(w.cub_tmp, tb, w.code_in, w.code, w.idx_in, w.perm, (int)n, 0, 32, s)) !=
        cudaSuccess)
        return e;
    k_tree_gather<<<nb, 256, 0, s>>>(Y, w.perm, n, w.xs);
    if ((e = cudaMemsetAsync(w.Px, 0, sizeof(double), s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(w.Py, 0, sizeof(double), s)) != cudaSuccess) return e;
    tb = w.cub_bytes;
    if ((e = cub::DeviceScan::InclusiveSum(w.cub_tmp, tb, w.xs, w.Px + 1, (int)n, s)) != cudaSuccess) return e;
    tb = w.cub_bytes;
    if ((e = cub::DeviceScan::InclusiveSum(w.cub_tmp, tb, w.xs + n, w.Py + 1, (int)n, s)) != cudaSuccess) return e;
    const int64_t ld = n + 1;
    for (int lev = 0; lev <= kTreeDepth; ++lev) {
        k_tree_flags<<<nb, 256, 0, s>>>(w.code, n, 2 * (kTreeDepth - lev), w.flag);
        tb = w.cub_bytes;
        if ((e = cub::DeviceScan::ExclusiveSum(w.cub_tmp, tb, w.flag, w.scan + lev * ld, (int)(n + 1), s)) !=
            cudaSuccess)
            return e;
        k_tree_starts<<<nb, 256, 0, s>>>(w.flag, w.scan + lev * ld, n, w.starts + lev * ld);
    }
    TreeView tv{w.perm, w.Px, w.Py, w.scan, w.starts, n};
    k_tree_walk<<<nb, 256, 0, s>>>(Y, tv, w.hdr, theta, eps, w.R, w.E);
    return cudaGetLastError();
}

}  // namespace tsnet

using namespace tsnet;

extern "C" {

size_t tsnet_tree_workspace_bytes(int64_t n) {
    if (n < 0) return 0;
    return tree_ws_map(nullptr, n).bytes;
}

}  // extern "C"

namespace tsnet {

int tree_gradient(const Ws& w, const GradArgs& a, double theta, int variant, float2* grad, double* Z_out,
                  void* tws, size_t tws_bytes, cudaStream_t s) {
    const int64_t n = a.n;
    TSNET_ARG(theta >= 0.0 && theta < 0.7 && std::isfinite(theta),
              "theta = %g must be in [0, 0.7) (a summary then never contains its own point)", theta);
    TSNET_ARG(variant == 0 || variant == 1, "variant must be 0 (BH-tsNET) or 1 (FIt-tsNET)");
    TSNET_ARG(n < ((int64_t)1 << 26), "the quadtree walk indexes nodes with 26 bits (n < 2^26)");
    const TreeWs tw = tree_ws_map(tws, n);
    TSNET_ARG(tws != nullptr && tws_bytes >= tw.bytes, "tree workspace too small (%zu < %zu bytes)", tws_bytes,
              tw.bytes);
    TSNET_CUDA(tree_sums(a.Y, n, theta, (double)a.eps, tws, s));
    const int nb = tree_blocks(n);
    if (variant == 0) {
        TSNET_CUDA(launch_spmv(w, a, s));
        k_tree_grad_bh<<<nb, 256, 0, s>>>(n, a.Y, w.f_attr, tw.R, tw.E, tw.hdr, a.lambda_kl, a.lambda_c, a.lambda_r,
                                         grad);
        TSNET_LAUNCH_CHECK();
    } else {
        GradArgs b = a;
        b.lambda_r = 0.0f;                                 // the grid carries the repulsion only
        TSNET_CUDA(launch_field_phase(w, b, s));
        TSNET_CUDA(launch_spmv(w, b, s));
        TSNET_CUDA(launch_grad_out(w, b, grad, nullptr, nullptr, s));
        k_tree_grad_fit<<<nb, 256, 0, s>>>(n, tw.E, a.lambda_r, grad);
        TSNET_LAUNCH_CHECK();
    }
    // Z of the gradient: the tree's (BH-tsNET) or the grid's (FIt-tsNET)
    if (Z_out)
        TSNET_CUDA(cudaMemcpyAsync(Z_out, variant == 0 ? &tw.hdr->Z : &w.geo->Z, sizeof(double),
                                   cudaMemcpyDeviceToDevice, s));
    return TSNET_OK;
}

}  // namespace tsnet
