// move.cuh -- step a7 pieces shared by the stand-alone move (k_update,
// iterate.cu) and the move fused into the sliced-ELL SpMV (attr_sell.cu):
// the field gather at a point and the gains/momentum update (reading R12).
#pragma once

#include "common.cuh"

namespace tsnet {

// a1: box of a point and its in-box coordinates (fp64 arithmetic, reading
// R16); shared by the box sort (field.cu) and the move, which recomputes it
// from the position it reads anyway instead of reading it back (12 B/point).
// (y - lo) / h_b is formed as (y - lo) * inv_h (inv_h = 1 / h_b, fp64): the
// product is within 1.5 ulp of the quotient, i.e. within 3.4e-13 of it for
// |r| <= I <= 1024, so the box (its floor) is the quotient's unless r lies
// within kBoxGuard of an integer -- then the quotient itself decides.
constexpr double kBoxGuard = 1e-10;
// out of line, so that the (rarely taken) exact division is a branch and not
// computed for every point and selected
static __device__ __noinline__ double box_coord_exact(double d, double h_b) { return d / h_b; }
// one axis: the interval b in [0, I) and the coordinate u in it
__device__ __forceinline__ void box_axis(float y, double lo, double h_b, double inv_h, int I, int& b, float& u) {
    const double d = (double)y - lo;          // exact: both are fp32 values
    double r = d * inv_h;
    double f = floor(r);
    double t = r - f;
    if (fabs(t - 0.5) > 0.5 - kBoxGuard) {    // within kBoxGuard of a boundary: the quotient decides
        r = box_coord_exact(d, h_b);
        f = floor(r);
        t = r - f;
    }
    const int bi = (int)f;
    b = min(max(bi, 0), I - 1);
    u = (float)t;
    if (b != bi) u = (float)(r - (double)b);  // clamped (a point on the far edge)
}
__device__ __forceinline__ void box_of(float2 y, double lo_x, double lo_y, double h_b, double inv_h, int I, int& b,
                                       float& ux, float& uy) {
    int bx, by;
    box_axis(y.x, lo_x, h_b, inv_h, I, bx, ux);
    box_axis(y.y, lo_y, h_b, inv_h, I, by, uy);
    b = by * I + bx;
}

__device__ __forceinline__ void lagrange3u(float u, float (&L)[3]) {
    const float s0 = 1.0f / 6.0f, s1 = 0.5f, s2 = 5.0f / 6.0f;
    L[0] = 4.5f * (u - s1) * (u - s2);
    L[1] = -9.0f * (u - s0) * (u - s2);
    L[2] = 4.5f * (u - s0) * (u - s1);
}

// f_field_i = sum_{a,c} L_a(u_x) L_c(u_y) [ (X_i - t_ac) P0 + Q ],  X_i - t_ac = (u - s) h_b,
// evaluated as  u h_b sum w P0 + sum w R  with R_x = Q_x - s_a h_b P0,
// R_y = Q_y - s_c h_b P0 per node (formed once per node by k_row_inv).
// The field grid is one record of kBoxRec float4 per box, box-major
// (field.cu, k_row_inv): node k = 3 c + a of box b has P0 at float k, R_x at
// 9 + k, R_y at 18 + k of record b (27 floats + 1 pad: 7 vector loads per
// point instead of 9 (P0, Q_x, Q_y, pad) nodes; random box gathers are
// shared-memory wavefront bound in the move).
constexpr int kBoxRec = 7;
// the node offsets s_t = (t + 1/2) / 3 of an interval
__device__ __forceinline__ float node_s(int t) { return t == 0 ? 1.0f / 6.0f : (t == 1 ? 0.5f : 5.0f / 6.0f); }
template <bool GLOBAL = false>
__device__ __forceinline__ float2 gather_field(const Geo& g, const float4* __restrict__ fgrid, int b, float2 u) {
    const float h_b = (float)g.h_b;
    float Lx[3], Ly[3];
    lagrange3u(u.x, Lx);
    lagrange3u(u.y, Ly);
    const float4* box = fgrid + (int64_t)b * kBoxRec;   // generic loads: fgrid may be the shared-memory copy
    float f[4 * kBoxRec];
#pragma unroll
    for (int q = 0; q < kBoxRec; ++q) {
        const float4 v = GLOBAL ? __ldg(box + q) : box[q];
        f[4 * q] = v.x;
        f[4 * q + 1] = v.y;
        f[4 * q + 2] = v.z;
        f[4 * q + 3] = v.w;
    }
    float sp = 0.f, sx = 0.f, sy = 0.f;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int k = 3 * c + a;
            const float wgt = Lx[a] * Ly[c];
            sp = fmaf(wgt, f[k], sp);
            sx = fmaf(wgt, f[9 + k], sx);
            sy = fmaf(wgt, f[18 + k], sy);
        }
    }
    return make_float2(fmaf(u.x * h_b, sp, sx), fmaf(u.y * h_b, sp, sy));
}

__device__ __forceinline__ float sgnf(float x) { return (float)((x > 0.f) - (x < 0.f)); }

__device__ __forceinline__ void gains_move(float gr, float& v, float& gn, float& y, const tsnet_step_params& sp) {
    gn = (sgnf(gr) != sgnf(v)) ? gn + sp.gain_inc : gn * sp.gain_dec;
    gn = fmaxf(gn, sp.gain_min);
    v = sp.momentum * v - sp.eta * gn * gr;
    y = y + v;
}

}  // namespace tsnet
