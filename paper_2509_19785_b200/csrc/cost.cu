// cost.cu -- the tsNET cost C = (C_KL, C_CMP, C_ENT*) (Eq. 1)
//   C_KL  = lambda_kl sum_{p_ij > 0} p_ij ln(p_ij Z / w_ij)
//         = lambda_kl [ sum p ln p + sum p ln(1 + r^2) + (sum p) ln Z ]
//   C_CMP = lambda_c / (2n) sum |X_i|^2
//   C_ENT* = -lambda_r / (4 n^2) sum_{i != j} ln(eps + r^2)      (reading R1)
// mode 0: exact O(n^2) tiles for Z and C_ENT*; mode 1: Z and the entropy sum
// from the interpolation grid (O(n): sparse pass + grid Parseval sums).
#include <algorithm>

#include "common.cuh"

namespace tsnet {

// acc[0] = sum p (ln p + ln(1 + r^2)), acc[1] = sum p, acc[2] = Z (pairs), acc[3] = sum ln(eps + r^2),
// acc[4] = sum |X|^2
__global__ void k_cost_zero(double* acc) {
    if (threadIdx.x < 8) acc[threadIdx.x] = 0.0;
}

__device__ __forceinline__ void block_add(double v, double* dst) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(dst, v);
}

__global__ void __launch_bounds__(256) k_cost_sparse(int64_t n, const int64_t* __restrict__ indptr,
                                                     const int32_t* __restrict__ indices,
                                                     const float* __restrict__ values, const float2* __restrict__ Y,
                                                     double* acc) {
    double s0 = 0.0, s1 = 0.0, s4 = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 yi = Y[i];
        s4 += (double)yi.x * yi.x + (double)yi.y * yi.y;
        for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
            const double p = values[e];
            if (!(p > 0.0)) continue;
            const float2 yj = Y[indices[e]];
            const double dx = (double)yi.x - yj.x, dy = (double)yi.y - yj.y;
            s0 += p * (log(p) + log1p(dx * dx + dy * dy));
            s1 += p;
        }
    }
    block_add(s0, acc + 0);
    block_add(s1, acc + 1);
    block_add(s4, acc + 4);
}

constexpr int kTile = 256;

__global__ void __launch_bounds__(kTile) k_cost_pairs(int64_t n, const float2* __restrict__ Y, float eps, double* acc) {
    __shared__ float2 tile[kTile];
    const int64_t i = blockIdx.x * (int64_t)kTile + threadIdx.x;
    const float2 yi = i < n ? Y[i] : make_float2(0.f, 0.f);
    double z = 0.0, ent = 0.0;
    for (int64_t j0 = 0; j0 < n; j0 += kTile) {
        __syncthreads();
        if (j0 + threadIdx.x < n) tile[threadIdx.x] = Y[j0 + threadIdx.x];
        __syncthreads();
        const int m = (int)std::min<int64_t>(kTile, n - j0);
        if (i < n) {
            float zt = 0.f;
            double et = 0.0;
            for (int t = 0; t < m; ++t) {
                if (j0 + t == i) continue;
                const float dx = yi.x - tile[t].x, dy = yi.y - tile[t].y;
                const float r2 = dx * dx + dy * dy;
                zt += 1.0f / (1.0f + r2);
                et += (double)logf(eps + r2);
            }
            z += zt;
            ent += et;
        }
    }
    block_add(z, acc + 2);
    block_add(ent, acc + 3);
}

__global__ void k_cost_final(int64_t n, const double* acc, const Geo* g, int mode, float lambda_kl, float lambda_c,
                             float lambda_r, float eps, double* out3) {
    const double nn = (double)n;
    const double Z = (mode == 0) ? acc[2] : g->Z;
    out3[0] = (double)lambda_kl * (acc[0] + acc[1] * log(Z));
    out3[1] = (double)lambda_c / (2.0 * nn) * acc[4];
    // mode 1: interpolated sum_{i != j} ln(eps + r^2) = <W1, K_ln * W1> - n ln(eps) (field.cu)
    const double M2 = (double)g->M * (double)g->M;
    const double ent = (mode == 0) ? acc[3] : g->eacc / M2 - nn * log((double)eps);
    out3[2] = -(double)lambda_r / (4.0 * nn * nn) * ent;
}

cudaError_t launch_cost(const Ws& w, const GradArgs& a, int mode, double* out3, cudaStream_t s) {
    k_cost_zero<<<1, 32, 0, s>>>(w.cost);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((a.n + 255) / 256, (int64_t)kNumSMs * 4));
    k_cost_sparse<<<blocks, 256, 0, s>>>(a.n, a.indptr, a.indices, a.values, a.Y, w.cost);
    if (mode == 0) k_cost_pairs<<<(int)((a.n + kTile - 1) / kTile), kTile, 0, s>>>(a.n, a.Y, a.eps, w.cost);
    k_cost_final<<<1, 1, 0, s>>>(a.n, w.cost, w.geo, mode, a.lambda_kl, a.lambda_c, a.lambda_r, a.eps, out3);
    return cudaGetLastError();
}

}  // namespace tsnet
