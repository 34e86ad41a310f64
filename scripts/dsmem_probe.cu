// Experiment: random float2 gather throughput on B200 from (a) global memory
// through L1/L2 (what k_spmv2 does for Y[j]), (b) distributed shared memory
// of a thread-block cluster (ld.shared::cluster), (c) local shared memory.
// Each gather index comes from a coalesced int32 stream, as in the SpMV.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_probe dsmem_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void k_global(const float2* __restrict__ tab, const int* __restrict__ idx, int64_t m, float* out) {
    float ax = 0.f, ay = 0.f;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < m; i += 4 * stride) {
        int j0 = __ldcs(idx + i), j1 = __ldcs(idx + i + stride), j2 = __ldcs(idx + i + 2 * stride), j3 = __ldcs(idx + i + 3 * stride);
        float2 a = __ldg(tab + j0), b = __ldg(tab + j1), c = __ldg(tab + j2), d = __ldg(tab + j3);
        ax += a.x + b.x + c.x + d.x;
        ay += a.y + b.y + c.y + d.y;
    }
    for (; i < m; i += stride) {
        float2 a = __ldg(tab + idx[i]);
        ax += a.x;
        ay += a.y;
    }
    if (ax == 12345.f) out[0] = ay;
}

// table slice per CTA: S float2; global index g -> rank g / S, offset g % S (S power of 2)
template <int LOG_S, bool REMOTE>
__global__ void k_dsmem(const float2* __restrict__ tab, const int* __restrict__ idx, int64_t m, float* out) {
    extern __shared__ float2 sl[];
    constexpr int S = 1 << LOG_S;
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    for (int t = threadIdx.x; t < S; t += blockDim.x) sl[t] = tab[(int64_t)rank * S + t];
    cl.sync();
    uint32_t base = (uint32_t)__cvta_generic_to_shared(sl);
    float ax = 0.f, ay = 0.f;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    auto gat = [&](int g) {
        float2 v;
        uint32_t a = base + (uint32_t)(g & (S - 1)) * 8u;
        if (REMOTE) {
            uint32_t r = (uint32_t)g >> LOG_S, ra;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(r));
            asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(ra));
        } else {
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
        }
        return v;
    };
    for (; i + 3 * stride < m; i += 4 * stride) {
        int j0 = __ldcs(idx + i), j1 = __ldcs(idx + i + stride), j2 = __ldcs(idx + i + 2 * stride), j3 = __ldcs(idx + i + 3 * stride);
        float2 a = gat(j0), b = gat(j1), c = gat(j2), d = gat(j3);
        ax += a.x + b.x + c.x + d.x;
        ay += a.y + b.y + c.y + d.y;
    }
    for (; i < m; i += stride) {
        float2 a = gat(idx[i]);
        ax += a.x;
        ay += a.y;
    }
    cl.sync();
    if (ax == 12345.f) out[0] = ay;
}

template <typename K>
float time_launch(K kern, dim3 grid, dim3 block, size_t smem, int cluster, const float2* tab, const int* idx, int64_t m, float* out) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int w = 0; w < 2; ++w) CK(cudaLaunchKernelEx(&cfg, kern, tab, idx, m, out));
    CK(cudaEventRecord(e0));
    const int reps = 5;
    for (int w = 0; w < reps; ++w) CK(cudaLaunchKernelEx(&cfg, kern, tab, idx, m, out));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms / reps;
}

template <int LOG_S, bool REMOTE>
void run_dsmem(int cluster, int threads, const float2* tab, int* idx_dev, const std::vector<int>& idx_host_full, int64_t m,
               float* out, int sms) {
    auto kern = k_dsmem<LOG_S, REMOTE>;
    size_t smem = (size_t)8 << LOG_S;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (cluster > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(cluster);
    int ncl = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
    if (e != cudaSuccess || ncl == 0) {
        printf("cluster %d S=%d: not launchable (%s)\n", cluster, 1 << LOG_S, cudaGetErrorString(e));
        cudaGetLastError();
        return;
    }
    // indices restricted to the cluster's table: remap the host stream
    const int64_t span = (int64_t)(REMOTE ? cluster : 1) << LOG_S;
    std::vector<int> h(m);
    for (int64_t i = 0; i < m; ++i) h[i] = (int)((uint32_t)idx_host_full[i] % (uint32_t)span);
    CK(cudaMemcpy(idx_dev, h.data(), m * 4, cudaMemcpyHostToDevice));
    int grid = ncl * cluster;
    float ms = time_launch(kern, dim3(grid), dim3(threads), smem, cluster, tab, idx_dev, m, out);
    printf("%s cluster %2d slice %6d float2 (%3zu KB) clusters %3d CTAs %3d thr %4d: %.3f ms  %.1f G gathers/s  %.2f per SM-cycle\n",
           REMOTE ? "dsmem " : "local ", cluster, 1 << LOG_S, smem >> 10, ncl, grid, threads, ms, m / ms / 1e6,
           m / (ms * 1e-3) / sms / 1.9e9);
}

int main() {
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int64_t m = 200'000'000;
    const int T = 950'000;
    std::mt19937_64 rng(1);
    std::vector<int> ih(m);
    for (int64_t i = 0; i < m; ++i) ih[i] = (int)(rng() & 0x7fffffff);
    std::vector<int> ig(m);
    for (int64_t i = 0; i < m; ++i) ig[i] = ih[i] % T;
    float2* tab;
    int* idx;
    float* out;
    CK(cudaMalloc(&tab, sizeof(float2) * 4'200'000));
    CK(cudaMemset(tab, 0, sizeof(float2) * 4'200'000));
    CK(cudaMalloc(&idx, m * 4));
    CK(cudaMalloc(&out, 4));
    CK(cudaMemcpy(idx, ig.data(), m * 4, cudaMemcpyHostToDevice));
    for (int thr : {256, 512, 1024}) {
        int occ;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_global, thr, 0));
        float ms = time_launch(k_global, dim3(sms * occ), dim3(thr), 0, 1, tab, idx, m, out);
        printf("global T=%d thr %d: %.3f ms  %.1f G gathers/s  %.2f per SM-cycle\n", T, thr, ms, m / ms / 1e6,
               m / (ms * 1e-3) / sms / 1.9e9);
    }
    for (int thr : {512, 1024}) {
        run_dsmem<14, false>(1, thr, tab, idx, ih, m, out, sms);
        run_dsmem<14, true>(2, thr, tab, idx, ih, m, out, sms);
        run_dsmem<14, true>(4, thr, tab, idx, ih, m, out, sms);
        run_dsmem<14, true>(8, thr, tab, idx, ih, m, out, sms);
        run_dsmem<14, true>(16, thr, tab, idx, ih, m, out, sms);
        run_dsmem<13, true>(8, thr, tab, idx, ih, m, out, sms);
        run_dsmem<13, true>(16, thr, tab, idx, ih, m, out, sms);
    }
    return 0;
}
