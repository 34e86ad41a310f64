// Probe (not product code): random-row gather throughput on B200 through the
// TMA unit (cp.async.bulk.tensor.2d ... tile::gather4: 4 rows of a 2-D tensor
// per instruction, into shared memory, mbarrier completion) against plain
// LSU loads of the same rows (ld.global.v4 / v2).  The layout Y viewed as
// 16-byte rows (2 points per row), cfg-4 size (474k rows, 7.6 MB: L2-resident).
// Question: can the TMA route exceed the LSU's ~1 random gather
// per SM-cycle that caps a row-wise SpMV at 0.35 of the HBM peak?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4_probe gather4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));     \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}

constexpr int kIssuers = 4;     // issuing warps per CTA (lane 0 each), one ring each
constexpr int kDepth = 32;      // gather4s in flight per ring
constexpr int kRow = 16;        // bytes per row

// Each issuer streams `per` gather4s of 4 hashed random rows.
__global__ void __launch_bounds__(32 * kIssuers) k_tma_g4(const __grid_constant__ CUtensorMap tm, int rows, int per,
                                                          float* out) {
    __shared__ __align__(128) uint8_t ring[kIssuers][kDepth][128];   // TMA destinations: 128-byte aligned
    __shared__ __align__(8) uint64_t bar[kIssuers][kDepth];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
        for (int s = 0; s < kDepth; ++s) mbar_init(&bar[w][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    float acc = 0.f;
    if (lane == 0) {
        const uint32_t seed = (blockIdx.x * kIssuers + w) * 0x9e3779b9U;
        for (int q = 0; q < per; ++q) {
            const int s = q % kDepth;
            if (q >= kDepth) {
                mbar_wait(&bar[w][s], ((q / kDepth) - 1) & 1);
                acc += *reinterpret_cast<const float*>(&ring[w][s][0]);
            }
            int r[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) r[t] = (int)(hash32(seed + 4u * q + t) % (uint32_t)rows);
            mbar_expect(&bar[w][s], 4 * kRow);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(&ring[w][s][0])),
                "l"(&tm), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(smem_u32(&bar[w][s]))
                : "memory");
        }
        for (int q = per; q < per + kDepth; ++q) {
            const int s = q % kDepth;
            if (q >= kDepth) mbar_wait(&bar[w][s], ((q / kDepth) - 1) & 1);
        }
    }
    if (lane == 0 && acc == 1.2345f) out[blockIdx.x] = acc;
}

// LSU baseline: every thread `per` random 16-byte (v4) or 8-byte (v2) loads,
// 8 in flight
template <int BYTES>
__global__ void __launch_bounds__(256) k_lsu(const float4* __restrict__ Y, int rows, int per, float* out) {
    const uint32_t seed = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9e3779b9U;
    float acc = 0.f;
    for (int q = 0; q < per; q += 8) {
        float v[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const int r = (int)(hash32(seed + q + t) % (uint32_t)rows);
            if (BYTES == 16) {
                const float4 f = __ldg(Y + r);
                v[t] = f.x + f.w;
            } else {
                const float2 f = __ldg(reinterpret_cast<const float2*>(Y) + 2 * r);
                v[t] = f.x + f.y;
            }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) acc += v[t];
    }
    if (acc == 1.2345f) out[0] = acc;
}

int main(int argc, char** argv) {
    const int rows = argc > 1 ? atoi(argv[1]) : 473987;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    float4* Y = nullptr;
    float* out = nullptr;
    CK(cudaMalloc(&Y, (size_t)rows * kRow));
    CK(cudaMalloc(&out, 1 << 20));
    CK(cudaMemset(Y, 0, (size_t)rows * kRow));
    CUtensorMap tm;
    const cuuint64_t dims[2] = {4, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {kRow};
    const cuuint32_t box[2] = {4, 1};
    const cuuint32_t estr[2] = {1, 1};
    CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Y, dims, strides, box, estr,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) {
        printf("cuTensorMapEncodeTiled failed: %d\n", (int)cr);
        return 1;
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int ctas_per_sm : {1, 2, 4, 8}) {
        const int grid = sms * ctas_per_sm, per = 4096;
        k_tma_g4<<<grid, 32 * kIssuers>>>(tm, rows, per, out);
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        for (int it = 0; it < 5; ++it) k_tma_g4<<<grid, 32 * kIssuers>>>(tm, rows, per, out);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double g4 = 5.0 * grid * kIssuers * (double)per;
        printf("{\"path\": \"tma_gather4\", \"ctas_per_sm\": %d, \"issuers_per_cta\": %d, \"depth\": %d, "
               "\"rows_per_s\": %.4g, \"gather4_per_s\": %.4g, \"rows_per_sm_cycle\": %.3f}\n",
               ctas_per_sm, kIssuers, kDepth, 4.0 * g4 / (ms * 1e-3), g4 / (ms * 1e-3),
               4.0 * g4 / (ms * 1e-3) / (sms * 1.965e9));
    }
    for (int bytes : {16, 8}) {
        const int grid = sms * 8, per = 1024;
        auto launch = [&]() {
            if (bytes == 16) k_lsu<16><<<grid, 256>>>(Y, rows, per, out);
            else k_lsu<8><<<grid, 256>>>(Y, rows, per, out);
        };
        launch();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        for (int it = 0; it < 5; ++it) launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double n = 5.0 * grid * 256.0 * per;
        printf("{\"path\": \"lsu_ld_v%d\", \"rows_per_s\": %.4g, \"rows_per_sm_cycle\": %.3f}\n", bytes / 4,
               n / (ms * 1e-3), n / (ms * 1e-3) / (sms * 1.965e9));
    }
    return 0;
}
