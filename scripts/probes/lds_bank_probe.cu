// Probe: shared-memory wavefronts of 64-bit loads for chosen per-lane address
// patterns (is the conflict degree counted per half-warp or over the warp?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 lds_bank_probe.cu -o lds_bank_probe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
__global__ void k_probe(const unsigned* __restrict__ offs, float* out, int iters) {
    __shared__ __align__(16) float s[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i;
    __syncthreads();
    unsigned o = offs[threadIdx.x & 31];
    float ax = 0.f, ay = 0.f;
    for (int it = 0; it < iters; ++it) {
        float x, y;
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"((unsigned)__cvta_generic_to_shared(s) + o));
        ax += x; ay += y;
    }
    out[threadIdx.x] = ax + ay;
}
int main() {
    std::vector<std::vector<unsigned>> pats;
    std::vector<unsigned> p(32);
    for (int l = 0; l < 32; ++l) p[l] = (l % 16) * 8 + (l / 16) * 128;  pats.push_back(p);          // 0: each pair twice, once per half
    for (int l = 0; l < 32; ++l) p[l] = (l < 16) ? ((l % 8) * 8 + (l / 8) * 128) : ((8 + l % 8) * 8 + ((l - 16) / 8) * 128); pats.push_back(p); // 1: halves in disjoint pairs, 2-way within half
    for (int l = 0; l < 32; ++l) p[l] = l * 8; pats.push_back(p);                                    // 2: consecutive
    for (int l = 0; l < 32; ++l) p[l] = (l < 16) ? l * 8 : (l - 16) * 128; pats.push_back(p);         // 3: half1 all in pair 0
    for (int l = 0; l < 32; ++l) p[l] = (l % 16) * 8 + (l / 16) * 1024 + ((l % 16) < 8 ? 0 : 0); pats.push_back(p); // 4: like 0, far
    for (int l = 0; l < 32; ++l) p[l] = (l < 16) ? ((l % 4) * 8 + (l / 4) * 128) : ((4 + (l - 16) % 12) * 8 + ((l - 16) / 12) * 256); pats.push_back(p); // 5: half0 4-way in pairs 0-3, half1 pairs 4-15 (one 2-way)
    std::mt19937 g(1);
    for (int r = 0; r < 4; ++r) { for (int l = 0; l < 32; ++l) p[l] = (g() % 4096) * 8; pats.push_back(p); }  // 6-9 random
    unsigned* d; float* out;
    cudaMalloc(&d, 32 * 4); cudaMalloc(&out, 128 * 4);
    for (size_t i = 0; i < pats.size(); ++i) {
        // model predictions: per-half sum of max occupancy, and whole-warp max occupancy (distinct addresses)
        int half_sum = 0, whole = 0;
        for (int h = 0; h < 3; ++h) {
            int mx = 0;
            for (int b = 0; b < 16; ++b) {
                std::vector<unsigned> seen;
                for (int l = (h == 2 ? 0 : 16 * h); l < (h == 2 ? 32 : 16 * h + 16); ++l)
                    if ((pats[i][l] / 8) % 16 == (unsigned)b) { bool f = false; for (auto v : seen) f |= v == pats[i][l]; if (!f) seen.push_back(pats[i][l]); }
                mx = std::max<int>(mx, seen.size());
            }
            if (h < 2) half_sum += mx; else whole = mx;
        }
        cudaMemcpy(d, pats[i].data(), 32 * 4, cudaMemcpyHostToDevice);
        k_probe<<<1, 32>>>(d, out, 1000);
        cudaDeviceSynchronize();
        printf("pattern %zu: per-half model %d, whole-warp model %d\n", i, half_sum, whole);
    }
    return 0;
}
