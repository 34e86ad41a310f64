// Probe 2: shared-memory wavefronts of 64-bit loads with repeated (broadcast)
// addresses and of predicated 64-bit stores.  Each launch: one LDS.64 and one
// STS.64 per lane (store predicated off where the offset is ~0u).
#include <cstdio>
#include <random>
#include <vector>
__global__ void k_probe(const unsigned* __restrict__ lo, const unsigned* __restrict__ so, float* out) {
    __shared__ __align__(16) float s[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i;
    __syncthreads();
    const unsigned base = (unsigned)__cvta_generic_to_shared(s);
    const unsigned o = lo[threadIdx.x], w = so[threadIdx.x];
    float x, y;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(base + o));
    if (w != ~0u) asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(base + w), "f"(x), "f"(y));
    __syncthreads();
    out[threadIdx.x] = s[threadIdx.x * 2];
}
int main() {
    std::vector<std::pair<std::vector<unsigned>, std::vector<unsigned>>> pats;
    std::vector<unsigned> L(32), S(32, ~0u);
    std::mt19937 g(7);
    auto add = [&]() { pats.push_back({L, S}); };
    for (int l = 0; l < 32; ++l) L[l] = 4096; add();                                           // 0: all one address
    for (int l = 0; l < 32; ++l) L[l] = (l % 16 < 8) ? (l % 16) * 8 + 512 * (l / 16) : 4096 + 64; add();  // 1: 8 distinct (pairs 0-7) + 8 same (pair 8) per half
    for (int l = 0; l < 32; ++l) L[l] = (l % 16 < 8) ? (l % 16) * 8 + 512 * (l / 16) : 4096; add();  // 2: 8 distinct (pairs 0-7) + 8 same in pair 0
    for (int l = 0; l < 32; ++l) L[l] = (l % 2) ? (g() % 2048) * 8 : 8192 * 2; add();           // 3: 8 random + 8 same per half
    for (int l = 0; l < 32; ++l) L[l] = (l % 2) ? (g() % 2048) * 8 : 8192 * 2; add();           // 4: again
    for (int l = 0; l < 32; ++l) { L[l] = 16384; S[l] = (l % 3 == 0) ? (g() % 2048) * 8 : ~0u; } add();   // 5: stores: ~11 random lanes
    for (int l = 0; l < 32; ++l) { L[l] = 16384; S[l] = (l % 3 == 0) ? (g() % 2048) * 8 : ~0u; } add();   // 6: again
    for (int l = 0; l < 32; ++l) { L[l] = 16384; S[l] = (l < 16) ? l * 8 : ~0u; } add();        // 7: 16 lanes of half 0, distinct pairs
    for (int l = 0; l < 32; ++l) { L[l] = 16384; S[l] = (l % 2 == 0) ? (l / 2) * 8 : ~0u; } add();  // 8: even lanes, pairs 0-15 (8 per half)
    unsigned *dl, *ds; float* out;
    cudaMalloc(&dl, 128); cudaMalloc(&ds, 128); cudaMalloc(&out, 128 * 4);
    for (size_t i = 0; i < pats.size(); ++i) {
        auto model = [&](const std::vector<unsigned>& v) {
            int sum = 0;
            for (int h = 0; h < 2; ++h) {
                int mx = 0;
                for (int b = 0; b < 16; ++b) {
                    std::vector<unsigned> seen;
                    for (int l = 16 * h; l < 16 * h + 16; ++l)
                        if (v[l] != ~0u && (v[l] / 8) % 16 == (unsigned)b) {
                            bool f = false;
                            for (auto x : seen) f |= x == v[l];
                            if (!f) seen.push_back(v[l]);
                        }
                    mx = std::max<int>(mx, seen.size());
                }
                sum += mx;
            }
            return sum;
        };
        cudaMemcpy(dl, pats[i].first.data(), 128, cudaMemcpyHostToDevice);
        cudaMemcpy(ds, pats[i].second.data(), 128, cudaMemcpyHostToDevice);
        k_probe<<<1, 32>>>(dl, ds, out);
        cudaDeviceSynchronize();
        printf("pattern %zu: load per-half model %d, store per-half model %d\n", i, model(pats[i].first), model(pats[i].second));
    }
    return 0;
}
