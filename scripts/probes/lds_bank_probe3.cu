// Probe 3: wavefronts of one LDS.64 per lane for patterns with repeated
// addresses, and of predicated LDS.64 (offset ~0u = lane off).
#include <cstdio>
#include <random>
#include <vector>
__global__ void k_probe(const unsigned* __restrict__ lo, float* out) {
    __shared__ __align__(16) float s[8192];
    const unsigned base = (unsigned)__cvta_generic_to_shared(s);
    const unsigned o = lo[threadIdx.x];
    float x = 0.f, y = 0.f;
    asm volatile("{\n.reg .pred p;\nsetp.ne.u32 p, %2, -1;\n@p ld.shared.v2.f32 {%0, %1}, [%3];\n}" : "+f"(x), "+f"(y) : "r"(o), "r"(base + o));
    out[threadIdx.x] = x + y;
}
int main() {
    std::vector<std::vector<unsigned>> pats;
    std::vector<unsigned> L(32);
    std::mt19937 g(11);
    auto distinct = [&]() { for (int l = 0; l < 32; ++l) L[l] = (l % 16) * 8 + (l / 16) * 1024; };
    distinct(); pats.push_back(L);                                   // 0: distinct pairs per half (2)
    distinct(); L[1] = L[0]; pats.push_back(L);                      // 1: one repeat in half 0
    distinct(); L[1] = L[0]; L[17] = L[16]; pats.push_back(L);       // 2: one repeat per half
    distinct(); L[16] = L[0]; pats.push_back(L);                     // 3: repeat across halves
    distinct(); L[1] = L[2] = L[0]; pats.push_back(L);               // 4: 3 lanes same in half 0
    for (int l = 0; l < 32; ++l) L[l] = (l < 16) ? 4096 : 8192; pats.push_back(L);   // 5: each half one address
    distinct(); for (int l = 8; l < 16; ++l) L[l] = ~0u; pats.push_back(L);          // 6: half 0 lanes 8-15 off
    for (int l = 0; l < 32; ++l) L[l] = (l % 2) ? (g() % 2048) * 8 : ~0u; pats.push_back(L);  // 7: 8 random per half, others off
    for (int l = 0; l < 32; ++l) L[l] = (l % 2) ? (g() % 2048) * 8 : ~0u; pats.push_back(L);  // 8
    for (int l = 0; l < 32; ++l) L[l] = (l % 2) ? (g() % 2048) * 8 : 16384; pats.push_back(L); // 9: 8 random + 8 dummy per half
    distinct(); L[5] = L[0] + 128; pats.push_back(L);                // 10: 2-way conflict in half 0 (model 3)
    unsigned* dl; float* out;
    cudaMalloc(&dl, 128); cudaMalloc(&out, 128 * 4);
    for (size_t i = 0; i < pats.size(); ++i) {
        int sum = 0;
        for (int h = 0; h < 2; ++h) {
            int mx = 0;
            for (int b = 0; b < 16; ++b) {
                std::vector<unsigned> seen;
                for (int l = 16 * h; l < 16 * h + 16; ++l)
                    if (pats[i][l] != ~0u && (pats[i][l] / 8) % 16 == (unsigned)b) {
                        bool f = false;
                        for (auto x : seen) f |= x == pats[i][l];
                        if (!f) seen.push_back(pats[i][l]);
                    }
                mx = std::max<int>(mx, seen.size());
            }
            sum += mx;
        }
        cudaMemcpy(dl, pats[i].data(), 128, cudaMemcpyHostToDevice);
        k_probe<<<1, 32>>>(dl, out);
        cudaDeviceSynchronize();
        printf("pattern %zu: per-half model %d\n", i, sum);
    }
    return 0;
}
