// Probe 4: how a predicated LDS.64 with some lanes off is split into
// wavefronts: by warp halves, or the active lanes taken 16 at a time?
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
static int occ(const std::vector<unsigned>& v, const std::vector<int>& lanes) {
    int mx = 0;
    for (int b = 0; b < 16; ++b) {
        std::vector<unsigned> seen;
        for (int l : lanes)
            if (v[l] != ~0u && (v[l] / 8) % 16 == (unsigned)b) {
                bool f = false;
                for (auto x : seen) f |= x == v[l];
                if (!f) seen.push_back(v[l]);
            }
        mx = std::max<int>(mx, seen.size());
    }
    return mx;
}
int main() {
    std::vector<std::vector<unsigned>> pats;
    std::vector<unsigned> L(32);
    std::mt19937 g(5);
    auto off = [&]() { for (auto& x : L) x = ~0u; };
    off(); for (int l = 0; l < 8; ++l) { L[l] = l * 8; L[16 + l] = (8 + l) * 8 + 1024; } pats.push_back(L);      // b
    off(); for (int l = 0; l < 4; ++l) { L[l] = l * 8; L[16 + l] = (4 + l) * 8 + 1024; } pats.push_back(L);      // c
    off(); for (int l = 0; l < 8; ++l) { L[l] = l * 8; L[16 + l] = (8 + l) * 8 + 1024; L[24 + l] = (8 + l) * 8 + 2048; } pats.push_back(L);  // h
    off(); for (int l = 0; l < 8; ++l) { L[2 * l + 1] = l * 8; L[16 + 2 * l + 1] = (8 + l) * 8 + 1024; } pats.push_back(L);  // b on odd lanes
    for (int r = 0; r < 12; ++r) {      // random: k active lanes at random positions, random addresses
        off();
        int k = 6 + r * 2;
        for (int t = 0; t < k; ++t) { int l; do l = g() % 32; while (L[l] != ~0u); L[l] = (g() % 2048) * 8; }
        pats.push_back(L);
    }
    unsigned* dl; float* out;
    cudaMalloc(&dl, 128); cudaMalloc(&out, 128 * 4);
    for (size_t i = 0; i < pats.size(); ++i) {
        const auto& v = pats[i];
        std::vector<int> h0, h1, act;
        for (int l = 0; l < 32; ++l) { if (l < 16) h0.push_back(l); else h1.push_back(l); if (v[l] != ~0u) act.push_back(l); }
        const int halves = occ(v, h0) + occ(v, h1);
        const int whole = occ(v, act);
        std::vector<int> g1(act.begin(), act.begin() + std::min<size_t>(16, act.size())), g2(act.begin() + g1.size(), act.end());
        const int first16 = occ(v, g1) + occ(v, g2);
        cudaMemcpy(dl, v.data(), 128, cudaMemcpyHostToDevice);
        k_probe<<<1, 32>>>(dl, out);
        cudaDeviceSynchronize();
        printf("pattern %zu active %zu: halves %d whole %d first16 %d\n", i, act.size(), halves, whole, first16);
    }
    return 0;
}
