// fft.cuh -- batched mixed-radix (4/2/3/5) Stockham FFT on shared memory,
// one CTA cooperating on B transforms of length M.
//
// Convolution step of the FFT-accelerated interpolation (PAPER.md:187-188,
// "The computation of the interpolation is accelerated using FFT"; Alg. 3
// l.400, l.403).  M = 6 I is 5-smooth (grid policy R9), read from the
// workspace at run time, so one compiled kernel serves every grid size.
//
// Stage s with radix R and span Ns (product of earlier radices), butterfly j:
//   inputs  x[j + r M/R], r < R, times twiddle w_M^{r (j mod Ns) M/(Ns R)}
//   R-point DFT
//   outputs y[(j / Ns) Ns R + (j mod Ns) + r Ns]
// Out of place (ping-pong between the data and a scratch buffer of the same
// shape), one barrier per stage for the whole batch.
#pragma once
#include "common.cuh"

namespace tsnet {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
// -i * a and +i * a
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }
__device__ __forceinline__ float2 mul_pi(float2 a) { return make_float2(-a.y, a.x); }

// R-point DFT in registers; forward = exp(-2 pi i r k / R), inverse = conjugate.
template <int R>
__device__ __forceinline__ void dft(float2 (&v)[R], bool inv);

template <>
__device__ __forceinline__ void dft<2>(float2 (&v)[2], bool) {
    float2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
}

template <>
__device__ __forceinline__ void dft<3>(float2 (&v)[3], bool inv) {
    const float s = 0.86602540378443864676f;  // sin(2 pi / 3)
    float2 t = cadd(v[1], v[2]);
    float2 m = make_float2(v[0].x - 0.5f * t.x, v[0].y - 0.5f * t.y);
    float2 d = cscale(csub(v[1], v[2]), s);
    v[0] = cadd(v[0], t);
    float2 x1 = cadd(m, mul_mi(d)), x2 = cadd(m, mul_pi(d));
    v[1] = inv ? x2 : x1;
    v[2] = inv ? x1 : x2;
}

template <>
__device__ __forceinline__ void dft<4>(float2 (&v)[4], bool inv) {
    float2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    float2 u0 = cadd(v[1], v[3]), u1 = csub(v[1], v[3]);
    v[0] = cadd(t0, u0);
    v[2] = csub(t0, u0);
    float2 x1 = cadd(t1, mul_mi(u1)), x3 = cadd(t1, mul_pi(u1));
    v[1] = inv ? x3 : x1;
    v[3] = inv ? x1 : x3;
}

template <>
__device__ __forceinline__ void dft<5>(float2 (&v)[5], bool inv) {
    const float c1 = 0.30901699437494742410f;   // cos(2 pi / 5)
    const float c2 = -0.80901699437494742410f;  // cos(4 pi / 5)
    const float s1 = 0.95105651629515357212f;   // sin(2 pi / 5)
    const float s2 = 0.58778525229247312917f;   // sin(4 pi / 5)
    float2 t1 = cadd(v[1], v[4]), t2 = cadd(v[2], v[3]);
    float2 d1 = csub(v[1], v[4]), d2 = csub(v[2], v[3]);
    float2 b1 = make_float2(v[0].x + c1 * t1.x + c2 * t2.x, v[0].y + c1 * t1.y + c2 * t2.y);
    float2 b2 = make_float2(v[0].x + c2 * t1.x + c1 * t2.x, v[0].y + c2 * t1.y + c1 * t2.y);
    float2 e1 = make_float2(s1 * d1.x + s2 * d2.x, s1 * d1.y + s2 * d2.y);
    float2 e2 = make_float2(s2 * d1.x - s1 * d2.x, s2 * d1.y - s1 * d2.y);
    v[0] = cadd(v[0], cadd(t1, t2));
    float2 x1 = cadd(b1, mul_mi(e1)), x4 = cadd(b1, mul_pi(e1));
    float2 x2 = cadd(b2, mul_mi(e2)), x3 = cadd(b2, mul_pi(e2));
    v[1] = inv ? x4 : x1;
    v[4] = inv ? x1 : x4;
    v[2] = inv ? x3 : x2;
    v[3] = inv ? x2 : x3;
}

// One Stockham stage over B transforms: src + b*ld -> dst + b*ld.
template <int R>
__device__ __forceinline__ void fft_stage(const float2* __restrict__ src, float2* __restrict__ dst, int ld, int B,
                                          int M, int Ns, const float2* __restrict__ tw, bool inv) {
    const int nb = M / R;
    const int total = B * nb;
    const int stride = M / (Ns * R);
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
        const int b = t / nb;
        const int j = t - b * nb;
        const int k = j % Ns;
        const float2* s = src + b * ld;
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = s[j + r * nb];
#pragma unroll
        for (int r = 1; r < R; ++r) {
            float2 w = tw[r * k * stride];
            if (inv) w.y = -w.y;
            v[r] = cmul(v[r], w);
        }
        dft<R>(v, inv);
        float2* d = dst + b * ld + (j - k) * R + k;   // (j / Ns) Ns R + (j mod Ns)
#pragma unroll
        for (int r = 0; r < R; ++r) d[r * Ns] = v[r];
    }
    __syncthreads();
}

// Full transform of B length-M sequences stored at buf + b*ld (M = product of
// the plan's radices), ping-ponging through `scratch` (same shape).  The
// result is left in buf (a copy-back pass runs when the stage count is odd).
// plan: radix of stage s in bits [2s, 2s+2) as R - 2; nrad stages.  Caller
// synchronises before; the routine ends with a barrier.
__device__ void fft_block(float2* buf, float2* scratch, int ld, int B, int M, unsigned long long plan, int nrad,
                          const float2* tw, bool inv) {
    int Ns = 1;
    float2* src = buf;
    float2* dst = scratch;
    for (int s = 0; s < nrad; ++s) {
        const int R = (int)((plan >> (2 * s)) & 3ull) + 2;
        if (R == 4)
            fft_stage<4>(src, dst, ld, B, M, Ns, tw, inv);
        else if (R == 2)
            fft_stage<2>(src, dst, ld, B, M, Ns, tw, inv);
        else if (R == 3)
            fft_stage<3>(src, dst, ld, B, M, Ns, tw, inv);
        else
            fft_stage<5>(src, dst, ld, B, M, Ns, tw, inv);
        Ns *= R;
        float2* tmp = src;
        src = dst;
        dst = tmp;
    }
    if (src != buf) {
        for (int t = threadIdx.x; t < B * M; t += blockDim.x) {
            const int b = t / M, x = t - b * M;
            buf[b * ld + x] = src[b * ld + x];
        }
        __syncthreads();
    }
}

}  // namespace tsnet
