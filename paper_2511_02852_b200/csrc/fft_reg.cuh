// Register-blocked inverse FFT for one power-of-two length N (64..4096)
// held in shared memory, T = N/16 threads per transform, each thread owning
// 16 elements per pass.
//
// Pass structure (in place, natural-order input): with current sub-length M
// and radix R (M' = M/R), every (group g, n2 < M') item does
//     y[k1] = sum_{n1} x[g M + M' n1 + n2] w_R^{n1 k1}      (R-point DFT in registers)
//     y[k1] *= w_M^{n2 k1}                                   (twiddle)
// and writes y[k1] back to g M + M' k1 + n2 -- the same R addresses it read,
// so items never conflict and one barrier separates passes.  After the last
// pass position sum_p d_p M_p holds X[sum_p d_p R_1..R_{p-1}]: the caller
// reads outputs through `out_pos`.  w = exp(+2 pi i / .) (inverse DFT, as
// numpy ifft * n; reference fft_background.py:191).
#pragma once
#include "hs_common.cuh"

namespace hs {

// XOR swizzle of a transform's float2 slots: permutes within aligned groups
// of 16 so that every pass's strided loads / stores and the digit-reversed
// output read hit 16 distinct 8-byte bank pairs per half warp (model and
// check: tools/fft_banks.py); no padding, the layout stays N slots
__device__ __forceinline__ int fpad(int i) { return i ^ (((i >> 4) ^ (i >> 8)) & 15); }

template <int N> struct FftPlan;
// radices per pass; the product is N, every radix divides 16
template <> struct FftPlan<64> { static constexpr int P = 2; __host__ __device__ static constexpr int R(int p) { return p == 0 ? 16 : p == 1 ? 4 : 1; } };
template <> struct FftPlan<128> { static constexpr int P = 2; __host__ __device__ static constexpr int R(int p) { return p == 0 ? 16 : p == 1 ? 8 : 1; } };
template <> struct FftPlan<256> { static constexpr int P = 2; __host__ __device__ static constexpr int R(int p) { return p == 0 ? 16 : p == 1 ? 16 : 1; } };
template <> struct FftPlan<512> { static constexpr int P = 3; __host__ __device__ static constexpr int R(int p) { return p == 0 ? 16 : p == 1 ? 16 : 2; } };
template <> struct FftPlan<1024> { static constexpr int P = 3; __host__ __device__ static constexpr int R(int p) { return p == 0 ? 16 : p == 1 ? 16 : 4; } };
template <> struct FftPlan<2048> { static constexpr int P = 3; __host__ __device__ static constexpr int R(int p) { return p == 0 ? 16 : p == 1 ? 16 : 8; } };
template <> struct FftPlan<4096> { static constexpr int P = 3; __host__ __device__ static constexpr int R(int p) { return p == 0 ? 16 : p == 1 ? 16 : 16; } };

__device__ __forceinline__ float2 cfma_tw(float2 v, float2 w) {   // v * w with FMAs
    return make_float2(fmaf(v.x, w.x, -v.y * w.y), fmaf(v.x, w.y, v.y * w.x));
}

template <int R> __device__ __forceinline__ void dft_reg(float2* v);

template <> __device__ __forceinline__ void dft_reg<1>(float2*) {}

template <> __device__ __forceinline__ void dft_reg<2>(float2* v) {
    const float2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
}

template <> __device__ __forceinline__ void dft_reg<4>(float2* v) {
    const float2 a = cadd(v[0], v[2]), b = csub(v[0], v[2]);
    const float2 c = cadd(v[1], v[3]), d = cmul_i(csub(v[1], v[3]));   // i (x1 - x3)
    v[0] = cadd(a, c);
    v[2] = csub(a, c);
    v[1] = cadd(b, d);
    v[3] = csub(b, d);
}

// radix 4 x 2: a[n2][k1] = DFT4(x[n2 + 2 n1]); a[1][k1] *= w8^k1; X[k1 + 4 k2]
template <> __device__ __forceinline__ void dft_reg<8>(float2* v) {
    const float s = 0.70710678118654752440f;
    float2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
    dft_reg<4>(e);
    dft_reg<4>(o);
    o[1] = make_float2((o[1].x - o[1].y) * s, (o[1].x + o[1].y) * s);    // * e^{i pi/4}
    o[2] = cmul_i(o[2]);                                               // * i
    o[3] = make_float2((-o[3].x - o[3].y) * s, (o[3].x - o[3].y) * s);   // * e^{3 i pi/4}
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = cadd(e[k], o[k]);
        v[k + 4] = csub(e[k], o[k]);
    }
}

// radix 4 x 4: a[n2][k1] = DFT4(x[n2 + 4 n1]); a[n2][k1] *= w16^(n2 k1); X[k1 + 4 k2] = DFT4_n2
template <> __device__ __forceinline__ void dft_reg<16>(float2* v) {
    // w16^m for m = 0..9 (cos, sin of 2 pi m / 16)
    const float c1 = 0.92387953251128675613f, s1 = 0.38268343236508977173f;
    const float c2 = 0.70710678118654752440f;
    float2 a[4][4];
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
#pragma unroll
        for (int n1 = 0; n1 < 4; ++n1) a[n2][n1] = v[n2 + 4 * n1];
        dft_reg<4>(a[n2]);
    }
    // twiddles w16^(n2 k1)
    const float2 w1 = make_float2(c1, s1), w2 = make_float2(c2, c2), w3 = make_float2(s1, c1);
    const float2 w6 = make_float2(-c2, c2), w9 = make_float2(-c1, -s1);
    a[1][1] = cfma_tw(a[1][1], w1);
    a[1][2] = cfma_tw(a[1][2], w2);
    a[1][3] = cfma_tw(a[1][3], w3);
    a[2][1] = cfma_tw(a[2][1], w2);
    a[2][2] = cmul_i(a[2][2]);                    // w16^4 = i
    a[2][3] = cfma_tw(a[2][3], w6);
    a[3][1] = cfma_tw(a[3][1], w3);
    a[3][2] = cfma_tw(a[3][2], w6);
    a[3][3] = cfma_tw(a[3][3], w9);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
        float2 t[4] = {a[0][k1], a[1][k1], a[2][k1], a[3][k1]};
        dft_reg<4>(t);
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = t[k2];
    }
}

// One pass of radix R over sub-length M for transform `f` (T threads, tt = lane in transform).
template <int N, int R>
__device__ __forceinline__ void fft_pass(float2* __restrict__ buf, const float2* __restrict__ twN, int M, int tt) {
    constexpr int T = N / 16;
    const int Mp = M / R;
#pragma unroll
    for (int q = 0; q < 16 / R; ++q) {
        const int item = tt + q * T;                  // 0 .. N/R - 1
        const int g = item / Mp, n2 = item - g * Mp;
        const int base = g * M + n2;
        float2 v[R];
#pragma unroll
        for (int n1 = 0; n1 < R; ++n1) v[n1] = buf[fpad(base + n1 * Mp)];
        dft_reg<R>(v);
        if (Mp > 1) {
            const int step = n2 * (N / M);            // w_M^(n2 k1) = w_N^(n2 k1 N/M)
#pragma unroll
            for (int k1 = 1; k1 < R; ++k1) v[k1] = cfma_tw(v[k1], twN[(step * k1) & (N - 1)]);
        }
#pragma unroll
        for (int k1 = 0; k1 < R; ++k1) buf[fpad(base + k1 * Mp)] = v[k1];
    }
}

// All passes of one transform; every thread of the CTA must call this
// (barriers inside).  `active` is false for threads without a transform.
template <int N>
__device__ __forceinline__ void fft_inplace(float2* __restrict__ buf, const float2* __restrict__ twN, int tt, bool active) {
    using Pl = FftPlan<N>;
    int M = N;
#pragma unroll
    for (int p = 0; p < Pl::P; ++p) {
        if (active) {
            if (Pl::R(p) == 16) fft_pass<N, 16>(buf, twN, M, tt);
            else if (Pl::R(p) == 8) fft_pass<N, 8>(buf, twN, M, tt);
            else if (Pl::R(p) == 4) fft_pass<N, 4>(buf, twN, M, tt);
            else if (Pl::R(p) == 2) fft_pass<N, 2>(buf, twN, M, tt);
        }
        M /= Pl::R(p);
        __syncthreads();
    }
}

// shared-memory position holding output X[k] after fft_inplace
template <int N>
__device__ __forceinline__ int out_pos(int k) {
    using Pl = FftPlan<N>;
    int pos = 0, M = N, rem = k;
#pragma unroll
    for (int p = 0; p < Pl::P; ++p) {
        const int R = Pl::R(p);
        M /= R;
        pos += (rem % R) * M;
        rem /= R;
    }
    return pos;
}

}  // namespace hs
