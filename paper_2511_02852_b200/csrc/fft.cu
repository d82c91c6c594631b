// FFT background: per-frame dispersion rotation + inverse 2-D FFT to height,
// choppy displacement and (optionally) periodic normals.
//
// Replaces evolve_and_synthesize (reference fft_background.py:181-208), which
// runs spectral_at (:155-159) and three complex128 np.fft.ifft2 calls.
//
// B200 design:
//   * the three real outputs ride on 1.5 complex transforms:
//       A = hh * (1 + lambda kx/|k|)         -> IFFT2(A) = height + i dx
//       B = -i lambda (ky/|k|) hh            -> IFFT2(B) = dy (real)
//     (the imaginary part of the displacement spectra is dropped at the four
//     self-conjugate bins first -- the Hermitian part the reference's .real
//     keeps);
//   * pass 1 (rows, axis 1): one CTA per row pair (i, n-i) so the h0(-k)
//     gather stays in shared memory; h0 is read exactly once (8 B/bin).  B is
//     only transformed for rows 0..n/2: rows n-i are conj of rows i;
//   * pass 2 (columns, axis 0): A columns in tiles; B columns two at a time
//     packed as Y[:,j1] + i Y[:,j2] (each column of Y is Hermitian in i, so
//     one complex IFFT yields two real dy columns);
//   * in-place radix-2/4 DIT in shared memory (two radix-2 stages fused into
//     a radix-4 butterfly per thread, one barrier per pair of stages) with an
//     fp64-accurate fp32 twiddle table;
//   * the phase omega*t is formed and reduced mod 2 pi in fp64 before the
//     fp32 sincos.
#include "fft_reg.cuh"

namespace hs {

__device__ __forceinline__ int bitrev(int x, int logn) { return (int)(__brev((unsigned)x) >> (32 - logn)); }

// In-place inverse DFT (e^{+i}) of `count` sequences of length n stored at
// buf + f*stride in bit-reversed order; result in natural order.
__device__ void ifft_smem(float2* buf, int count, int stride, int n, int logn, const float2* tw) {
    int s = 0;
    if (logn & 1) {
        const int half = n >> 1;
        const int items = count * half;
        for (int it = threadIdx.x; it < items; it += blockDim.x) {
            int f = it >> (logn - 1), k = it & (half - 1);
            float2* p = buf + f * stride + 2 * k;
            float2 a = p[0], b = p[1];
            p[0] = cadd(a, b);
            p[1] = csub(a, b);
        }
        __syncthreads();
        s = 1;
    }
    const int quarter = n >> 2;
    for (; s < logn; s += 2) {
        const int m = 1 << s;
        const int items = count * quarter;
        for (int it = threadIdx.x; it < items; it += blockDim.x) {
            int f = it >> (logn - 2), r = it & (quarter - 1);
            int q = r & (m - 1);
            int base = ((r >> s) << (s + 2)) + q;
            float2* p = buf + f * stride + base;
            float2 x0 = p[0], x1 = p[m], x2 = p[2 * m], x3 = p[3 * m];
            float2 w1 = tw[q << (logn - s - 1)];
            float2 t = cmul(x1, w1);
            float2 y0 = cadd(x0, t), y1 = csub(x0, t);
            t = cmul(x3, w1);
            float2 y2 = cadd(x2, t), y3 = csub(x2, t);
            float2 w2 = tw[q << (logn - s - 2)];
            t = cmul(y2, w2);
            p[0] = cadd(y0, t);
            p[2 * m] = csub(y0, t);
            t = cmul_i(cmul(y3, w2));
            p[m] = cadd(y1, t);
            p[3 * m] = csub(y1, t);
        }
        __syncthreads();
    }
}

struct FftDev {
    int n, logn, chop_on;
    double g, t, chop, dt;
    const long long* frame_ptr;
    double* sumsq_zero;
    const double* kf;
    const double* omega;      // [(n/2+1)^2] or NULL
    const float2* h0;
    const float2* tw;
    float2* wa;
    float2* wb;
};

// ---------------------------------------------------------------- pass 1 --
__global__ void __launch_bounds__(256) fft_rows_kernel(FftDev d) {
    extern __shared__ float2 sm[];
    const int n = d.n, logn = d.logn, half = n >> 1;
    float2* tw = sm;               // n/2
    float2* r0 = tw + half;        // h0 row i
    float2* r1 = r0 + n;           // h0 row i'
    float2* A0 = r1 + n;           // A row i   (bit reversed)
    float2* A1 = A0 + n;           // A row i'
    float2* B0 = A1 + n;           // B row i
    const int i = blockIdx.x;
    const int ip = (n - i) & (n - 1);
    const bool self = (i == ip);
    if (d.sumsq_zero && i == 0 && threadIdx.x == 0) *d.sumsq_zero = 0.0;   // accumulated by pass 2
    for (int k = threadIdx.x; k < half / 2; k += blockDim.x) cp_async16(tw + 2 * k, d.tw + 2 * k);
    for (int k = threadIdx.x; k < half; k += blockDim.x) {
        cp_async16(r0 + 2 * k, d.h0 + (size_t)i * n + 2 * k);
        cp_async16(r1 + 2 * k, d.h0 + (size_t)ip * n + 2 * k);
    }
    cp_async_wait_all();
    __syncthreads();
    const double kxi = d.kf[i], kxip = d.kf[ip];
    const double t = d.frame_ptr ? dmul((double)(*d.frame_ptr), d.dt) : d.t;   // t = frame*dt
    const bool row_sc = (i == 0) || (i == half);
    const double two_pi = 6.283185307179586476925286766559;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const int jm = (n - j) & (n - 1);
        const double kyj = d.kf[j];
        const double km = hypot(kxi, kyj);
        const double w = sqrt(d.g * km);
        double ph = w * t;
        ph -= two_pi * rint(ph * (1.0 / two_pi));
        float s, c;
        sincosf((float)ph, &s, &c);
        const float2 rot = make_float2(c, -s);    // e^{-i w t}
        const float2 rotc = make_float2(c, s);    // e^{+i w t}
        const int jr = bitrev(j, logn);
        // hh(i, j) = h0(i,j) rot + conj(h0(-i,-j)) conj(rot)
        float2 hh0 = cadd(cmul(r0[j], rot), cmul(cconj(r1[jm]), rotc));
        const bool sc = row_sc && (j == 0 || j == half);   // self-conjugate bin
        const double kinv = km > 0.0 ? 1.0 / km : 1.0;       // k_safe (fft_background.py:194-195)
        if (d.chop_on) {
            float fa = sc ? 1.f : (float)(1.0 + d.chop * kxi * kinv);
            A0[jr] = make_float2(hh0.x * fa, hh0.y * fa);
            float fb = sc ? 0.f : (float)(d.chop * kyj * kinv);
            // -i * fb * hh = fb * (hh.y, -hh.x)
            B0[jr] = make_float2(fb * hh0.y, -fb * hh0.x);
        } else {
            A0[jr] = hh0;
        }
        if (!self) {
            float2 hh1 = cadd(cmul(r1[j], rot), cmul(cconj(r0[jm]), rotc));
            float fa = d.chop_on ? (float)(1.0 + d.chop * kxip * kinv) : 1.f;
            A1[jr] = make_float2(hh1.x * fa, hh1.y * fa);
        }
    }
    __syncthreads();
    // A0, A1 are contiguous (count 2, stride n); B0 follows A1
    if (self) {
        ifft_smem(A0, 1, n, n, logn, tw);
        if (d.chop_on) ifft_smem(B0, 1, n, n, logn, tw);
    } else {
        ifft_smem(A0, d.chop_on ? 3 : 2, n, n, logn, tw);
    }
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        d.wa[(size_t)i * n + j] = A0[j];
        if (!self) d.wa[(size_t)ip * n + j] = A1[j];
        if (d.chop_on) d.wb[(size_t)i * n + j] = B0[j];
    }
}

// ---------------------------------------------------------------- pass 2 --
struct ColOut {
    float* h; float* dx; float* dy; double* sumsq; long long* frame_advance; int fixed_point;
};

template <int CA, int CBP>
__global__ void __launch_bounds__(256) fft_cols_kernel(FftDev d, ColOut o, int n_a_tiles) {
    extern __shared__ float2 sm[];
    __shared__ double red[8];
    const int n = d.n, logn = d.logn, half = n >> 1;
    const int stride = n + 1;                 // padded column stride
    float2* tw = sm;
    float2* cols = tw + half;
    if (o.frame_advance && blockIdx.x == 0 && threadIdx.x == 0) *o.frame_advance += 1;
    for (int k = threadIdx.x; k < half / 2; k += blockDim.x) cp_async16(tw + 2 * k, d.tw + 2 * k);
    double acc = 0.0;
    if ((int)blockIdx.x < n_a_tiles) {
        const int j0 = blockIdx.x * CA;
        for (int e = threadIdx.x; e < n * CA; e += blockDim.x) {
            int i = e / CA, c = e - i * CA;
            cp_async8(cols + c * stride + bitrev(i, logn), d.wa + (size_t)i * n + j0 + c, true);
        }
        cp_async_wait_all();
        __syncthreads();
        ifft_smem(cols, CA, stride, n, logn, tw);
        for (int e = threadIdx.x; e < n * CA; e += blockDim.x) {
            int i = e / CA, c = e - i * CA;
            float2 v = cols[c * stride + i];
            size_t o_idx = (size_t)i * n + j0 + c;
            o.h[o_idx] = v.x;
            o.dx[o_idx] = d.chop_on ? v.y : 0.f;
            acc += (double)v.x * (double)v.x;
        }
    } else {
        const int j0 = (blockIdx.x - n_a_tiles) * (2 * CBP);
        if (!d.chop_on) {
            for (int e = threadIdx.x; e < n * 2 * CBP; e += blockDim.x) {
                int i = e / (2 * CBP), c = e - i * (2 * CBP);
                o.dy[(size_t)i * n + j0 + c] = 0.f;
            }
            cp_async_wait_all();
            return;
        }
        cp_async_wait_all();
        for (int e = threadIdx.x; e < n * CBP; e += blockDim.x) {
            int i = e / CBP, q = e - i * CBP;
            int src = i <= half ? i : n - i;
            float2 y1 = d.wb[(size_t)src * n + j0 + 2 * q];
            float2 y2 = d.wb[(size_t)src * n + j0 + 2 * q + 1];
            if (i == 0 || i == half) { y1.y = 0.f; y2.y = 0.f; }   // rows are real there
            else if (i > half) { y1.y = -y1.y; y2.y = -y2.y; }     // Y[-i] = conj(Y[i])
            cols[q * stride + bitrev(i, logn)] = make_float2(y1.x - y2.y, y1.y + y2.x);
        }
        __syncthreads();
        ifft_smem(cols, CBP, stride, n, logn, tw);
        for (int e = threadIdx.x; e < n * 2 * CBP; e += blockDim.x) {
            int i = e / (2 * CBP), c = e - i * (2 * CBP);
            float2 v = cols[(c >> 1) * stride + i];
            o.dy[(size_t)i * n + j0 + c] = (c & 1) ? v.y : v.x;
        }
    }
    if (o.sumsq) {
        acc = warp_sum(acc);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
            if (t != 0.0) sumsq_add(o.sumsq, t, o.fixed_point);
        }
    }
}

// -------------------------------------------------------------- normals --
__global__ void normals_periodic_kernel(const float* __restrict__ h, float* __restrict__ nrm,
                                        int n, float inv2s) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    if (j >= n) return;
    const int ip = (i + 1) & (n - 1), im = (i - 1) & (n - 1);
    const int jp = (j + 1) & (n - 1), jm = (j - 1) & (n - 1);
    float hx = (h[(size_t)ip * n + j] - h[(size_t)im * n + j]) * inv2s;
    float hy = (h[(size_t)i * n + jp] - h[(size_t)i * n + jm]) * inv2s;
    float r = rsqrtf(hx * hx + hy * hy + 1.f);
    float* o = nrm + ((size_t)i * n + j) * 3;
    o[0] = -hx * r;
    o[1] = -hy * r;
    o[2] = r;
}

// ------------------------------------------------ register-FFT kernels --
// n >= 64: each transform is N/16 threads x 16 register elements per pass
// (fft_reg.cuh).  Same data flow as the radix-2/4 kernels above.
// om_row: this CTA's row |i| of the host omega table staged in shared memory
// (or NULL: formed from kf); kxi, kxip = kf[i], kf[ip]; dk = kf[1]
// The dispersion w depends on |j| only, so columns j and -j share the phase
// and its sincos: one call forms both (jm = -j mod n; j == jm writes once).
// Every output is the same arithmetic as a per-column formation.
__device__ __forceinline__ void spectrum_cols(const FftDev& d, const float2* r0, const float2* r1, int i, int j,
                                              double t, const double* om_row, double kxi, double kxip, double dk,
                                              float2* A0, float2* A1, float2* B0) {
    const int n = d.n, half = n >> 1;
    const int jm = (n - j) & (n - 1);
    double w;
    if (om_row) {    // host table, numpy's sqrt(g hypot(kx, ky)) (fft_background.py:40-47)
        w = om_row[j <= half ? j : n - j];
    } else {
        const double kyj = dk * (double)(j <= half ? j : j - n);
        w = sqrt(d.g * sqrt(fma(kxi, kxi, kyj * kyj)));
    }
    const double two_pi = 6.283185307179586476925286766559;
    double ph = w * t;
    ph -= two_pi * rint(ph * (1.0 / two_pi));       // reduce in fp64, |ph| <= pi (App. B.2)
    float s, c;
    __sincosf((float)ph, &s, &c);                   // |err| < 4e-7 on [-pi, pi]
    const float2 rot = make_float2(c, -s), rotc = make_float2(c, s);
    // lambda k / |k| only scales fp32 values: fp32 reciprocal
    const float wf = (float)w;
    const float kinv = wf > 0.f ? (float)d.g / (wf * wf) : 1.f;    // 1/|k| = g / w^2
    const float ch = (float)d.chop;
    const float2 a0 = r0[j], a1 = r1[j], m0 = r0[jm], m1 = r1[jm];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int jj = q ? jm : j;
        if (q && jm == j) break;
        const double kyj = dk * (double)(jj <= half ? jj : jj - n);     // the chop factors use it in fp32
        const float2 hh0 = q ? cadd(cmul(m0, rot), cmul(cconj(a1), rotc)) : cadd(cmul(a0, rot), cmul(cconj(m1), rotc));
        const float2 hh1 = q ? cadd(cmul(m1, rot), cmul(cconj(a0), rotc)) : cadd(cmul(a1, rot), cmul(cconj(m0), rotc));
        const bool sc = ((i == 0) || (i == half)) && (jj == 0 || jj == half);   // self-conjugate bin
        float2 x0, x1, y0;
        if (d.chop_on) {
            const float fa = sc ? 1.f : 1.f + ch * (float)kxi * kinv;
            x0 = make_float2(hh0.x * fa, hh0.y * fa);
            const float fb = sc ? 0.f : ch * (float)kyj * kinv;
            y0 = make_float2(fb * hh0.y, -fb * hh0.x);
            const float fa1 = 1.f + ch * (float)kxip * kinv;
            x1 = make_float2(hh1.x * fa1, hh1.y * fa1);
        } else {
            x0 = hh0;
            x1 = hh1;
            y0 = make_float2(0.f, 0.f);
        }
        const int o = fpad(jj);
        A0[o] = x0;
        A1[o] = x1;
        B0[o] = y0;
    }
}

#ifdef HS_FFT_TRACE
__device__ unsigned long long g_ftrace[2048 * 8];
__device__ __forceinline__ unsigned long long fgtime() {
    unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}
#define FTRACE(k) do { if (threadIdx.x == 0 && blockIdx.x < 2048) g_ftrace[blockIdx.x * 8 + (k)] = fgtime(); } while (0)
#else
#define FTRACE(k) do {} while (0)
#endif

#ifdef HS_FFT_ROWS_MINB
#define HS_FFT_ROWS_LB(n) __launch_bounds__(3 * ((n) / 16) < 32 ? 32 : 3 * ((n) / 16), HS_FFT_ROWS_MINB)
#else
#define HS_FFT_ROWS_LB(n)
#endif
#ifdef HS_FFT_COLS_MINB
#define HS_FFT_COLS_LB(n, ct) __launch_bounds__((ct) * ((n) / 16) < 32 ? 32 : (ct) * ((n) / 16), HS_FFT_COLS_MINB)
#else
#define HS_FFT_COLS_LB(n, ct)
#endif
template <int N>
__global__ void HS_FFT_ROWS_LB(N) fft_rows_reg_kernel(FftDev d) {
    FTRACE(0);
    constexpr int T = N / 16, NP = N + 4;   // transform stride: lanes on different transforms hit different banks
    extern __shared__ float2 sm[];
    float2* tw = sm;            // N
    float2* r0 = tw + N;        // h0 row i
    float2* r1 = r0 + N;        // h0 row i'
    float2* buf = r1 + N;       // 3 transforms of NP: A(i), A(i'), B(i)
    double* om = reinterpret_cast<double*>(buf + 3 * NP);   // omega row |i| (N/2 + 1)
    const int i = blockIdx.x, ip = (N - i) & (N - 1);
    const bool self = (i == ip);
    if (d.sumsq_zero && i == 0 && threadIdx.x == 0) *d.sumsq_zero = 0.0;
    // every input of the row pair at once: twiddles and h0 rows i and -i as three
    // bulk copies (one thread, completion on an mbarrier), the dispersion row by
    // cp.async (its rows are only 8-byte aligned); the frame counter and
    // wavenumbers load meanwhile
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_expect_tx(&bar, 3u * N * (unsigned)sizeof(float2));
        bulk_g2s(tw, d.tw, N * sizeof(float2), &bar);
        bulk_g2s(r0, d.h0 + (size_t)i * N, N * sizeof(float2), &bar);
        bulk_g2s(r1, d.h0 + (size_t)ip * N, N * sizeof(float2), &bar);
    }
    if (d.omega) {
        const double* orow = d.omega + (size_t)(i <= N / 2 ? i : N - i) * (N / 2 + 1);
        for (int k = threadIdx.x; k <= N / 2; k += blockDim.x) cp_async8(om + k, orow + k, true);
    }
    const double t = d.frame_ptr ? dmul((double)(*d.frame_ptr), d.dt) : d.t;   // t = frame * dt
    const double kxi = __ldg(d.kf + i), kxip = __ldg(d.kf + ip), dk = __ldg(d.kf + 1);
    cp_async_wait_all();
    __syncthreads();                                // (also publishes the barrier's init)
    mbar_wait(&bar, 0);
    FTRACE(1);
    for (int j = threadIdx.x; j <= N / 2; j += blockDim.x)
        spectrum_cols(d, r0, r1, i, j, t, d.omega ? om : nullptr, kxi, kxip, dk, buf, buf + NP, buf + 2 * NP);
    __syncthreads();
    FTRACE(2);
    const int f = threadIdx.x / T, tt = threadIdx.x - f * T;
    const bool active = (f == 0) || (f == 1 && !self) || (f == 2 && d.chop_on);
    fft_inplace<N>(buf + (f < 3 ? f : 0) * NP, tw, tt, active && f < 3);
    FTRACE(3);
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        const int pos = fpad(out_pos<N>(k));
        d.wa[(size_t)i * N + k] = buf[pos];
        if (!self) d.wa[(size_t)ip * N + k] = buf[NP + pos];
        if (d.chop_on) d.wb[(size_t)i * N + k] = buf[2 * NP + pos];
    }
    FTRACE(4);
}

// columns: CT transforms per CTA; blocks < n_a_tiles do A (height + i dx),
// the rest do B (two real dy columns per transform)
template <int N, int CT>
__global__ void HS_FFT_COLS_LB(N, CT) fft_cols_reg_kernel(FftDev d, ColOut o, int n_a_tiles) {
    constexpr int T = N / 16, NP = N + 4;   // transform stride: lanes on different transforms hit different banks
    extern __shared__ float2 sm[];
    __shared__ double red[32];
    float2* tw = sm;
    float2* buf = tw + N;       // CT transforms of NP
    if (o.frame_advance && blockIdx.x == 0 && threadIdx.x == 0) *o.frame_advance += 1;
    __shared__ __align__(8) unsigned long long bar;  // the twiddles: one bulk copy
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_expect_tx(&bar, N * (unsigned)sizeof(float2));
        bulk_g2s(tw, d.tw, N * sizeof(float2), &bar);
    }
    const bool is_a = (int)blockIdx.x < n_a_tiles;
    double acc = 0.0;
    if (is_a) {
        const int j0 = blockIdx.x * CT;
        if constexpr (CT % 2 == 0) {
            // two adjacent columns per 16-byte load, scattered to their transforms
            for (int e = threadIdx.x; e < N * (CT / 2); e += blockDim.x) {
                const int i = e / (CT / 2), c = 2 * (e - i * (CT / 2));
                const float4 w = __ldg(reinterpret_cast<const float4*>(d.wa + (size_t)i * N + j0 + c));
                const int pi = fpad(i);
                buf[c * NP + pi] = make_float2(w.x, w.y);
                buf[(c + 1) * NP + pi] = make_float2(w.z, w.w);
            }
        } else {
            for (int e = threadIdx.x; e < N * CT; e += blockDim.x) {
                const int i = e / CT, c = e - i * CT;
                cp_async8(buf + c * NP + fpad(i), d.wa + (size_t)i * N + j0 + c, true);
            }
        }
    } else if (d.chop_on) {
        const int j0 = (blockIdx.x - n_a_tiles) * (2 * CT);
        const int half = N >> 1;
        for (int e = threadIdx.x; e < N * CT; e += blockDim.x) {
            const int i = e / CT, q = e - i * CT;
            const int src = i <= half ? i : N - i;
            const float4 w = __ldg(reinterpret_cast<const float4*>(d.wb + (size_t)src * N + j0 + 2 * q));
            float2 y1 = make_float2(w.x, w.y);
            float2 y2 = make_float2(w.z, w.w);
            if (i == 0 || i == half) { y1.y = 0.f; y2.y = 0.f; }      // rows 0, n/2 are real
            else if (i > half) { y1.y = -y1.y; y2.y = -y2.y; }        // Y[-i] = conj(Y[i])
            buf[q * NP + fpad(i)] = make_float2(y1.x - y2.y, y1.y + y2.x);
        }
    }
    cp_async_wait_all();
    __syncthreads();                                // (also publishes the barrier's init)
    mbar_wait(&bar, 0);                             // before any exit: the copy targets this CTA's smem
    if (!is_a && !d.chop_on) {
        const int j0 = (blockIdx.x - n_a_tiles) * (2 * CT);
        for (int e = threadIdx.x; e < N * 2 * CT; e += blockDim.x) {
            const int i = e / (2 * CT), c = e - i * (2 * CT);
            o.dy[(size_t)i * N + j0 + c] = 0.f;
        }
        return;
    }
    const int f = threadIdx.x / T, tt = threadIdx.x - f * T;
    fft_inplace<N>(buf + (f < CT ? f : 0) * NP, tw, tt, f < CT);
    if (is_a) {
        const int j0 = blockIdx.x * CT;
        if constexpr (CT % 4 == 0) {
            // one output row position per 4 columns: 16-byte height and dx stores
            for (int e = threadIdx.x; e < N * (CT / 4); e += blockDim.x) {
                const int i = e / (CT / 4), c = 4 * (e - i * (CT / 4));
                const int pos = fpad(out_pos<N>(i));
                const float2 v0 = buf[c * NP + pos], v1 = buf[(c + 1) * NP + pos];
                const float2 v2 = buf[(c + 2) * NP + pos], v3 = buf[(c + 3) * NP + pos];
                const size_t oi = (size_t)i * N + j0 + c;
                *reinterpret_cast<float4*>(o.h + oi) = make_float4(v0.x, v1.x, v2.x, v3.x);
                *reinterpret_cast<float4*>(o.dx + oi) =
                    d.chop_on ? make_float4(v0.y, v1.y, v2.y, v3.y) : make_float4(0.f, 0.f, 0.f, 0.f);
                acc += (double)v0.x * (double)v0.x;
                acc += (double)v1.x * (double)v1.x;
                acc += (double)v2.x * (double)v2.x;
                acc += (double)v3.x * (double)v3.x;
            }
        } else {
            for (int e = threadIdx.x; e < N * CT; e += blockDim.x) {
                const int i = e / CT, c = e - i * CT;
                const float2 v = buf[c * NP + fpad(out_pos<N>(i))];
                const size_t oi = (size_t)i * N + j0 + c;
                o.h[oi] = v.x;
                o.dx[oi] = d.chop_on ? v.y : 0.f;
                acc += (double)v.x * (double)v.x;
            }
        }
    } else {
        const int j0 = (blockIdx.x - n_a_tiles) * (2 * CT);
        if constexpr (CT % 2 == 0) {
            // two transforms (four dy columns) per 16-byte store
            for (int e = threadIdx.x; e < N * (CT / 2); e += blockDim.x) {
                const int i = e / (CT / 2), q = 2 * (e - i * (CT / 2));
                const int pos = fpad(out_pos<N>(i));
                const float2 v0 = buf[q * NP + pos], v1 = buf[(q + 1) * NP + pos];
                *reinterpret_cast<float4*>(o.dy + (size_t)i * N + j0 + 2 * q) = make_float4(v0.x, v0.y, v1.x, v1.y);
            }
        } else {
            for (int e = threadIdx.x; e < N * 2 * CT; e += blockDim.x) {
                const int i = e / (2 * CT), c = e - i * (2 * CT);
                const float2 v = buf[(c >> 1) * NP + fpad(out_pos<N>(i))];
                o.dy[(size_t)i * N + j0 + c] = (c & 1) ? v.y : v.x;
            }
        }
    }
    if (o.sumsq) {
        acc = warp_sum(acc);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tsum = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tsum += red[w];
            if (tsum != 0.0) sumsq_add(o.sumsq, tsum, o.fixed_point);
        }
    }
}

// kernel attributes, once per device: set by hs_configure_device before any
// graph capture (attribute calls inside a capture invalidate it), or lazily
// here on first eager use
template <int N, int CT>
int fft_reg_attrs(size_t sm_rows, size_t sm_cols) {
    static PerDevice<bool> attr_done{};
    bool& attr = attr_done.get();
    if (!attr) {
        HS_CUDA(cudaFuncSetAttribute(fft_rows_reg_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_rows));
        HS_CUDA(cudaFuncSetAttribute(fft_cols_reg_kernel<N, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_cols));
        attr = true;
    }
    return 0;
}

template <int N>
int launch_fft_reg(const FftDev& d, const ColOut& o, cudaStream_t st) {
    constexpr int T = N / 16, NP = N + 4;   // transform stride: lanes on different transforms hit different banks
    // transforms per column CTA (B needs 2 CT <= N): 256 threads, so that the
    // 1.5 N column transforms spread evenly over the SMs (all CTAs resident)
#ifndef HS_FFT_COLS_MIN_CT
#define HS_FFT_COLS_MIN_CT 4
#endif
    // at least HS_FFT_COLS_MIN_CT columns per CTA where the CTA stays <= 512
    // threads: 4 adjacent float2 columns fill a 32-byte sector per row read
    constexpr int CT0 = (256 / T) < 1 ? 1 : ((256 / T) < N / 2 ? (256 / T) : N / 2);
    constexpr int CT = (CT0 < HS_FFT_COLS_MIN_CT && HS_FFT_COLS_MIN_CT * T <= 512) ? HS_FFT_COLS_MIN_CT : CT0;
    const int rows_threads = 3 * T < 32 ? 32 : 3 * T;
    const size_t sm_rows = (size_t)(3 * N + 3 * NP) * sizeof(float2) + (size_t)(N / 2 + 1) * sizeof(double);
    const size_t sm_cols = (size_t)(N + CT * NP) * sizeof(float2);
    if (int rc = fft_reg_attrs<N, CT>(sm_rows, sm_cols)) return rc;
    fft_rows_reg_kernel<N><<<N / 2 + 1, rows_threads, sm_rows, st>>>(d);
    HS_LAUNCH_CHECK();
    const int n_a = N / CT, n_b = N / (2 * CT);
    const int cols_threads = CT * T < 32 ? 32 : CT * T;
    fft_cols_reg_kernel<N, CT><<<n_a + n_b, cols_threads, sm_cols, st>>>(d, o, n_a);
    HS_LAUNCH_CHECK();
    return 0;
}

template <int N>
int fft_reg_configure() {
    constexpr int T = N / 16, NP = N + 4;
    constexpr int CT0 = (256 / T) < 1 ? 1 : ((256 / T) < N / 2 ? (256 / T) : N / 2);
    constexpr int CT = (CT0 < HS_FFT_COLS_MIN_CT && HS_FFT_COLS_MIN_CT * T <= 512) ? HS_FFT_COLS_MIN_CT : CT0;
    const size_t sm_rows = (size_t)(3 * N + 3 * NP) * sizeof(float2) + (size_t)(N / 2 + 1) * sizeof(double);
    const size_t sm_cols = (size_t)(N + CT * NP) * sizeof(float2);
    return fft_reg_attrs<N, CT>(sm_rows, sm_cols);
}

int fft_configure() {
    int rc = 0;
    if (!rc) rc = fft_reg_configure<64>();
    if (!rc) rc = fft_reg_configure<128>();
    if (!rc) rc = fft_reg_configure<256>();
    if (!rc) rc = fft_reg_configure<512>();
    if (!rc) rc = fft_reg_configure<1024>();
    if (!rc) rc = fft_reg_configure<2048>();
    if (!rc) rc = fft_reg_configure<4096>();
    return rc;
}

}  // namespace hs

using namespace hs;

#ifdef HS_FFT_TRACE
extern "C" HS_API int hs_debug_ftrace(void* dst) {
    return (int)cudaMemcpyFromSymbol(dst, hs::g_ftrace, sizeof(hs::g_ftrace));
}
#endif

extern "C" int hs_periodic_normals(const float* height, float* normal, int n, double spacing, void* stream) {
    HS_CHECK_ARG(height && normal, "hs_periodic_normals: null buffer");
    HS_CHECK_ARG(n >= 2 && (n & (n - 1)) == 0, "hs_periodic_normals: n=%d must be a power of two", n);
    dim3 grid((n + 127) / 128, n);
    normals_periodic_kernel<<<grid, 128, 0, as_stream(stream)>>>(height, normal, n, (float)(1.0 / (2.0 * spacing)));
    HS_LAUNCH_CHECK();
    return 0;
}

extern "C" int hs_fft_evolve(const HsFftArgs* a, void* stream) {
    HS_EXP_SKIP_POINT("fft");
    HS_CHECK_ARG(a != nullptr, "hs_fft_evolve: null args");
    const int n = a->n;
    HS_CHECK_ARG(n >= 4 && n <= 4096 && (n & (n - 1)) == 0, "hs_fft_evolve: n=%d must be a power of two in [4, 4096]", n);
    HS_CHECK_ARG(a->kf && a->h0 && a->twiddle && a->work_a && a->height && a->dx && a->dy,
                 "hs_fft_evolve: missing buffer");
    const int chop_on = a->choppiness != 0.0;
    HS_CHECK_ARG(!chop_on || a->work_b, "hs_fft_evolve: work_b required when choppiness != 0");
    HS_CHECK_ARG(!a->emit_normals || a->normal, "hs_fft_evolve: normal buffer required");
    HS_CHECK_ARG((((uintptr_t)a->height | (uintptr_t)a->dx | (uintptr_t)a->dy | (uintptr_t)a->work_a |
                   (uintptr_t)a->work_b) & 15u) == 0, "hs_fft_evolve: field and work buffers must be 16-byte aligned");
    cudaStream_t st = as_stream(stream);
    FftDev d;
    d.n = n;
    d.logn = 31 - __builtin_clz((unsigned)n);
    d.chop_on = chop_on;
    d.g = a->g; d.t = a->t; d.chop = a->choppiness; d.dt = a->dt; d.frame_ptr = a->frame_ptr;
    d.sumsq_zero = a->sumsq;
    d.kf = a->kf;
    d.omega = a->omega;
    d.h0 = reinterpret_cast<const float2*>(a->h0);
    d.tw = reinterpret_cast<const float2*>(a->twiddle);
    d.wa = reinterpret_cast<float2*>(a->work_a);
    d.wb = reinterpret_cast<float2*>(a->work_b);

    ColOut oreg{a->height, a->dx, a->dy, a->sumsq, a->frame_advance, a->fixed_point};
    int rc_reg = -1;
    switch (n) {
        case 64: rc_reg = launch_fft_reg<64>(d, oreg, st); break;
        case 128: rc_reg = launch_fft_reg<128>(d, oreg, st); break;
        case 256: rc_reg = launch_fft_reg<256>(d, oreg, st); break;
        case 512: rc_reg = launch_fft_reg<512>(d, oreg, st); break;
        case 1024: rc_reg = launch_fft_reg<1024>(d, oreg, st); break;
        case 2048: rc_reg = launch_fft_reg<2048>(d, oreg, st); break;
        case 4096: rc_reg = launch_fft_reg<4096>(d, oreg, st); break;
        default: break;
    }
    if (rc_reg > 0) return rc_reg;
    if (rc_reg == 0) {
        if (a->emit_normals) {
            dim3 grid((n + 127) / 128, n);
            normals_periodic_kernel<<<grid, 128, 0, st>>>(a->height, a->normal, n, (float)(1.0 / (2.0 * a->spacing)));
            HS_LAUNCH_CHECK();
        }
        return 0;
    }

    size_t sm_rows = (size_t)(n / 2 + 5 * n) * sizeof(float2);
    static PerDevice<size_t> rows_attr_d{};   // attribute calls stay out of graph capture after the first frame
    size_t& rows_attr = rows_attr_d.get();
    if (rows_attr == 0) rows_attr = 48 * 1024;
    if (sm_rows > rows_attr) {
        HS_CUDA(cudaFuncSetAttribute(fft_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_rows));
        rows_attr = sm_rows;
    }
    fft_rows_kernel<<<n / 2 + 1, 256, sm_rows, st>>>(d);
    HS_LAUNCH_CHECK();

    ColOut o{a->height, a->dx, a->dy, a->sumsq, a->frame_advance, a->fixed_point};
    // columns per CTA: keep a tile <= 64 KiB of complex64
    auto launch_cols = [&](auto kern, int ca, int cbp) -> int {
        int n_a = n / ca;
        int n_b = n / (2 * cbp);
        size_t sm = (size_t)(n / 2 + (size_t)(ca > cbp ? ca : cbp) * (n + 1)) * sizeof(float2);
        static PerDevice<size_t> cols_attr_d[2]{};
        size_t& cols_attr = cols_attr_d[ca == 8 ? 0 : 1].get();
        if (cols_attr == 0) cols_attr = 48 * 1024;
        if (sm > cols_attr) {
            HS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            cols_attr = sm;
        }
        kern<<<n_a + n_b, 256, sm, st>>>(d, o, n_a);
        HS_LAUNCH_CHECK();
        return 0;
    };
    int rc;
    if (n <= 8) rc = launch_cols(fft_cols_kernel<4, 2>, 4, 2);
    else if (n <= 512) rc = launch_cols(fft_cols_kernel<8, 4>, 8, 4);
    else if (n <= 1024) rc = launch_cols(fft_cols_kernel<8, 4>, 8, 4);
    else rc = launch_cols(fft_cols_kernel<4, 2>, 4, 2);
    if (rc) return rc;

    if (a->emit_normals) {
        dim3 grid((n + 127) / 128, n);
        normals_periodic_kernel<<<grid, 128, 0, st>>>(a->height, a->normal, n, (float)(1.0 / (2.0 * a->spacing)));
        HS_LAUNCH_CHECK();
    }
    return 0;
}
