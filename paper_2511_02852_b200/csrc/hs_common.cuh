// Shared device helpers for the hybridsea_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "hybridsea_b200.h"

namespace hs {

// ---------------------------------------------------------------- errors --
void set_error(const char* fmt, ...);

#define HS_CHECK_ARG(cond, ...)                \
    do {                                       \
        if (!(cond)) {                         \
            ::hs::set_error(__VA_ARGS__);      \
            return 1;                          \
        }                                      \
    } while (0)

#define HS_CUDA(call)                                                              \
    do {                                                                           \
        cudaError_t _e = (call);                                                   \
        if (_e != cudaSuccess) {                                                   \
            ::hs::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,             \
                            cudaGetErrorString(_e));                               \
            return 2;                                                              \
        }                                                                          \
    } while (0)

#define HS_LAUNCH_CHECK()                                                          \
    do {                                                                           \
        cudaError_t _e = cudaGetLastError();                                       \
        if (_e != cudaSuccess) {                                                   \
            ::hs::set_error("%s:%d launch: %s", __FILE__, __LINE__,                \
                            cudaGetErrorString(_e));                               \
            return 2;                                                              \
        }                                                                          \
    } while (0)

// deterministic-mode sum of squares: fp64 partial -> int64 fixed point
__device__ __forceinline__ void sumsq_add(double* dst, double v, int fixed_point) {
    if (fixed_point)
        atomicAdd(reinterpret_cast<unsigned long long*>(dst),
                  (unsigned long long)__double2ll_rn(v * (double)(1ull << HS_FIXED_SUMSQ_BITS)));
    else
        atomicAdd(dst, v);
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Experiment builds only (-DHS_EXP_SKIP): HS_EXP_SKIP=<stage>[,<stage>...]
// makes that stage's entry point return without launching, to measure how
// much of the frame a stage holds (tools/gpu/skip.sh).  Never in the product.
#ifdef HS_EXP_SKIP
bool hs_exp_skip(const char* tag);
#define HS_EXP_SKIP_POINT(tag) do { if (hs_exp_skip(tag)) return 0; } while (0)
#else
#define HS_EXP_SKIP_POINT(tag) do {} while (0)
#endif
// Launch state kept per device (function attributes and occupancy are per
// device), so one process may drive several GPUs.
constexpr int HS_MAX_DEVICES = 64;
int current_device();   // cudaGetDevice, clamped to [0, HS_MAX_DEVICES)
template <typename T>
struct PerDevice {
    T v[HS_MAX_DEVICES];
    T& get() { return v[current_device()]; }
};
// one-time per-device kernel configuration (attributes, occupancy), run by
// hs_configure_device before graph capture and lazily on first eager use
int fft_configure();
int smooth_configure();
int compose_configure();
int particles_configure();
int num_sms();

// ---------------------------------------------------------------- complex --
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// multiply by +i
__device__ __forceinline__ float2 cmul_i(float2 a) { return make_float2(-a.y, a.x); }
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }

// ------------------------------------------------- exact fp64 (no FMA) --
// The reference evaluates with separate IEEE mul/add (numpy); contraction to
// FMA would change positions and flip cull decisions, so spell them out.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// ------------------------------------------------------ Philox4x64-10 --
struct U256 { unsigned long long w[4]; };

__device__ __forceinline__ void philox_round(unsigned long long c[4], unsigned long long k0,
                                             unsigned long long k1) {
    const unsigned long long M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
    unsigned long long lo0 = M0 * c[0], hi0 = __umul64hi(M0, c[0]);
    unsigned long long lo1 = M1 * c[2], hi1 = __umul64hi(M1, c[2]);
    unsigned long long n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
}

// word (d % 4) of block counter0 + 1 + d/4  -- numpy Philox stream layout
__device__ __forceinline__ unsigned long long philox_draw(const unsigned long long* st,
                                                          unsigned long long d) {
    unsigned long long c[4];
    unsigned long long add = 1ULL + (d >> 2);
    // 256-bit add with carry
    unsigned long long s0 = st[2] + add;
    unsigned long long carry = s0 < add ? 1ULL : 0ULL;
    c[0] = s0;
    for (int i = 1; i < 4; ++i) {
        unsigned long long v = st[2 + i] + carry;
        carry = (carry && v == 0ULL) ? 1ULL : 0ULL;
        c[i] = v;
    }
    unsigned long long k0 = st[0], k1 = st[1];
    const unsigned long long W0 = 0x9E3779B97F4A7C15ULL, W1 = 0xBB67AE8584CAA73BULL;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += W0; k1 += W1; }
        philox_round(c, k0, k1);
    }
    return c[d & 3];
}

// ------------------------------------------------------------ PCG64 --
// numpy's PCG64 (XSL-RR 128/64): step the 128-bit LCG, output XSL-RR of the
// new state; default_rng's bit generator (reference harness.py:79).
typedef unsigned __int128 u128;
typedef unsigned long long u64;

__device__ __forceinline__ u128 pcg_mult() {
    return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

__device__ __forceinline__ u64 pcg_output(u128 s) {
    const u64 hi = (u64)(s >> 64), lo = (u64)s;
    const unsigned rot = (unsigned)(hi >> 58);
    const u64 x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

// One PCG64 draw: step the LCG, output XSL-RR of the new state.
__device__ __forceinline__ u64 pcg_next(u128& s, u128 inc) {
    s = s * pcg_mult() + inc;
    return pcg_output(s);
}

// LCG jump-ahead by `delta` steps (Brown, "Random number generation with
// arbitrary strides", 1994).
__device__ __forceinline__ u128 pcg_advance(u128 s, u128 inc, u64 delta) {
    u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
    while (delta) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * s + acc_plus;
}

// Raw draw d (counted from the stream state) of an injection stream
// (HsInjectArgs.rng, 8 words): word 7 = 0 -> Philox4x64-10 [key, counter0,
// draw index]; word 7 = 1 -> PCG64 [state hi, lo, inc hi, lo, -, -, draw index]
__device__ __forceinline__ u64 stream_draw(const u64* st, u64 d) {
    if (st[7] == 1ull) {
        const u128 s0 = ((u128)st[0] << 64) | st[1], inc = ((u128)st[2] << 64) | st[3];
        return pcg_output(pcg_advance(s0, inc, d + 1));
    }
    return philox_draw(st, d);
}

// numpy: lo + (hi - lo) * ((raw >> 11) * 2^-53)
__device__ __forceinline__ double uniform_from(unsigned long long raw, double lo, double range) {
    double unit = (double)(raw >> 11) * (1.0 / 9007199254740992.0);
    return dadd(lo, dmul(range, unit));
}

// ------------------------------------------------------------ reductions --
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Block-wide exclusive scan of one int per thread; returns the exclusive
// prefix and writes the block total to *total.  `sm` needs 33 ints.
__device__ __forceinline__ int block_excl_scan(int v, int* sm, int* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    int inc = warp_incl_scan(v, lane);
    if (lane == 31) sm[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int w = lane < nw ? sm[lane] : 0;
        int wi = warp_incl_scan(w, lane);
        if (lane < nw) sm[lane] = wi - w;
        if (lane == nw - 1) sm[32] = wi;
    }
    __syncthreads();
    int res = inc - v + sm[wid];
    *total = sm[32];
    __syncthreads();
    return res;
}

// ------------------------------------------------------------ cp.async --
// Asynchronous global -> shared copies (LDGSTS): a thread issues all of its
// tile loads back to back and waits once, so a CTA keeps KBs in flight
// instead of one dependent load per loop trip.  `valid == false` zero-fills.
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 4 : 0));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 8 : 0));
}
// 16-byte copy, zero-filled when !valid (src-size 0)
__device__ __forceinline__ void cp_async16z(void* smem, const void* gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// ------------------------------------------------- bulk copy (TMA, 1-D) --
// One thread moves a whole contiguous block global -> shared with
// cp.async.bulk (the Hopper/Blackwell tensor-memory-access engine, no
// per-element instructions); completion is counted in bytes on an mbarrier
// that every consumer waits on.  Addresses 16-byte aligned, sizes multiples
// of 16.
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(b), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, unsigned long long* bar) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem), b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(s), "l"(gmem), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 ::"r"(b), "r"(parity) : "memory");
}

// The patch as its synthesised surface sees it: the rectangle at the
// synthesis origin (HsPatch.sx0/sy0; max corner = min + (l1, l2) as
// PatchRegion.max_corner, particles.py:63-65)
__device__ __forceinline__ HsPatch synth_view(HsPatch P) {
    P.x0 = P.sx0;
    P.y0 = P.sy0;
    P.x1 = P.sx0 + P.l1;
    P.y1 = P.sy0 + P.l2;
    return P;
}

__device__ __forceinline__ float smoothstep01(float t) {
    t = fminf(fmaxf(t, 0.f), 1.f);
    return t * t * (3.f - 2.f * t);
}

}  // namespace hs
