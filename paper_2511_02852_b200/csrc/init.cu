// Device init of the background spectral amplitudes h0 (hs_init_h0).
//
// Replaces the host fp64 init_fft (reference fft_background.py:102-146):
//   * Gaussian pairs of np.random.default_rng(seed).standard_normal((n,n,2))
//     (fft_background.py:136-137): the same PCG64 XSL-RR 128/64 raw stream,
//     turned into draws by numpy's 52-bit 256-strip ziggurat (strip tables
//     constructed on the host, normal_draws.py);
//   * band mask (fft_background.py:119-125) and the variance
//     S(omega, theta) g / (2 omega) / k dk^2 / 2 (fft_background.py:127-132,
//     77-87; spectrum.py:108-121, 124-132), fp64 in the reference's order.
//
// Parallel parse of a rejection sampler.  An attempt starting at raw
// position p consumes 1 raw (fast accept), 2 (wedge test, accept or reject)
// or 1 + 2m (exponential tail, m tries) and yields at most one draw; the
// draws are the accepted attempts along the chain p0 = 0, p' = p + consumed.
//   1. classify: one thread per chunk of HS_ZIG_CHUNK positions jumps the
//      LCG to its chunk, classifies every position and summarises the chunk
//      as a map entry offset e (< HS_ZIG_ENTRIES) -> (draws, exit offset into
//      the next chunk).  Chains from different entries merge within a few
//      positions, so the map is formed from the chain of entry 0 plus a short
//      walk per other entry.
//   2. group: one warp per HS_ZIG_GROUP chunks composes the maps (lane e
//      follows entry e; each chunk's 32-entry row is read coalesced and
//      picked with a shuffle, so the loads do not depend on the chain).
//   3. scan: one warp follows the chain through the groups from entry 0.
//   4. chunks: one warp per group resolves each chunk's entry and first draw.
//   5. draws: one thread per chunk writes its accepted values in order.
//   6. h0: one thread per grid cell forms the mask, the variance and h0.
#include "hs_common.cuh"

namespace hs {
namespace {

constexpr int ZL = HS_ZIG_CHUNK;
constexpr int ZE = HS_ZIG_ENTRIES;
constexpr int ZG = HS_ZIG_GROUP;
constexpr int CLASSIFY_THREADS = 128;

__device__ __forceinline__ double unit53(u64 r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

struct Work {
    double* val;        // [P] value of an accepted attempt
    uint8_t* cons;      // [P] consumed raws | 0x80 if accepted
    uint32_t* summ;     // [C * ZE] chunk maps: draws << 8 | exit
    uint32_t* gsum;     // [NG * ZE] group maps
    uint32_t* gentry;   // [NG]
    uint32_t* gbase;    // [NG]
    uint32_t* centry;   // [C]
    uint32_t* cbase;    // [C]
    double* xi;         // [2 n^2]
};

struct Sizes {
    long long total;    // draws needed: 2 n^2
    long long P;        // raw positions classified
    long long C, NG;    // chunks, groups
};

Sizes sizes_for(int n) {
    Sizes z;
    z.total = 2LL * n * n;
    // ~1.02 raws per draw on average; 6% + 8192 slack is > 100 sigma
    const long long want = z.total + z.total / 16 + 8192;
    const long long per_group = (long long)ZL * ZG;
    z.NG = (want + per_group - 1) / per_group;
    z.C = z.NG * ZG;
    z.P = z.C * ZL;
    return z;
}

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

size_t carve(const Sizes& z, void* base, Work* w) {
    size_t off = 0;
    char* p = (char*)base;
    auto take = [&](size_t bytes) { void* r = p ? p + off : nullptr; off += align256(bytes); return r; };
    void* val = take(sizeof(double) * z.P);
    void* cons = take(z.P);
    void* summ = take(sizeof(uint32_t) * z.C * ZE);
    void* gsum = take(sizeof(uint32_t) * z.NG * ZE);
    void* gentry = take(sizeof(uint32_t) * z.NG);
    void* gbase = take(sizeof(uint32_t) * z.NG);
    void* centry = take(sizeof(uint32_t) * z.C);
    void* cbase = take(sizeof(uint32_t) * z.C);
    void* xi = take(sizeof(double) * z.total);
    if (w) {
        w->val = (double*)val; w->cons = (uint8_t*)cons; w->summ = (uint32_t*)summ; w->gsum = (uint32_t*)gsum;
        w->gentry = (uint32_t*)gentry; w->gbase = (uint32_t*)gbase; w->centry = (uint32_t*)centry;
        w->cbase = (uint32_t*)cbase; w->xi = (double*)xi;
    }
    return off;
}

struct Zig {
    const u64* k;
    const double* w;
    const double* f;
    double r, inv_r;
};

// One ziggurat attempt at the position whose raw is the next draw of `s`
// (numpy random_standard_normal, one loop iteration).  Returns the raws
// consumed; `ok` / `x` the outcome.  `s` is advanced by one raw only.
__device__ __forceinline__ int zig_attempt(u128& s, u128 inc, const Zig& Z, bool& ok, double& x) {
    const u64 r0 = pcg_next(s, inc);
    const int idx = (int)(r0 & 0xff);
    const u64 r = r0 >> 8;
    const u64 rabs = (r >> 1) & 0x000fffffffffffffull;
    x = __dmul_rn((double)rabs, __ldg(Z.w + idx));
    if (r & 1) x = -x;
    if (rabs < __ldg(Z.k + idx)) { ok = true; return 1; }
    u128 t = s;                                   // look-ahead copy for the slow paths
    if (idx == 0) {                               // exponential tail beyond r
        for (int q = 1; q < 127; q += 2) {
            const double xx = __dmul_rn(-Z.inv_r, log1p(-unit53(pcg_next(t, inc))));
            const double yy = -log1p(-unit53(pcg_next(t, inc)));
            if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
                const double v = __dadd_rn(Z.r, xx);
                x = ((rabs >> 8) & 1) ? -v : v;
                ok = true;
                return q + 2;
            }
        }
        ok = false;
        return 127 | 0x100;                       // flagged: run longer than the window
    }
    const double u = unit53(pcg_next(t, inc));    // wedge test
    const double fi = __ldg(Z.f + idx), fim = __ldg(Z.f + idx - 1);
    ok = __dadd_rn(__dmul_rn(__dsub_rn(fim, fi), u), fi) < exp(__dmul_rn(__dmul_rn(-0.5, x), x));
    return 2;
}

__global__ void __launch_bounds__(CLASSIFY_THREADS)
zig_classify_kernel(Work W, long long C, u128 s0, u128 inc, Zig Z, int* status) {
    __shared__ uint8_t cons_s[ZL][CLASSIFY_THREADS];
    __shared__ uint8_t cum_s[ZL][CLASSIFY_THREADS];   // draws before position p on the entry-0 chain
    const int t = threadIdx.x;
    const long long c = (long long)blockIdx.x * CLASSIFY_THREADS + t;
    if (c >= C) return;
    u128 s = pcg_advance(s0, inc, (u64)c * ZL);
    const long long base = c * ZL;
    bool bad = false;
    for (int p = 0; p < ZL; ++p) {
        bool ok;
        double x;
        int k = zig_attempt(s, inc, Z, ok, x);
        if (k & 0x100) { bad = true; k &= 0xff; }
        const uint8_t b = (uint8_t)(k | (ok ? 0x80 : 0));
        cons_s[p][t] = b;
        W.cons[base + p] = b;
        W.val[base + p] = ok ? x : 0.0;
    }
    // chain of entry 0: mark its positions with the draws before them
    uint32_t on0[ZL / 32] = {};
    int pos = 0, cnt = 0;
    while (pos < ZL) {
        on0[pos >> 5] |= 1u << (pos & 31);
        cum_s[pos][t] = (uint8_t)cnt;
        const uint8_t b = cons_s[pos][t];
        cnt += b >> 7;
        pos += b & 0x7f;
    }
    const int total0 = cnt, exit0 = pos - ZL;
    for (int e = 0; e < ZE; ++e) {
        int q = e, extra = 0, draws, ex;
        while (q < ZL && !((on0[q >> 5] >> (q & 31)) & 1)) {
            const uint8_t b = cons_s[q][t];
            extra += b >> 7;
            q += b & 0x7f;
        }
        if (q < ZL) { draws = extra + total0 - cum_s[q][t]; ex = exit0; }
        else { draws = extra; ex = q - ZL; }
        if (ex >= ZE) { bad = true; ex = ZE - 1; }
        W.summ[c * ZE + e] = ((uint32_t)draws << 8) | (uint32_t)ex;
    }
    if (bad) atomicOr(status, 1);
}

// Compose HS_ZIG_GROUP chunk maps per warp; lane = entry offset.
__global__ void zig_group_kernel(Work W, long long NG) {
    const int lane = threadIdx.x & 31;
    const long long g = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (g >= NG) return;
    uint32_t st = lane, cnt = 0;
    const uint32_t* row = W.summ + g * ZG * ZE + lane;
#pragma unroll 8
    for (int k = 0; k < ZG; ++k) {
        const uint32_t v = __shfl_sync(0xffffffffu, row[k * ZE], st);
        cnt += v >> 8;
        st = v & 0xff;
    }
    W.gsum[g * ZE + lane] = (cnt << 8) | st;
}

// Follow the chain from position 0 through the group maps (one warp).  Rows
// are fetched 8 groups ahead of the chain (their addresses do not depend on it).
__global__ void zig_scan_kernel(Work W, long long NG, long long total, int* status) {
    const int lane = threadIdx.x;
    uint32_t st = 0;
    unsigned long long base = 0;
    for (long long g0 = 0; g0 < NG; g0 += 8) {
        uint32_t rows[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) rows[u] = g0 + u < NG ? __ldg(W.gsum + (g0 + u) * ZE + lane) : 0u;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (g0 + u >= NG) break;
            const uint32_t v = __shfl_sync(0xffffffffu, rows[u], st);
            if (lane == 0) { W.gentry[g0 + u] = st; W.gbase[g0 + u] = (uint32_t)min(base, 0xffffffffull); }
            base += v >> 8;
            st = v & 0xff;
        }
    }
    if (lane == 0 && base < (unsigned long long)total) atomicOr(status, 2);
}

// Entry offset and first draw index of every chunk (one warp per group).
__global__ void zig_chunks_kernel(Work W, long long NG) {
    const int lane = threadIdx.x & 31;
    const long long g = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (g >= NG) return;
    uint32_t st = W.gentry[g], base = W.gbase[g];
    const uint32_t* row = W.summ + g * ZG * ZE + lane;
    for (int k0 = 0; k0 < ZG; k0 += 8) {
        uint32_t rows[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) rows[u] = __ldg(row + (k0 + u) * ZE);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t v = __shfl_sync(0xffffffffu, rows[u], st);
            if (lane == 0) { W.centry[g * ZG + k0 + u] = st; W.cbase[g * ZG + k0 + u] = base; }
            base += v >> 8;
            st = v & 0xff;
        }
    }
}

__global__ void zig_draws_kernel(Work W, long long C, long long total) {
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    int pos = (int)W.centry[c];
    long long j = W.cbase[c];
    const long long base = c * ZL;
    while (pos < ZL && j < total) {
        const uint8_t b = W.cons[base + pos];
        if (b & 0x80) W.xi[j++] = W.val[base + pos];
        pos += b & 0x7f;
    }
}

// S_J(omega) (spectrum.py:108-121) in numpy's evaluation order.
__device__ double jonswap(const HsInitArgs& a, double w) {
    const double wp = a.omega_p;
    const double sig = w <= wp ? a.sigma_low : a.sigma_high;
    const double d = __dsub_rn(w, wp);
    const double r = exp(__ddiv_rn(-__dmul_rn(d, d), __dmul_rn(__dmul_rn(2.0, __dmul_rn(sig, sig)), __dmul_rn(wp, wp))));
    double s = __dmul_rn(__dmul_rn(a.alpha, __dmul_rn(a.g, a.g)), pow(w, -5.0));
    s = __dmul_rn(s, exp(__dmul_rn(-1.25, pow(__ddiv_rn(wp, w), 4.0))));
    return __dmul_rn(s, pow(a.gamma, r));
}

__global__ void h0_kernel(HsInitArgs a, const double* __restrict__ xi) {
    const int n = a.n;
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (long long)n * n) return;
    const int i = (int)(q / n), j = (int)(q % n);
    const double kx = a.kf[i], ky = a.kf[j];
    const double k = hypot(kx, ky);
    bool live = k >= a.k_lo && k <= a.k_hi && q != 0;
    if (a.kb_hi > 0.0) live = live && k >= a.kb_lo && k < a.kb_hi;
    double re = 0.0, im = 0.0;
    if (live) {
        const double om = __dsqrt_rn(__dmul_rn(a.g, k));
        const double theta = __dsub_rn(atan2(ky, kx), a.mean_direction);
        const double s = a.spread_const ? a.spread_s
                                        : __dmul_rn(16.0, pow(__ddiv_rn(om, a.omega_p), om <= a.omega_p ? 5.0 : -2.5));
        const double c = __ddiv_rn(exp(__dsub_rn(lgamma(__dadd_rn(s, 1.0)), lgamma(__dadd_rn(s, 0.5)))),
                                   __dmul_rn(2.0, __dsqrt_rn(3.141592653589793)));
        const double th = atan2(sin(theta), cos(theta));
        const double dir = pow(fabs(cos(__dmul_rn(0.5, th))), __dmul_rn(2.0, s));
        const double dd = __dmul_rn(__dmul_rn(jonswap(a, om), c), dir);
        double var = __ddiv_rn(__dmul_rn(dd, __ddiv_rn(a.g, __dmul_rn(2.0, om))), k);
        var = __ddiv_rn(__dmul_rn(__dmul_rn(var, a.dk), a.dk), 2.0);
        const double amp = __dsqrt_rn(__ddiv_rn(var, 2.0));
        re = __dmul_rn(amp, xi[2 * q]);
        im = __dmul_rn(amp, xi[2 * q + 1]);
    }
    if (a.h0) { a.h0[2 * q] = re; a.h0[2 * q + 1] = im; }
    if (a.h0_f32) { a.h0_f32[2 * q] = __double2float_rn(re); a.h0_f32[2 * q + 1] = __double2float_rn(im); }
}

}  // namespace
}  // namespace hs

using namespace hs;

extern "C" long long hs_init_workspace_bytes(int n) {
    if (n < 2 || (n & (n - 1)) != 0 || n > 4096) return -1;
    return (long long)carve(sizes_for(n), nullptr, nullptr);
}

extern "C" int hs_init_h0(const HsInitArgs* a, void* stream) {
    HS_CHECK_ARG(a != nullptr, "hs_init_h0: null args");
    HS_CHECK_ARG(a->n >= 4 && (a->n & (a->n - 1)) == 0 && a->n <= 4096, "hs_init_h0: n=%d must be a power of two in [4, 4096]", a->n);
    HS_CHECK_ARG(a->work && a->kf && a->zig_k && a->zig_w && a->zig_f && a->status, "hs_init_h0: missing buffer");
    HS_CHECK_ARG(a->h0 || a->h0_f32, "hs_init_h0: no output");
    cudaStream_t st = as_stream(stream);
    const Sizes z = sizes_for(a->n);
    Work W;
    carve(z, a->work, &W);
    if (a->xi) W.xi = a->xi;
    const u128 s0 = ((u128)a->pcg_state[0] << 64) | a->pcg_state[1];
    const u128 inc = ((u128)a->pcg_inc[0] << 64) | a->pcg_inc[1];
    Zig Z{a->zig_k, a->zig_w, a->zig_f, a->zig_r, 1.0 / a->zig_r};
    HS_CUDA(cudaMemsetAsync(a->status, 0, sizeof(int), st));
    zig_classify_kernel<<<(unsigned)((z.C + CLASSIFY_THREADS - 1) / CLASSIFY_THREADS), CLASSIFY_THREADS, 0, st>>>(
        W, z.C, s0, inc, Z, a->status);
    HS_LAUNCH_CHECK();
    const unsigned warps_blocks = (unsigned)((z.NG + 7) / 8);
    zig_group_kernel<<<warps_blocks, 256, 0, st>>>(W, z.NG);
    HS_LAUNCH_CHECK();
    zig_scan_kernel<<<1, 32, 0, st>>>(W, z.NG, z.total, a->status);
    HS_LAUNCH_CHECK();
    zig_chunks_kernel<<<warps_blocks, 256, 0, st>>>(W, z.NG);
    HS_LAUNCH_CHECK();
    zig_draws_kernel<<<(unsigned)((z.C + 255) / 256), 256, 0, st>>>(W, z.C, z.total);
    HS_LAUNCH_CHECK();
    const long long nn = (long long)a->n * a->n;
    h0_kernel<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(*a, W.xi);
    HS_LAUNCH_CHECK();
    return 0;
}
