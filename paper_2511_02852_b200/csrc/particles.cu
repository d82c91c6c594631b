// Wave-particle pool kernels: boundary injection and the fused
// advect + cull + stable bucket-segmented compaction + layer splat.
//
// Replaces inject (reference particles.py:219-300), advect (:303-328),
// ParticleSet.extend/compact (:163-178) and the per-bucket _splat of
// synthesize (patch_synthesis.py:165-186, 298-310).
//
// Pool layout: SoA, fp64 position + direction,
// fp32 amplitude, no per-particle bucket id -- each patch region is
// bucket-segmented and each segment keeps the reference's stable birth
// order.  The advect kernel reads the virtual sequence
//     for b: [old segment b][new crests b][new troughs b]
// (exactly the reference pool order restricted to bucket b after
// pool.extend(inject(...))) and compacts it with a single-pass
// decoupled-look-back scan, so buckets stay contiguous and in order.
#include <stdlib.h>

#include "synth_common.cuh"

namespace hs {

// Bilinear scatter-add of one particle into its bucket layer
// (patch_synthesis.py:165-186 at gx/f, 298-310).  u = (x - x0)/(texel f) + pad
// in fp64 (index and clamp decision), weights in fp32.
struct SplatLayer {
    long long raw_off;
    double inv_tf;          // 1 / (texel * f)
    double umax, vmax;      // wx - 1, wy - 1
    int pitch, pad;         // raw row pitch (multiple of 4 floats), grid pad
};

__device__ __forceinline__ void red4(float* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" :: "l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ void red2(float* p, float a, float b) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" :: "l"(p), "f"(a), "f"(b) : "memory");
}
// add (v0, v1) at row[c], row[c + 1]; row is 16-byte aligned: one 16-byte
// reduction when the pair sits in one aligned float4, else two 8-byte ones
// (zero lanes leave their neighbours unchanged)
__device__ __forceinline__ void red_pair(float* row, int c, float v0, float v1) {
    const int s = c & 3;
    float* b = row + (c - s);
    if (s == 0) red4(b, v0, v1, 0.f, 0.f);
    else if (s == 1) red4(b, 0.f, v0, v1, 0.f);
    else if (s == 2) red2(b + 2, v0, v1);
    else { red2(b + 2, 0.f, v0); red2(b + 4, v1, 0.f); }
}

// deterministic mode: one int64 fixed-point slot per raw float slot
__device__ __forceinline__ void red_fixed(float* raw, long long e, float v) {
    atomicAdd(reinterpret_cast<unsigned long long*>(raw) + e,
              (unsigned long long)__float2ll_rn(v * (float)(1ull << HS_FIXED_SPLAT_BITS)));
}

template <bool FX>
__device__ __forceinline__ void splat_at(float* __restrict__ raw, const SplatLayer& L, double x0, double y0,
                                         double x, double y, float amp, int* clamp_acc) {
    double u = (x - x0) * L.inv_tf + (double)L.pad;
    double v = (y - y0) * L.inv_tf + (double)L.pad;
    if (u < 0.0 || u > L.umax || v < 0.0 || v > L.vmax) ++(*clamp_acc);
    u = fmin(fmax(u, 0.0), L.umax - 1e-9);
    v = fmin(fmax(v, 0.0), L.vmax - 1e-9);
    const int i0 = (int)u, j0 = (int)v;
    const float fu = (float)(u - i0), fv = (float)(v - j0);
    const float a1 = amp * fu, a0 = amp - a1;          // amp (1 - fu), amp fu
    if constexpr (FX) {
        const long long e = L.raw_off + (long long)i0 * L.pitch + j0;
        red_fixed(raw, e, a0 * (1.f - fv));
        red_fixed(raw, e + 1, a0 * fv);
        red_fixed(raw, e + L.pitch, a1 * (1.f - fv));
        red_fixed(raw, e + L.pitch + 1, a1 * fv);
    } else {
        float* row = raw + L.raw_off + (long long)i0 * L.pitch;
        red_pair(row, j0, a0 * (1.f - fv), a0 * fv);
        red_pair(row + L.pitch, j0, a1 * (1.f - fv), a1 * fv);
    }
}

__device__ __forceinline__ void splat_at(bool fx, float* __restrict__ raw, const SplatLayer& L, double x0, double y0,
                                         double x, double y, float amp, int* clamp_acc) {
    if (fx) splat_at<true>(raw, L, x0, y0, x, y, amp, clamp_acc);
    else splat_at<false>(raw, L, x0, y0, x, y, amp, clamp_acc);
}

// despawn-energy accumulation: fp64, or int64 fixed point (deterministic mode)
__device__ __forceinline__ long long energy_fixed(double e) {
    return __double2ll_rn(e * (double)(1ull << HS_FIXED_ENERGY_BITS));
}
__device__ __forceinline__ void energy_add(double* dst, double e, bool fx) {
    if (fx) atomicAdd(reinterpret_cast<unsigned long long*>(dst), (unsigned long long)energy_fixed(e));
    else atomicAdd(dst, e);
}
// add a (shared-memory) accumulator of the same mode into a global one
__device__ __forceinline__ void energy_flush(double* dst, const double& acc, bool fx) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(acc);
    if (!bits) return;
    if (fx) atomicAdd(reinterpret_cast<unsigned long long*>(dst), bits);
    else atomicAdd(dst, acc);
}

// ============================================================== inject ==
struct InjectDev {
    HsInjectArgs a;
};

__device__ __forceinline__ int find_cell(const int* gstart, int ncell, int g) {
    // largest c with gstart[c] <= g and gstart[c+1] > g
    int lo = 0, hi = ncell - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (gstart[mid] <= g) lo = mid; else hi = mid - 1;
    }
    return lo;
}

#ifdef HS_INJECT_TRACE
__device__ unsigned long long g_itrace[16];
#define ITRACE(k) do { if (threadIdx.x == 0 && blockIdx.x == 0) { unsigned long long t_; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_itrace[k] = t_; } } while (0)
#else
#define ITRACE(k) do {} while (0)
#endif

constexpr int INJ_SMEM_MEMBERS = 640;   // member records held in shared memory
constexpr int INJ_REC = 6;              // e, amp, x, y, ux, uy per member (doubles)

__global__ void __launch_bounds__(512) inject_kernel(HsInjectArgs a) {
    ITRACE(0);
    const int p = blockIdx.x;
    const int nb = a.nb, nth = a.n_theta, ncell = nb * 4;
    __shared__ int n_emit[HS_MAX_BUCKETS * 4];
    __shared__ int gstart[HS_MAX_BUCKETS * 4 + 1];
    __shared__ int live_cnt[HS_MAX_BUCKETS];
    __shared__ int live_before[HS_MAX_BUCKETS + 1];
    __shared__ int soff[HS_MAX_BUCKETS + 1];
    __shared__ int scan_sm[33];
    __shared__ int abort_s;
    const HsPatch P = a.patches[p];
    // resident append (a.append): per-bucket advection constants and segment tails
    __shared__ double ap_step[HS_MAX_BUCKETS], ap_r2[HS_MAX_BUCKETS], ap_eout[HS_MAX_BUCKETS];
    __shared__ long long ap_dst[HS_MAX_BUCKETS];
    __shared__ int ap_room[HS_MAX_BUCKETS], ap_kept[HS_MAX_BUCKETS], ap_clamp;
    __shared__ SplatLayer ap_sl[HS_MAX_BUCKETS];
    if (a.append && threadIdx.x >= 32 && threadIdx.x < 32 + nb) {
        const int b = threadIdx.x - 32, s = p * nb + b;
        const HsBucket Bk = a.buckets[b];
        ap_step[b] = dmul(Bk.speed, a.res.dt);            // speeds * dt (particles.py:312)
        ap_r2[b] = dmul(Bk.radius, Bk.radius);
        const int len = a.res.len_in[s];
        ap_dst[b] = (long long)a.res.seg_base[s] + len;
        ap_room[b] = a.res.seg_cap[s] - len;
        ap_kept[b] = 0;
        ap_eout[b] = 0.0;
        const HsLayer L = a.res.layers[P.layer_base + b];
        ap_sl[b] = SplatLayer{L.raw_off, 1.0 / (P.texel * (double)L.f), (double)(L.wx - 1), (double)(L.wy - 1),
                              L.raw_pitch, L.pad};
        if (b == 0) ap_clamp = 0;
    }
    // the bucket table, cached for the member passes (warps 2.., beside the ledger)
    __shared__ HsBucket Bs[HS_MAX_BUCKETS];
    if (threadIdx.x >= 64)
        for (int e = threadIdx.x - 64; e < nb * (int)(sizeof(HsBucket) / 8); e += blockDim.x - 64)
            reinterpret_cast<double*>(Bs)[e] = reinterpret_cast<const double*>(a.buckets)[e];
    double* acc = a.acc + (size_t)p * ncell;
    const double* hr = a.half_rate + (size_t)p * ncell;
    unsigned long long* rng = a.rng + (size_t)p * 8;

    if (p == 0)
        for (int w = threadIdx.x; w < a.n_zero_words; w += blockDim.x) a.zero_words[w] = 0;
    // 1. quota ledger: acc += half_rate; n = floor(acc); acc -= n   (particles.py:243-245)
    for (int c = threadIdx.x; c < ncell; c += blockDim.x) {
        double v = dadd(acc[c], hr[c]);
        double fl = floor(v);
        acc[c] = dsub(v, fl);
        n_emit[c] = (int)fl;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        // cell prefix (cell = 4 b + side): lane b owns bucket b's four cells
        const int lane = threadIdx.x;
        int e0 = 0, e1 = 0, e2 = 0, e3 = 0;
        if (lane < nb) { e0 = n_emit[4 * lane]; e1 = n_emit[4 * lane + 1]; e2 = n_emit[4 * lane + 2]; e3 = n_emit[4 * lane + 3]; }
        const int sb = e0 + e1 + e2 + e3;
        const int inc = warp_incl_scan(sb, lane);
        if (lane < nb) {
            const int g0 = inc - sb;
            gstart[4 * lane] = g0;
            gstart[4 * lane + 1] = g0 + e0;
            gstart[4 * lane + 2] = g0 + e0 + e1;
            gstart[4 * lane + 3] = g0 + e0 + e1 + e2;
            atomicAdd(reinterpret_cast<unsigned long long*>(&a.groups[(size_t)p * nb + lane]),
                      (unsigned long long)sb);            // result unused: no round trip
        }
        const int tot = __shfl_sync(0xffffffffu, inc, 31);
        if (lane == 0) {
            gstart[ncell] = tot;
            abort_s = (long long)tot * nth > a.member_capacity;
            if (abort_s) atomicOr(a.status, HS_STATUS_STAGE_OVERFLOW);
        }
    }
    __syncthreads();
    ITRACE(1);
    const int g_tot = gstart[ncell];
    int* scount = a.stage_count + (size_t)p * nb;
    if (g_tot == 0 || abort_s) {     // no groups: no RNG draws (particles.py:248-249)
        for (int b = threadIdx.x; b < nb; b += blockDim.x) {
            scount[b] = 0;
            if (a.append) a.res.len_out[p * nb + b] = a.res.len_in[p * nb + b];
        }
        return;
    }
    const int M = g_tot * nth;
    const double birth = a.birth_frame ? dmul((double)(*a.birth_frame), a.birth_dt) : a.birth_t;
    const double pi = 3.141592653589793;
    const double dth = dmul(2.0, pi) / (double)nth;
    const double j_lo = dmul(-0.5, dth), j_range = dsub(dmul(0.5, dth), j_lo);
    const unsigned long long D = rng[6];
    // member records (energy, amplitude, position, direction): shared memory
    // when they fit (the per-bucket sums below walk them serially), global
    // scratch otherwise
    __shared__ __align__(16) double scr_sm[INJ_REC * INJ_SMEM_MEMBERS];
    double* scr = M <= INJ_SMEM_MEMBERS ? scr_sm : a.scratch + (size_t)p * a.member_capacity * INJ_REC;

    // 2. every member: amplitude + booked energy (particles.py:256-264, 291-292)
    //    and its entry point and direction (:266-290), in one pass
    for (int m = threadIdx.x; m < M; m += blockDim.x) {
        const int g = m / nth, k = m - g * nth;
        const int cell = find_cell(gstart, ncell, g);
        const int s = cell & 3;
        const HsBucket& B = Bs[cell >> 2];
        double jit = uniform_from(stream_draw(rng, D + (unsigned long long)g), j_lo, j_range);
        double th0 = dadd(-pi, dmul((double)k + 0.5, dth));
        double th = dadd(th0, jit);
        double cv = fabs(cos(dmul(0.5, th)));
        double dv = dmul(B.spread_c, pow(cv, dmul(2.0, B.spread_s)));
        double amp = sqrt(dmul(dmul(dmul(dmul(2.0, B.s1d), dv), B.width), dth));
        double e = dmul(dmul(dmul(dmul(dmul(0.125, a.rho), a.g), dmul(amp, amp)), pi), dmul(B.radius, B.radius));
        double thw = dadd(th, a.mean_dir);
        double dx, dy;
        sincos(thw, &dy, &dx);                  // one argument reduction for both
        double dot = (s == 0) ? dx : (s == 1) ? -dx : (s == 2) ? dy : -dy;
        int side = dot > 0.0 ? s : (s ^ 1);
        double u = uniform_from(stream_draw(rng, D + (unsigned long long)g_tot + (unsigned long long)m), 0.0, 1.0);
        double px, py;
        if (side == 0)      { px = P.x0;                 py = dadd(P.y0, dmul(u, P.l2)); }
        else if (side == 1) { px = dadd(P.x0, P.l1);     py = dadd(P.y0, dmul(u, P.l2)); }
        else if (side == 2) { px = dadd(P.x0, dmul(u, P.l1)); py = P.y0; }
        else                { px = dadd(P.x0, dmul(u, P.l1)); py = dadd(P.y0, P.l2); }
        double* r = scr + INJ_REC * m;
        r[0] = e; r[1] = amp; r[2] = px; r[3] = py; r[4] = dx; r[5] = dy;
    }
    __syncthreads();
    ITRACE(2);
    // 3. per-bucket energy in member order (bincount order, a serial fp64 sum per
    //    bucket: lane b walks bucket b, loads four ahead) and live counts; prefixes
    const int per_live = a.beta != 0.0 ? 2 : 1;
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        double s = 0.0;
        int live = 0;
        if (lane < nb) {
            const int m0 = gstart[4 * lane] * nth, m1 = gstart[4 * lane + 4] * nth;
            int m = m0;
            for (; m + 4 <= m1; m += 4) {
                const double2 v0 = *reinterpret_cast<const double2*>(scr + INJ_REC * m);
                const double2 v1 = *reinterpret_cast<const double2*>(scr + INJ_REC * (m + 1));
                const double2 v2 = *reinterpret_cast<const double2*>(scr + INJ_REC * (m + 2));
                const double2 v3 = *reinterpret_cast<const double2*>(scr + INJ_REC * (m + 3));
                s = dadd(dadd(dadd(dadd(s, v0.x), v1.x), v2.x), v3.x);
                live += (v0.y > 0.0) + (v1.y > 0.0) + (v2.y > 0.0) + (v3.y > 0.0);
            }
            for (; m < m1; ++m) {
                s = dadd(s, scr[INJ_REC * m]);
                live += scr[INJ_REC * m + 1] > 0.0;
            }
            // e_in += s (one IEEE add, as the reference's ledger update); the
            // result is unused, so this is a fire-and-forget reduction
            atomicAdd(&a.e_in[(size_t)p * nb + lane], s);
            live_cnt[lane] = live;
        }
        const int inc = warp_incl_scan(live, lane);
        if (lane < nb) {
            live_before[lane + 1] = inc;
            soff[lane + 1] = per_live * inc;
        }
        const int tot = __shfl_sync(0xffffffffu, inc, 31);
        if (lane == 0) {
            live_before[0] = 0;
            soff[0] = 0;
            abort_s = per_live * tot > P.stage_capacity;
            if (abort_s) atomicOr(a.status, HS_STATUS_STAGE_OVERFLOW);
        }
    }
    __syncthreads();
    ITRACE(3);
    if (abort_s) {
        for (int b = threadIdx.x; b < nb; b += blockDim.x) {
            scount[b] = 0;
            if (a.append) a.res.len_out[p * nb + b] = a.res.len_in[p * nb + b];
        }
        if (threadIdx.x == 0) rng[6] = D + (unsigned long long)g_tot * (1 + nth);
        return;
    }
    // 4. positions / directions for live members, in order  (particles.py:266-299)
    const long long sb = P.stage_base;
    int carry = 0;
    for (int base = 0; base < M; base += blockDim.x) {
        const int m = base + threadIdx.x;
        double amp = 0.0;
        if (m < M) amp = scr[INJ_REC * m + 1];
        int live = (m < M) && amp > 0.0;
        int tot;
        int ex = block_excl_scan(live, scan_sm, &tot) + carry;
        if (live) {
            const int g = m / nth;
            const int b = find_cell(gstart, ncell, g) >> 2;
            const HsBucket& B = Bs[b];
            const double* r = scr + INJ_REC * m;
            const double px = r[2], py = r[3], dx = r[4], dy = r[5];
            const int rank = ex - live_before[b];
            if (a.append) {
                // advected in their birth frame (harness.py:142-152), culled, appended
                // in the stage's slot order [crests b][troughs b]; culled ones leave holes
                const double ph = dsub(px, dmul(B.radius, dx)), qh = dsub(py, dmul(B.radius, dy));
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                    if (m == 1 && per_live != 2) break;
                    const int j = rank + m * live_cnt[b];
                    const double x0 = m ? ph : px, y0 = m ? qh : py;
                    const float am = m ? (float)(-a.beta * amp) : (float)amp;
                    const double nx = dadd(x0, dmul(dx, ap_step[b]));      // pos += dir * (c dt) (:312-313)
                    const double ny = dadd(y0, dmul(dy, ap_step[b]));
                    const double ox = fmax(fmax(dsub(P.x0, nx), dsub(nx, P.x1)), 0.0);
                    const double oy = fmax(fmax(dsub(P.y0, ny), dsub(ny, P.y1)), 0.0);
                    const bool keep = dadd(dmul(ox, ox), dmul(oy, oy)) <= ap_r2[b];  // (:315-320)
                    if (j < ap_room[b]) {
                        const long long o = ap_dst[b] + j;
                        a.res.pool.x[o] = keep ? nx : __longlong_as_double(0x7ff8000000000000LL);
                        a.res.pool.y[o] = ny; a.res.pool.ux[o] = dx; a.res.pool.uy[o] = dy; a.res.pool.amp[o] = am;
                        if (a.res.pool.birth) a.res.pool.birth[o] = birth;
                    }
                    if (keep && j < ap_room[b]) {        // overflowed members are lost (status bit)
                        atomicAdd(&ap_kept[b], 1);
                        int cl = 0;
                        splat_at(a.res.fixed_point, a.res.raw_layers, ap_sl[b], P.sx0, P.sy0, nx, ny, am, &cl);
                        if (cl) atomicAdd(&ap_clamp, cl);
                    } else if (am > 0.f) {
                        const double e2 = (double)am;                  // crest despawn energy (:322-327)
                        energy_add(&ap_eout[b], 0.125 * a.rho * a.g * (e2 * e2) * 3.141592653589793 * ap_r2[b],
                                   a.res.fixed_point);
                    }
                }
            } else {
                long long o = sb + soff[b] + rank;
                a.stage.x[o] = px; a.stage.y[o] = py; a.stage.ux[o] = dx; a.stage.uy[o] = dy;
                a.stage.amp[o] = (float)amp;
                if (a.stage.birth) a.stage.birth[o] = birth;
                if (per_live == 2) {
                    o += live_cnt[b];
                    a.stage.x[o] = dsub(px, dmul(B.radius, dx));
                    a.stage.y[o] = dsub(py, dmul(B.radius, dy));
                    a.stage.ux[o] = dx; a.stage.uy[o] = dy;
                    a.stage.amp[o] = (float)(-a.beta * amp);
                    if (a.stage.birth) a.stage.birth[o] = birth;
                }
            }
        }
        carry += tot;
    }
    ITRACE(4);
    for (int b = threadIdx.x; b < nb; b += blockDim.x) scount[b] = per_live * live_cnt[b];
    if (threadIdx.x == 0) rng[6] = D + (unsigned long long)g_tot * (1 + nth);
    if (a.append) {
        __syncthreads();
        for (int b = threadIdx.x; b < nb; b += blockDim.x) {
            const int s = p * nb + b, n = per_live * live_cnt[b];
            // an overflowing segment keeps only the members that fit: its length
            // never runs past seg_cap into the next bucket's segment
            a.res.len_out[s] = a.res.len_in[s] + min(n, ap_room[b]);
            if (n > ap_room[b]) atomicOr(a.status, HS_STATUS_POOL_OVERFLOW);
            if (ap_kept[b]) atomicAdd(&a.res.live[s], ap_kept[b]);
            energy_flush(&a.res.e_out[s], ap_eout[b], a.res.fixed_point);
        }
        if (threadIdx.x == 0 && ap_clamp && a.res.clamped) atomicAdd(&a.res.clamped[p], ap_clamp);
    }
    ITRACE(5);
}

#ifdef HS_INJECT_TRACE
extern "C" HS_API int hs_debug_itrace(void* dst) {
    return (int)cudaMemcpyFromSymbol(dst, g_itrace, sizeof(g_itrace));
}
#endif

// ============================================================== advect ==
constexpr int ADV_THREADS = 256;
constexpr int ADV_ITEMS = 4;                        // items per thread per chunk
constexpr int ADV_CHUNK = ADV_THREADS * ADV_ITEMS;  // 1024
constexpr unsigned long long FLAG_AGG = 1ULL << 32;
constexpr unsigned long long FLAG_PRE = 2ULL << 32;

__device__ __forceinline__ int find_seg(const int* off, int nseg, int v) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= v) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ void splat_one(float* __restrict__ raw, const HsLayer& L, const HsPatch& P,
                                          double x, double y, float amp, int* clamp_acc) {
    SplatLayer S{L.raw_off, 1.0 / (P.texel * (double)L.f), (double)(L.wx - 1), (double)(L.wy - 1), L.raw_pitch, L.pad};
    splat_at<false>(raw, S, P.sx0, P.sy0, x, y, amp, clamp_acc);
}

// Persistent CTAs take tiles of ADV_TILE virtual items in order from a global
// counter; tiles never straddle patches.  Two phases per tile:
//   1. stream the tile's items from HBM: advect in fp64 with the reference's
//      operation order, keep test, one ballot word per (chunk, item, warp);
//      publish the tile's survivor count and resolve its prefix with a
//      warp-parallel decoupled look-back (32 predecessors per round);
//   2. re-read the items (L2-resident now), recompute the same positions and
//      scatter survivors stably (ballot ranks) + the fused layer splat; the
//      dropped are optionally scattered the same way.
// Large tiles keep the look-back chain short (~210 tiles at C3).
__device__ __forceinline__ void adv_item(const HsAdvectArgs& a, const HsPatch& P, const long long* in_base,
                                         const int* st_off, const int* voff, const int* in_cnt, const double* step_s,
                                         int v, int b, double& x, double& y, double& ux, double& uy,
                                         const float** amp_ptr, double* birth = nullptr) {
    const int local = v - voff[b];
    const bool from_pool = local < in_cnt[b];
    const long long src = from_pool ? in_base[b] + local
                                    : P.stage_base + st_off[b] + (local - in_cnt[b]);
    const HsPool& S = from_pool ? a.in : a.stage;
    const double step = step_s[b];
    ux = S.ux[src];
    uy = S.uy[src];
    x = dadd(S.x[src], dmul(ux, step));        // pos += dir * (c dt)  (particles.py:312-313)
    y = dadd(S.y[src], dmul(uy, step));
    *amp_ptr = S.amp + src;
    if (birth && S.birth) *birth = S.birth[src];
}

template <int ADV_CHUNKS>
__global__ void __launch_bounds__(ADV_THREADS, 3) advect_kernel(HsAdvectArgs a) {
    constexpr int ADV_TILE = ADV_CHUNK * ADV_CHUNKS;                        // items per look-back tile
    constexpr int ADV_WORDS = ADV_CHUNKS * ADV_ITEMS * (ADV_THREADS / 32);  // ballot words per tile
    const int nb = a.nb;
    __shared__ int tile_prefix[HS_MAX_PATCHES + 1];
    __shared__ int in_off[HS_MAX_BUCKETS + 1];
    __shared__ long long in_base[HS_MAX_BUCKETS];
    __shared__ int st_off[HS_MAX_BUCKETS + 1];
    __shared__ int voff[HS_MAX_BUCKETS + 1];
    __shared__ int in_cnt_s[HS_MAX_BUCKETS];
    __shared__ double step_s[HS_MAX_BUCKETS], r2_s[HS_MAX_BUCKETS];
    __shared__ SplatLayer sl_s[HS_MAX_BUCKETS];
    __shared__ int keep_hist[HS_MAX_BUCKETS];
    __shared__ int drop_hist[HS_MAX_BUCKETS];
    __shared__ double eout_s[HS_MAX_BUCKETS];
    __shared__ unsigned keepw[ADV_WORDS];
    __shared__ int wpre[ADV_WORDS];
    __shared__ unsigned char bk_s[ADV_TILE];
    __shared__ int tile_s, prefix_s, clamp_s, cur_p_s, seg_b_s, seg_end_s;
    __shared__ HsPatch P_s;

    if (threadIdx.x == 0) {
        cur_p_s = -1;
        tile_prefix[0] = 0;
        for (int p = 0; p < a.n_patches; ++p) {
            const HsPatch& P = a.patches[p];
            int cap = P.pool_capacity + (a.stage_count ? P.stage_capacity : 0);
            tile_prefix[p + 1] = tile_prefix[p] + (cap + ADV_TILE - 1) / ADV_TILE;
        }
    }
    __syncthreads();
    const int total_tiles = tile_prefix[a.n_patches];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

    while (true) {
        if (threadIdx.x == 0) tile_s = atomicAdd(a.tile_counter, 1);
        __syncthreads();
        const int tile = tile_s;
        if (tile >= total_tiles) break;
        const int p = find_seg(tile_prefix, a.n_patches + 1, tile);
        const int ltile = tile - tile_prefix[p];
        if (p != cur_p_s && wid == 0) {
            // per-patch tables (warp 0; reused while tiles stay in patch p)
            const HsPatch P = a.patches[p];
            if (lane == 0) P_s = P;
            const int ci = lane < nb ? a.in_count[(size_t)p * nb + lane] : 0;
            const int cs = (lane < nb && a.stage_count) ? a.stage_count[(size_t)p * nb + lane] : 0;
            const int si = warp_incl_scan(ci, lane), ss = warp_incl_scan(cs, lane);
            if (lane < nb) {
                in_off[lane] = si - ci; st_off[lane] = ss - cs; voff[lane] = si - ci + ss - cs; in_cnt_s[lane] = ci;
                in_base[lane] = P.pool_base + si - ci;
                const HsBucket B = a.buckets[lane];
                step_s[lane] = dmul(B.speed, a.dt);                   // speeds * dt
                r2_s[lane] = dmul(B.radius, B.radius);
                if (a.splat) {
                    const HsLayer L = a.layers[P.layer_base + lane];
                    sl_s[lane] = SplatLayer{L.raw_off, 1.0 / (P.texel * (double)L.f), (double)(L.wx - 1),
                                            (double)(L.wy - 1), L.raw_pitch, L.pad};
                }
            }
            if (lane == nb - 1) { in_off[nb] = si; st_off[nb] = ss; voff[nb] = si + ss; }
            if (lane == 0) cur_p_s = p;
        }
        if (threadIdx.x < nb) { keep_hist[threadIdx.x] = 0; drop_hist[threadIdx.x] = 0; eout_s[threadIdx.x] = 0.0; }
        __syncthreads();
        const int N = voff[nb];
        const int tbase = ltile * ADV_TILE;
        if (tbase >= N) {               // empty tile (the patch's later tiles are empty too)
            __syncthreads();
            continue;
        }
        if (threadIdx.x == 0) {
            const int b = find_seg(voff, nb + 1, tbase);
            seg_b_s = b;
            seg_end_s = voff[b + 1];
            clamp_s = 0;
        }
        __syncthreads();
        const HsPatch P = P_s;
        const int seg_b = seg_b_s, seg_end = seg_end_s;

        // ---- phase 1: keep flags (HBM stream) ----
#pragma unroll
        for (int c = 0; c < ADV_CHUNKS; ++c) {
            int keep[ADV_ITEMS];
#pragma unroll
            for (int it = 0; it < ADV_ITEMS; ++it) {
                const int li = c * ADV_CHUNK + it * ADV_THREADS + threadIdx.x;
                const int v = tbase + li;
                keep[it] = 0;
                if (v < N) {
                    const int b = v < seg_end ? seg_b : find_seg(voff, nb + 1, v);
                    bk_s[li] = (unsigned char)b;
                    double x, y, ux, uy;
                    const float* ap;
                    adv_item(a, P, in_base, st_off, voff, in_cnt_s, step_s, v, b, x, y, ux, uy, &ap);
                    const double ox = fmax(fmax(dsub(P.x0, x), dsub(x, P.x1)), 0.0);
                    const double oy = fmax(fmax(dsub(P.y0, y), dsub(y, P.y1)), 0.0);
                    keep[it] = dadd(dmul(ox, ox), dmul(oy, oy)) <= r2_s[b];   // support disk (:315-320)
                }
            }
#pragma unroll
            for (int it = 0; it < ADV_ITEMS; ++it) {
                const unsigned bal = __ballot_sync(0xffffffffu, keep[it]);
                if (lane == 0) keepw[(c * ADV_ITEMS + it) * (ADV_THREADS / 32) + wid] = bal;
            }
        }
        __syncthreads();
        if (wid == 0) {
            // exclusive scan of the tile's ballot-word popcounts (item order)
            constexpr int PER = (ADV_WORDS + 31) / 32;
            int cnt[PER], loc = 0;
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                cnt[q] = lane * PER + q < ADV_WORDS ? __popc(keepw[lane * PER + q]) : 0;
                loc += cnt[q];
            }
            const int inc = warp_incl_scan(loc, lane);
            const int agg = __shfl_sync(0xffffffffu, inc, 31);
            int run = inc - loc;
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                if (lane * PER + q < ADV_WORDS) wpre[lane * PER + q] = run;
                run += cnt[q];
            }
            // decoupled look-back over this patch's earlier tiles, 32 at a time
            unsigned long long* ts = a.tile_state;
            const int first = tile - ltile;
            unsigned long long prefix = 0;
            if (ltile == 0) {
                if (lane == 0) atomicExch(&ts[tile], FLAG_PRE | (unsigned long long)agg);
            } else {
                if (lane == 0) atomicExch(&ts[tile], FLAG_AGG | (unsigned long long)agg);
                int hi = tile - 1;
                while (true) {
                    const int j = hi - lane;
                    unsigned long long sv = FLAG_PRE;     // before the patch: prefix 0
                    if (j >= first) {
                        do { sv = *((volatile unsigned long long*)&ts[j]); } while ((sv >> 32) == 0);
                    }
                    const unsigned pre = __ballot_sync(0xffffffffu, (sv & (3ULL << 32)) == FLAG_PRE);
                    const int stop = pre ? __ffs(pre) - 1 : 31;          // closest full prefix
                    unsigned long long val = lane <= stop ? (sv & 0xffffffffULL) : 0ULL;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                    prefix += val;
                    if (pre) break;
                    hi -= 32;
                }
                if (lane == 0) atomicExch(&ts[tile], FLAG_PRE | (prefix + (unsigned long long)agg));
            }
            if (lane == 0) prefix_s = (int)prefix;
        }
        __syncthreads();
        const int tprefix = prefix_s;

        // ---- phase 2: stable scatter + splat (L2 re-read) ----
        int clamp_local = 0;
        float* raw = a.raw_layers;
#pragma unroll
        for (int c = 0; c < ADV_CHUNKS; ++c) {
#pragma unroll
            for (int it = 0; it < ADV_ITEMS; ++it) {
                const int li = c * ADV_CHUNK + it * ADV_THREADS + threadIdx.x;
                const int v = tbase + li;
                if (v >= N) continue;
                const int w = (c * ADV_ITEMS + it) * (ADV_THREADS / 32) + wid;
                const unsigned bal = keepw[w];
                const bool kept = (bal >> lane) & 1u;
                const int rank = tprefix + wpre[w] + __popc(bal & ((1u << lane) - 1u));
                const int b = bk_s[li];
                double x, y, ux, uy, bt = 0.0;
                const float* ap;
                adv_item(a, P, in_base, st_off, voff, in_cnt_s, step_s, v, b, x, y, ux, uy, &ap, &bt);
                const float am = *ap;
                if (kept) {
                    if (rank < P.pool_capacity) {
                        const long long o = P.pool_base + rank;
                        a.out.x[o] = x; a.out.y[o] = y; a.out.ux[o] = ux; a.out.uy[o] = uy; a.out.amp[o] = am;
                        if (a.out.birth) a.out.birth[o] = bt;
                    } else {
                        atomicOr(a.status, HS_STATUS_POOL_OVERFLOW);
                    }
                    atomicAdd(&keep_hist[b], 1);
                    if (a.splat) splat_at(a.fixed_point, raw, sl_s[b], P.sx0, P.sy0, x, y, am, &clamp_local);
                } else {
                    if (am > 0.f) {
                        // crest despawn energy rho g A^2 pi r^2 / 8 (particles.py:322-327)
                        const double amp = (double)am;
                        const double e = 0.125 * a.rho * a.g * (amp * amp) * 3.141592653589793 * r2_s[b];
                        atomicAdd(&eout_s[b], e);
                    }
                    if (a.dropped.x) {
                        const long long o = P.pool_base + (v - rank);       // stable among the dropped
                        a.dropped.x[o] = x; a.dropped.y[o] = y; a.dropped.ux[o] = ux; a.dropped.uy[o] = uy;
                        a.dropped.amp[o] = am;
                        if (a.dropped.birth) a.dropped.birth[o] = bt;
                        atomicAdd(&drop_hist[b], 1);
                    }
                }
            }
        }
        if (clamp_local) atomicAdd(&clamp_s, clamp_local);
        __syncthreads();
        if (threadIdx.x < nb) {
            const int b = threadIdx.x;
            if (keep_hist[b]) atomicAdd(&a.out_count[(size_t)p * nb + b], keep_hist[b]);
            if (drop_hist[b]) atomicAdd(&a.dropped_count[(size_t)p * nb + b], drop_hist[b]);
            energy_flush(&a.e_out[(size_t)p * nb + b], eout_s[b], a.fixed_point);
        }
        if (threadIdx.x == 0 && clamp_s && a.clamped) atomicAdd(&a.clamped[p], clamp_s);
        __syncthreads();
    }
}

// ------------------------------------------------ two-kernel compaction --
// Count + scatter (used when HsAdvectArgs.keep_words is set): no serial
// look-back chain -- the scatter kernel sums the per-tile survivor counts of
// its patch's earlier tiles directly (a few hundred ints, L2-resident).
struct AdvTables {
    long long in_base[HS_MAX_BUCKETS];
    int slack[HS_MAX_BUCKETS];
    int in_off[HS_MAX_BUCKETS + 1], st_off[HS_MAX_BUCKETS + 1], voff[HS_MAX_BUCKETS + 1];
    int in_cnt[HS_MAX_BUCKETS];
    double step[HS_MAX_BUCKETS], r2[HS_MAX_BUCKETS];
    SplatLayer sl[HS_MAX_BUCKETS];
    HsPatch P;
    int p, ltile, first, seg_b, seg_end;
};

// every thread calls; returns false when the block's tile is empty
__device__ __forceinline__ bool adv_setup(const HsAdvectArgs& a, AdvTables& T, int tile) {
    const int nb = a.nb, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        int pre = 0, p = 0;
        for (; p < a.n_patches; ++p) {
            const HsPatch& Pq = a.patches[p];
            const int cap = Pq.pool_capacity + (a.stage_count ? Pq.stage_capacity : 0);
            const int nt = (cap + ADV_CHUNK - 1) / ADV_CHUNK;
            if (tile < pre + nt) break;
            pre += nt;
        }
        T.p = p;
        T.first = pre;
        T.ltile = tile - pre;
    }
    __syncthreads();
    const int p = T.p;
    if (p >= a.n_patches) return false;
    if (wid == 0) {
        const HsPatch P = a.patches[p];
        if (lane == 0) T.P = P;
        const int ci = lane < nb ? a.in_count[(size_t)p * nb + lane] : 0;
        const int cs = (lane < nb && a.stage_count) ? a.stage_count[(size_t)p * nb + lane] : 0;
        const int si = warp_incl_scan(ci, lane), ss = warp_incl_scan(cs, lane);
        if (lane < nb) {
            T.in_off[lane] = si - ci; T.st_off[lane] = ss - cs; T.voff[lane] = si - ci + ss - cs; T.in_cnt[lane] = ci;
            T.in_base[lane] = a.in_seg_base ? (long long)a.in_seg_base[(size_t)p * nb + lane] : P.pool_base + si - ci;
            T.slack[lane] = a.out_slack_prefix ? a.out_slack_prefix[(size_t)p * nb + lane] : 0;
            const HsBucket B = a.buckets[lane];
            T.step[lane] = dmul(B.speed, a.dt);
            T.r2[lane] = dmul(B.radius, B.radius);
            if (a.splat) {
                const HsLayer L = a.layers[P.layer_base + lane];
                T.sl[lane] = SplatLayer{L.raw_off, 1.0 / (P.texel * (double)L.f), (double)(L.wx - 1),
                                        (double)(L.wy - 1), L.raw_pitch, L.pad};
            }
        }
        if (lane == nb - 1) { T.in_off[nb] = si; T.st_off[nb] = ss; T.voff[nb] = si + ss; }
        __syncwarp();
        if (lane == 0) {
            const int tb = T.ltile * ADV_CHUNK;
            if (tb < T.voff[nb]) {
                const int b = find_seg(T.voff, nb + 1, tb);
                T.seg_b = b;
                T.seg_end = T.voff[b + 1];
            }
        }
    }
    __syncthreads();
    return T.ltile * ADV_CHUNK < T.voff[nb];
}

__global__ void __launch_bounds__(ADV_THREADS) advect_count_kernel(HsAdvectArgs a) {
    __shared__ AdvTables T;
    __shared__ int wsum[ADV_THREADS / 32];
    const int tile = blockIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // the scatter kernel's accumulators, cleared here instead of by memset nodes
    {
        const long long gt = (long long)blockIdx.x * ADV_THREADS + threadIdx.x;
        const long long nthreads = (long long)gridDim.x * ADV_THREADS;
        const long long ncnt = (long long)a.n_patches * a.nb;
        if (gt < ncnt) {
            a.out_count[gt] = 0;
            if (a.dropped.x) a.dropped_count[gt] = 0;
        }
        if (a.splat && !a.raw_is_clear) {
            float* r = a.raw_layers;
            const long long n = a.raw_layers_len;
            const long long head = min(n, (long long)((16 - ((size_t)r & 15)) & 15) / 4);
            if (gt < head) r[gt] = 0.f;
            float4* r4 = reinterpret_cast<float4*>(r + head);
            const long long n4 = (n - head) / 4;
            for (long long k = gt; k < n4; k += nthreads) r4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
            const long long tail = head + n4 * 4;
            if (gt < n - tail) r[tail + gt] = 0.f;
        }
    }
    const bool live = adv_setup(a, T, tile);
    unsigned* words = a.keep_words + (size_t)tile * (ADV_ITEMS * ADV_THREADS / 32);
    if (!live) {
        if (threadIdx.x == 0) a.tile_state[tile] = 0ULL;
        return;
    }
    const int nb = a.nb, N = T.voff[nb], tbase = T.ltile * ADV_CHUNK;
    const HsPatch& P = T.P;
    int mine = 0;
#pragma unroll
    for (int it = 0; it < ADV_ITEMS; ++it) {
        const int v = tbase + it * ADV_THREADS + threadIdx.x;
        int keep = 0;
        if (v < N) {
            const int b = v < T.seg_end ? T.seg_b : find_seg(T.voff, nb + 1, v);
            double x, y, ux, uy;
            const float* ap;
            adv_item(a, P, T.in_base, T.st_off, T.voff, T.in_cnt, T.step, v, b, x, y, ux, uy, &ap);
            const double ox = fmax(fmax(dsub(P.x0, x), dsub(x, P.x1)), 0.0);
            const double oy = fmax(fmax(dsub(P.y0, y), dsub(y, P.y1)), 0.0);
            keep = dadd(dmul(ox, ox), dmul(oy, oy)) <= T.r2[b] && x == x;   // support disk (:315-320); NaN = hole
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) { words[it * (ADV_THREADS / 32) + wid] = bal; mine += __popc(bal); }
    }
    if (lane == 0) wsum[wid] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < ADV_THREADS / 32; ++w) t += wsum[w];
        a.tile_state[tile] = (unsigned long long)t;
    }
}

__global__ void __launch_bounds__(ADV_THREADS) advect_scatter_kernel(HsAdvectArgs a) {
    __shared__ AdvTables T;
    __shared__ int wpre[ADV_ITEMS * ADV_THREADS / 32];
    __shared__ unsigned wbits[ADV_ITEMS * ADV_THREADS / 32];
    __shared__ int red[ADV_THREADS / 32];
    __shared__ int keep_hist[HS_MAX_BUCKETS], drop_hist[HS_MAX_BUCKETS], clamp_s;
    __shared__ double eout_s[HS_MAX_BUCKETS];
    const int tile = blockIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nb = a.nb;
    if (threadIdx.x < nb) { keep_hist[threadIdx.x] = 0; drop_hist[threadIdx.x] = 0; eout_s[threadIdx.x] = 0.0; }
    if (threadIdx.x == 0) clamp_s = 0;
    if (!adv_setup(a, T, tile)) return;
    const int N = T.voff[nb], tbase = T.ltile * ADV_CHUNK, p = T.p;
    const HsPatch& P = T.P;
    // tile prefix: survivors of this patch's earlier tiles
    int acc = 0;
    for (int q = T.first + threadIdx.x; q < tile; q += ADV_THREADS) acc += (int)a.tile_state[q];
    acc = warp_sum(acc);
    if (lane == 0) red[wid] = acc;
    const unsigned* words = a.keep_words + (size_t)tile * (ADV_ITEMS * ADV_THREADS / 32);
    if (wid == 0) {
        const unsigned wv = words[lane];              // 32 = ADV_ITEMS * 8 words, item order
        const int c = __popc(wv);
        wbits[lane] = wv;
        wpre[lane] = warp_incl_scan(c, lane) - c;
    }
    __syncthreads();
    int tprefix = 0;
#pragma unroll
    for (int w = 0; w < ADV_THREADS / 32; ++w) tprefix += red[w];
    int clamp_local = 0;
    float* raw = a.raw_layers;
#pragma unroll
    for (int it = 0; it < ADV_ITEMS; ++it) {
        const int v = tbase + it * ADV_THREADS + threadIdx.x;
        const int w = it * (ADV_THREADS / 32) + wid;
        const unsigned bal = wbits[w];
        const int b = v < N ? (v < T.seg_end ? T.seg_b : find_seg(T.voff, nb + 1, v)) : -1;
        // per-bucket survivor counts, warp-aggregated (a warp's items nearly always share a bucket)
        {
            const int b0 = __shfl_sync(0xffffffffu, b, 0);
            if (__all_sync(0xffffffffu, b == b0 || b < 0)) {
                if (lane == 0 && bal) atomicAdd(&keep_hist[b0], __popc(bal));
            } else if (b >= 0 && ((bal >> lane) & 1u)) {
                atomicAdd(&keep_hist[b], 1);
            }
        }
        if (v >= N) continue;
        const bool kept = (bal >> lane) & 1u;
        const int rank = tprefix + wpre[w] + __popc(bal & ((1u << lane) - 1u));
        double x, y, ux, uy, bt = 0.0;
        const float* ap;
        adv_item(a, P, T.in_base, T.st_off, T.voff, T.in_cnt, T.step, v, b, x, y, ux, uy, &ap, &bt);
        const float am = *ap;
        if (kept) {
            const int slot = rank + T.slack[b];
            if (slot < P.pool_capacity) {
                const long long o = P.pool_base + slot;
                a.out.x[o] = x; a.out.y[o] = y; a.out.ux[o] = ux; a.out.uy[o] = uy; a.out.amp[o] = am;
                if (a.out.birth) a.out.birth[o] = bt;
            } else {
                atomicOr(a.status, HS_STATUS_POOL_OVERFLOW);
            }
            if (a.splat) splat_at(a.fixed_point, raw, T.sl[b], P.sx0, P.sy0, x, y, am, &clamp_local);
        } else if (x == x) {                             // a despawn (NaN marks a resident-pool hole)
            if (am > 0.f) {
                const double amp = (double)am;          // crest despawn energy (particles.py:322-327)
                energy_add(&eout_s[b], 0.125 * a.rho * a.g * (amp * amp) * 3.141592653589793 * T.r2[b], a.fixed_point);
            }
            if (a.dropped.x) {
                const long long o = P.pool_base + (v - rank);
                a.dropped.x[o] = x; a.dropped.y[o] = y; a.dropped.ux[o] = ux; a.dropped.uy[o] = uy;
                a.dropped.amp[o] = am;
                if (a.dropped.birth) a.dropped.birth[o] = bt;
                atomicAdd(&drop_hist[b], 1);
            }
        }
    }
    if (clamp_local) atomicAdd(&clamp_s, clamp_local);
    __syncthreads();
    if (threadIdx.x < nb) {
        const int b = threadIdx.x;
        if (keep_hist[b]) atomicAdd(&a.out_count[(size_t)p * nb + b], keep_hist[b]);
        if (drop_hist[b]) atomicAdd(&a.dropped_count[(size_t)p * nb + b], drop_hist[b]);
        energy_flush(&a.e_out[(size_t)p * nb + b], eout_s[b], a.fixed_point);
    }
    if (threadIdx.x == 0 && clamp_s && a.clamped) atomicAdd(&a.clamped[p], clamp_s);
}

// ======================================================== splat only ==
__global__ void __launch_bounds__(256) splat_kernel(HsSplatArgs a) {
    const int p = blockIdx.y;
    const int nb = a.nb;
    __shared__ int off[HS_MAX_BUCKETS + 1];
    __shared__ int clamp_s;
    if (threadIdx.x == 0) {
        int s = 0;
        for (int b = 0; b < nb; ++b) { off[b] = s; s += a.count[(size_t)p * nb + b]; }
        off[nb] = s;
        clamp_s = 0;
    }
    __syncthreads();
    const HsPatch P = a.patches[p];
    const int N = off[nb];
    int cl = 0;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < N; v += gridDim.x * blockDim.x) {
        const int b = find_seg(off, nb + 1, v);
        const long long src = P.pool_base + v;
        splat_one(a.raw_layers, a.layers[P.layer_base + b], P, a.pool.x[src], a.pool.y[src], a.pool.amp[src], &cl);
    }
    if (cl) atomicAdd(&clamp_s, cl);
    __syncthreads();
    if (threadIdx.x == 0 && clamp_s && a.clamped) atomicAdd(&a.clamped[p], clamp_s);
}

// ====================================================== resident pool ==
// In-place frame path (HsResidentArgs, include/hybridsea_b200.h).  A tile is
// 1024 consecutive slots of ONE (patch, bucket) segment, so every CTA works
// on a single bucket: one step, one support radius, one splat layer, and one
// atomic per counter at the end.
#ifndef HS_RES_THREADS
#define HS_RES_THREADS 256
#endif
constexpr int RES_THREADS = HS_RES_THREADS;
constexpr int RES_ITEMS = 1024 / RES_THREADS;   // a tile is 1024 slots (harness.RES_TILE)
constexpr int RES_TILE = RES_THREADS * RES_ITEMS;

// Slots k = k0 + it * STRIDE + lane_k (it < ITEMS) of the resident tile m =
// (segment, tile in segment, absolute first slot): advect in place, cull to a
// NaN hole, splat; per-warp totals of drops, clamps and despawn energy.
// Slot loads issue before the segment length is known: slots past len (up to
// the tile end, inside the pool arrays) are read and ignored.
template <bool FX, int ITEMS, int STRIDE>
__device__ __forceinline__ void resident_slots(const HsResidentArgs& a, int4 m, int k0, int lane_k) {
    double* __restrict__ px = a.pool.x;
    double* __restrict__ py = a.pool.y;
    const double* __restrict__ pux = a.pool.ux;
    const double* __restrict__ puy = a.pool.uy;
    const float* __restrict__ pam = a.pool.amp;
    const int s = m.x;
    const long long base = (long long)m.z;
    double x[ITEMS], y[ITEMS], ux[ITEMS], uy[ITEMS];
    float am[ITEMS];
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
        const long long o = base + k0 + it * STRIDE + lane_k;
        x[it] = px[o]; y[it] = py[o]; ux[it] = __ldg(pux + o); uy[it] = __ldg(puy + o); am[it] = __ldg(pam + o);
    }
    const int n = min(RES_TILE, a.len_in[s] - m.y * RES_TILE);
    const int p = s / a.nb, b = s - p * a.nb;
    const HsPatch* P = a.patches + p;
    const double x0 = __ldg(&P->x0), y0 = __ldg(&P->y0), x1 = __ldg(&P->x1), y1 = __ldg(&P->y1);
    const double sx0 = __ldg(&P->sx0), sy0 = __ldg(&P->sy0);     // synthesis origin (tracking patches)
    const HsBucket* Bk = a.buckets + b;
    const double step = dmul(__ldg(&Bk->speed), a.dt);            // speeds * dt (particles.py:312)
    const double rad = __ldg(&Bk->radius);
    const double r2 = dmul(rad, rad);
    const HsLayer* L = a.layers + __ldg(&P->layer_base) + b;
    const SplatLayer sl{__ldg(&L->raw_off), 1.0 / (__ldg(&P->texel) * (double)__ldg(&L->f)),
                        (double)(__ldg(&L->wx) - 1), (double)(__ldg(&L->wy) - 1), __ldg(&L->raw_pitch),
                        __ldg(&L->pad)};
    int drops = 0, clamp_local = 0;
    double e = 0.0;
    long long efx = 0;
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
        const int k = k0 + it * STRIDE + lane_k;
        if (k >= n || x[it] != x[it]) continue;                     // beyond len, or a hole
        const long long o = base + k;
        const double nx = dadd(x[it], dmul(ux[it], step));           // pos += dir * (c dt)  (:312-313)
        const double ny = dadd(y[it], dmul(uy[it], step));
        const double ox = fmax(fmax(dsub(x0, nx), dsub(nx, x1)), 0.0);
        const double oy = fmax(fmax(dsub(y0, ny), dsub(ny, y1)), 0.0);
        if (dadd(dmul(ox, ox), dmul(oy, oy)) <= r2) {                // support disk (:315-320)
            px[o] = nx;
            py[o] = ny;
#ifndef HS_EXP_NOSPLAT
            splat_at<FX>(a.raw_layers, sl, sx0, sy0, nx, ny, am[it], &clamp_local);
#endif
        } else {
            px[o] = __longlong_as_double(0x7ff8000000000000LL);       // hole: stable compaction is deferred
            ++drops;
            if (am[it] > 0.f) {                                       // crest despawn energy (:322-327)
                const double amp = (double)am[it];
                const double ep = 0.125 * a.rho * a.g * (amp * amp) * 3.141592653589793 * r2;
                if constexpr (FX) efx += energy_fixed(ep); else e += ep;
            }
        }
    }
    // per-warp totals (drops and despawns are rare: most warps skip the atomics)
    if (__any_sync(0xffffffffu, drops != 0 || clamp_local != 0)) {
        drops = warp_sum(drops);
        clamp_local = warp_sum(clamp_local);
        if constexpr (FX) efx = warp_sum(efx); else e = warp_sum(e);
        if ((threadIdx.x & 31) == 0) {
            if (drops) atomicSub(&a.live[s], drops);
            if constexpr (FX) {
                if (efx) atomicAdd(reinterpret_cast<unsigned long long*>(&a.e_out[s]), (unsigned long long)efx);
            } else if (e != 0.0) {
                atomicAdd(&a.e_out[s], e);
            }
            if (clamp_local && a.clamped) atomicAdd(&a.clamped[p], clamp_local);
        }
    }
}

// Persistent CTAs walk the tile list with stride gridDim.x; a tile-map entry
// is prefetched one tile ahead, so each tile costs one memory round trip.
// Every warp retires its slots independently (no barrier).  (A dynamic
// variant -- atomic tile claims plus a shared-memory splat of small layers --
// measured slower on C3 and C5 once the FFT branch forks after inject.)
#ifndef HS_RES_MINB
#define HS_RES_MINB 3          // 3 CTAs/SM: 80 registers, no inner-loop spills
#endif
template <bool FX>
__global__ void __launch_bounds__(RES_THREADS, HS_RES_MINB) advect_resident_kernel(HsResidentArgs a) {
    const int4* __restrict__ tmap = reinterpret_cast<const int4*>(a.tile_map);
    int t = blockIdx.x;
    int4 m = t < a.max_tiles ? __ldg(tmap + t) : make_int4(-1, 0, 0, 0);
    while (m.x >= 0) {
        const int tn = t + gridDim.x;
        const int4 mn = tn < a.max_tiles ? __ldg(tmap + tn) : make_int4(-1, 0, 0, 0);
        resident_slots<FX, RES_ITEMS, RES_THREADS>(a, m, 0, threadIdx.x);
        t = tn;
        m = mn;
    }
}

// One CTA per patch: advect + cull + splat this frame's injected particles
// (the virtual [new crests b][new troughs b] of particles.py:296-299, advected
// in their birth frame, harness.py:142-152) and append them at the tails of
// their bucket segments; culled ones become holes so slots stay in order.
__global__ void __launch_bounds__(RES_THREADS) append_resident_kernel(HsResidentArgs a) {
    const int p = blockIdx.x, nb = a.nb;
    __shared__ int soff[HS_MAX_BUCKETS + 1];
    __shared__ int kept_s[HS_MAX_BUCKETS];
    __shared__ double eout_s[HS_MAX_BUCKETS];
    __shared__ long long dst_s[HS_MAX_BUCKETS];
    __shared__ int room_s[HS_MAX_BUCKETS];
    __shared__ double step_s[HS_MAX_BUCKETS], r2_s[HS_MAX_BUCKETS];
    __shared__ SplatLayer sl_s[HS_MAX_BUCKETS];
    __shared__ int clamp_s;
    __shared__ HsPatch P_s;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
        const HsPatch P = a.patches[p];
        if (lane == 0) { P_s = P; clamp_s = 0; }
        const int s = p * nb + lane;
        const int c = lane < nb ? a.stage_count[s] : 0;
        const int inc = warp_incl_scan(c, lane);
        if (lane < nb) {
            soff[lane] = inc - c;
            const int len = a.len_in[s];
            a.len_out[s] = len + min(c, a.seg_cap[s] - len);      // clamped on overflow (status bit)
            dst_s[lane] = (long long)a.seg_base[s] + len;
            room_s[lane] = a.seg_cap[s] - len;
            kept_s[lane] = 0;
            eout_s[lane] = 0.0;
            const HsBucket Bk = a.buckets[lane];
            step_s[lane] = dmul(Bk.speed, a.dt);
            r2_s[lane] = dmul(Bk.radius, Bk.radius);
            const HsLayer L = a.layers[P.layer_base + lane];
            sl_s[lane] = SplatLayer{L.raw_off, 1.0 / (P.texel * (double)L.f), (double)(L.wx - 1),
                                    (double)(L.wy - 1), L.raw_pitch, L.pad};
            if (c > a.seg_cap[s] - len) atomicOr(a.status, HS_STATUS_POOL_OVERFLOW);
        }
        if (lane == 31) soff[nb] = inc;
    }
    __syncthreads();
    const int N = soff[nb];
    const HsPatch& P = P_s;
    int clamp_local = 0;
    for (int v = threadIdx.x; v < N; v += RES_THREADS) {
        const int b = find_seg(soff, nb + 1, v);
        const int j = v - soff[b];
        const long long src = P.stage_base + v;
        const double ux = a.stage.ux[src], uy = a.stage.uy[src];
        const float am = a.stage.amp[src];
        const double nx = dadd(a.stage.x[src], dmul(ux, step_s[b]));
        const double ny = dadd(a.stage.y[src], dmul(uy, step_s[b]));
        const double ox = fmax(fmax(dsub(P.x0, nx), dsub(nx, P.x1)), 0.0);
        const double oy = fmax(fmax(dsub(P.y0, ny), dsub(ny, P.y1)), 0.0);
        const bool keep = dadd(dmul(ox, ox), dmul(oy, oy)) <= r2_s[b];
        if (j < room_s[b]) {
            const long long o = dst_s[b] + j;
            a.pool.x[o] = keep ? nx : __longlong_as_double(0x7ff8000000000000LL);
            a.pool.y[o] = ny; a.pool.ux[o] = ux; a.pool.uy[o] = uy; a.pool.amp[o] = am;
            if (a.pool.birth) a.pool.birth[o] = a.stage.birth ? a.stage.birth[src] : 0.0;
        }
        if (keep && j < room_s[b]) {
            atomicAdd(&kept_s[b], 1);
            splat_at(a.fixed_point, a.raw_layers, sl_s[b], P.sx0, P.sy0, nx, ny, am, &clamp_local);
        } else if (am > 0.f) {
            const double amp = (double)am;
            energy_add(&eout_s[b], 0.125 * a.rho * a.g * (amp * amp) * 3.141592653589793 * r2_s[b], a.fixed_point);
        }
    }
    if (clamp_local) atomicAdd(&clamp_s, clamp_local);
    __syncthreads();
    if (threadIdx.x < nb) {
        const int s = p * nb + threadIdx.x;
        if (kept_s[threadIdx.x]) atomicAdd(&a.live[s], kept_s[threadIdx.x]);
        energy_flush(&a.e_out[s], eout_s[threadIdx.x], a.fixed_point);
    }
    if (threadIdx.x == 0 && clamp_s && a.clamped) atomicAdd(&a.clamped[p], clamp_s);
}

// Segment table (HsLayoutArgs).  One CTA: warp w lays out patch w (strided),
// lane b = bucket b; then a block scan of per-patch tile totals places every
// segment's tiles in tile_map.
__global__ void __launch_bounds__(1024) resident_layout_kernel(HsLayoutArgs a) {
    const int nb = a.nb, lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __shared__ int ptiles[HS_MAX_PATCHES];
    __shared__ int pfirst[HS_MAX_PATCHES];
    __shared__ int scan_sm[33];
    for (int p = wid; p < a.n_patches; p += nw) {
        const HsPatch P = a.patches[p];
        const int s = p * nb + lane;
        const int c = (lane < nb && a.count) ? a.count[s] : 0;
        const int inc = warp_incl_scan(c, lane);
        int nt = 0;
        if (lane < nb) {
            const long long base = P.pool_base + (inc - c) + a.slack_prefix[s];
            const int cap = c + a.slack[s];
            if (base + cap > P.pool_base + P.pool_capacity) atomicOr(a.status, HS_STATUS_POOL_OVERFLOW);
            a.seg_base[s] = (int)base;
            a.seg_cap[s] = cap;
            a.len[s] = c;
            a.live[s] = c;
            nt = (cap + RES_TILE - 1) / RES_TILE;
        }
        const int tinc = warp_incl_scan(nt, lane);
        if (lane == 31) ptiles[p] = tinc;
    }
    __syncthreads();
    // exclusive scan of ptiles over patches (<= HS_MAX_PATCHES <= blockDim.x)
    {
        const int v = threadIdx.x < a.n_patches ? ptiles[threadIdx.x] : 0;
        int tot;
        const int ex = block_excl_scan(v, scan_sm, &tot);
        if (threadIdx.x < a.n_patches) pfirst[threadIdx.x] = ex;
        if (threadIdx.x == 0 && tot > a.max_tiles) atomicOr(a.status, HS_STATUS_POOL_OVERFLOW);
    }
    __syncthreads();
    int4* tmap = reinterpret_cast<int4*>(a.tile_map);
    for (int t = threadIdx.x; t < a.max_tiles; t += blockDim.x) tmap[t] = make_int4(-1, 0, 0, 0);
    __syncthreads();
    for (int p = wid; p < a.n_patches; p += nw) {
        const int s = p * nb + lane;
        const int nt = lane < nb ? (a.seg_cap[s] + RES_TILE - 1) / RES_TILE : 0;
        const int first = pfirst[p] + warp_incl_scan(nt, lane) - nt;
        if (lane < nb)
            for (int k = 0; k < nt && first + k < a.max_tiles; ++k)
                tmap[first + k] = make_int4(s, k, a.seg_base[s] + k * RES_TILE, 0);
    }
}

// ============================================================ emission ==
// Kinematic emitting bodies (HsEmitArgs).  Positions follow the reference's
// buoyancy_step update for a constant velocity, position += velocity * dt
// (interaction.py:140), in fp64 without contraction.
__device__ __forceinline__ void source_step(const HsEmitArgs& a, int s, double& px, double& py) {
    const HsSource& S = a.sources[s];
    if (S.body >= 0) {                              // a floating body: hs_bodies moved it
        px = a.bodies[S.body].pos[0];
        py = a.bodies[S.body].pos[1];
        return;
    }
    px = dadd(a.pos_in[2 * s], dmul(S.vx, a.dt));
    py = dadd(a.pos_in[2 * s + 1], dmul(S.vy, a.dt));
}

// This frame's emission plan of source s (emit_from_motion, interaction.py:
// 185-230): kinematic sources carry it precomputed; a body's comes from its
// state after hs_bodies (energy split by |v_z| : |v_h|, signed amplitudes,
// the wake fan turned to -v_h).
struct SrcPlan {
    double e_ring, e_wake, amp_ring, amp_wake, back;
    int n_ring, n_wake;
};

__device__ __forceinline__ SrcPlan source_plan(const HsEmitArgs& a, int s) {
    const HsSource& S = a.sources[s];
    SrcPlan q{S.e_ring, S.e_wake, S.amp_ring, S.amp_wake, 0.0, S.n_ring, S.n_wake};
    if (S.body < 0) return q;
    const HsBody& B = a.bodies[S.body];
    const double d_v = dsub(B.submerged, B.prev_submerged);
    const double budget = dmul(dmul(dmul(dmul(1.0, a.rho), a.g), fabs(d_v)), B.mean_submersion);
    q.e_ring = q.e_wake = 0.0;
    if (!(budget > 0.0)) return q;
    const double v_z = fabs(B.vel[2]), v_h = hypot(B.vel[0], B.vel[1]);
    const double rw = dadd(v_z, v_h) == 0.0 ? 1.0 : __ddiv_rn(v_z, dadd(v_z, v_h));
    const double sign = d_v >= 0.0 ? 1.0 : -1.0;
    const double rgp = dmul(dmul(a.rho, a.g), 3.141592653589793);
    const double er = dmul(rw, budget);
    if (er > 0.0) {
        const double r = a.buckets[S.ring_bucket].radius;
        q.e_ring = er;
        q.amp_ring = dmul(sign, sqrt(__ddiv_rn(dmul(8.0, __ddiv_rn(er, (double)S.n_ring)), dmul(rgp, dmul(r, r)))));
    }
    const double ew = dmul(dsub(1.0, rw), budget);
    if (ew > 0.0 && v_h > 0.0) {
        const double r = a.buckets[S.wake_bucket].radius;
        q.e_wake = ew;
        q.amp_wake = dmul(sign, sqrt(__ddiv_rn(dmul(8.0, __ddiv_rn(ew, (double)S.n_wake)), dmul(rgp, dmul(r, r)))));
        q.back = atan2(-B.vel[1], -B.vel[0]);
    }
    return q;
}

// owning patch: the first whose region contains the point, inclusive
// (Simulation.owning_patch, harness.py:125-129; PatchRegion.contains, particles.py:71-74)
__device__ __forceinline__ int owner_of(const HsEmitArgs& a, double px, double py) {
    for (int p = 0; p < a.n_patches; ++p) {
        const HsPatch& P = a.patches[p];
        if (px >= P.x0 && px <= P.x1 && py >= P.y0 && py <= P.y1) return p;
    }
    return -1;
}

// Frame start (one thread per patch): a tracking patch's region becomes last
// frame's synthesis origin, and its synthesis origin moves to
// _snap(p - l/2, texel) of its source's new position (harness.py:65-66,115-123).
__global__ void track_kernel(HsEmitArgs a) {
    for (int p = threadIdx.x; p < a.n_patches; p += blockDim.x) {
        HsPatch* P = a.patches + p;
        const int s = P->track;
        if (s < 0 || s >= a.n_sources) continue;
        const double x0 = P->sx0, y0 = P->sy0;
        P->x0 = x0;
        P->y0 = y0;
        P->x1 = dadd(x0, P->l1);
        P->y1 = dadd(y0, P->l2);
        double px, py;
        source_step(a, s, px, py);
        P->sx0 = dmul(rint(__ddiv_rn(dsub(px, dmul(P->l1, 0.5)), P->texel)), P->texel);
        P->sy0 = dmul(rint(__ddiv_rn(dsub(py, dmul(P->l2, 0.5)), P->texel)), P->texel);
    }
}

// buoyancy_step (interaction.py:105-149) for every body, one warp each: lane
// p samples the previous frame's blended surface at probe p, lane 0 then
// integrates in the reference's operation order (fp64, no contraction).
__global__ void __launch_bounds__(128) bodies_kernel(HsBodyArgs a) {
    const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (w >= a.n_bodies) return;
    HsBody& B = a.bodies[w];
    const int np = B.n_probes;
    const double c = cos(B.yaw), sn = sin(B.yaw);
    double wx = 0.0, wy = 0.0, wz = 0.0, hgt = 0.0, nx = 0.0, ny = 0.0, nz = 1.0;
    if (lane < np) {
        const double* o = B.probe_off[lane];
        wx = dsub(dadd(B.pos[0], dmul(c, o[0])), dmul(sn, o[1]));     // interaction.py:72-76
        wy = dadd(dadd(B.pos[1], dmul(sn, o[0])), dmul(c, o[1]));
        wz = dadd(B.pos[2], o[2]);
        const bool flat = a.frame ? (*a.frame == 0) : (a.flat != 0);
        if (!flat) {
            float h; float3 n;
            sample_surface_heights(a.bg_height, a.bg_n, a.bg_spacing, a.n_extra_bg, a.extra_bg, a.n_patches,
                                   a.patches, a.patch_height, wx, wy, h, n);
            hgt = (double)h; nx = (double)n.x; ny = (double)n.y; nz = (double)n.z;
        }
    }
    if (lane != 0) {
        // lane 0 gathers every probe below
    }
    double Wx[HS_MAX_PROBES], Wy[HS_MAX_PROBES], D[HS_MAX_PROBES], Nx[HS_MAX_PROBES], Ny[HS_MAX_PROBES], Nz[HS_MAX_PROBES];
#pragma unroll
    for (int q = 0; q < HS_MAX_PROBES; ++q) {
        Wx[q] = __shfl_sync(0xffffffffu, wx, q);
        Wy[q] = __shfl_sync(0xffffffffu, wy, q);
        D[q] = __shfl_sync(0xffffffffu, dsub(hgt, wz), q);            // depth = h - z
        Nx[q] = __shfl_sync(0xffffffffu, nx, q);
        Ny[q] = __shfl_sync(0xffffffffu, ny, q);
        Nz[q] = __shfl_sync(0xffffffffu, nz, q);
    }
    if (lane != 0) return;
    double frac[HS_MAX_PROBES];
    double submerged = 0.0;
    for (int q = 0; q < np; ++q) {
        frac[q] = fmin(fmax(__ddiv_rn(D[q], B.draft), 0.0), 1.0);
        submerged = dadd(submerged, dmul(B.probe_vol[q], frac[q]));
    }
    double F[3] = {0.0, 0.0, 0.0}, torque_z = 0.0;
    const double rg = dmul(a.rho, a.g);
    for (int q = 0; q < np; ++q) {
        const double sc = dmul(dmul(rg, B.probe_vol[q]), frac[q]);   // rho g vol frac (:126)
        const double f0 = dmul(sc, Nx[q]), f1 = dmul(sc, Ny[q]), f2 = dmul(sc, Nz[q]);
        F[0] = dadd(F[0], f0); F[1] = dadd(F[1], f1); F[2] = dadd(F[2], f2);
        const double r0 = dsub(Wx[q], B.pos[0]), r1 = dsub(Wy[q], B.pos[1]);
        torque_z = dadd(torque_z, dsub(dmul(r0, f1), dmul(r1, f0)));
    }
    const double wet = B.displaced > 0.0 ? __ddiv_rn(submerged, B.displaced) : 0.0;
    const double dl = dmul(B.drag_linear, wet);
    for (int k = 0; k < 3; ++k) F[k] = dsub(F[k], dmul(dl, B.vel[k]));
    F[0] = dadd(F[0], dmul(B.thrust_force, cos(B.yaw)));
    F[1] = dadd(F[1], dmul(B.thrust_force, sin(B.yaw)));
    F[2] = dadd(F[2], dmul(B.thrust_force, 0.0));
    torque_z = dadd(torque_z, dsub(B.yaw_torque, dmul(dmul(B.drag_yaw, wet), B.yaw_rate)));
    const double inertia = dmul(dmul(0.5, B.mass), dmul(B.hull_extent, B.hull_extent));
    const double gz[3] = {0.0, 0.0, -a.g};
    for (int k = 0; k < 3; ++k) B.vel[k] = dadd(B.vel[k], dmul(dadd(__ddiv_rn(F[k], B.mass), gz[k]), a.dt));
    for (int k = 0; k < 3; ++k) B.pos[k] = dadd(B.pos[k], dmul(B.vel[k], a.dt));
    B.yaw_rate = dadd(B.yaw_rate, dmul(__ddiv_rn(torque_z, inertia), a.dt));
    B.yaw = dadd(B.yaw, dmul(B.yaw_rate, a.dt));
    B.prev_submerged = B.submerged;
    B.submerged = submerged;
    double ws = 0.0;
    int nw = 0;
    for (int q = 0; q < np; ++q)
        if (D[q] > 0.0) { ws = dadd(ws, fmin(D[q], B.draft)); ++nw; }
    B.mean_submersion = nw ? __ddiv_rn(ws, (double)nw) : 0.0;
}

// One CTA per source: find its owner and where its fans go (after the
// fans of earlier sources with the same owner and bucket, ring before wake,
// interaction.py:218-230), then write crests and troughs
// (interaction.py:203-216) and splat them at the synthesis origin.
__global__ void __launch_bounds__(256) emit_kernel(HsEmitArgs a) {
    const int s = blockIdx.x, nb = a.nb;
    __shared__ int before[HS_MAX_BUCKETS];
    __shared__ int own_s, clamp_s;
    __shared__ double px_s, py_s;
    const int m = a.beta != 0.0 ? 2 : 1;
    if (threadIdx.x < HS_MAX_BUCKETS) before[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        double px, py;
        source_step(a, s, px, py);
        px_s = px; py_s = py;
        own_s = owner_of(a, px, py);
        clamp_s = 0;
    }
    __syncthreads();
    const int own = own_s;
    if (own < 0) return;
    for (int q = threadIdx.x; q < s; q += blockDim.x) {
        double qx, qy;
        source_step(a, q, qx, qy);
        if (owner_of(a, qx, qy) != own) continue;
        const HsSource& Q = a.sources[q];
        const SrcPlan qp = source_plan(a, q);
        if (qp.e_ring > 0.0) atomicAdd(&before[Q.ring_bucket], m * qp.n_ring);
        if (qp.e_wake > 0.0) atomicAdd(&before[Q.wake_bucket], m * qp.n_wake);
    }
    __syncthreads();
    const HsSource S = a.sources[s];
    const SrcPlan pl = source_plan(a, s);
    const HsPatch& P = a.patches[own];
    const double px = px_s, py = py_s;
    int clamp_local = 0;
#pragma unroll 1
    for (int branch = 0; branch < 2; ++branch) {
        const bool ring = branch == 0;
        if ((ring ? pl.e_ring : pl.e_wake) <= 0.0) continue;
        const int b = ring ? S.ring_bucket : S.wake_bucket;
        const int n = ring ? pl.n_ring : pl.n_wake;
        const double amp = ring ? pl.amp_ring : pl.amp_wake;
        const int seg = own * nb + b;
        int off = before[b];
        if (!ring && pl.e_ring > 0.0 && S.ring_bucket == b) off += m * pl.n_ring;
        const long long base = (long long)a.seg_base[seg] + a.len[seg] + off;
        if (a.len[seg] + off + m * n > a.seg_cap[seg]) {
            if (threadIdx.x == 0) atomicOr(a.status, HS_STATUS_POOL_OVERFLOW);
            continue;
        }
        const double r = a.buckets[b].radius;
        const HsLayer L = a.layers[P.layer_base + b];
        const SplatLayer sl{L.raw_off, 1.0 / (P.texel * (double)L.f), (double)(L.wx - 1), (double)(L.wy - 1),
                            L.raw_pitch, L.pad};
        const double* dirs = a.dirs + 2 * (S.dir_off + (ring ? 0 : S.n_ring));
        const float ca = (float)amp, ta = (float)dmul(-a.beta, amp);
        const bool turn = !ring && S.body >= 0;         // a body's wake: back + linspace offset
        for (int k = threadIdx.x; k < n; k += blockDim.x) {
            double ux, uy;
            if (turn) {
                const double ang = dadd(pl.back, dirs[2 * k]);
                ux = cos(ang);
                uy = sin(ang);
            } else {
                ux = dirs[2 * k];
                uy = dirs[2 * k + 1];
            }
            const double cx = dadd(px, dmul(S.hull_extent, ux));      // center + hull * dirs
            const double cy = dadd(py, dmul(S.hull_extent, uy));
            long long o = base + k;
            a.pool.x[o] = cx; a.pool.y[o] = cy; a.pool.ux[o] = ux; a.pool.uy[o] = uy; a.pool.amp[o] = ca;
            if (a.pool.birth) a.pool.birth[o] = 0.0;          // emitted: birth 0 (interaction.py:210-213)
            splat_at(a.fixed_point, a.raw_layers, sl, P.sx0, P.sy0, cx, cy, ca, &clamp_local);
            if (m == 2) {                                              // trailing trough, -beta * amp
                const double tx = dsub(cx, dmul(r, ux)), ty = dsub(cy, dmul(r, uy));
                o += n;
                a.pool.x[o] = tx; a.pool.y[o] = ty; a.pool.ux[o] = ux; a.pool.uy[o] = uy; a.pool.amp[o] = ta;
                if (a.pool.birth) a.pool.birth[o] = 0.0;
                splat_at(a.fixed_point, a.raw_layers, sl, P.sx0, P.sy0, tx, ty, ta, &clamp_local);
            }
        }
    }
    if (clamp_local) atomicAdd(&clamp_s, clamp_local);
    __syncthreads();
    if (threadIdx.x == 0 && clamp_s && a.clamped) atomicAdd(&a.clamped[own], clamp_s);
}

// After every emit CTA: positions, segment lengths, live counts and the
// energy books, sources in order, ring before wake (harness.py:155-167).
__global__ void emit_commit_kernel(HsEmitArgs a) {
    if (threadIdx.x != 0) return;
    const int m = a.beta != 0.0 ? 2 : 1;
    for (int s = 0; s < a.n_sources; ++s) {
        double px, py;
        source_step(a, s, px, py);
        a.pos_out[2 * s] = px;
        a.pos_out[2 * s + 1] = py;
        const int own = owner_of(a, px, py);
        if (own < 0) continue;
        const HsSource& S = a.sources[s];
        const SrcPlan pl = source_plan(a, s);
        for (int branch = 0; branch < 2; ++branch) {
            const double e = branch == 0 ? pl.e_ring : pl.e_wake;
            if (e <= 0.0) continue;
            const int seg = own * a.nb + (branch == 0 ? S.ring_bucket : S.wake_bucket);
            const int cnt = m * (branch == 0 ? pl.n_ring : pl.n_wake);
            if (a.len[seg] + cnt > a.seg_cap[seg]) continue;          // overflow flagged by emit_kernel
            a.len[seg] += cnt;
            atomicAdd(&a.live[seg], cnt);   // advect_resident decrements live concurrently (other stream)
            a.e_in[seg] = dadd(a.e_in[seg], e);
        }
    }
}

}  // namespace hs

using namespace hs;

namespace hs {
// persistent grids: resident CTAs per SM of the advect kernels, once per device
static PerDevice<int> adv_occ_d{}, res_occ_d{};
int particles_configure() {
    int& a = adv_occ_d.get();
    if (a == 0) {
        HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, advect_kernel<1>, ADV_THREADS, 0));
        if (a < 1) a = 1;
    }
    int& r = res_occ_d.get();
    if (r == 0) {
        HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, advect_resident_kernel<false>, RES_THREADS, 0));
        if (r < 1) r = 1;
    }
    return 0;
}
}  // namespace hs

extern "C" int hs_inject(const HsInjectArgs* a, void* stream) {
    HS_EXP_SKIP_POINT("inject");
    HS_CHECK_ARG(a != nullptr, "hs_inject: null args");
    HS_CHECK_ARG(a->nb >= 1 && a->nb <= HS_MAX_BUCKETS, "hs_inject: nb=%d out of range", a->nb);
    HS_CHECK_ARG(a->n_theta >= 1, "hs_inject: n_theta must be >= 1");
    HS_CHECK_ARG(a->n_patches >= 0 && a->n_patches <= HS_MAX_PATCHES, "hs_inject: n_patches out of range");
    if (a->n_patches == 0) return 0;
    HS_CHECK_ARG(a->buckets && a->patches && a->half_rate && a->acc && a->groups && a->e_in && a->rng &&
                 a->stage_count && a->scratch && a->status && a->stage.x && a->stage.amp,
                 "hs_inject: missing buffer");
    if (a->append)
        HS_CHECK_ARG(a->res.pool.x && a->res.pool.amp && a->res.seg_base && a->res.seg_cap && a->res.len_in &&
                     a->res.len_out && a->res.live && a->res.e_out && a->res.raw_layers && a->res.layers,
                     "hs_inject: append needs the resident pool");
    inject_kernel<<<a->n_patches, 512, 0, as_stream(stream)>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}

extern "C" int hs_advect(const HsAdvectArgs* a, void* stream) {
    HS_CHECK_ARG(a != nullptr, "hs_advect: null args");
    HS_CHECK_ARG(a->nb >= 1 && a->nb <= HS_MAX_BUCKETS, "hs_advect: nb=%d out of range", a->nb);
    HS_CHECK_ARG(a->n_patches >= 0 && a->n_patches <= HS_MAX_PATCHES, "hs_advect: n_patches out of range");
    HS_CHECK_ARG(a->dt >= 0.0, "hs_advect: dt must be nonnegative");
    if (a->n_patches == 0) return 0;
    HS_CHECK_ARG(a->buckets && a->patches && a->in_count && a->out_count && a->e_out && a->tile_state &&
                 a->tile_counter && a->status, "hs_advect: missing buffer");
    HS_CHECK_ARG(!a->splat || (a->raw_layers && a->layers), "hs_advect: splat needs layers");
    cudaStream_t st = as_stream(stream);
    if (a->dropped.x)
        HS_CHECK_ARG(a->dropped_count && a->dropped.y && a->dropped.ux && a->dropped.uy && a->dropped.amp,
                     "hs_advect: incomplete dropped pool");
    if (a->keep_words) {
        // count kernel: clears out/dropped counts and the raw layers, writes every tile's
        // state; scatter kernel: tiles of every patch, 1024 items each (empty tiles exit at once)
        HS_CHECK_ARG((long long)a->max_tiles * ADV_THREADS >= (long long)a->n_patches * a->nb,
                     "hs_advect: max_tiles too small");
        advect_count_kernel<<<a->max_tiles, ADV_THREADS, 0, st>>>(*a);
        HS_LAUNCH_CHECK();
        advect_scatter_kernel<<<a->max_tiles, ADV_THREADS, 0, st>>>(*a);
        HS_LAUNCH_CHECK();
        return 0;
    }
    HS_CUDA(cudaMemsetAsync(a->out_count, 0, sizeof(int) * (size_t)a->n_patches * a->nb, st));
    if (a->dropped.x) HS_CUDA(cudaMemsetAsync(a->dropped_count, 0, sizeof(int) * (size_t)a->n_patches * a->nb, st));
    HS_CUDA(cudaMemsetAsync(a->tile_state, 0, sizeof(unsigned long long) * (size_t)a->max_tiles, st));
    HS_CUDA(cudaMemsetAsync(a->tile_counter, 0, sizeof(int), st));
    if (a->splat) HS_CUDA(cudaMemsetAsync(a->raw_layers, 0, sizeof(float) * (size_t)a->raw_layers_len, st));
    if (int rc = particles_configure()) return rc;
    const int occ = adv_occ_d.get();
    advect_kernel<1><<<num_sms() * occ, ADV_THREADS, 0, st>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}

extern "C" int hs_splat(const HsSplatArgs* a, void* stream) {
    HS_CHECK_ARG(a != nullptr, "hs_splat: null args");
    HS_CHECK_ARG(a->nb >= 1 && a->nb <= HS_MAX_BUCKETS, "hs_splat: nb out of range");
    if (a->n_patches == 0) return 0;
    cudaStream_t st = as_stream(stream);
    HS_CUDA(cudaMemsetAsync(a->raw_layers, 0, sizeof(float) * (size_t)a->raw_layers_len, st));
    int bx = (a->max_count + 255) / 256;
    if (bx < 1) bx = 1;
    if (bx > 4096) bx = 4096;
    dim3 grid(bx, a->n_patches);
    splat_kernel<<<grid, 256, 0, st>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}

static int check_resident(const HsResidentArgs* a, const char* who) {
    HS_CHECK_ARG(a != nullptr, "%s: null args", who);
    HS_CHECK_ARG(a->nb >= 1 && a->nb <= HS_MAX_BUCKETS, "%s: nb=%d out of range", who, a->nb);
    HS_CHECK_ARG(a->n_patches >= 0 && a->n_patches <= HS_MAX_PATCHES, "%s: n_patches out of range", who);
    HS_CHECK_ARG(a->dt >= 0.0, "%s: dt must be nonnegative", who);
    HS_CHECK_ARG(a->buckets && a->patches && a->pool.x && a->pool.y && a->pool.ux && a->pool.uy && a->pool.amp &&
                 a->seg_base && a->seg_cap && a->len_in && a->live && a->e_out && a->raw_layers && a->layers &&
                 a->status, "%s: missing buffer", who);
    return 0;
}

extern "C" int hs_advect_resident(const HsResidentArgs* a, void* stream) {
    HS_EXP_SKIP_POINT("advect");
    if (int rc = check_resident(a, "hs_advect_resident")) return rc;
    if (a->n_patches == 0) return 0;
    HS_CHECK_ARG(a->tile_map && a->max_tiles > 0, "hs_advect_resident: missing tile map");
    HS_CHECK_ARG(((size_t)a->tile_map & 15) == 0, "hs_advect_resident: tile_map must be 16-byte aligned");
    if (int rc = particles_configure()) return rc;
    const int occ = res_occ_d.get();
    const int grid = min(a->max_tiles, num_sms() * occ);
    cudaStream_t st = as_stream(stream);
    if (a->fixed_point) advect_resident_kernel<true><<<grid, RES_THREADS, 0, st>>>(*a);
    else advect_resident_kernel<false><<<grid, RES_THREADS, 0, st>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}

extern "C" int hs_append_resident(const HsResidentArgs* a, void* stream) {
    if (int rc = check_resident(a, "hs_append_resident")) return rc;
    if (a->n_patches == 0) return 0;
    HS_CHECK_ARG(a->stage.x && a->stage.amp && a->stage_count && a->len_out, "hs_append_resident: missing stage");
    append_resident_kernel<<<a->n_patches, RES_THREADS, 0, as_stream(stream)>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}

extern "C" int hs_resident_layout(const HsLayoutArgs* a, void* stream) {
    HS_CHECK_ARG(a != nullptr, "hs_resident_layout: null args");
    HS_CHECK_ARG(a->nb >= 1 && a->nb <= HS_MAX_BUCKETS, "hs_resident_layout: nb out of range");
    HS_CHECK_ARG(a->n_patches >= 0 && a->n_patches <= HS_MAX_PATCHES, "hs_resident_layout: n_patches out of range");
    if (a->n_patches == 0) return 0;
    HS_CHECK_ARG(a->patches && a->slack && a->slack_prefix && a->seg_base && a->seg_cap && a->len && a->live &&
                 a->tile_map && a->status && a->max_tiles > 0, "hs_resident_layout: missing buffer");
    resident_layout_kernel<<<1, 1024, 0, as_stream(stream)>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}

static int check_emit(const HsEmitArgs* a, const char* who) {
    HS_CHECK_ARG(a != nullptr, "%s: null args", who);
    HS_CHECK_ARG(a->n_sources >= 0 && a->n_sources <= HS_MAX_SOURCES, "%s: n_sources out of range", who);
    HS_CHECK_ARG(a->n_patches >= 0 && a->n_patches <= HS_MAX_PATCHES, "%s: n_patches out of range", who);
    HS_CHECK_ARG(a->nb >= 1 && a->nb <= HS_MAX_BUCKETS, "%s: nb out of range", who);
    HS_CHECK_ARG(a->dt > 0.0, "%s: dt must be positive", who);
    HS_CHECK_ARG(a->n_sources == 0 || (a->sources && a->pos_in && a->pos_out), "%s: missing source buffers", who);
    HS_CHECK_ARG(a->n_patches == 0 || a->patches, "%s: missing patches", who);
    return 0;
}

extern "C" int hs_track(const HsEmitArgs* a, void* stream) {
    if (int rc = check_emit(a, "hs_track")) return rc;
    if (a->n_patches == 0 || a->n_sources == 0) return 0;
    track_kernel<<<1, 256, 0, as_stream(stream)>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}

extern "C" int hs_emit(const HsEmitArgs* a, void* stream) {
    if (int rc = check_emit(a, "hs_emit")) return rc;
    if (a->n_sources == 0 || a->n_patches == 0) return 0;
    HS_CHECK_ARG(a->dirs && a->buckets && a->pool.x && a->pool.amp && a->seg_base && a->seg_cap && a->len &&
                 a->live && a->e_in && a->raw_layers && a->layers && a->status, "hs_emit: missing buffer");
    cudaStream_t st = as_stream(stream);
    emit_kernel<<<a->n_sources, 256, 0, st>>>(*a);
    HS_LAUNCH_CHECK();
    emit_commit_kernel<<<1, 32, 0, st>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}

extern "C" int hs_bodies(const HsBodyArgs* a, void* stream) {
    HS_CHECK_ARG(a != nullptr, "hs_bodies: null args");
    if (a->n_bodies == 0) return 0;
    HS_CHECK_ARG(a->bodies && a->dt > 0.0, "hs_bodies: missing bodies or dt <= 0");
    HS_CHECK_ARG(a->n_extra_bg >= 0 && a->n_extra_bg < HS_MAX_CASCADES, "hs_bodies: n_extra_bg out of range");
    HS_CHECK_ARG(a->flat || a->n_patches == 0 || (a->patches && a->patch_height), "hs_bodies: missing patch surfaces");
    bodies_kernel<<<(a->n_bodies + 3) / 4, 128, 0, as_stream(stream)>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}
