// Patch synthesis and blending kernels.
//
//   hs_smooth    separable raised-cosine smoothing of every (patch, bucket)
//                layer, raw padded layer -> cropped smoothed layer
//                (reference patch_synthesis.py:105-130, 206-209, 311-312)
//   hs_compose   gain-sum of bilinearly upsampled layers (:261-274, 301-313)
//                + clamped-border normals (finish_field :323-340)
//                + smoothstep blend with the periodic background at the patch
//                nodes (coupling.py:37-40, 120-141; fft_background.py:222-249)
//                in ONE pass over the patch grid (heights staged in shared
//                memory with a 1-texel halo for the finite differences)
//   hs_sample    SurfaceSampler.sample at arbitrary points (coupling.py:143-161)
//   hs_composite Simulation.stitched_heights (harness.py:219-241)
//   hs_finish    finish_field on a standalone grid
#include "synth_common.cuh"

namespace hs {

// =============================================================== smooth ==
constexpr int SM_TILE = 32;             // wide-kernel tiles
constexpr int SM_TX = 32;               // fused tile: rows (x, axis 0)
constexpr int SM_TY = 64;               // fused tile: columns (y, axis 1) -- wider tiles: less halo
                                        // recomputed in the x pass, less staging per output

constexpr int SM_RB = 8;                 // outputs per thread along the convolution axis

// x pass of one tile, register-blocked: thread item = (column c, block of 8
// output rows); the K taps live in registers and each input value is loaded
// once and feeds up to 8 accumulators.
#ifdef HS_SMOOTH_TRACE
__device__ unsigned long long g_strace[4096 * 4];
__device__ __forceinline__ unsigned long long sgtime() {
    unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}
#define STRACE(k) do { if (threadIdx.x == 0 && blockIdx.x < 4096) g_strace[blockIdx.x * 4 + (k)] = sgtime(); } while (0)
#else
#define STRACE(k) do {} while (0)
#endif

template <int H>
__device__ __forceinline__ void smooth_tile_unrolled(const HsSmoothArgs& a, const HsLayer& L, int cx0, int cy0,
                                                     float* __restrict__ smem) {
    constexpr int K = 2 * H + 1;
    constexpr int W = SM_TY + 2 * H;           // staged columns (y halo)
    constexpr int MS = W | 1;                  // odd row stride: conflict-free column walks
    constexpr int NV = (W + 1 + 3) >> 2;       // float4s per staged row
    constexpr int IS = 4 * NV;                 // staged row stride (floats)
    constexpr int ROWS = SM_TX + 2 * H;
    float* const in0 = smem;                   // ROWS x IS
    float* const mid = in0 + ROWS * IS;        // SM_TX x MS
    float* const ot = in0;                     // the y pass's output reuses the staging rows
    // the halo's first column ry0 = cy0 + pad - H = cy0 + 1 (pad = H + 1); loading
    // from cy0 instead makes every staged row 16-byte aligned in global memory
    // (raw_off and raw_pitch are multiples of 4 floats), so rows move as float4s
    {
        const float* raw = a.raw_layers + L.raw_off;
        const int rx0 = cx0 + L.pad - H;
        for (int e = threadIdx.x; e < ROWS * NV; e += blockDim.x) {
            const int r = e / NV, c4 = e - r * NV;
            const int gx = rx0 + r, gy = cy0 + 4 * c4;
            // columns in [wy, raw_pitch) are zero; beyond the pitch is the next row
            const bool ok = gx >= 0 && gx < L.wx && gy < L.raw_pitch;
            cp_async16z(in0 + r * IS + 4 * c4, ok ? raw + (long long)gx * L.raw_pitch + gy : raw, ok);
        }
    }
    float t[K];
#pragma unroll
    for (int m = 0; m < K; ++m) t[m] = __ldg(a.taps + L.taps_off + m);
    cp_async_wait_all();
    __syncthreads();
    STRACE(1);
    const float* in = in0 + 1;                 // staged column 1 = halo column 0
    // x pass (axis 0): mid[r][c] = sum_m t[m] in[r + m][c]; thread item =
    // (column c, block of 8 output rows): each input value is loaded once and
    // feeds up to 8 accumulators
    for (int item = threadIdx.x; item < W * (SM_TX / SM_RB); item += blockDim.x) {
        const int c = item % W, rb = item / W;
        float acc[SM_RB];
#pragma unroll
        for (int k = 0; k < SM_RB; ++k) acc[k] = 0.f;
        const float* col = in + (rb * SM_RB) * IS + c;
#pragma unroll
        for (int u = 0; u < SM_RB + 2 * H; ++u) {
            const float v = col[u * IS];
#pragma unroll
            for (int k = 0; k < SM_RB; ++k) {
                const int m = u - k;
                if (m >= 0 && m < K) acc[k] = fmaf(t[m], v, acc[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < SM_RB; ++k) mid[(rb * SM_RB + k) * MS + c] = acc[k];
    }
    __syncthreads();
    // y pass (axis 1): thread item = (row r, block of 8 output columns)
    for (int item = threadIdx.x; item < SM_TX * (SM_TY / SM_RB); item += blockDim.x) {
        const int r = item % SM_TX, cb = item / SM_TX;
        float acc[SM_RB];
#pragma unroll
        for (int k = 0; k < SM_RB; ++k) acc[k] = 0.f;
        const float* row = mid + r * MS + cb * SM_RB;
#pragma unroll
        for (int u = 0; u < SM_RB + 2 * H; ++u) {
            const float v = row[u];
#pragma unroll
            for (int k = 0; k < SM_RB; ++k) {
                const int m = u - k;
                if (m >= 0 && m < K) acc[k] = fmaf(t[m], v, acc[k]);
            }
        }
        // through shared memory (row stride SM_TY + 4: 16-byte rows) so the global
        // stores below are whole coalesced row segments
#pragma unroll
        for (int k = 0; k < SM_RB; ++k) ot[r * (SM_TY + 4) + cb * SM_RB + k] = acc[k];
    }
    __syncthreads();
    float* out = a.smooth_layers + L.sm_off + (long long)cx0 * L.ncy + cy0;
    const int rv = min(SM_TX, L.ncx - cx0), cv = min(SM_TY, L.ncy - cy0);
    if ((((uintptr_t)out | (uintptr_t)L.ncy * 4u) & 15u) == 0 && cv == SM_TY) {
        // float4 rows (the full-size layers: 16-byte aligned crop rows)
        for (int e = threadIdx.x; e < SM_TX * (SM_TY / 4); e += blockDim.x) {
            const int r = e / (SM_TY / 4), c4 = e - r * (SM_TY / 4);
            if (r < rv)
                *reinterpret_cast<float4*>(out + (long long)r * L.ncy + 4 * c4) =
                    *reinterpret_cast<const float4*>(ot + r * (SM_TY + 4) + 4 * c4);
        }
    } else {
        for (int e = threadIdx.x; e < SM_TX * SM_TY; e += blockDim.x) {
            const int r = e / SM_TY, c = e - r * SM_TY;
            if (r < rv && c < cv) out[(long long)r * L.ncy + c] = ot[r * (SM_TY + 4) + c];
        }
    }
}

// the unrolled form for half widths up to HS_SMOOTH_UNROLL_MAX; wider
// kernels take the runtime-H loop.  Each instantiation adds to the kernel's
// instruction footprint, and in the frame (smooth beside the FFT) that costs
// more than the unrolling saves on the few wide tiles: frame time C3 96.9 ->
// 95.6 us, PR1 55.3 -> 51.9, C4 241 -> 240 going from 24 to 8 (alone, the C3
// smooth is 21.5 -> 26.8 us); 6 takes PR1 to 51.2 with C3 unchanged, 5 or 4
// send C3's H = 6 full-resolution layer to the loop (101 us).
#ifndef HS_SMOOTH_UNROLL_MAX
#define HS_SMOOTH_UNROLL_MAX 6
#endif
template <int H>
__device__ __forceinline__ bool smooth_try_unrolled(const HsSmoothArgs& a, const HsLayer& L, int cx0, int cy0,
                                                    float* __restrict__ smem) {
    if constexpr (H <= HS_SMOOTH_UNROLL_MAX) {
        smooth_tile_unrolled<H>(a, L, cx0, cy0, smem);
        return true;
    } else {
        return false;
    }
}

__device__ __forceinline__ void smooth_tile_generic(const float* __restrict__ in, int IS, float* __restrict__ mid,
                                                    const float* __restrict__ taps, int H, int W, int MS,
                                                    float* __restrict__ out, long long out_base, int ncy,
                                                    int rows_valid, int cols_valid) {
    const int K = 2 * H + 1;
    for (int e = threadIdx.x; e < SM_TX * W; e += blockDim.x) {
        const int r = e / W, c = e - r * W;
        const float* col = in + r * IS + c;
        float s = 0.f;
        for (int m = 0; m < K; ++m) s = fmaf(taps[m], col[m * IS], s);
        mid[r * MS + c] = s;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < SM_TX * SM_TY; e += blockDim.x) {
        const int r = e / SM_TY, c = e - r * SM_TY;
        if (r >= rows_valid || c >= cols_valid) continue;
        const float* row = mid + r * MS + c;
        float s = 0.f;
        for (int m = 0; m < K; ++m) s = fmaf(taps[m], row[m], s);
        out[out_base + (long long)r * ncy + c] = s;
    }
}


// Layer groups (HsLayer.group): every member smooths into its own crop in
// its own CTA; the CTA that finishes a group's tile last (ticket) folds the
// members' tiles, in member order, into the first layer's crop as
// sum_m gain_m smooth_m -- so the compose upsamples the group once
// (bilinear upsampling is linear, patch_synthesis.py:261-274, 301-313), the
// members still run in parallel, and the sum is order-fixed (deterministic).
__device__ __forceinline__ void group_sum_tile(const HsSmoothArgs& a, int l, const HsLayer& L, int cx0, int cy0) {
    __shared__ int s_last;
    const int lead = L.group > 1 ? l : l + L.group;
    const int n = a.layers[lead].group;
    __threadfence();                           // this CTA's crop stores, device-visible
    __syncthreads();
    if (threadIdx.x == 0) {
        const int tix = L.ticket + (cx0 / SM_TX) * ((L.ncy + SM_TY - 1) / SM_TY) + cy0 / SM_TY;
        const int prev = atomicAdd(&a.tickets[tix], 1);
        s_last = prev == n - 1;
        if (s_last) a.tickets[tix] = 0;        // re-armed for the next frame / graph replay
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int rv = min(SM_TX, L.ncx - cx0), cv = min(SM_TY, L.ncy - cy0);
    for (int e = threadIdx.x; e < rv * cv; e += blockDim.x) {
        const int r = e / cv, c = e - r * cv;
        const long long o = (long long)(cx0 + r) * L.ncy + cy0 + c;
        // eight members' values in flight at once, summed in member order
        float s = 0.f;
        for (int m0 = 0; m0 < n; m0 += 8) {
            float v[8];
#pragma unroll
            for (int m = 0; m < 8; ++m)
                if (m0 + m < n) v[m] = __ldcg(a.smooth_layers + a.layers[lead + m0 + m].sm_off + o);
#pragma unroll
            for (int m = 0; m < 8; ++m)
                if (m0 + m < n) s = fmaf(a.layers[lead + m0 + m].gain, v[m], s);
        }
        a.smooth_layers[a.layers[lead].sm_off + o] = s;
    }
}

#ifndef HS_SMOOTH_MINB
#define HS_SMOOTH_MINB 5          // 48 registers, no spills: 5 CTAs per SM (C3 frame -0.8 us vs 4)
#endif
__global__ void __launch_bounds__(256, HS_SMOOTH_MINB) smooth_kernel(HsSmoothArgs a) {
    extern __shared__ __align__(16) float smem[];
    STRACE(0);
    const int* ti = a.tile_info + 3 * blockIdx.x;
    const int l = ti[0];
    const HsLayer L = a.layers[l];
    const int cx0 = ti[1], cy0 = ti[2];
    const int H = L.H;
    bool done = false;
    switch (H) {
#define HS_SM_CASE(h) case h: done = smooth_try_unrolled<h>(a, L, cx0, cy0, smem); break;
        HS_SM_CASE(1) HS_SM_CASE(2) HS_SM_CASE(3) HS_SM_CASE(4) HS_SM_CASE(5) HS_SM_CASE(6) HS_SM_CASE(7)
        HS_SM_CASE(8) HS_SM_CASE(9) HS_SM_CASE(10) HS_SM_CASE(11) HS_SM_CASE(12) HS_SM_CASE(13)
        HS_SM_CASE(14) HS_SM_CASE(15) HS_SM_CASE(16) HS_SM_CASE(17) HS_SM_CASE(18) HS_SM_CASE(19)
        HS_SM_CASE(20) HS_SM_CASE(21) HS_SM_CASE(22) HS_SM_CASE(23) HS_SM_CASE(24)
#undef HS_SM_CASE
        default: break;
    }
    if (!done) {
        {
            const int K = 2 * H + 1, W = SM_TY + 2 * H;
            const int MS = W | 1;
            const int NV = (W + 1 + 3) >> 2;
            const int IS = 4 * NV;
            float* taps = smem;                        // K (padded to 4)
            float* in = taps + ((K + 3) & ~3);         // (SM_TX + 2H) x IS
            float* mid = in + (SM_TX + 2 * H) * IS;    // SM_TX x MS
            for (int m = threadIdx.x; m < K; m += blockDim.x) taps[m] = a.taps[L.taps_off + m];
            const float* raw = a.raw_layers + L.raw_off;
            const int rx0 = cx0 + L.pad - H;
            for (int e = threadIdx.x; e < (SM_TX + 2 * H) * NV; e += blockDim.x) {
                const int r = e / NV, c4 = e - r * NV;
                const int gx = rx0 + r, gy = cy0 + 4 * c4;
                const bool ok = gx >= 0 && gx < L.wx && gy < L.raw_pitch;
                cp_async16z(in + r * IS + 4 * c4, ok ? raw + (long long)gx * L.raw_pitch + gy : raw, ok);
            }
            cp_async_wait_all();
            __syncthreads();
            STRACE(1);
            const long long ob = (long long)cx0 * L.ncy + cy0;
            const int rv = min(SM_TX, L.ncx - cx0), cv = min(SM_TY, L.ncy - cy0);
            smooth_tile_generic(in + 1, IS, mid, taps, H, W, MS, a.smooth_layers + L.sm_off, ob, L.ncy, rv, cv);
        }
    }
    if (L.group > 1 || L.group < 0) group_sum_tile(a, l, L, cx0, cy0);
    STRACE(2);
}

// Wide kernels (H > HS_SMOOTH_FUSED_MAX_H): two 1-D passes through `mid`.
// x pass: mid[r][c] = sum_m taps[m] raw[r + pad - H + m][c], r in crop rows,
// c over the full padded width; y pass: out[r][c] = sum_m taps[m] mid[r][c + pad - H + m].
__global__ void __launch_bounds__(256) smooth_wide_x_kernel(HsSmoothArgs a) {
    extern __shared__ float smem[];
    const int tile = blockIdx.x;
    const int l = find_seg_i(a.xtile_prefix, a.n_layers + 1, tile);
    const HsLayer L = a.layers[l];
    const int local = tile - a.xtile_prefix[l];
    const int tiles_c = (L.wy + SM_TILE - 1) / SM_TILE;
    const int r0 = (local / tiles_c) * SM_TILE, c0 = (local % tiles_c) * SM_TILE;
    const int H = L.H, K = 2 * H + 1, R = SM_TILE + 2 * H;
    float* taps = smem;
    float* in = taps + ((K + 3) & ~3);          // R x 32
    for (int m = threadIdx.x; m < K; m += blockDim.x) taps[m] = a.taps[L.taps_off + m];
    const float* raw = a.raw_layers + L.raw_off;
    for (int e = threadIdx.x; e < R * SM_TILE; e += blockDim.x) {
        int r = e / SM_TILE, c = e - r * SM_TILE;
        int gx = r0 + L.pad - H + r, gy = c0 + c;
        const bool ok = gx >= 0 && gx < L.wx && gy < L.wy;
        cp_async4(in + e, ok ? raw + (long long)gx * L.raw_pitch + gy : raw, ok);
    }
    cp_async_wait_all();
    __syncthreads();
    float* mid = a.mid + L.mid_off;
    for (int e = threadIdx.x; e < SM_TILE * SM_TILE; e += blockDim.x) {
        int r = e / SM_TILE, c = e - r * SM_TILE;
        if (r0 + r >= L.ncx || c0 + c >= L.wy) continue;
        float s = 0.f;
        for (int m = 0; m < K; ++m) s = fmaf(taps[m], in[(r + m) * SM_TILE + c], s);
        mid[(long long)(r0 + r) * L.wy + c0 + c] = s;
    }
}

__global__ void __launch_bounds__(256) smooth_wide_y_kernel(HsSmoothArgs a) {
    extern __shared__ float smem[];
    const int tile = blockIdx.x;
    const int l = find_seg_i(a.ytile_prefix, a.n_layers + 1, tile);
    const HsLayer L = a.layers[l];
    const int local = tile - a.ytile_prefix[l];
    const int tiles_c = (L.ncy + SM_TILE - 1) / SM_TILE;
    const int r0 = (local / tiles_c) * SM_TILE, c0 = (local % tiles_c) * SM_TILE;
    const int H = L.H, K = 2 * H + 1, C = SM_TILE + 2 * H;
    float* taps = smem;
    float* in = taps + ((K + 3) & ~3);          // 32 x C
    for (int m = threadIdx.x; m < K; m += blockDim.x) taps[m] = a.taps[L.taps_off + m];
    const float* mid = a.mid + L.mid_off;
    for (int e = threadIdx.x; e < SM_TILE * C; e += blockDim.x) {
        int r = e / C, c = e - r * C;
        int gx = r0 + r, gy = c0 + L.pad - H + c;
        const bool ok = gx < L.ncx && gy >= 0 && gy < L.wy;
        cp_async4(in + e, ok ? mid + (long long)gx * L.wy + gy : mid, ok);
    }
    cp_async_wait_all();
    __syncthreads();
    float* out = a.smooth_layers + L.sm_off;
    for (int e = threadIdx.x; e < SM_TILE * SM_TILE; e += blockDim.x) {
        int r = e / SM_TILE, c = e - r * SM_TILE;
        if (r0 + r >= L.ncx || c0 + c >= L.ncy) continue;
        float s = 0.f;
        const float* row = in + r * C + c;
        for (int m = 0; m < K; ++m) s = fmaf(taps[m], row[m], s);
        out[(long long)(r0 + r) * L.ncy + c0 + c] = s;
    }
}

// =============================================================== sample ==
// sample_clamped (coupling.py:63-82): bilinear on the node grid, clamped at borders
__device__ __forceinline__ void sample_clamped_at(const HsPatch& P, const float* __restrict__ ph,
                                                  const float* __restrict__ pn, double x, double y,
                                                  float& hp, float3& q) {
    const double u = fmin(fmax((x - P.x0) / P.texel, 0.0), (double)(P.res - 1));
    const double v = fmin(fmax((y - P.y0) / P.texel, 0.0), (double)(P.ny - 1));
    const int i = min((int)u, P.res - 2), j = min((int)v, P.ny - 2);
    const float fu = (float)(u - i), fv = (float)(v - j);
    const float w00 = (1.f - fu) * (1.f - fv), w10 = fu * (1.f - fv), w01 = (1.f - fu) * fv, w11 = fu * fv;
    const long long b = P.grid_base;
    const long long a00 = b + (long long)i * P.ny + j, a10 = a00 + P.ny, a01 = a00 + 1, a11 = a10 + 1;
    hp = ph[a00] * w00 + ph[a10] * w10 + ph[a01] * w01 + ph[a11] * w11;
    if (pn) {
        float qx = pn[3 * a00] * w00 + pn[3 * a10] * w10 + pn[3 * a01] * w01 + pn[3 * a11] * w11;
        float qy = pn[3 * a00 + 1] * w00 + pn[3 * a10 + 1] * w10 + pn[3 * a01 + 1] * w01 + pn[3 * a11 + 1] * w11;
        float qz = pn[3 * a00 + 2] * w00 + pn[3 * a10 + 2] * w10 + pn[3 * a01 + 2] * w01 + pn[3 * a11 + 2] * w11;
        float r = rsqrtf(qx * qx + qy * qy + qz * qz);
        q = make_float3(qx * r, qy * r, qz * r);
    } else {
        q = make_float3(0.f, 0.f, 1.f);
    }
}

__device__ void sample_surface(const BgView& bg, int n_extra, const HsBgTile* extra, int n_patches,
                               const HsPatch* __restrict__ patches,
                               const float* __restrict__ ph, const float* __restrict__ pn,
                               double x, double y, float& h, float3& nv) {
    sample_bg(bg, x, y, h, nv);
    if (bg.h) add_cascades(n_extra, extra, x, y, h, nv.x, nv.y, nv.z);
    for (int p = 0; p < n_patches; ++p) {
        const HsPatch P = synth_view(patches[p]);
        const double w = blend_w(P, x, y);
        if (!(w > 0.0)) continue;
        float hp; float3 q;
        sample_clamped_at(P, ph, pn, x, y, hp, q);
        const float wf = (float)w;
        h = wf * hp + (1.f - wf) * h;
        if (pn) {
            float mx = wf * q.x + (1.f - wf) * nv.x, my = wf * q.y + (1.f - wf) * nv.y, mz = wf * q.z + (1.f - wf) * nv.z;
            float rr = rsqrtf(mx * mx + my * my + mz * mz);
            nv = make_float3(mx * rr, my * rr, mz * rr);
        }
    }
}

__global__ void sample_kernel(HsSampleArgs a) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= a.n_points) return;
    BgView bg{a.bg_height, a.bg_normal, a.bg_n, a.bg_spacing, a.bg_x0, a.bg_y0};
    float h; float3 nv;
    if (a.from_heights) {
        sample_surface_heights(a.bg_height, a.bg_n, a.bg_spacing, a.n_extra_bg, a.extra_bg, a.n_patches, a.patches,
                               a.patch_height, a.points[2 * k], a.points[2 * k + 1], h, nv);
    } else if (a.clamped_only) {
        sample_clamped_at(synth_view(a.patches[0]), a.patch_height, a.patch_normal, a.points[2 * k], a.points[2 * k + 1], h, nv);
    } else {
        sample_surface(bg, a.n_extra_bg, a.extra_bg, a.n_patches, a.patches, a.patch_height, a.patch_normal,
                       a.points[2 * k], a.points[2 * k + 1], h, nv);
    }
    a.out_height[k] = h;
    if (a.out_normal) { a.out_normal[3 * k] = nv.x; a.out_normal[3 * k + 1] = nv.y; a.out_normal[3 * k + 2] = nv.z; }
}

__global__ void composite_kernel(HsCompositeArgs a) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= a.total_box) return;
    const int p = find_seg_i(a.box_prefix, a.n_patches + 1, k);
    const int local = k - a.box_prefix[p];
    const int i0 = a.box[4 * p], i1 = a.box[4 * p + 1], j0 = a.box[4 * p + 2], j1 = a.box[4 * p + 3];
    const int wj = j1 - j0;
    const int i = i0 + local / wj, j = j0 + local % wj;
    (void)i1;
    BgView bg{a.bg_height, a.bg_normal, a.n, a.spacing, 0.0, 0.0};
    float h; float3 nv;
    sample_surface(bg, a.n_extra_bg, a.extra_bg, a.n_patches, a.patches, a.patch_height, nullptr,
                   (double)i * a.spacing, (double)j * a.spacing, h, nv);
    a.out[(long long)i * a.n + j] = h;
}

// the summed-cascade background on cascade 0's grid (before the patch boxes)
__global__ void bg_sum_kernel(HsCompositeArgs a) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= (long long)a.n * a.n) return;
    const int i = (int)(k / a.n), j = (int)(k - (long long)i * a.n);
    float h = a.bg_height[k];
    for (int c = 0; c < a.n_extra_bg; ++c) {
        float hc, sx, sy;
        sample_tile(a.extra_bg[c], (double)i * a.spacing, (double)j * a.spacing, hc, sx, sy);
        h += hc;
    }
    a.out[k] = h;
}

// =============================================================== finish ==
__global__ void finish_kernel(HsFinishArgs a) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    if (j >= a.ny) return;
    const float* H = a.height;
    const long long o = (long long)i * a.ny + j;
    const float s = (float)a.spacing;
    float hx, hy;
    if (i == 0) hx = (H[o + a.ny] - H[o]) / s;
    else if (i == a.nx - 1) hx = (H[o] - H[o - a.ny]) / s;
    else hx = (H[o + a.ny] - H[o - a.ny]) / (2.f * s);
    if (j == 0) hy = (H[o + 1] - H[o]) / s;
    else if (j == a.ny - 1) hy = (H[o] - H[o - 1]) / s;
    else hy = (H[o + 1] - H[o - 1]) / (2.f * s);
    const float rn = rsqrtf(hx * hx + hy * hy + 1.f);
    if (a.normal) { a.normal[3 * o] = -hx * rn; a.normal[3 * o + 1] = -hy * rn; a.normal[3 * o + 2] = rn; }
    if (a.disp) { a.disp[2 * o] = (float)a.chop_scale * hx; a.disp[2 * o + 1] = (float)a.chop_scale * hy; }
}

__global__ void sumsq_kernel(const float* __restrict__ x, long long n, double* out) {
    __shared__ double red[32];
    double acc = 0.0;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        double v = x[k];
        acc += v * v;
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        atomicAdd(out, t);
    }
}

}  // namespace hs

using namespace hs;

#ifdef HS_SMOOTH_TRACE
extern "C" HS_API int hs_debug_strace(void* dst) {
    return (int)cudaMemcpyFromSymbol(dst, hs::g_strace, sizeof(hs::g_strace));
}
#endif

namespace hs {
// dynamic shared-memory limits of the smooth kernels, raised once per device
// (hs_configure_device raises them to the largest size any layout needs, so
// no attribute call lands inside a graph capture)
static PerDevice<size_t> smooth_attr_d{}, wide_attr_d{};

static size_t smooth_fused_smem(int max_H) {
    const int W = SM_TY + 2 * max_H, K = 2 * max_H + 1, IS = 4 * ((W + 4) >> 2);
    return (size_t)(((K + 3) & ~3) + (SM_TX + 2 * max_H) * IS + SM_TX * (W | 1)) * sizeof(float);
}
static size_t smooth_wide_smem(int max_H_wide) {
    const int K = 2 * max_H_wide + 1, R = SM_TILE + 2 * max_H_wide;
    return (size_t)(((K + 3) & ~3) + R * SM_TILE) * sizeof(float);
}

int smooth_attrs(size_t fused, size_t wide) {
    size_t& fa = smooth_attr_d.get();
    size_t& wa = wide_attr_d.get();
    if (fa == 0) fa = 48 * 1024;
    if (wa == 0) wa = 48 * 1024;
    if (fused > fa) {
        HS_CUDA(cudaFuncSetAttribute(smooth_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused));
        fa = fused;
    }
    if (wide > wa) {
        HS_CUDA(cudaFuncSetAttribute(smooth_wide_x_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wide));
        HS_CUDA(cudaFuncSetAttribute(smooth_wide_y_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wide));
        wa = wide;
    }
    return 0;
}

int smooth_configure() {
    return smooth_attrs(smooth_fused_smem(HS_SMOOTH_FUSED_MAX_H), smooth_wide_smem(780));
}
}  // namespace hs

extern "C" int hs_smooth(const HsSmoothArgs* a, void* stream) {
    HS_EXP_SKIP_POINT("smooth");
    HS_CHECK_ARG(a != nullptr, "hs_smooth: null args");
    HS_CHECK_ARG(a->layers && a->taps && a->raw_layers && a->smooth_layers && a->tile_info, "hs_smooth: missing buffer");
    cudaStream_t st = as_stream(stream);
    if (a->total_tiles > 0) {
        HS_CHECK_ARG(a->max_H >= 1 && a->max_H <= HS_SMOOTH_FUSED_MAX_H, "hs_smooth: max_H=%d out of range", a->max_H);
        const size_t sm = smooth_fused_smem(a->max_H);
        if (int rc = smooth_attrs(sm, 0)) return rc;
        smooth_kernel<<<a->total_tiles, 256, sm, st>>>(*a);
        HS_LAUNCH_CHECK();
    }
    if (a->total_xtiles > 0) {
        HS_CHECK_ARG(a->mid && a->xtile_prefix && a->ytile_prefix, "hs_smooth: wide layers need mid + tile prefixes");
        HS_CHECK_ARG(a->max_H_wide >= 1 && a->max_H_wide <= 780, "hs_smooth: max_H_wide=%d out of range", a->max_H_wide);
        const size_t sm = smooth_wide_smem(a->max_H_wide);
        if (int rc = smooth_attrs(0, sm)) return rc;
        smooth_wide_x_kernel<<<a->total_xtiles, 256, sm, st>>>(*a);
        HS_LAUNCH_CHECK();
        smooth_wide_y_kernel<<<a->total_ytiles, 256, sm, st>>>(*a);
        HS_LAUNCH_CHECK();
    }
    return 0;
}

extern "C" int hs_sample(const HsSampleArgs* a, void* stream) {
    HS_CHECK_ARG(a != nullptr, "hs_sample: null args");
    if (a->n_points == 0) return 0;
    HS_CHECK_ARG(a->points && a->out_height, "hs_sample: missing buffer");
    HS_CHECK_ARG(a->bg_height == nullptr || (a->bg_n >= 2 && (a->bg_n & (a->bg_n - 1)) == 0),
                 "hs_sample: background size must be a power of two");
    sample_kernel<<<(a->n_points + 255) / 256, 256, 0, as_stream(stream)>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}

extern "C" int hs_composite(const HsCompositeArgs* a, void* stream) {
    HS_EXP_SKIP_POINT("composite");
    HS_CHECK_ARG(a != nullptr, "hs_composite: null args");
    cudaStream_t st = as_stream(stream);
    HS_CHECK_ARG(a->out, "hs_composite: missing output");
    const size_t bytes = sizeof(float) * (size_t)a->n * a->n;
    HS_CHECK_ARG(a->n_extra_bg >= 0 && a->n_extra_bg < HS_MAX_CASCADES, "hs_composite: n_extra_bg out of range");
    if (a->bg_height && a->n_extra_bg > 0) {
        const long long nn = (long long)a->n * a->n;
        bg_sum_kernel<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(*a);
        HS_LAUNCH_CHECK();
    } else if (a->bg_height) {
        HS_CUDA(cudaMemcpyAsync(a->out, a->bg_height, bytes, cudaMemcpyDeviceToDevice, st));
    } else {
        HS_CUDA(cudaMemsetAsync(a->out, 0, bytes, st));
    }
    if (a->total_box == 0) return 0;
    composite_kernel<<<(a->total_box + 255) / 256, 256, 0, st>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}

namespace hs {
// ------------------------------------------------ composite box exchange --
__global__ void box_pack_kernel(HsBoxArgs a) {
    const int k = blockIdx.x;                       // local slot
    const int stride = 4 + a.bw * a.bh;
    float* slot = a.payload + ((size_t)a.rank * a.slots + k) * stride;
    int i0 = 0, i1 = 0, j0 = 0, j1 = 0;
    if (k < a.n_local) {
        // harness.py:230-233: [floor(min / spacing), ceil(max / spacing) + 1), clipped
        const HsPatch P = synth_view(a.patches[k]);
        i0 = (int)fmin(fmax(floor(P.x0 / a.spacing), 0.0), (double)a.n);
        i1 = (int)fmin(fmax(ceil(P.x1 / a.spacing) + 1.0, 0.0), (double)a.n);
        j0 = (int)fmin(fmax(floor(P.y0 / a.spacing), 0.0), (double)a.n);
        j1 = (int)fmin(fmax(ceil(P.y1 / a.spacing) + 1.0, 0.0), (double)a.n);
        if (i1 - i0 > a.bw || j1 - j0 > a.bh) {
            if (threadIdx.x == 0 && blockIdx.y == 0) atomicOr(a.status, HS_STATUS_BOX_OVERFLOW);
            i1 = min(i1, i0 + a.bw);
            j1 = min(j1, j0 + a.bh);
        }
    }
    if (threadIdx.x == 0 && blockIdx.y == 0) {
        slot[0] = __int_as_float(i0); slot[1] = __int_as_float(i1);
        slot[2] = __int_as_float(j0); slot[3] = __int_as_float(j1);
    }
    const int wj = j1 - j0;
    for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < (i1 - i0) * wj; e += gridDim.y * blockDim.x) {
        const int r = e / wj, c = e - r * wj;
        slot[4 + r * a.bh + c] = a.composite[(long long)(i0 + r) * a.n + j0 + c];
    }
}

__global__ void box_paste_kernel(HsBoxArgs a) {
    const int s = blockIdx.x;                       // global slot (rank-major = global patch order)
    if (s / a.slots == a.rank) return;              // this rank's own boxes are already in place
    const int stride = 4 + a.bw * a.bh;
    const float* slot = a.payload + (size_t)s * stride;
    const int i0 = __float_as_int(slot[0]), i1 = __float_as_int(slot[1]);
    const int j0 = __float_as_int(slot[2]), j1 = __float_as_int(slot[3]);
    const int wj = j1 - j0, total = a.world * a.slots;
    for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < (i1 - i0) * wj; e += gridDim.y * blockDim.x) {
        const int r = e / wj, c = e - r * wj;
        const int i = i0 + r, j = j0 + c;
        bool later = false;                         // a later box covering this node wins
        for (int t = s + 1; t < total && !later; ++t) {
            const float* h = a.payload + (size_t)t * stride;
            later = i >= __float_as_int(h[0]) && i < __float_as_int(h[1]) && j >= __float_as_int(h[2]) &&
                    j < __float_as_int(h[3]);
        }
        if (!later) a.composite[(long long)i * a.n + j] = slot[4 + r * a.bh + c];
    }
}

// deterministic-mode raw layers: int64 fixed point -> float, 4 slots per thread
__global__ void fixed_to_float_kernel(const long long* __restrict__ src, float* __restrict__ dst, long long n,
                                      double scale) {
    const long long i = 4 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
    if (i + 3 < n) {
        const longlong2 a = *reinterpret_cast<const longlong2*>(src + i);
        const longlong2 b = *reinterpret_cast<const longlong2*>(src + i + 2);
        *reinterpret_cast<float4*>(dst + i) = make_float4((float)((double)a.x * scale), (float)((double)a.y * scale),
                                                          (float)((double)b.x * scale), (float)((double)b.y * scale));
    } else {
        for (long long k = i; k < n; ++k) dst[k] = (float)((double)src[k] * scale);
    }
}
}  // namespace hs

extern "C" int hs_fixed_to_float(const long long* src, float* dst, long long n, int bits, void* stream) {
    HS_CHECK_ARG(n >= 0 && (n == 0 || (src && dst)), "hs_fixed_to_float: bad buffers");
    HS_CHECK_ARG(((size_t)src & 15) == 0 && ((size_t)dst & 15) == 0, "hs_fixed_to_float: buffers must be 16-byte aligned");
    HS_CHECK_ARG(bits >= 0 && bits < 63, "hs_fixed_to_float: bits=%d", bits);
    if (n == 0) return 0;
    const long long threads = (n + 3) / 4;
    fixed_to_float_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, as_stream(stream)>>>(src, dst, n, ldexp(1.0, -bits));
    HS_LAUNCH_CHECK();
    return 0;
}

extern "C" int hs_finish(const HsFinishArgs* a, void* stream) {
    HS_CHECK_ARG(a != nullptr, "hs_finish: null args");
    HS_CHECK_ARG(a->nx >= 2 && a->ny >= 2, "hs_finish: grid must be at least 2x2");
    dim3 grid((a->ny + 127) / 128, a->nx);
    finish_kernel<<<grid, 128, 0, as_stream(stream)>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}

namespace hs {
__global__ void advance_frame_kernel(long long* f) { *f += 1; }
}  // namespace hs

extern "C" int hs_clear(void* p, long long bytes, void* stream) {
    HS_EXP_SKIP_POINT("clear");
    HS_CHECK_ARG(bytes >= 0 && (bytes == 0 || p), "hs_clear: bad buffer");
    if (bytes) HS_CUDA(cudaMemsetAsync(p, 0, (size_t)bytes, as_stream(stream)));
    return 0;
}

extern "C" int hs_advance_frame(long long* frame, void* stream) {
    HS_CHECK_ARG(frame != nullptr, "hs_advance_frame: null counter");
    hs::advance_frame_kernel<<<1, 1, 0, as_stream(stream)>>>(frame);
    HS_LAUNCH_CHECK();
    return 0;
}

extern "C" int hs_sumsq(const float* x, long long n, double* out, void* stream) {
    HS_CHECK_ARG(out != nullptr, "hs_sumsq: null output");
    if (n <= 0) return 0;
    int grid = (int)((n + 255) / 256);
    if (grid > 4 * num_sms()) grid = 4 * num_sms();
    sumsq_kernel<<<grid, 256, 0, as_stream(stream)>>>(x, n, out);
    HS_LAUNCH_CHECK();
    return 0;
}

static int check_box(const HsBoxArgs* a, const char* who) {
    HS_CHECK_ARG(a != nullptr, "%s: null args", who);
    HS_CHECK_ARG(a->n >= 1 && a->spacing > 0.0 && a->composite && a->payload && a->status, "%s: missing buffer", who);
    HS_CHECK_ARG(a->bw >= 1 && a->bh >= 1 && a->slots >= 1 && a->world >= 1 && a->rank >= 0 && a->rank < a->world,
                 "%s: bad slot geometry", who);
    return 0;
}

extern "C" int hs_box_pack(const HsBoxArgs* a, void* stream) {
    if (int rc = check_box(a, "hs_box_pack")) return rc;
    HS_CHECK_ARG(a->n_local >= 0 && a->n_local <= a->slots && (a->n_local == 0 || a->patches),
                 "hs_box_pack: n_local=%d out of range", a->n_local);
    const int ny = min(16, (a->bw * a->bh + 255) / 256);
    box_pack_kernel<<<dim3(a->slots, ny), 256, 0, as_stream(stream)>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}

extern "C" int hs_box_paste(const HsBoxArgs* a, void* stream) {
    if (int rc = check_box(a, "hs_box_paste")) return rc;
    if (a->world == 1) return 0;
    const int ny = min(16, (a->bw * a->bh + 255) / 256);
    box_paste_kernel<<<dim3(a->world * a->slots, ny), 256, 0, as_stream(stream)>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}

namespace hs {
__global__ void spectral_at_kernel(const double2* __restrict__ h0, const double* __restrict__ omega, int n, double t,
                                   double2* __restrict__ out) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= (long long)n * n) return;
    const int i = (int)(k / n), j = (int)(k - (long long)i * n), half = n / 2;
    const int ia = i <= half ? i : n - i, ja = j <= half ? j : n - j;
    const double ph = omega[(long long)ia * (half + 1) + ja] * t;
    double s, c;
    sincos(ph, &s, &c);
    const double2 a = h0[k];
    const double2 b = h0[(long long)((n - i) % n) * n + (n - j) % n];       // h0(-k), conjugated below
    // a (c - i s) + conj(b) (c + i s)
    out[k] = make_double2(a.x * c + a.y * s + b.x * c + b.y * s, a.y * c - a.x * s + b.x * s - b.y * c);
}

__global__ void conv1d_zero_kernel(const double* __restrict__ in, double* __restrict__ out, long long outer, int n,
                                   long long inner, const double* __restrict__ taps, int H) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= outer * n * inner) return;
    const long long o = k / ((long long)n * inner), rem = k - o * n * inner;
    const int i = (int)(rem / inner);
    const long long q = rem - (long long)i * inner;
    const double* row = in + o * n * inner + q;
    double s = 0.0;
    for (int m = -H; m <= H; ++m) {
        const int ii = i + m;
        if (ii >= 0 && ii < n) s += taps[m + H] * row[(long long)ii * inner];
    }
    out[k] = s;
}
}  // namespace hs

extern "C" int hs_spectral_at(const double* h0, const double* omega, int n, double t, double* out, void* stream) {
    HS_CHECK_ARG(h0 && omega && out && n >= 2, "hs_spectral_at: bad arguments");
    const long long nn = (long long)n * n;
    spectral_at_kernel<<<(unsigned)((nn + 255) / 256), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const double2*>(h0), omega, n, t, reinterpret_cast<double2*>(out));
    HS_LAUNCH_CHECK();
    return 0;
}

extern "C" int hs_conv1d_zero(const double* in, double* out, long long outer, int n, long long inner,
                              const double* taps, int H, void* stream) {
    HS_CHECK_ARG(in && out && taps && outer >= 0 && n >= 1 && inner >= 0 && H >= 0, "hs_conv1d_zero: bad arguments");
    HS_CHECK_ARG(2 * H + 1 <= n, "hs_conv1d_zero: kernel of %d taps wider than grid axis of %d", 2 * H + 1, n);
    const long long total = outer * n * inner;
    if (total == 0) return 0;
    conv1d_zero_kernel<<<(unsigned)((total + 255) / 256), 256, 0, as_stream(stream)>>>(in, out, outer, n, inner, taps, H);
    HS_LAUNCH_CHECK();
    return 0;
}
