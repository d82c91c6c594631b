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
#include "hs_common.cuh"

namespace hs {

__device__ __forceinline__ int find_seg_i(const int* off, int nseg, int v) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= v) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// =============================================================== smooth ==
constexpr int SM_TILE = 32;

__global__ void __launch_bounds__(256) smooth_kernel(HsSmoothArgs a) {
    extern __shared__ float smem[];
    const int tile = blockIdx.x;
    const int l = find_seg_i(a.tile_prefix, a.n_layers + 1, tile);
    const HsLayer L = a.layers[l];
    const int local = tile - a.tile_prefix[l];
    const int tiles_y = (L.ncy + SM_TILE - 1) / SM_TILE;
    const int cx0 = (local / tiles_y) * SM_TILE, cy0 = (local % tiles_y) * SM_TILE;
    const int H = L.H, K = 2 * H + 1, W = SM_TILE + 2 * H;
    float* taps = smem;            // K (padded to 4)
    float* in = taps + ((K + 3) & ~3);
    float* mid = in + W * W;
    for (int m = threadIdx.x; m < K; m += blockDim.x) taps[m] = a.taps[L.taps_off + m];
    const float* raw = a.raw_layers + L.raw_off;
    const int rx0 = cx0 + L.pad - H, ry0 = cy0 + L.pad - H;
    for (int e = threadIdx.x; e < W * W; e += blockDim.x) {
        int r = e / W, c = e - r * W;
        int gx = rx0 + r, gy = ry0 + c;
        in[e] = (gx >= 0 && gx < L.wx && gy >= 0 && gy < L.wy) ? raw[(long long)gx * L.wy + gy] : 0.f;
    }
    __syncthreads();
    // pass along axis 0 (x): mid[r][c] = sum_m taps[m] in[r+m][c]
    for (int e = threadIdx.x; e < SM_TILE * W; e += blockDim.x) {
        int r = e / W, c = e - r * W;
        const float* col = in + r * W + c;
        float s = 0.f;
        for (int m = 0; m < K; ++m) s = fmaf(taps[m], col[m * W], s);
        mid[e] = s;
    }
    __syncthreads();
    // pass along axis 1 (y)
    float* out = a.smooth_layers + L.sm_off;
    for (int e = threadIdx.x; e < SM_TILE * SM_TILE; e += blockDim.x) {
        int r = e / SM_TILE, c = e - r * SM_TILE;
        int ox = cx0 + r, oy = cy0 + c;
        if (ox >= L.ncx || oy >= L.ncy) continue;
        const float* row = mid + r * W + c;
        float s = 0.f;
        for (int m = 0; m < K; ++m) s = fmaf(taps[m], row[m], s);
        out[(long long)ox * L.ncy + oy] = s;
    }
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
        in[e] = (gx >= 0 && gx < L.wx && gy < L.wy) ? raw[(long long)gx * L.wy + gy] : 0.f;
    }
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
        in[e] = (gx < L.ncx && gy >= 0 && gy < L.wy) ? mid[(long long)gx * L.wy + gy] : 0.f;
    }
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

// ============================================================== compose ==
__device__ __forceinline__ float upsample_at(const float* __restrict__ S, const HsLayer& L, int i, int j) {
    if (L.f == 1) return S[(long long)i * L.ncy + j];
    const int ci = i / L.f, cj = j / L.f;
    const float wi = (float)((double)(i - ci * L.f) / (double)L.f);
    const float wj = (float)((double)(j - cj * L.f) / (double)L.f);
    const int ci1 = min(ci + 1, L.ncx - 1), cj1 = min(cj + 1, L.ncy - 1);
    const float* r0 = S + (long long)ci * L.ncy;
    const float* r1 = S + (long long)ci1 * L.ncy;
    float a0 = r0[cj] * (1.f - wi) + r1[cj] * wi;
    float a1 = r0[cj1] * (1.f - wi) + r1[cj1] * wi;
    return a0 * (1.f - wj) + a1 * wj;
}

struct BgView {
    const float* h; const float* nrm; int n; double spacing; double x0, y0;
};

// periodic bilinear (fft_background.py:222-249)
__device__ __forceinline__ void sample_bg(const BgView& bg, double x, double y, float& h, float3& nv) {
    if (!bg.h) { h = 0.f; nv = make_float3(0.f, 0.f, 1.f); return; }
    const double u = (x - bg.x0) / bg.spacing, v = (y - bg.y0) / bg.spacing;
    const double fi = floor(u), fj = floor(v);
    const float fu = (float)(u - fi), fv = (float)(v - fj);
    const int m = bg.n - 1;
    const int i0 = ((long long)fi) & m, j0 = ((long long)fj) & m;
    const int i1 = (i0 + 1) & m, j1 = (j0 + 1) & m;
    const float w00 = (1.f - fu) * (1.f - fv), w10 = fu * (1.f - fv), w01 = (1.f - fu) * fv, w11 = fu * fv;
    const long long a00 = (long long)i0 * bg.n + j0, a10 = (long long)i1 * bg.n + j0;
    const long long a01 = (long long)i0 * bg.n + j1, a11 = (long long)i1 * bg.n + j1;
    h = bg.h[a00] * w00 + bg.h[a10] * w10 + bg.h[a01] * w01 + bg.h[a11] * w11;
    if (bg.nrm) {
        const float* N = bg.nrm;
        float nx = N[3 * a00] * w00 + N[3 * a10] * w10 + N[3 * a01] * w01 + N[3 * a11] * w11;
        float ny = N[3 * a00 + 1] * w00 + N[3 * a10 + 1] * w10 + N[3 * a01 + 1] * w01 + N[3 * a11 + 1] * w11;
        float nz = N[3 * a00 + 2] * w00 + N[3 * a10 + 2] * w10 + N[3 * a01 + 2] * w01 + N[3 * a11 + 2] * w11;
        float r = rsqrtf(nx * nx + ny * ny + nz * nz);
        nv = make_float3(nx * r, ny * r, nz * r);
    } else {
        nv = make_float3(0.f, 0.f, 1.f);
    }
}

// smoothstep weight from inward boundary depth (coupling.py:27-40)
__device__ __forceinline__ double blend_w(const HsPatch& P, double x, double y) {
    double d = fmin(fmin(x - P.x0, P.x1 - x), fmin(y - P.y0, P.y1 - y));
    if (!(d > 0.0)) return 0.0;
    double t = fmin(fmax(d / P.margin, 0.0), 1.0);
    return t * t * (3.0 - 2.0 * t);
}

constexpr int CT = 32;

__global__ void __launch_bounds__(256) compose_kernel(HsComposeArgs a) {
    __shared__ float hs_[CT + 2][CT + 3];
    __shared__ double red_s[8];
    __shared__ long long redc_s[8];
    const int tile = blockIdx.x;
    const int p = find_seg_i(a.tile_prefix, a.n_patches + 1, tile);
    const HsPatch P = a.patches[p];
    const int local = tile - a.tile_prefix[p];
    const int tiles_y = (P.ny + CT - 1) / CT;
    const int i0 = (local / tiles_y) * CT, j0 = (local % tiles_y) * CT;
    const HsLayer* Ls = a.layers + P.layer_base;
    const int nb = a.nb;
    // 1. patch heights with a 1-texel halo
    for (int e = threadIdx.x; e < (CT + 2) * (CT + 2); e += blockDim.x) {
        int r = e / (CT + 2), c = e - r * (CT + 2);
        int i = i0 - 1 + r, j = j0 - 1 + c;
        float h = 0.f;
        if (i >= 0 && i < P.res && j >= 0 && j < P.ny) {
            for (int b = 0; b < nb; ++b) {
                const HsLayer L = Ls[b];
                h += L.gain * upsample_at(a.smooth_layers + L.sm_off, L, i, j);
            }
        }
        hs_[r][c] = h;
    }
    __syncthreads();
    BgView bg{a.bg_height, a.bg_normal, a.bg_n, a.bg_spacing, 0.0, 0.0};
    const float s = (float)P.texel;
    const int inset = max(1, (int)rint(P.margin / P.texel));
    double acc = 0.0;
    long long cnt = 0;
    const long long gb = P.grid_base;
    for (int e = threadIdx.x; e < CT * CT; e += blockDim.x) {
        int r = e / CT, c = e - r * CT;
        int i = i0 + r, j = j0 + c;
        if (i >= P.res || j >= P.ny) continue;
        const float h = hs_[r + 1][c + 1];
        float hx, hy;
        if (i == 0) hx = (hs_[r + 2][c + 1] - h) / s;
        else if (i == P.res - 1) hx = (h - hs_[r][c + 1]) / s;
        else hx = (hs_[r + 2][c + 1] - hs_[r][c + 1]) / (2.f * s);
        if (j == 0) hy = (hs_[r + 1][c + 2] - h) / s;
        else if (j == P.ny - 1) hy = (h - hs_[r + 1][c]) / s;
        else hy = (hs_[r + 1][c + 2] - hs_[r + 1][c]) / (2.f * s);
        const float rn = rsqrtf(hx * hx + hy * hy + 1.f);
        const float3 pn = make_float3(-hx * rn, -hy * rn, rn);
        const long long o = gb + (long long)i * P.ny + j;
        if (a.patch_height) a.patch_height[o] = h;
        if (a.patch_normal) { a.patch_normal[3 * o] = pn.x; a.patch_normal[3 * o + 1] = pn.y; a.patch_normal[3 * o + 2] = pn.z; }
        if (i >= inset && i < P.res - inset && j >= inset && j < P.ny - inset) {
            acc += (double)h * (double)h;
            ++cnt;
        }
        if (a.blend_mode) {
            const double x = P.x0 + (double)i * P.texel;     // patch nodes (coupling.py:57-59)
            const double y = P.y0 + (double)j * P.texel;
            float hb; float3 nb3;
            sample_bg(bg, x, y, hb, nb3);
            const double w = blend_w(P, x, y);
            if (w > 0.0) {
                const float wf = (float)w;
                hb = wf * h + (1.f - wf) * hb;
                float mx = wf * pn.x + (1.f - wf) * nb3.x;
                float my = wf * pn.y + (1.f - wf) * nb3.y;
                float mz = wf * pn.z + (1.f - wf) * nb3.z;
                float rr = rsqrtf(mx * mx + my * my + mz * mz);
                nb3 = make_float3(mx * rr, my * rr, mz * rr);
            }
            if (a.blend_height) a.blend_height[o] = hb;
            if (a.blend_normal) { a.blend_normal[3 * o] = nb3.x; a.blend_normal[3 * o + 1] = nb3.y; a.blend_normal[3 * o + 2] = nb3.z; }
        }
    }
    if (a.interior_sumsq) {
        acc = warp_sum(acc);
        long long c2 = cnt;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c2 += __shfl_xor_sync(0xffffffffu, c2, o);
        if ((threadIdx.x & 31) == 0) { red_s[threadIdx.x >> 5] = acc; redc_s[threadIdx.x >> 5] = c2; }
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0; long long tc = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { t += red_s[w]; tc += redc_s[w]; }
            if (tc) {
                atomicAdd(&a.interior_sumsq[p], t);
                if (a.interior_count) atomicAdd((unsigned long long*)&a.interior_count[p], (unsigned long long)tc);
            }
        }
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

__device__ void sample_surface(const BgView& bg, int n_patches, const HsPatch* __restrict__ patches,
                               const float* __restrict__ ph, const float* __restrict__ pn,
                               double x, double y, float& h, float3& nv) {
    sample_bg(bg, x, y, h, nv);
    for (int p = 0; p < n_patches; ++p) {
        const HsPatch P = patches[p];
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
    if (a.clamped_only) {
        sample_clamped_at(a.patches[0], a.patch_height, a.patch_normal, a.points[2 * k], a.points[2 * k + 1], h, nv);
    } else {
        sample_surface(bg, a.n_patches, a.patches, a.patch_height, a.patch_normal,
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
    sample_surface(bg, a.n_patches, a.patches, a.patch_height, nullptr,
                   (double)i * a.spacing, (double)j * a.spacing, h, nv);
    a.out[(long long)i * a.n + j] = h;
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

extern "C" int hs_smooth(const HsSmoothArgs* a, void* stream) {
    HS_CHECK_ARG(a != nullptr, "hs_smooth: null args");
    HS_CHECK_ARG(a->layers && a->taps && a->raw_layers && a->smooth_layers && a->tile_prefix, "hs_smooth: missing buffer");
    cudaStream_t st = as_stream(stream);
    if (a->total_tiles > 0) {
        HS_CHECK_ARG(a->max_H >= 1 && a->max_H <= HS_SMOOTH_FUSED_MAX_H, "hs_smooth: max_H=%d out of range", a->max_H);
        const int W = SM_TILE + 2 * a->max_H, K = 2 * a->max_H + 1;
        size_t sm = (size_t)(((K + 3) & ~3) + W * W + SM_TILE * W) * sizeof(float);
        static size_t smooth_attr = 48 * 1024;
        if (sm > smooth_attr) {
            HS_CUDA(cudaFuncSetAttribute(smooth_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            smooth_attr = sm;
        }
        smooth_kernel<<<a->total_tiles, 256, sm, st>>>(*a);
        HS_LAUNCH_CHECK();
    }
    if (a->total_xtiles > 0) {
        HS_CHECK_ARG(a->mid && a->xtile_prefix && a->ytile_prefix, "hs_smooth: wide layers need mid + tile prefixes");
        HS_CHECK_ARG(a->max_H_wide >= 1 && a->max_H_wide <= 780, "hs_smooth: max_H_wide=%d out of range", a->max_H_wide);
        const int K = 2 * a->max_H_wide + 1, R = SM_TILE + 2 * a->max_H_wide;
        size_t sm = (size_t)(((K + 3) & ~3) + R * SM_TILE) * sizeof(float);
        static size_t wide_attr = 48 * 1024;
        if (sm > wide_attr) {
            HS_CUDA(cudaFuncSetAttribute(smooth_wide_x_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            HS_CUDA(cudaFuncSetAttribute(smooth_wide_y_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            wide_attr = sm;
        }
        smooth_wide_x_kernel<<<a->total_xtiles, 256, sm, st>>>(*a);
        HS_LAUNCH_CHECK();
        smooth_wide_y_kernel<<<a->total_ytiles, 256, sm, st>>>(*a);
        HS_LAUNCH_CHECK();
    }
    return 0;
}

extern "C" int hs_compose(const HsComposeArgs* a, void* stream) {
    HS_CHECK_ARG(a != nullptr, "hs_compose: null args");
    if (a->total_tiles == 0) return 0;
    HS_CHECK_ARG(a->patches && a->layers && a->smooth_layers && a->tile_prefix, "hs_compose: missing buffer");
    HS_CHECK_ARG(!a->blend_mode || a->bg_height == nullptr || (a->bg_n >= 2 && (a->bg_n & (a->bg_n - 1)) == 0),
                 "hs_compose: background size must be a power of two");
    compose_kernel<<<a->total_tiles, 256, 0, as_stream(stream)>>>(*a);
    HS_LAUNCH_CHECK();
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
    HS_CHECK_ARG(a != nullptr, "hs_composite: null args");
    HS_CHECK_ARG(a->out, "hs_composite: missing output");
    cudaStream_t st = as_stream(stream);
    const size_t bytes = sizeof(float) * (size_t)a->n * a->n;
    if (a->bg_height) HS_CUDA(cudaMemcpyAsync(a->out, a->bg_height, bytes, cudaMemcpyDeviceToDevice, st));
    else HS_CUDA(cudaMemsetAsync(a->out, 0, bytes, st));
    if (a->total_box == 0) return 0;
    composite_kernel<<<(a->total_box + 255) / 256, 256, 0, st>>>(*a);
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
