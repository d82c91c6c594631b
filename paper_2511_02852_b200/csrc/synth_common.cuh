// Helpers shared by the synthesis / blend kernels.
#pragma once
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

// One further cascade of a summed background (HsBgTile): bilinear periodic
// height and the slope (n.x/n.z, n.y/n.z) of the renormalised bilinear node
// normal, node normals from periodic central differences of the tile's
// heights (fft_background.py:162-178, 222-249).
__device__ __forceinline__ float3 tile_node_normal(const float* __restrict__ H, int n, int i, int j, float inv2s) {
    const int m = n - 1;
    const float hx = (__ldg(H + (long long)((i + 1) & m) * n + (j & m)) - __ldg(H + (long long)((i - 1) & m) * n + (j & m))) * inv2s;
    const float hy = (__ldg(H + (long long)(i & m) * n + ((j + 1) & m)) - __ldg(H + (long long)(i & m) * n + ((j - 1) & m))) * inv2s;
    const float r = rsqrtf(hx * hx + hy * hy + 1.f);
    return make_float3(-hx * r, -hy * r, r);
}

__device__ __forceinline__ void sample_tile(const HsBgTile& T, double x, double y, float& h, float& sx, float& sy) {
    const double u = x / T.spacing, v = y / T.spacing;
    const double fi = floor(u), fj = floor(v);
    const float fu = (float)(u - fi), fv = (float)(v - fj);
    const int m = T.n - 1;
    const int i0 = (int)((long long)fi & m), j0 = (int)((long long)fj & m);
    const int i1 = (i0 + 1) & m, j1 = (j0 + 1) & m;
    const float w00 = (1.f - fu) * (1.f - fv), w10 = fu * (1.f - fv), w01 = (1.f - fu) * fv, w11 = fu * fv;
    const float* H = T.height;
    h = __ldg(H + (long long)i0 * T.n + j0) * w00 + __ldg(H + (long long)i1 * T.n + j0) * w10
      + __ldg(H + (long long)i0 * T.n + j1) * w01 + __ldg(H + (long long)i1 * T.n + j1) * w11;
    const float inv2s = (float)(0.5 / T.spacing);
    const float3 a = tile_node_normal(H, T.n, i0, j0, inv2s), b = tile_node_normal(H, T.n, i1, j0, inv2s);
    const float3 c = tile_node_normal(H, T.n, i0, j1, inv2s), d = tile_node_normal(H, T.n, i1, j1, inv2s);
    const float nx = a.x * w00 + b.x * w10 + c.x * w01 + d.x * w11;
    const float ny = a.y * w00 + b.y * w10 + c.y * w01 + d.y * w11;
    const float nz = a.z * w00 + b.z * w10 + c.z * w01 + d.z * w11;
    sx = nx / nz;                              // renormalisation cancels in the slope
    sy = ny / nz;
}

// add the extra cascades at (x, y) to a cascade-0 sample (h, unit normal n)
__device__ __forceinline__ void add_cascades(int n_extra, const HsBgTile* extra, double x, double y, float& h,
                                             float& nx, float& ny, float& nz) {
    if (n_extra <= 0) return;
    float sx = nx / nz, sy = ny / nz;
    for (int c = 0; c < n_extra; ++c) {
        float hc, sxc, syc;
        sample_tile(extra[c], x, y, hc, sxc, syc);
        h += hc;
        sx += sxc;
        sy += syc;
    }
    const float r = rsqrtf(sx * sx + sy * sy + 1.f);
    nx = sx * r; ny = sy * r; nz = r;
}

// SurfaceSampler._raw (coupling.py:120-141, normal_mode "blend") from height
// grids only, as the frame leaves them: the periodic background (cascade 0
// at origin 0, + further cascades) with central-difference node normals, then
// every patch (synthesis rectangle) by clamped bilinear heights and
// clamped-border finite-difference node normals (finish_field, :323-340)
// under its smoothstep weight.
__device__ __forceinline__ float3 patch_node_normal(const float* __restrict__ H, int nx, int ny, int i, int j, float s) {
    float hx, hy;
    if (i == 0) hx = (H[(long long)ny + j] - H[j]) / s;
    else if (i == nx - 1) hx = (H[(long long)i * ny + j] - H[(long long)(i - 1) * ny + j]) / s;
    else hx = (H[(long long)(i + 1) * ny + j] - H[(long long)(i - 1) * ny + j]) / (2.f * s);
    const long long r = (long long)i * ny;
    if (j == 0) hy = (H[r + 1] - H[r]) / s;
    else if (j == ny - 1) hy = (H[r + j] - H[r + j - 1]) / s;
    else hy = (H[r + j + 1] - H[r + j - 1]) / (2.f * s);
    const float rn = rsqrtf(hx * hx + hy * hy + 1.f);
    return make_float3(-hx * rn, -hy * rn, rn);
}

__device__ __forceinline__ void sample_surface_heights(const float* bg_h, int bg_n, double bg_sp, int n_extra,
                                                       const HsBgTile* extra, int n_patches,
                                                       const HsPatch* __restrict__ patches,
                                                       const float* __restrict__ patch_h, double x, double y,
                                                       float& h, float3& nv) {
    h = 0.f;
    nv = make_float3(0.f, 0.f, 1.f);
    if (bg_h) {
        const HsBgTile T0{bg_h, bg_n, 0, bg_sp};
        float sx, sy;
        sample_tile(T0, x, y, h, sx, sy);            // renormalised bilinear normal as a slope
        float nx = sx, ny = sy, nz = 1.f;            // the normal's direction
        add_cascades(n_extra, extra, x, y, h, nx, ny, nz);
        const float r = rsqrtf(nx * nx + ny * ny + nz * nz);
        nv = make_float3(nx * r, ny * r, nz * r);
    }
    for (int p = 0; p < n_patches; ++p) {
        const HsPatch P = synth_view(patches[p]);
        double d = fmin(fmin(x - P.x0, P.x1 - x), fmin(y - P.y0, P.y1 - y));
        if (!(d > 0.0)) continue;
        double t = fmin(fmax(d / P.margin, 0.0), 1.0);
        const float w = (float)(t * t * (3.0 - 2.0 * t));
        const double u = fmin(fmax((x - P.x0) / P.texel, 0.0), (double)(P.res - 1));
        const double v = fmin(fmax((y - P.y0) / P.texel, 0.0), (double)(P.ny - 1));
        const int i = min((int)u, P.res - 2), j = min((int)v, P.ny - 2);
        const float fu = (float)(u - i), fv = (float)(v - j);
        const float w00 = (1.f - fu) * (1.f - fv), w10 = fu * (1.f - fv), w01 = (1.f - fu) * fv, w11 = fu * fv;
        const float* H = patch_h + P.grid_base;
        const long long a00 = (long long)i * P.ny + j;
        const float hp = H[a00] * w00 + H[a00 + P.ny] * w10 + H[a00 + 1] * w01 + H[a00 + P.ny + 1] * w11;
        const float s = (float)P.texel;
        const float3 n00 = patch_node_normal(H, P.res, P.ny, i, j, s), n10 = patch_node_normal(H, P.res, P.ny, i + 1, j, s);
        const float3 n01 = patch_node_normal(H, P.res, P.ny, i, j + 1, s), n11 = patch_node_normal(H, P.res, P.ny, i + 1, j + 1, s);
        float qx = n00.x * w00 + n10.x * w10 + n01.x * w01 + n11.x * w11;
        float qy = n00.y * w00 + n10.y * w10 + n01.y * w01 + n11.y * w11;
        float qz = n00.z * w00 + n10.z * w10 + n01.z * w01 + n11.z * w11;
        const float rq = rsqrtf(qx * qx + qy * qy + qz * qz);
        qx *= rq; qy *= rq; qz *= rq;
        h = w * hp + (1.f - w) * h;
        const float mx = w * qx + (1.f - w) * nv.x, my = w * qy + (1.f - w) * nv.y, mz = w * qz + (1.f - w) * nv.z;
        const float rm = rsqrtf(mx * mx + my * my + mz * mz);
        nv = make_float3(mx * rm, my * rm, mz * rm);
    }
}

// smoothstep weight from inward boundary depth (coupling.py:27-40)
__device__ __forceinline__ double blend_w(const HsPatch& P, double x, double y) {
    double d = fmin(fmin(x - P.x0, P.x1 - x), fmin(y - P.y0, P.y1 - y));
    if (!(d > 0.0)) return 0.0;
    double t = fmin(fmax(d / P.margin, 0.0), 1.0);
    return t * t * (3.0 - 2.0 * t);
}

}  // namespace hs
