// hs_compose: the per-patch output pass of the hybrid step.
//
//   heights  sum_b gain_b * bilinear_upsample_b     (patch_synthesis.py:261-274, 301-313)
//   normals  clamped-border central differences     (finish_field :323-340,
//                                                     fft_background.py:168-178)
//   blend    w = smoothstep(d / margin) at the patch nodes,
//            h = w h_patch + (1 - w) bilinear_periodic(h_fft),
//            n = normalize(w n_patch + (1 - w) n_fft)  (coupling.py:37-40, 120-141)
//   stats    interior sum of h^2 for FrameStats.patch_variance (harness.py:176-178)
//
// One CTA per 32x32 output tile (+1-texel halo).  Per CTA the coarse (f > 1)
// smoothed layers' footprint under the tile is staged in shared memory and
// the bilinear row / column indices and weights are tabulated once; f == 1
// layers are read straight from L2 with coalesced rows.  Blend distances and
// background sample positions are formed per row / column in fp64 (world
// coordinates, as the reference) and applied per texel in fp32.
#include "synth_common.cuh"

namespace hs {

constexpr int CT = 30;            // output tile edge
constexpr int CH = CT + 2;        // haloed height tile (32): lane = haloed row, 32 columns in registers
constexpr int WPB = 2;            // warps (tiles) per block
constexpr int BG_CAP = 8;         // staged background footprint per axis (+1 halo each side)
constexpr int CS_WARP = 1536;     // floats of staged coarse footprints per warp

__device__ __forceinline__ float lerpf(float a, float b, float w) { return fmaf(w, b - a, a); }

__device__ __forceinline__ float3 bg_node_normal(const float* H, int n, long long i, long long j, float inv2s) {
    const int m = n - 1;
    const float hx = (H[((i + 1) & m) * n + (j & m)] - H[((i - 1) & m) * n + (j & m)]) * inv2s;
    const float hy = (H[(i & m) * n + ((j + 1) & m)] - H[(i & m) * n + ((j - 1) & m)]) * inv2s;
    const float r = rsqrtf(hx * hx + hy * hy + 1.f);
    return make_float3(-hx * r, -hy * r, r);
}

struct WarpSmem {
    float hs[CH][CH + 1];             // haloed patch heights
    float tcol[20][CH];               // row-interpolated coarse rows of one layer (lane = column)
    float4 rw[CH];                    // per haloed row: coarse row (rel), g0, g1, unused
    float cs[CS_WARP];                // staged coarse footprints of all layers
    HsLayer Ls[HS_MAX_BUCKETS];
    int st[HS_MAX_BUCKETS][4];        // per layer: staged offset (-1: none), cr0, cc0, ncol
    float bgh[(BG_CAP + 2) * (BG_CAP + 2)];
    float bgn[BG_CAP * BG_CAP * 3];
    float row_d[CT], col_d[CT], row_fu[CT], col_fv[CT];
    int row_q0[CT], row_q1[CT], col_q0[CT], col_q1[CT];
    int bg_q[4];
};

// One warp per 30 x 30 output tile (32 x 32 haloed heights):
//   heights  lane = haloed row; per layer the warp walks the row's coarse
//            cells left to right (cell boundaries are warp-uniform), forms the
//            two row-interpolated coarse values per cell and lerps them into
//            32 register accumulators: sum_b gain_b upsample_b
//            (patch_synthesis.py:261-274, 301-313); f == 1 layers are staged
//            through shared memory (coalesced) and read transposed
//   epilogue clamped FD normals (finish_field :323-340) and the smoothstep
//            blend against the periodic background at the patch nodes
//            (coupling.py:37-40, 120-141), background footprint staged
// Warps never synchronise with each other.
__global__ void __launch_bounds__(32 * WPB) compose_kernel(HsComposeArgs a) {
    __shared__ WarpSmem wsm[WPB];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int tile = blockIdx.x * WPB + wid;
    if (a.frame_advance && blockIdx.x == 0 && threadIdx.x == 0) *a.frame_advance += 1;
    if (tile >= a.total_tiles) return;
    WarpSmem& W = wsm[wid];
    const int* ti = a.tile_info + 3 * tile;
    const int p = ti[0], i0 = ti[1], j0 = ti[2];
    const HsPatch P = a.patches[p];
    const int nb = a.nb;
    const bool have_bg = a.bg_height != nullptr;
    const int bm = a.bg_n - 1;
    const double inv_sp = have_bg ? 1.0 / a.bg_spacing : 0.0;

    // background footprint of the output tile (+1 halo for the node normals)
    if (lane == 0) {
        W.bg_q[0] = W.bg_q[1] = W.bg_q[2] = W.bg_q[3] = 0;
        if (have_bg) {
            const int il = min(i0 + CT - 1, P.res - 1), jl = min(j0 + CT - 1, P.ny - 1);
            const long long qa = (long long)floor((P.x0 + (double)i0 * P.texel) * inv_sp);
            const long long qb = (long long)floor((P.x0 + (double)il * P.texel) * inv_sp) + 1;
            const long long qc = (long long)floor((P.y0 + (double)j0 * P.texel) * inv_sp);
            const long long qd = (long long)floor((P.y0 + (double)jl * P.texel) * inv_sp) + 1;
            if (qb - qa + 1 <= BG_CAP && qd - qc + 1 <= BG_CAP) {
                W.bg_q[0] = (int)(qa & bm); W.bg_q[1] = (int)(qb - qa + 1);
                W.bg_q[2] = (int)(qc & bm); W.bg_q[3] = (int)(qd - qc + 1);
            }
        }
    }
    __syncwarp();
    const bool bg_staged = W.bg_q[1] > 0;
    const bool own_normals = a.bg_normal == nullptr;
    if (bg_staged) {
        const int nr = W.bg_q[1] + 2, nc = W.bg_q[3] + 2;
        for (int e = lane; e < nr * nc; e += 32) {
            const int rr = e / nc, cc = e - rr * nc;
            const long long g = (long long)((W.bg_q[0] - 1 + rr) & bm) * a.bg_n + ((W.bg_q[2] - 1 + cc) & bm);
            cp_async4(W.bgh + e, a.bg_height + g, true);
        }
        if (!own_normals) {
            const int nr0 = W.bg_q[1], nc0 = W.bg_q[3];
            for (int e = lane; e < nr0 * nc0; e += 32) {
                const int rr = e / nc0, cc = e - rr * nc0;
                const long long g = (long long)((W.bg_q[0] + rr) & bm) * a.bg_n + ((W.bg_q[2] + cc) & bm);
                cp_async4(W.bgn + 3 * e, a.bg_normal + 3 * g, true);
                cp_async4(W.bgn + 3 * e + 1, a.bg_normal + 3 * g + 1, true);
                cp_async4(W.bgn + 3 * e + 2, a.bg_normal + 3 * g + 2, true);
            }
        }
    }
    // blend / background tables: lane k < 30 does output row k and column k (fp64 world coordinates)
    if (lane < CT) {
#pragma unroll
        for (int axis = 0; axis < 2; ++axis) {
            const int idx = (axis == 0 ? i0 : j0) + lane;
            const double lo = axis == 0 ? P.x0 : P.y0, hi = axis == 0 ? P.x1 : P.y1;
            const double x = lo + (double)idx * P.texel;        // node positions (coupling.py:57-59)
            const float d = (float)fmin(x - lo, hi - x);        // boundary_depth (coupling.py:27-34)
            int q0 = 0, q1 = 0;
            float fr = 0.f;
            if (have_bg) {
                const double u = x * inv_sp;                     // background origin (0, 0)
                const double fl = floor(u);
                fr = (float)(u - fl);
                const long long q = (long long)fl;
                if (bg_staged) {
                    const long long base = axis == 0 ? (long long)floor((P.x0 + (double)i0 * P.texel) * inv_sp)
                                                     : (long long)floor((P.y0 + (double)j0 * P.texel) * inv_sp);
                    q0 = (int)(q - base);
                    q1 = q0 + 1;
                } else {
                    q0 = (int)(q & bm);
                    q1 = (q0 + 1) & bm;
                }
            }
            if (axis == 0) { W.row_d[lane] = d; W.row_fu[lane] = fr; W.row_q0[lane] = q0; W.row_q1[lane] = q1; }
            else           { W.col_d[lane] = d; W.col_fv[lane] = fr; W.col_q0[lane] = q0; W.col_q1[lane] = q1; }
        }
    }

    // ---- heights: lane = haloed column c, acc[r] = haloed row r ----
    // all global reads are batched: layer descriptors (one round trip), then
    // every coarse footprint by cp.async while the f == 1 layers stream in
    const int c = lane;
    const int j_raw = j0 - 1 + c;
    const int j = min(max(j_raw, 0), P.ny - 1);
    const int ib = i0 - 1;                         // haloed row 0
    const int ilo = min(max(ib, 0), P.res - 1), ihi = min(max(ib + CH - 1, 0), P.res - 1);
    const int jlo = min(max(j0 - 1, 0), P.ny - 1), jhi = min(max(j0 - 1 + CH - 1, 0), P.ny - 1);
    if (lane < nb) W.Ls[lane] = a.layers[P.layer_base + lane];
    __syncwarp();
    {
        // staging plan: lane b sizes layer b's footprint; offsets by a warp scan
        int need = 0, cr0 = 0, cc0 = 0, ncol = 0;
        if (lane < nb && W.Ls[lane].f > 1) {
            const HsLayer& L = W.Ls[lane];
            cr0 = ilo / L.f;
            const int nr = min(ihi / L.f + 1, L.ncx - 1) - cr0 + 1;
            cc0 = jlo / L.f;
            ncol = min(jhi / L.f + 1, L.ncy - 1) - cc0 + 1;
            need = nr * ncol;
        }
        const int inc = warp_incl_scan(need, lane);
        if (lane < nb) {
            W.st[lane][0] = (need > 0 && inc <= CS_WARP) ? inc - need : -1;
            W.st[lane][1] = cr0; W.st[lane][2] = cc0; W.st[lane][3] = ncol;
        }
    }
    __syncwarp();
    for (int b = 0; b < nb; ++b) {
        const HsLayer& L = W.Ls[b];
        const int off = W.st[b][0];
        if (off < 0) continue;
        const int cr0 = W.st[b][1], cc0 = W.st[b][2], ncol = W.st[b][3];
        const int nr = min(ihi / L.f + 1, L.ncx - 1) - cr0 + 1;
        const float* S = a.smooth_layers + L.sm_off;
        for (int e = lane; e < nr * ncol; e += 32) {
            const int rr = e / ncol, cc = e - rr * ncol;
            cp_async4(W.cs + off + e, S + (long long)(cr0 + rr) * L.ncy + cc0 + cc, true);
        }
    }
    float acc[CH];
#pragma unroll
    for (int q = 0; q < CH; ++q) acc[q] = 0.f;
    for (int b = 0; b < nb; ++b) {                 // f == 1 layers: coalesced rows, 32 loads in flight
        const HsLayer& L = W.Ls[b];
        if (L.f != 1) continue;
        const float* S = a.smooth_layers + L.sm_off;
        float v[CH];
#pragma unroll
        for (int q = 0; q < CH; ++q) v[q] = S[(long long)min(max(ib + q, 0), P.res - 1) * L.ncy + j];
#pragma unroll
        for (int q = 0; q < CH; ++q) acc[q] = fmaf(L.gain, v[q], acc[q]);
    }
    cp_async_wait_all();
    __syncwarp();
    for (int b = 0; b < nb; ++b) {
        const HsLayer& L = W.Ls[b];
        if (L.f == 1) continue;
        const int f = L.f;
        const float inv_f = 1.f / (float)f;
        const int cr0 = ilo / f, nr = min(ihi / f + 1, L.ncx - 1) - cr0 + 1;
        const int cj = j / f;
        const int cj1 = min(cj + 1, L.ncy - 1);
        const float wj = (float)(j - cj * f) * inv_f;
        {   // per haloed row (lane = row): coarse row offset and gain-folded weights
            const int ii = min(max(ib + lane, 0), P.res - 1);
            const int ci = ii / f;
            const float wi = (float)(ii - ci * f) * inv_f;
            const float g1 = L.gain * wi;
            W.rw[lane] = make_float4(__int_as_float(ci - cr0), L.gain - g1, g1, 0.f);
        }
        const int off = W.st[b][0];
        if (off >= 0 && nr <= 20) {
            // x-first bilinear (:270-273): interpolate this lane's column on each staged coarse row
            const int ncol = W.st[b][3], cc0 = W.st[b][2];
            const float* src = W.cs + off + (cj - cc0);
            const int d1 = cj1 - cj;
            for (int rr = 0; rr < nr; ++rr) W.tcol[rr][c] = lerpf(src[rr * ncol], src[rr * ncol + d1], wj);
            __syncwarp();
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const float4 e = W.rw[q];
                const int rr = __float_as_int(e.x);
                const int rn = min(rr + 1, nr - 1);
                acc[q] = fmaf(e.y, W.tcol[rr][c], fmaf(e.z, W.tcol[rn][c], acc[q]));
            }
        } else {                                   // not staged: direct reads (rare)
            __syncwarp();
            const float* S = a.smooth_layers + L.sm_off;
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const float4 e = W.rw[q];
                const int ci = cr0 + __float_as_int(e.x), ci1 = min(ci + 1, L.ncx - 1);
                const float* r0 = S + (long long)ci * L.ncy;
                const float* r1 = S + (long long)ci1 * L.ncy;
                acc[q] = fmaf(e.y, lerpf(r0[cj], r0[cj1], wj), fmaf(e.z, lerpf(r1[cj], r1[cj1], wj), acc[q]));
            }
        }
        __syncwarp();
    }
    {
        const bool jok = j_raw >= 0 && j_raw < P.ny;
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            const int ii = ib + q;
            W.hs[q][c] = (jok && ii >= 0 && ii < P.res) ? acc[q] : 0.f;
        }
    }
    cp_async_wait_all();
    __syncwarp();
    if (bg_staged && own_normals) {
        const int nr0 = W.bg_q[1], nc0 = W.bg_q[3], ncs = nc0 + 2;
        const float inv2s = (float)(0.5 / a.bg_spacing);
        for (int e = lane; e < nr0 * nc0; e += 32) {
            const int rr = e / nc0 + 1, cc = e % nc0 + 1;
            const float hx = (W.bgh[(rr + 1) * ncs + cc] - W.bgh[(rr - 1) * ncs + cc]) * inv2s;
            const float hy = (W.bgh[rr * ncs + cc + 1] - W.bgh[rr * ncs + cc - 1]) * inv2s;
            const float rn = rsqrtf(hx * hx + hy * hy + 1.f);
            W.bgn[3 * e] = -hx * rn; W.bgn[3 * e + 1] = -hy * rn; W.bgn[3 * e + 2] = rn;
        }
        __syncwarp();
    }

    // ---- normals, blend, outputs ----
    const float inv_s = (float)(1.0 / P.texel), inv_2s = (float)(0.5 / P.texel);
    const float inv_margin = (float)(1.0 / P.margin);
    const float inv2sp = have_bg ? (float)(0.5 / a.bg_spacing) : 0.f;
    const int inset = max(1, (int)rint(P.margin / P.texel));
    double accv = 0.0;
    int cnt = 0;
    const long long gb = P.grid_base;
    const int bn = a.bg_n, bnc = W.bg_q[3], bnh = W.bg_q[3] + 2;
    for (int e = lane; e < CT * CT; e += 32) {
        const int rr = e / CT, c = e - rr * CT;
        const int ii = i0 + rr, j = j0 + c;
        if (ii >= P.res || j >= P.ny) continue;
        const float h = W.hs[rr + 1][c + 1];
        float hx, hy;
        if (ii == 0) hx = (W.hs[rr + 2][c + 1] - h) * inv_s;
        else if (ii == P.res - 1) hx = (h - W.hs[rr][c + 1]) * inv_s;
        else hx = (W.hs[rr + 2][c + 1] - W.hs[rr][c + 1]) * inv_2s;
        if (j == 0) hy = (W.hs[rr + 1][c + 2] - h) * inv_s;
        else if (j == P.ny - 1) hy = (h - W.hs[rr + 1][c]) * inv_s;
        else hy = (W.hs[rr + 1][c + 2] - W.hs[rr + 1][c]) * inv_2s;
        const float rn = rsqrtf(hx * hx + hy * hy + 1.f);
        const float pnx = -hx * rn, pny = -hy * rn, pnz = rn;
        const long long o = gb + (long long)ii * P.ny + j;
        if (a.patch_height) a.patch_height[o] = h;
        if (a.patch_normal) { a.patch_normal[3 * o] = pnx; a.patch_normal[3 * o + 1] = pny; a.patch_normal[3 * o + 2] = pnz; }
        if (ii >= inset && ii < P.res - inset && j >= inset && j < P.ny - inset) {
            accv += (double)h * (double)h;
            ++cnt;
        }
        if (a.blend_mode) {
            float hb = 0.f, nx = 0.f, ny = 0.f, nz = 1.f;
            if (have_bg) {
                const float fu = W.row_fu[rr], fv = W.col_fv[c];
                const float w00 = (1.f - fu) * (1.f - fv), w10 = fu * (1.f - fv), w01 = (1.f - fu) * fv, w11 = fu * fv;
                const int q0 = W.row_q0[rr], q1 = W.row_q1[rr], p0 = W.col_q0[c], p1 = W.col_q1[c];
                if (bg_staged) {
                    hb = W.bgh[(q0 + 1) * bnh + p0 + 1] * w00 + W.bgh[(q1 + 1) * bnh + p0 + 1] * w10
                       + W.bgh[(q0 + 1) * bnh + p1 + 1] * w01 + W.bgh[(q1 + 1) * bnh + p1 + 1] * w11;
                    const int a00 = q0 * bnc + p0, a10 = q1 * bnc + p0, a01 = q0 * bnc + p1, a11 = q1 * bnc + p1;
                    nx = W.bgn[3 * a00] * w00 + W.bgn[3 * a10] * w10 + W.bgn[3 * a01] * w01 + W.bgn[3 * a11] * w11;
                    ny = W.bgn[3 * a00 + 1] * w00 + W.bgn[3 * a10 + 1] * w10 + W.bgn[3 * a01 + 1] * w01 + W.bgn[3 * a11 + 1] * w11;
                    nz = W.bgn[3 * a00 + 2] * w00 + W.bgn[3 * a10 + 2] * w10 + W.bgn[3 * a01 + 2] * w01 + W.bgn[3 * a11 + 2] * w11;
                } else {
                    const float* B = a.bg_height;
                    hb = B[(long long)q0 * bn + p0] * w00 + B[(long long)q1 * bn + p0] * w10
                       + B[(long long)q0 * bn + p1] * w01 + B[(long long)q1 * bn + p1] * w11;
                    float3 n00, n10, n01, n11;
                    if (own_normals) {
                        n00 = bg_node_normal(B, bn, q0, p0, inv2sp); n10 = bg_node_normal(B, bn, q1, p0, inv2sp);
                        n01 = bg_node_normal(B, bn, q0, p1, inv2sp); n11 = bg_node_normal(B, bn, q1, p1, inv2sp);
                    } else {
                        const float* Nn = a.bg_normal;
                        const long long a00 = 3 * ((long long)q0 * bn + p0), a10 = 3 * ((long long)q1 * bn + p0);
                        const long long a01 = 3 * ((long long)q0 * bn + p1), a11 = 3 * ((long long)q1 * bn + p1);
                        n00 = make_float3(Nn[a00], Nn[a00 + 1], Nn[a00 + 2]); n10 = make_float3(Nn[a10], Nn[a10 + 1], Nn[a10 + 2]);
                        n01 = make_float3(Nn[a01], Nn[a01 + 1], Nn[a01 + 2]); n11 = make_float3(Nn[a11], Nn[a11 + 1], Nn[a11 + 2]);
                    }
                    nx = n00.x * w00 + n10.x * w10 + n01.x * w01 + n11.x * w11;
                    ny = n00.y * w00 + n10.y * w10 + n01.y * w01 + n11.y * w11;
                    nz = n00.z * w00 + n10.z * w10 + n01.z * w01 + n11.z * w11;
                }
                const float rr2 = rsqrtf(nx * nx + ny * ny + nz * nz);
                nx *= rr2; ny *= rr2; nz *= rr2;
            }
            const float d = fminf(W.row_d[rr], W.col_d[c]);
            if (d > 0.f) {
                const float w = smoothstep01(d * inv_margin);
                hb = w * h + (1.f - w) * hb;
                const float mx = w * pnx + (1.f - w) * nx, my = w * pny + (1.f - w) * ny, mz = w * pnz + (1.f - w) * nz;
                const float rr2 = rsqrtf(mx * mx + my * my + mz * mz);
                nx = mx * rr2; ny = my * rr2; nz = mz * rr2;
            }
            if (a.blend_height) a.blend_height[o] = hb;
            if (a.blend_normal) { a.blend_normal[3 * o] = nx; a.blend_normal[3 * o + 1] = ny; a.blend_normal[3 * o + 2] = nz; }
        }
    }
    if (a.interior_sumsq) {
        accv = warp_sum(accv);
        cnt = warp_sum(cnt);
        if (lane == 0 && cnt) {
            atomicAdd(&a.interior_sumsq[p], accv);
            if (a.interior_count) atomicAdd((unsigned long long*)&a.interior_count[p], (unsigned long long)cnt);
        }
    }
}

}  // namespace hs

using namespace hs;

extern "C" int hs_compose(const HsComposeArgs* a, void* stream) {
    HS_CHECK_ARG(a != nullptr, "hs_compose: null args");
    HS_CHECK_ARG(a->nb >= 1 && a->nb <= HS_MAX_BUCKETS, "hs_compose: nb out of range");
    if (a->total_tiles == 0) {
        if (a->frame_advance) HS_CHECK_ARG(false, "hs_compose: frame_advance needs at least one tile");
        return 0;
    }
    HS_CHECK_ARG(a->patches && a->layers && a->smooth_layers && a->tile_info, "hs_compose: missing buffer");
    HS_CHECK_ARG(!a->blend_mode || a->bg_height == nullptr || (a->bg_n >= 2 && (a->bg_n & (a->bg_n - 1)) == 0),
                 "hs_compose: background size must be a power of two");
    compose_kernel<<<(a->total_tiles + WPB - 1) / WPB, 32 * WPB, 0, as_stream(stream)>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}
