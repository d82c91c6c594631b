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

constexpr int CT = 32;            // output tile edge
constexpr int CH = CT + 2;        // with halo
constexpr int CS_CAP = 4096;      // floats of staged coarse layers per CTA
constexpr int BG_CAP = 8;         // staged background footprint per axis
constexpr int RPT = 5;            // haloed rows per thread in the height pass

// Bilinear-upsampling table entries (patch_synthesis.py:261-274), one per
// (layer, haloed row) and (layer, haloed column) of the tile:
//   row: x = staged offset of coarse row ci (pre-multiplied by the row
//        pitch), y = pitch to row ci + 1 (0 on the last coarse row), w = k/f
//   col: x = staged coarse column cj, y = 1 (0 on the last column), w = k/f
struct UpEnt { short x, y; float w; };

__device__ __forceinline__ float lerpf(float a, float b, float w) { return a * (1.f - w) + b * w; }

__global__ void __launch_bounds__(256) compose_kernel(HsComposeArgs a) {
    __shared__ float hs_[CH][CH + 1];
    __shared__ HsLayer Ls[HS_MAX_BUCKETS];
    __shared__ UpEnt rtab[HS_MAX_BUCKETS][CH];
    __shared__ UpEnt ctab[HS_MAX_BUCKETS][CH];
    __shared__ int st_r0[HS_MAX_BUCKETS], st_c0[HS_MAX_BUCKETS], st_nr[HS_MAX_BUCKETS], st_nc[HS_MAX_BUCKETS],
        st_off[HS_MAX_BUCKETS];
    __shared__ float cs[CS_CAP];
    __shared__ float bgh[BG_CAP * BG_CAP], bgn[BG_CAP * BG_CAP * 3];
    __shared__ float row_d[CT], col_d[CT], row_fu[CT], col_fv[CT];
    __shared__ int row_q0[CT], row_q1[CT], col_q0[CT], col_q1[CT];
    __shared__ int bg_q[4];            // staged background row / col origin and extent (0 extent: not staged)
    __shared__ double red_s[8];
    __shared__ long long redc_s[8];

    const int* ti = a.tile_info + 3 * blockIdx.x;
    const int p = ti[0], i0 = ti[1], j0 = ti[2];
    const HsPatch P = a.patches[p];
    const int nb = a.nb;
    const bool have_bg = a.bg_height != nullptr;
    const int bm = a.bg_n - 1;
    const double inv_sp = have_bg ? 1.0 / a.bg_spacing : 0.0;
    if (a.frame_advance && blockIdx.x == 0 && threadIdx.x == 0) *a.frame_advance += 1;

    for (int b = threadIdx.x; b < nb; b += blockDim.x) Ls[b] = a.layers[P.layer_base + b];
    __syncthreads();
    // 1. staging plan: coarse-layer footprints and the background footprint
    const int ilo = max(i0 - 1, 0), ihi = min(i0 + CT, P.res - 1);
    const int jlo = max(j0 - 1, 0), jhi = min(j0 + CT, P.ny - 1);
    if (threadIdx.x == 0) {
        int off = 0;
        for (int b = 0; b < nb; ++b) {
            const HsLayer& L = Ls[b];
            st_off[b] = -1;
            st_r0[b] = st_c0[b] = 0;
            if (L.f == 1) continue;
            const int r0 = ilo / L.f, r1 = min(ihi / L.f + 1, L.ncx - 1);
            const int c0 = jlo / L.f, c1 = min(jhi / L.f + 1, L.ncy - 1);
            const int nr = r1 - r0 + 1, nc = c1 - c0 + 1;
            st_nr[b] = nr; st_nc[b] = nc;
            if (off + nr * nc <= CS_CAP) {
                st_off[b] = off; st_r0[b] = r0; st_c0[b] = c0;
                off += nr * nc;
            }
        }
        bg_q[0] = bg_q[1] = bg_q[2] = bg_q[3] = 0;
        if (have_bg) {
            // node positions are monotone: the footprint spans the first and last output row / column
            const int il = min(i0 + CT - 1, P.res - 1), jl = min(j0 + CT - 1, P.ny - 1);
            const long long qa = (long long)floor((P.x0 + (double)i0 * P.texel) * inv_sp);
            const long long qb = (long long)floor((P.x0 + (double)il * P.texel) * inv_sp) + 1;
            const long long qc = (long long)floor((P.y0 + (double)j0 * P.texel) * inv_sp);
            const long long qd = (long long)floor((P.y0 + (double)jl * P.texel) * inv_sp) + 1;
            if (qb - qa + 1 <= BG_CAP && qd - qc + 1 <= BG_CAP) {
                bg_q[0] = (int)(qa & bm); bg_q[1] = (int)(qb - qa + 1);
                bg_q[2] = (int)(qc & bm); bg_q[3] = (int)(qd - qc + 1);
            }
        }
    }
    __syncthreads();
    // 2. tables and staging (all global -> shared copies asynchronous)
    for (int e = threadIdx.x; e < nb * CH; e += blockDim.x) {
        const int b = e / CH, r = e - b * CH;
        const HsLayer& L = Ls[b];
        if (L.f == 1 || st_off[b] < 0) continue;
        const float inv_f = 1.f / (float)L.f;
        const int i = min(max(i0 - 1 + r, 0), P.res - 1);
        const int j = min(max(j0 - 1 + r, 0), P.ny - 1);
        const int ci = i / L.f, cj = j / L.f;
        const int nc = st_nc[b];
        rtab[b][r] = UpEnt{(short)(st_off[b] + (ci - st_r0[b]) * nc), (short)(ci + 1 < L.ncx ? nc : 0),
                           (float)(i - ci * L.f) * inv_f};
        ctab[b][r] = UpEnt{(short)(cj - st_c0[b]), (short)(cj + 1 < L.ncy ? 1 : 0), (float)(j - cj * L.f) * inv_f};
    }
    for (int b = 0; b < nb; ++b) {
        if (Ls[b].f == 1 || st_off[b] < 0) continue;
        const int r0 = st_r0[b], c0 = st_c0[b], nc = st_nc[b], n = st_nr[b] * nc;
        const float* S = a.smooth_layers + Ls[b].sm_off;
        const int ncy = Ls[b].ncy;
        for (int e = threadIdx.x; e < n; e += blockDim.x) {
            const int rr = e / nc, cc = e - rr * nc;
            cp_async4(cs + st_off[b] + e, S + (long long)(r0 + rr) * ncy + c0 + cc, true);
        }
    }
    const bool bg_staged = bg_q[1] > 0;
    if (bg_staged) {
        const int nr = bg_q[1], nc = bg_q[3];
        for (int e = threadIdx.x; e < nr * nc; e += blockDim.x) {
            const int rr = e / nc, cc = e - rr * nc;
            const long long g = (long long)((bg_q[0] + rr) & bm) * a.bg_n + ((bg_q[2] + cc) & bm);
            cp_async4(bgh + e, a.bg_height + g, true);
            if (a.bg_normal) {
                cp_async4(bgn + 3 * e, a.bg_normal + 3 * g, true);
                cp_async4(bgn + 3 * e + 1, a.bg_normal + 3 * g + 1, true);
                cp_async4(bgn + 3 * e + 2, a.bg_normal + 3 * g + 2, true);
            }
        }
    }
    for (int e = threadIdx.x; e < 2 * CT; e += blockDim.x) {
        const bool is_row = e < CT;
        const int k = is_row ? e : e - CT;
        const int idx = (is_row ? i0 : j0) + k;
        const double lo = is_row ? P.x0 : P.y0, hi = is_row ? P.x1 : P.y1;
        const double x = lo + (double)idx * P.texel;        // node positions (coupling.py:57-59)
        const float d = (float)fmin(x - lo, hi - x);        // boundary_depth (coupling.py:27-34)
        int q0 = 0, q1 = 0;
        float fr = 0.f;
        if (have_bg) {
            const double u = x * inv_sp;                     // background origin (0, 0)
            const double fl = floor(u);
            fr = (float)(u - fl);
            const long long q = (long long)fl;
            if (bg_staged) {                                 // relative to the staged footprint
                const long long base = is_row ? (long long)floor((P.x0 + (double)i0 * P.texel) * inv_sp)
                                              : (long long)floor((P.y0 + (double)j0 * P.texel) * inv_sp);
                q0 = (int)(q - base);
                q1 = q0 + 1;
            } else {
                q0 = (int)(q & bm);
                q1 = (q0 + 1) & bm;
            }
        }
        if (is_row) { row_d[k] = d; row_fu[k] = fr; row_q0[k] = q0; row_q1[k] = q1; }
        else        { col_d[k] = d; col_fv[k] = fr; col_q0[k] = q0; col_q1[k] = q1; }
    }
    cp_async_wait_all();
    __syncthreads();
    // 3. patch heights on the haloed tile: thread = (column c, block of RPT rows)
    {
        const int c = threadIdx.x % CH, rb = threadIdx.x / CH;
        const int j = j0 - 1 + c;
        const bool jok = j >= 0 && j < P.ny;
        float acc[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) acc[q] = 0.f;
        if (rb * RPT < CH) {
            for (int b = 0; b < nb; ++b) {
                const HsLayer& L = Ls[b];
                if (L.f == 1) {
                    const float* S = a.smooth_layers + L.sm_off + j;
                    float v[RPT];
#pragma unroll
                    for (int q = 0; q < RPT; ++q) {
                        const int i = i0 - 1 + rb * RPT + q;
                        v[q] = (jok && i >= 0 && i < P.res && rb * RPT + q < CH) ? S[(long long)i * L.ncy] : 0.f;
                    }
#pragma unroll
                    for (int q = 0; q < RPT; ++q) acc[q] = fmaf(L.gain, v[q], acc[q]);
                } else if (st_off[b] >= 0) {
                    const UpEnt ce = ctab[b][c];
#pragma unroll
                    for (int q = 0; q < RPT; ++q) {
                        const int r = min(rb * RPT + q, CH - 1);
                        const UpEnt re = rtab[b][r];
                        const float* S = cs + re.x + ce.x;
                        const float v = lerpf(lerpf(S[0], S[re.y], re.w), lerpf(S[ce.y], S[re.y + ce.y], re.w), ce.w);
                        acc[q] = fmaf(L.gain, v, acc[q]);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < RPT; ++q) {
                        const int i = i0 - 1 + rb * RPT + q;
                        if (jok && i >= 0 && i < P.res)
                            acc[q] = fmaf(L.gain, upsample_at(a.smooth_layers + L.sm_off, L, i, j), acc[q]);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const int r = rb * RPT + q, i = i0 - 1 + r;
                if (r < CH) hs_[r][c] = (jok && i >= 0 && i < P.res) ? acc[q] : 0.f;
            }
        }
    }
    __syncthreads();
    // 4. normals, blend, outputs
    const float inv_s = (float)(1.0 / P.texel), inv_2s = (float)(0.5 / P.texel);
    const float inv_margin = (float)(1.0 / P.margin);
    const int inset = max(1, (int)rint(P.margin / P.texel));
    double accv = 0.0;
    long long cnt = 0;
    const long long gb = P.grid_base;
    const int bn = a.bg_n, bnc = bg_q[3];
#pragma unroll 4
    for (int e = threadIdx.x; e < CT * CT; e += blockDim.x) {
        const int r = e / CT, c = e - r * CT;
        const int i = i0 + r, j = j0 + c;
        if (i >= P.res || j >= P.ny) continue;
        const float h = hs_[r + 1][c + 1];
        float hx, hy;
        if (i == 0) hx = (hs_[r + 2][c + 1] - h) * inv_s;
        else if (i == P.res - 1) hx = (h - hs_[r][c + 1]) * inv_s;
        else hx = (hs_[r + 2][c + 1] - hs_[r][c + 1]) * inv_2s;
        if (j == 0) hy = (hs_[r + 1][c + 2] - h) * inv_s;
        else if (j == P.ny - 1) hy = (h - hs_[r + 1][c]) * inv_s;
        else hy = (hs_[r + 1][c + 2] - hs_[r + 1][c]) * inv_2s;
        const float rn = rsqrtf(hx * hx + hy * hy + 1.f);
        const float pnx = -hx * rn, pny = -hy * rn, pnz = rn;
        const long long o = gb + (long long)i * P.ny + j;
        if (a.patch_height) a.patch_height[o] = h;
        if (a.patch_normal) { a.patch_normal[3 * o] = pnx; a.patch_normal[3 * o + 1] = pny; a.patch_normal[3 * o + 2] = pnz; }
        if (i >= inset && i < P.res - inset && j >= inset && j < P.ny - inset) {
            accv += (double)h * (double)h;
            ++cnt;
        }
        if (a.blend_mode) {
            float hb = 0.f, nx = 0.f, ny = 0.f, nz = 1.f;
            if (have_bg) {
                const float fu = row_fu[r], fv = col_fv[c];
                const float w00 = (1.f - fu) * (1.f - fv), w10 = fu * (1.f - fv), w01 = (1.f - fu) * fv, w11 = fu * fv;
                const float* B;
                const float* Nn;
                long long a00, a10, a01, a11;
                if (bg_staged) {
                    B = bgh; Nn = bgn;
                    a00 = row_q0[r] * bnc + col_q0[c]; a10 = row_q1[r] * bnc + col_q0[c];
                    a01 = row_q0[r] * bnc + col_q1[c]; a11 = row_q1[r] * bnc + col_q1[c];
                } else {
                    B = a.bg_height; Nn = a.bg_normal;
                    a00 = (long long)row_q0[r] * bn + col_q0[c]; a10 = (long long)row_q1[r] * bn + col_q0[c];
                    a01 = (long long)row_q0[r] * bn + col_q1[c]; a11 = (long long)row_q1[r] * bn + col_q1[c];
                }
                hb = B[a00] * w00 + B[a10] * w10 + B[a01] * w01 + B[a11] * w11;
                if (a.bg_normal) {
                    nx = Nn[3 * a00] * w00 + Nn[3 * a10] * w10 + Nn[3 * a01] * w01 + Nn[3 * a11] * w11;
                    ny = Nn[3 * a00 + 1] * w00 + Nn[3 * a10 + 1] * w10 + Nn[3 * a01 + 1] * w01 + Nn[3 * a11 + 1] * w11;
                    nz = Nn[3 * a00 + 2] * w00 + Nn[3 * a10 + 2] * w10 + Nn[3 * a01 + 2] * w01 + Nn[3 * a11 + 2] * w11;
                    const float rr = rsqrtf(nx * nx + ny * ny + nz * nz);
                    nx *= rr; ny *= rr; nz *= rr;
                }
            }
            const float d = fminf(row_d[r], col_d[c]);
            if (d > 0.f) {
                const float w = smoothstep01(d * inv_margin);
                hb = w * h + (1.f - w) * hb;
                const float mx = w * pnx + (1.f - w) * nx, my = w * pny + (1.f - w) * ny, mz = w * pnz + (1.f - w) * nz;
                const float rr = rsqrtf(mx * mx + my * my + mz * mz);
                nx = mx * rr; ny = my * rr; nz = mz * rr;
            }
            if (a.blend_height) a.blend_height[o] = hb;
            if (a.blend_normal) { a.blend_normal[3 * o] = nx; a.blend_normal[3 * o + 1] = ny; a.blend_normal[3 * o + 2] = nz; }
        }
    }
    if (a.interior_sumsq) {
        accv = warp_sum(accv);
        long long c2 = cnt;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c2 += __shfl_xor_sync(0xffffffffu, c2, o);
        if ((threadIdx.x & 31) == 0) { red_s[threadIdx.x >> 5] = accv; redc_s[threadIdx.x >> 5] = c2; }
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
    compose_kernel<<<a->total_tiles, 256, 0, as_stream(stream)>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}
