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
// One CTA per 30x30 output tile (+1-texel halo).  The coarse (f > 1)
// smoothed layers' footprint under the tile is staged in shared memory in
// one cp.async batch; f == 1 layers are read straight from L2 with coalesced
// rows.  Blend distances and background sample positions are formed per row
// / column in fp64 (world coordinates, as the reference) and applied per
// texel in fp32.
#include "synth_common.cuh"

namespace hs {

#ifdef HS_COMPOSE_TRACE
// per-phase globaltimer stamps of thread 0 of each CTA (tools/compose_trace.py)
__device__ unsigned long long g_trace[4096 * 8];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}
#define TRACE(k) do { if (threadIdx.x == 0 && blockIdx.x < 4096) g_trace[blockIdx.x * 8 + (k)] = gtime(); } while (0)
#else
#define TRACE(k) do {} while (0)
#endif

constexpr int CT = 30;            // output tile edge
constexpr int CH = CT + 2;        // haloed height tile (32): lane = haloed column
#ifndef HS_COMPOSE_NW
#define HS_COMPOSE_NW 4
#endif
constexpr int NW = HS_COMPOSE_NW;  // warps per tile (CTA)
constexpr int NT = 32 * NW;
constexpr int RPW = CH / NW;      // haloed rows per warp in the height pass
constexpr int BG_CAP = 8;         // staged background footprint per axis (+1 halo each side)
constexpr int TCP = 36;           // tc row pitch: float4 rows; 8 lanes on distinct rows -> distinct 4-bank groups
constexpr int TC_ROWS = 72;       // row-interpolated coarse rows per tile, all coarse layers (C3: <= 64)
constexpr int TC_CAP = TC_ROWS * TCP;
constexpr int CPT = CH / NW;      // haloed columns per thread in the coarse pass (thread = haloed row)

__device__ __forceinline__ float lerpf(float a, float b, float w) { return fmaf(w, b - a, a); }

// 16-byte shared load from a 32-bit shared-window address (keeps the tile's
// table base a plain register instead of a generic pointer)
__device__ __forceinline__ float4 lds128(unsigned addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

// floor(x / f) for 0 <= x < 2^22, f >= 1, from the fp32 reciprocal: the
// quotient of x + 1/2 sits >= 1/(2f) from an integer, far above the rounding
// error, so the truncation is exact
__device__ __forceinline__ int fdiv(int x, float inv_f) { return (int)(((float)x + 0.5f) * inv_f); }

__device__ __forceinline__ float3 bg_node_normal(const float* H, int n, long long i, long long j, float inv2s) {
    const int m = n - 1;
    const float hx = (H[((i + 1) & m) * n + (j & m)] - H[((i - 1) & m) * n + (j & m)]) * inv2s;
    const float hy = (H[(i & m) * n + ((j + 1) & m)] - H[(i & m) * n + ((j - 1) & m)]) * inv2s;
    const float r = rsqrtf(hx * hx + hy * hy + 1.f);
    return make_float3(-hx * r, -hy * r, r);
}

// per-tile plan of one smoothed layer
struct LayerPlan {
    long long sm_off;
    int f, ncx, ncy;
    int cr0, cc0;                     // coarse footprint origin (f > 1)
    int tc_off;                       // row table offset in tc (-1: not tabulated, rows read from global)
    float inv_f, gain;
};

// one row of the tc table: a coarse layer's footprint row (shared-window byte
// addresses, so the per-row work decodes nothing)
struct RowEnt {
    unsigned src;                     // first footprint element of the row in smooth_layers (< 2^32 floats)
    unsigned tca;                     // tc row
    unsigned cola;                    // the layer's column table | ncol << 24
    float inv_f;
};

struct TileSmem {
    union {
        float tc[TC_CAP];             // coarse rows of every layer interpolated at the 32 haloed columns
        float4 trow[CT][BG_CAP];      // background (h, nx, ny, nz) x-lerped per output row (epilogue)
    } u2;
    float hs[CH][CH + 1];             // haloed patch heights
    float bgh[(BG_CAP + 2) * (BG_CAP + 2)];   // background heights (+1 halo)
    float bgn[BG_CAP * BG_CAP * 3];           // background node normals (given ones)
    float row_d[CT], col_d[CT], col_fv[CT];
    int col_p0[CT];
    double red[NW];
    int redc[NW];
    int nc, n1, nrows;                // coarse layers, f == 1 layers (group members folded), tc rows
    // dynamic tail:
    //   LayerPlan pl[nb]       coarse layers from the front, f == 1 layers at the back (layer order)
    //   RowEnt rows[TC_ROWS]
    //   unsigned col[nb][32]   per coarse layer and haloed column: byte offsets in the footprint row of
    //                          its two columns (4 col | 4 (col + d1) << 8) | in-cell remainder << 16
    //   int2 rowp[nb][32]      per coarse layer and haloed row: tc offset of its coarse row | next-row step << 16
    //                          (-1: not tabulated), row weight g1
};

__host__ __device__ constexpr size_t compose_smem_bytes(int nb) {
    return sizeof(TileSmem) + (size_t)nb * sizeof(LayerPlan) + TC_ROWS * sizeof(RowEnt) + (size_t)nb * 32 * 4 +
           (size_t)nb * 32 * 8;
}

// background footprint of an output tile: first node and node count per
// axis (0 counts: not stageable, read from global)
__device__ __forceinline__ int4 bg_footprint(const HsPatch& P, int i0, int j0, double inv_sp, int bm) {
    const int il = min(i0 + CT - 1, P.res - 1), jl = min(j0 + CT - 1, P.ny - 1);
    const long long qa = (long long)floor((P.x0 + (double)i0 * P.texel) * inv_sp);
    const long long qb = (long long)floor((P.x0 + (double)il * P.texel) * inv_sp) + 1;
    const long long qc = (long long)floor((P.y0 + (double)j0 * P.texel) * inv_sp);
    const long long qd = (long long)floor((P.y0 + (double)jl * P.texel) * inv_sp) + 1;
    if (qb - qa + 1 <= BG_CAP && qd - qc + 1 <= BG_CAP)
        return make_int4((int)(qa & bm), (int)(qb - qa + 1), (int)(qc & bm), (int)(qd - qc + 1));
    return make_int4(0, 0, 0, 0);
}

// One CTA (4 warps) per 30 x 30 output tile (32 x 32 haloed heights).
//   heights  sum_b gain_b upsample_b (patch_synthesis.py:261-274, 301-313),
//            x-first bilinear: every coarse (f > 1) layer's footprint is
//            staged by one cp.async batch, its rows are interpolated once at
//            the 32 haloed columns (tc table), and each haloed texel then
//            sums two table entries per layer (lane = column, warp w = rows
//            8w..8w+7); f == 1 layers are read as coalesced rows
//   epilogue clamped FD normals (finish_field :323-340) and the smoothstep
//            blend against the periodic background at the patch nodes
//            (coupling.py:37-40, 120-141); the background bilinear is done
//            separably from per-row x-lerped tables
#ifndef HS_COMPOSE_MINB
#define HS_COMPOSE_MINB 9         // one wave of 30x30 tiles at C3 (9 x 148 >= 1225); 6..8 measured slower
#endif
__global__ void __launch_bounds__(NT, HS_COMPOSE_MINB) compose_kernel(HsComposeArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TileSmem& W = *reinterpret_cast<TileSmem*>(smem_raw);
    const int nb = a.nb;
    LayerPlan* const Wpl = reinterpret_cast<LayerPlan*>(smem_raw + sizeof(TileSmem));
    RowEnt* const Wrow = reinterpret_cast<RowEnt*>(Wpl + nb);
    unsigned* const Wcol = reinterpret_cast<unsigned*>(Wrow + TC_ROWS);
    int2* const Wrowp = reinterpret_cast<int2*>(Wcol + nb * 32);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int tile = blockIdx.x;
    TRACE(0);
    if (a.frame_advance && tile == 0 && tid == 0) *a.frame_advance += 1;
    const int* ti = a.tile_info + 3 * tile;
    const int p = ti[0], i0 = ti[1], j0 = ti[2];
    const HsPatch P = synth_view(a.patches[p]);   // the retracked rectangle (tracking patches)
    // the background only enters texels inside the blend band (w < 1): a tile
    // whose every output texel sits deeper than the margin skips it.  The
    // depth min(x - x0, x1 - x) is concave along a row / column, so its
    // minimum over the tile is at the first or last row / column.
    bool in_band = false;
    {
        const float inv_m = (float)(1.0 / P.margin);
        const int rl = min(CT, P.res - i0) - 1, cl = min(CT, P.ny - j0) - 1;
        const double xa = P.x0 + (double)i0 * P.texel, xb = P.x0 + (double)(i0 + rl) * P.texel;
        const double ya = P.y0 + (double)j0 * P.texel, yb = P.y0 + (double)(j0 + cl) * P.texel;
        const float dx = fminf((float)fmin(xa - P.x0, P.x1 - xa), (float)fmin(xb - P.x0, P.x1 - xb));
        const float dy = fminf((float)fmin(ya - P.y0, P.y1 - ya), (float)fmin(yb - P.y0, P.y1 - yb));
        in_band = fminf(dx, dy) * inv_m < 1.f;
    }
    const bool have_bg = a.bg_height != nullptr && a.blend_mode && in_band;
    const int bm = a.bg_n - 1;
    const double inv_sp = have_bg ? 1.0 / a.bg_spacing : 0.0;
    const int4 bq = have_bg ? bg_footprint(P, i0, j0, inv_sp, bm) : make_int4(0, 0, 0, 0);
    const bool bg_staged = bq.y > 0;
    const bool own_normals = a.bg_normal == nullptr;

    const int ib = i0 - 1;                         // haloed row 0 / column 0
    const int jb = j0 - 1;
    const int ilo = min(max(ib, 0), P.res - 1), ihi = min(max(ib + CH - 1, 0), P.res - 1);
    const int jlo = min(max(jb, 0), P.ny - 1), jhi = min(max(jb + CH - 1, 0), P.ny - 1);

    if (wid == 0 || wid >= 2) {
        // layer plans (lane b: layer b).  Layer-group members (HsLayer.group < 0)
        // have no crop of their own: their smoothed sum sits in the group's
        // first layer, already gain-weighted
        LayerPlan pl{};
        int nr = 0, ncol = 0;
        bool coarse = false, fine = false;
        if (lane < nb) {
            const HsLayer L = a.layers[P.layer_base + lane];
            coarse = L.group >= 0 && L.f > 1;
            fine = L.group >= 0 && L.f == 1;
            pl.sm_off = L.sm_off; pl.f = L.f; pl.ncx = L.ncx; pl.ncy = L.ncy;
            pl.inv_f = 1.f / (float)L.f; pl.gain = L.group > 1 ? 1.f : L.gain;
            if (coarse) {
                pl.cr0 = ilo / L.f;
                nr = min(ihi / L.f + 1, L.ncx - 1) - pl.cr0 + 1;
                pl.cc0 = jlo / L.f;
                ncol = min(jhi / L.f + 1, L.ncy - 1) - pl.cc0 + 1;
            }
        }
        const unsigned mc = __ballot_sync(0xffffffffu, coarse);
        const unsigned lt = (1u << lane) - 1u;
        const int cix = __popc(mc & lt);
        if (wid == 0) {
            // a layer is tabulated only if every coarse layer before it was
            const int inc = warp_incl_scan(nr, lane);
            const bool fits = coarse && inc <= TC_ROWS;
            pl.tc_off = fits ? (inc - nr) * TCP : -1;
            const unsigned m1 = __ballot_sync(0xffffffffu, fine);
            if (coarse) Wpl[cix] = pl;
            if (fine) Wpl[nb - __popc(m1) + __popc(m1 & lt)] = pl;
            const int nrows = __reduce_max_sync(0xffffffffu, fits ? inc : 0);
            if (lane == 0) { W.nc = __popc(mc); W.n1 = __popc(m1); W.nrows = nrows; }
            if (fits) {
                RowEnt e;
                e.inv_f = pl.inv_f;
                e.cola = (unsigned)__cvta_generic_to_shared(Wcol + cix * 32) | ((unsigned)ncol << 24);
                const unsigned tca = (unsigned)__cvta_generic_to_shared(W.u2.tc + pl.tc_off);
                for (int r = 0; r < nr; ++r) {
                    e.src = (unsigned)(pl.sm_off + (long long)(pl.cr0 + r) * pl.ncy + pl.cc0);
                    e.tca = tca + (unsigned)(4 * TCP * r);
                    Wrow[inc - nr + r] = e;
                }
            }
        } else {
            // column table (warps 2 and 3: alternate coarse layers; lane = haloed
            // column): the footprint column, the clamped step to the next one and
            // the in-cell remainder (x-first bilinear, patch_synthesis.py:270-273)
            const int jj = min(max(jb + lane, 0), P.ny - 1);
            unsigned m = mc;
            for (int k = 0; m; ++k) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                const int f = __shfl_sync(0xffffffffu, pl.f, b), ncy = __shfl_sync(0xffffffffu, pl.ncy, b);
                const int cc0 = __shfl_sync(0xffffffffu, pl.cc0, b);
                const float inv_f = __shfl_sync(0xffffffffu, pl.inv_f, b);
                if ((k & 1) == (wid & 1)) {
                    const int cj = fdiv(jj, inv_f);
                    const int d1 = min(cj + 1, ncy - 1) - cj;
                    Wcol[k * 32 + lane] = (unsigned)(4 * (cj - cc0)) | ((unsigned)(4 * (cj - cc0 + d1)) << 8) |
                                          ((unsigned)(jj - cj * f) << 16);
                }
            }
        }
    } else if (lane < CT) {
        // per output row / column (fp64 world coordinates, coupling.py:57-59): boundary
        // depth (coupling.py:27-34) and the column-side background lerp
        const double yy = P.y0 + (double)(j0 + lane) * P.texel;
        W.col_d[lane] = (float)fmin(yy - P.y0, P.y1 - yy);
        const double xx = P.x0 + (double)(i0 + lane) * P.texel;
        W.row_d[lane] = (float)fmin(xx - P.x0, P.x1 - xx);
        if (have_bg) {
            const double v = yy * inv_sp, fl = floor(v);
            W.col_fv[lane] = (float)(v - fl);
            const long long q = (long long)fl;
            W.col_p0[lane] = bg_staged ? (int)(q - (long long)floor((P.y0 + (double)j0 * P.texel) * inv_sp)) : (int)(q & bm);
        }
    }
    // background footprint (+1 halo) by cp.async; independent of the plans
    if (bg_staged) {
        const int nr = bq.y + 2, nc = bq.w + 2;
        for (int e = tid; e < nr * nc; e += NT) {
            const int rr = e / nc, cc = e - rr * nc;
            const long long g = (long long)((bq.x - 1 + rr) & bm) * a.bg_n + ((bq.z - 1 + cc) & bm);
            cp_async4(W.bgh + e, a.bg_height + g, true);
        }
        if (!own_normals) {
            for (int e = tid; e < bq.y * bq.w; e += NT) {
                const int rr = e / bq.w, cc = e - rr * bq.w;
                const long long g = 3 * ((long long)((bq.x + rr) & bm) * a.bg_n + ((bq.z + cc) & bm));
                cp_async4(W.bgn + 3 * e, a.bg_normal + g, true);
                cp_async4(W.bgn + 3 * e + 1, a.bg_normal + g + 1, true);
                cp_async4(W.bgn + 3 * e + 2, a.bg_normal + g + 2, true);
            }
        }
    }
    __syncthreads();
    TRACE(1);
    const int nc = W.nc, n1 = W.n1, nrows = W.nrows;
    const float* __restrict__ SL = a.smooth_layers;
    // tc rows of this warp (wid, wid + NW, ...): each footprint row is staged
    // by cp.async into the start of its own tc row (lane = footprint column),
    // then lerped in place at the 32 haloed columns:
    //   tc[row][c] = lerp(row[col(c)], row[col(c) + d1], rem(c) / f)
    const unsigned lane4 = 4u * (unsigned)lane;
    for (int g = wid; g < nrows; g += NW) {
        const RowEnt e = Wrow[g];
        if (lane < (int)(e.cola >> 24)) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(e.tca + lane4), "l"(SL + e.src + lane));
        }
    }
    // row table: per coarse layer and haloed row, the tc row offset, the clamped
    // step to the next coarse row and the row weight
    for (int e = tid; e < nc * 32; e += NT) {
        const LayerPlan& L = Wpl[e >> 5];
        const int ii = min(max(ib + (e & 31), 0), P.res - 1);
        const int ci = fdiv(ii, L.inv_f);
        const float g1 = L.gain * ((float)(ii - ci * L.f) * L.inv_f);
        const int d1 = min(ci + 1, L.ncx - 1) - ci;
        Wrowp[e] = make_int2(L.tc_off >= 0 ? (L.tc_off + (ci - L.cr0) * TCP) | (d1 << 16) : -1, __float_as_int(g1));
    }
    // f == 1 layers straight into the haloed heights (lane = haloed column, coalesced rows)
    {
        const int c = lane;
        const int j = min(max(jb + c, 0), P.ny - 1);
        const int qb = RPW * wid;                  // first haloed row of this warp
        float acc[RPW];
#pragma unroll
        for (int k = 0; k < RPW; ++k) acc[k] = 0.f;
        for (int b = nb - n1; b < nb; ++b) {
            const LayerPlan& L = Wpl[b];
            const float* Sg = SL + L.sm_off;
            float u[RPW];
#pragma unroll
            for (int k = 0; k < RPW; ++k) u[k] = Sg[min(max(ib + qb + k, 0), P.res - 1) * L.ncy + j];
#pragma unroll
            for (int k = 0; k < RPW; ++k) acc[k] = fmaf(L.gain, u[k], acc[k]);
        }
        const int jr = jb + c;
        const bool jok = jr >= 0 && jr < P.ny;
#pragma unroll
        for (int k = 0; k < RPW; ++k) {
            const int ii = ib + qb + k;
            W.hs[qb + k][c] = (jok && ii >= 0 && ii < P.res) ? acc[k] : 0.f;
        }
    }
    cp_async_wait_all();                           // this warp's rows (and the background footprint)
    __syncwarp();
    TRACE(2);
    for (int g = wid; g < nrows; g += NW) {
        const RowEnt e = Wrow[g];
        unsigned pk;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(pk) : "r"((e.cola & 0xffffffu) + lane4));
        float x0, x1;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x0) : "r"(e.tca + (pk & 0xffu)));
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x1) : "r"(e.tca + ((pk >> 8) & 0xffu)));
        __syncwarp();
        const float v = lerpf(x0, x1, (float)(pk >> 16) * e.inv_f);
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(e.tca + lane4), "f"(v) : "memory");
    }
    __syncthreads();
    TRACE(3);
    // ---- coarse layers: thread = haloed row q, columns c0 .. c0+7; per layer
    // two float4 pairs of table reads and 16 FMAs ----
    {
        const int q = lane, c0 = CPT * wid;
        const unsigned tcs = (unsigned)__cvta_generic_to_shared(W.u2.tc) + 4u * (unsigned)c0;
        float h[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) h[k] = W.hs[q][c0 + k];
        for (int b = 0; b < nc; ++b) {
            const int2 rp = Wrowp[b * 32 + q];
            const float gain = Wpl[b].gain;
            const float g1 = __int_as_float(rp.y), g0 = gain - g1;
            if (rp.x >= 0) {
                const unsigned s0 = tcs + 4u * (unsigned)(rp.x & 0xffff), s1 = s0 + (unsigned)(4 * TCP) * (unsigned)(rp.x >> 16);
                const float4 a0 = lds128(s0), a1 = lds128(s0 + 16u), b0 = lds128(s1), b1 = lds128(s1 + 16u);
                const float t0[CPT] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float t1[CPT] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int k = 0; k < CPT; ++k) h[k] = fmaf(g0, t0[k], fmaf(g1, t1[k], h[k]));
            } else {                               // layer not tabulated: rows from global (rare)
                const LayerPlan& L = Wpl[b];
                const int ii = min(max(ib + q, 0), P.res - 1);
                const int ci = fdiv(ii, L.inv_f), ci1 = min(ci + 1, L.ncx - 1);
                const float* R0 = SL + L.sm_off + (long long)ci * L.ncy;
                const float* R1 = SL + L.sm_off + (long long)ci1 * L.ncy;
#pragma unroll
                for (int k = 0; k < CPT; ++k) {
                    const int jj = min(max(jb + c0 + k, 0), P.ny - 1);
                    const int cj = fdiv(jj, L.inv_f), cj1 = min(cj + 1, L.ncy - 1);
                    const float wj = (float)(jj - cj * L.f) * L.inv_f;
                    h[k] = fmaf(g0, lerpf(R0[cj], R0[cj1], wj), fmaf(g1, lerpf(R1[cj], R1[cj1], wj), h[k]));
                }
            }
        }
        const bool iok = ib + q >= 0 && ib + q < P.res;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const int jr = jb + c0 + k;
            W.hs[q][c0 + k] = (iok && jr >= 0 && jr < P.ny) ? h[k] : 0.f;
        }
    }
    __syncthreads();                               // tc dead: trow may overwrite it
    TRACE(4);
    // background: node normals (given, or from the staged heights), x-lerped per output row
    const float inv2sp = have_bg ? (float)(0.5 / a.bg_spacing) : 0.f;
    if (bg_staged) {
        const int ncs = bq.w + 2;
        const long long base_x = (long long)floor((P.x0 + (double)i0 * P.texel) * inv_sp);
        for (int e = tid; e < CT * bq.w; e += NT) {
            const int rr = e / bq.w, pc = e - rr * bq.w;
            const double u = (P.x0 + (double)(i0 + rr) * P.texel) * inv_sp, fl = floor(u);
            const float fu = (float)(u - fl);
            const int q0 = (int)((long long)fl - base_x);
            float4 n0, n1;
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const int qr = q0 + s;
                float4 v;
                v.x = W.bgh[(qr + 1) * ncs + pc + 1];
                if (own_normals) {
                    const float hx = (W.bgh[(qr + 2) * ncs + pc + 1] - W.bgh[qr * ncs + pc + 1]) * inv2sp;
                    const float hy = (W.bgh[(qr + 1) * ncs + pc + 2] - W.bgh[(qr + 1) * ncs + pc]) * inv2sp;
                    const float rn = rsqrtf(hx * hx + hy * hy + 1.f);
                    v.y = -hx * rn; v.z = -hy * rn; v.w = rn;
                } else {
                    const int ai = 3 * (qr * bq.w + pc);
                    v.y = W.bgn[ai]; v.z = W.bgn[ai + 1]; v.w = W.bgn[ai + 2];
                }
                if (s == 0) n0 = v; else n1 = v;
            }
            W.u2.trow[rr][pc] = make_float4(lerpf(n0.x, n1.x, fu), lerpf(n0.y, n1.y, fu), lerpf(n0.z, n1.z, fu),
                                            lerpf(n0.w, n1.w, fu));
        }
    }
    __syncthreads();
    TRACE(5);

    // ---- normals, blend, outputs ----
    const float inv_s = (float)(1.0 / P.texel), inv_2s = (float)(0.5 / P.texel);
    const float inv_margin = (float)(1.0 / P.margin);
    const int inset = max(1, (int)rint(P.margin / P.texel));
    double accv = 0.0;
    int cnt = 0;
    const long long gb = P.grid_base;
    const int bn = a.bg_n;
    const bool pure = !in_band && a.bg_height != nullptr && a.blend_mode && i0 >= inset && j0 >= inset &&
                      i0 + CT <= P.res - inset && j0 + CT <= P.ny - inset;
    if (pure) {
        // deep interior tile: every texel deeper than the margin (blend weight
        // 1: the blend is the patch), inside the variance inset, and off the
        // border (central differences) -- no per-texel tests at all
        for (int e = tid; e < CT * CT; e += NT) {
            const int rr = e / CT, cc = e - rr * CT;
            const int ii = i0 + rr, jj = j0 + cc;
            const float h = W.hs[rr + 1][cc + 1];
            const float hx = (W.hs[rr + 2][cc + 1] - W.hs[rr][cc + 1]) * inv_2s;
            const float hy = (W.hs[rr + 1][cc + 2] - W.hs[rr + 1][cc]) * inv_2s;
            const float rn = rsqrtf(hx * hx + hy * hy + 1.f);
            const float pnx = -hx * rn, pny = -hy * rn, pnz = rn;
            const int o = (int)gb + ii * P.ny + jj;
            if (a.patch_height) a.patch_height[o] = h;
            if (a.patch_normal) { a.patch_normal[3 * o] = pnx; a.patch_normal[3 * o + 1] = pny; a.patch_normal[3 * o + 2] = pnz; }
            accv = fma((double)h, (double)h, accv);
            ++cnt;
            if (a.blend_height) a.blend_height[o] = h;
            if (a.blend_normal) { a.blend_normal[3 * o] = pnx; a.blend_normal[3 * o + 1] = pny; a.blend_normal[3 * o + 2] = pnz; }
        }
    } else if (!have_bg && a.blend_mode) {
        // interior tile (every texel deeper than the margin, or no background):
        // the blend is the patch itself -- a light loop without the background
        // state, so the common case carries no spilled registers
        const bool bg_any = a.bg_height != nullptr;
        for (int e = tid; e < CT * CT; e += NT) {
            const int rr = e / CT, cc = e - rr * CT;
            const int ii = i0 + rr, jj = j0 + cc;
            if (ii >= P.res || jj >= P.ny) continue;
            const float h = W.hs[rr + 1][cc + 1];
            const float hu = ii == P.res - 1 ? h : W.hs[rr + 2][cc + 1];
            const float hd = ii == 0 ? h : W.hs[rr][cc + 1];
            const float hr = jj == P.ny - 1 ? h : W.hs[rr + 1][cc + 2];
            const float hl = jj == 0 ? h : W.hs[rr + 1][cc];
            const float hx = (hu - hd) * ((ii == 0 || ii == P.res - 1) ? inv_s : inv_2s);
            const float hy = (hr - hl) * ((jj == 0 || jj == P.ny - 1) ? inv_s : inv_2s);
            const float rn = rsqrtf(hx * hx + hy * hy + 1.f);
            const float pnx = -hx * rn, pny = -hy * rn, pnz = rn;
            const int o = (int)gb + ii * P.ny + jj;
            if (a.patch_height) a.patch_height[o] = h;
            if (a.patch_normal) { a.patch_normal[3 * o] = pnx; a.patch_normal[3 * o + 1] = pny; a.patch_normal[3 * o + 2] = pnz; }
            if (ii >= inset && ii < P.res - inset && jj >= inset && jj < P.ny - inset) {
                accv = fma((double)h, (double)h, accv);
                ++cnt;
            }
            float hb = h, nx = pnx, ny = pny, nz = pnz;
            const float d = fminf(W.row_d[rr], W.col_d[cc]);
            if (!bg_any || d * inv_margin < 1.f) {     // no background at all: blend with the flat sea
                const float w = d > 0.f ? smoothstep01(d * inv_margin) : 0.f;
                if (w < 1.f) {
                    hb = lerpf(0.f, h, w);
                    const float mx = lerpf(0.f, pnx, w), my = lerpf(0.f, pny, w), mz = lerpf(1.f, pnz, w);
                    const float r2 = rsqrtf(mx * mx + my * my + mz * mz);
                    nx = mx * r2; ny = my * r2; nz = mz * r2;
                    if (d <= 0.f) { hb = 0.f; nx = 0.f; ny = 0.f; nz = 1.f; }
                }
            }
            if (a.blend_height) a.blend_height[o] = hb;
            if (a.blend_normal) { a.blend_normal[3 * o] = nx; a.blend_normal[3 * o + 1] = ny; a.blend_normal[3 * o + 2] = nz; }
        }
    } else
    for (int e = tid; e < CT * CT; e += NT) {
        const int rr = e / CT, cc = e - rr * CT;
        const int ii = i0 + rr, jj = j0 + cc;
        if (ii >= P.res || jj >= P.ny) continue;
        const float h = W.hs[rr + 1][cc + 1];
        const float hu = ii == P.res - 1 ? h : W.hs[rr + 2][cc + 1];
        const float hd = ii == 0 ? h : W.hs[rr][cc + 1];
        const float hr = jj == P.ny - 1 ? h : W.hs[rr + 1][cc + 2];
        const float hl = jj == 0 ? h : W.hs[rr + 1][cc];
        const float hx = (hu - hd) * ((ii == 0 || ii == P.res - 1) ? inv_s : inv_2s);
        const float hy = (hr - hl) * ((jj == 0 || jj == P.ny - 1) ? inv_s : inv_2s);
        const float rn = rsqrtf(hx * hx + hy * hy + 1.f);
        const float pnx = -hx * rn, pny = -hy * rn, pnz = rn;
        const int o = (int)gb + ii * P.ny + jj;         // 32-bit: the harness keeps 3 x texels < 2^31
        if (a.patch_height) a.patch_height[o] = h;
        if (a.patch_normal) { a.patch_normal[3 * o] = pnx; a.patch_normal[3 * o + 1] = pny; a.patch_normal[3 * o + 2] = pnz; }
        if (ii >= inset && ii < P.res - inset && jj >= inset && jj < P.ny - inset) {
            accv = fma((double)h, (double)h, accv);
            ++cnt;
        }
        if (a.blend_mode) {
            const float d = fminf(W.row_d[rr], W.col_d[cc]);
            const float w = d > 0.f ? smoothstep01(d * inv_margin) : 0.f;
            float hb = h, nx = pnx, ny = pny, nz = pnz;    // w == 1: the patch alone (coupling.py:37-40)
            if (w < 1.f) {
            hb = 0.f; nx = 0.f; ny = 0.f; nz = 1.f;
            if (have_bg) {
                const float fv = W.col_fv[cc];
                if (bg_staged) {
                    const int p0 = W.col_p0[cc];
                    const float4 t0 = W.u2.trow[rr][p0], t1 = W.u2.trow[rr][p0 + 1];
                    hb = lerpf(t0.x, t1.x, fv);
                    nx = lerpf(t0.y, t1.y, fv); ny = lerpf(t0.z, t1.z, fv); nz = lerpf(t0.w, t1.w, fv);
                } else {
                    const double u = (P.x0 + (double)ii * P.texel) * inv_sp, fl = floor(u);
                    const float fu = (float)(u - fl);
                    const int q0 = (int)((long long)fl & bm), q1 = (q0 + 1) & bm;
                    const int p0 = W.col_p0[cc], p1 = (p0 + 1) & bm;
                    const float w00 = (1.f - fu) * (1.f - fv), w10 = fu * (1.f - fv), w01 = (1.f - fu) * fv, w11 = fu * fv;
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
                const float r2 = rsqrtf(nx * nx + ny * ny + nz * nz);
                nx *= r2; ny *= r2; nz *= r2;
                if (a.n_extra_bg > 0)                 // summed cascades (fft.cascades)
                    add_cascades(a.n_extra_bg, a.extra_bg, P.x0 + (double)ii * P.texel, P.y0 + (double)jj * P.texel,
                                 hb, nx, ny, nz);
            }
            if (d > 0.f) {
                hb = lerpf(hb, h, w);
                const float mx = lerpf(nx, pnx, w), my = lerpf(ny, pny, w), mz = lerpf(nz, pnz, w);
                const float r2 = rsqrtf(mx * mx + my * my + mz * mz);
                nx = mx * r2; ny = my * r2; nz = mz * r2;
            }
            }
            if (a.blend_height) a.blend_height[o] = hb;
            if (a.blend_normal) { a.blend_normal[3 * o] = nx; a.blend_normal[3 * o + 1] = ny; a.blend_normal[3 * o + 2] = nz; }
        }
    }
    TRACE(7);
    // FFT-resolution composite (stitched_heights, harness.py:219-241): the
    // composite nodes whose patch-grid row/column falls in this tile, strictly
    // inside the patch, get w h_patch + (1 - w) h_bg (the patch step of
    // sample_surface_heights / SurfaceSampler._raw) from the staged tile; the
    // grid already holds the background (every other node keeps it)
    if (a.composite && a.bg_height) {
        const double sp = a.bg_spacing;
        const int n = a.bg_n;
        const double xa = P.x0 + (double)i0 * P.texel, xb = P.x0 + (double)(i0 + CT) * P.texel;
        const double ya = P.y0 + (double)j0 * P.texel, yb = P.y0 + (double)(j0 + CT) * P.texel;
        const int ga0 = max((int)ceil(xa / sp), 0), ga1 = min((int)ceil(xb / sp), n);
        const int gb0 = max((int)ceil(ya / sp), 0), gb1 = min((int)ceil(yb / sp), n);
        const int cols = gb1 - gb0, tot = max(ga1 - ga0, 0) * max(cols, 0);
        for (int e = tid; e < tot; e += NT) {
            const int gi = ga0 + e / cols, gj = gb0 + e % cols;
            const double x = gi * sp, y = gj * sp;
            const double d = fmin(fmin(x - P.x0, P.x1 - x), fmin(y - P.y0, P.y1 - y));
            if (!(d > 0.0)) continue;
            const double t = fmin(fmax(d / P.margin, 0.0), 1.0);
            const float w = (float)(t * t * (3.0 - 2.0 * t));
            const double u = fmin(fmax((x - P.x0) / P.texel, 0.0), (double)(P.res - 1));
            const double v = fmin(fmax((y - P.y0) / P.texel, 0.0), (double)(P.ny - 1));
            const int i = min(max(min((int)u, P.res - 2), ib), ib + CH - 2);
            const int j = min(max(min((int)v, P.ny - 2), jb), jb + CH - 2);
            const float fu = (float)(u - i), fv = (float)(v - j);
            const float w00 = (1.f - fu) * (1.f - fv), w10 = fu * (1.f - fv), w01 = (1.f - fu) * fv, w11 = fu * fv;
            const int r = i - ib, q = j - jb;
            const float hp = W.hs[r][q] * w00 + W.hs[r + 1][q] * w10 + W.hs[r][q + 1] * w01 + W.hs[r + 1][q + 1] * w11;
            float* c = a.composite + (long long)gi * n + gj;
            *c = w * hp + (1.f - w) * *c;
        }
    }
    TRACE(6);
    if (a.interior_sumsq) {
        accv = warp_sum(accv);
        cnt = warp_sum(cnt);
        if (lane == 0) { W.red[wid] = accv; W.redc[wid] = cnt; }
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            int n = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) { s += W.red[w]; n += W.redc[w]; }
            if (n) {
                sumsq_add(&a.interior_sumsq[p], s, a.fixed_point);
                if (a.interior_count) atomicAdd((unsigned long long*)&a.interior_count[p], (unsigned long long)n);
            }
        }
    }
}

}  // namespace hs

using namespace hs;

#ifdef HS_COMPOSE_TRACE
extern "C" HS_API int hs_debug_trace(void* dst) {
    return (int)cudaMemcpyFromSymbol(dst, hs::g_trace, sizeof(hs::g_trace));
}
#endif

namespace hs {
// the whole 228 KB as shared memory (9 tiles per SM), once per device
int compose_configure() {
    static PerDevice<bool> carve_done{};
    bool& carve = carve_done.get();
    if (!carve) {
        HS_CUDA(cudaFuncSetAttribute(compose_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        carve = true;
    }
    return 0;
}
}  // namespace hs

extern "C" int hs_compose(const HsComposeArgs* a, void* stream) {
    HS_EXP_SKIP_POINT("compose");
    HS_CHECK_ARG(a != nullptr, "hs_compose: null args");
    HS_CHECK_ARG(a->nb >= 1 && a->nb <= HS_MAX_BUCKETS, "hs_compose: nb out of range");
    if (a->total_tiles == 0) {
        if (a->frame_advance) HS_CHECK_ARG(false, "hs_compose: frame_advance needs at least one tile");
        return 0;
    }
    HS_CHECK_ARG(a->patches && a->layers && a->smooth_layers && a->tile_info, "hs_compose: missing buffer");
    HS_CHECK_ARG(!a->blend_mode || a->bg_height == nullptr || (a->bg_n >= 2 && (a->bg_n & (a->bg_n - 1)) == 0),
                 "hs_compose: background size must be a power of two");
    if (int rc = compose_configure()) return rc;
    compose_kernel<<<a->total_tiles, NT, compose_smem_bytes(a->nb), as_stream(stream)>>>(*a);
    HS_LAUNCH_CHECK();
    return 0;
}
