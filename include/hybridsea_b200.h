/*
 * hybridsea_b200 -- C ABI of the B200-native hybrid ocean step.
 *
 * The reference (`hybridsea` 0.1.0, pure Python + numpy) has no FFI layer:
 * its operator API is the set of Python functions re-exported by
 * `pkg/src/hybridsea/__init__.py:8-59`.  Each entry point below replaces one
 * of those functions on the per-frame hot path; the
 * Python package `paper_2511_02852_b200` keeps the reference signatures and
 * calls these through ctypes.
 *
 * Conventions
 *   - every pointer named in an args struct is a DEVICE pointer unless the
 *     comment says "host"; the caller (PyTorch's caching allocator) owns all
 *     memory, kernels never allocate;
 *   - `stream` is a cudaStream_t passed as void*; every call only enqueues
 *     work (memsets + kernels) on it, never synchronises, so a whole frame is
 *     CUDA-graph capturable;
 *   - return 0 on success, nonzero on a host-side validation or launch error;
 *     hs_last_error() then describes it (thread-local).
 *   - arrays of per-patch / per-bucket descriptors are device arrays of the
 *     structs below (plain-old-data, 8-byte aligned).
 */
#ifndef HYBRIDSEA_B200_H
#define HYBRIDSEA_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define HS_API __attribute__((visibility("default")))
#else
#define HS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define HS_ABI_VERSION 1
#define HS_MAX_BUCKETS 32
#define HS_MAX_PATCHES 256

/* status word bits written by kernels (device int, checked by the host
 * outside the captured graph) */
#define HS_STATUS_POOL_OVERFLOW  1
#define HS_STATUS_STAGE_OVERFLOW 2
#define HS_STATUS_NONFINITE      4
#define HS_STATUS_BOX_OVERFLOW   8   /* a composite box exceeded HsBoxArgs' capacity */

/* Deterministic mode (fixed_point = 1 in the args below).  Every float sum
 * whose order depends on scheduling is taken in int64 fixed point, whose
 * addition is associative, so reruns are byte-identical (the reference's
 * determinism contract, test_acceptance.py:293-311):
 *   raw layers   value * 2^HS_FIXED_SPLAT_BITS, one int64 per raw float slot
 *                (same element offsets); hs_fixed_to_float turns them into the
 *                float raw layers hs_smooth reads;
 *   e_out        J * 2^HS_FIXED_ENERGY_BITS (the double slots hold int64);
 *   sumsq        m^2 * 2^HS_FIXED_SUMSQ_BITS (hs_fft_evolve.sumsq,
 *                hs_compose.interior_sumsq).                                 */
#define HS_FIXED_SPLAT_BITS 32
#define HS_FIXED_ENERGY_BITS 24
#define HS_FIXED_SUMSQ_BITS 32

HS_API int hs_abi_version(void);
HS_API const char* hs_last_error(void);
/* sizeof of ABI struct `which` (0 HsBucket, 1 HsPatch, 2 HsLayer, 3 HsPool,
 * 4..12 the args structs in declaration order); -1 if unknown */
HS_API int hs_struct_size(int which);

/* One-time configuration of the current device's kernels (shared-memory
 * limits, carve-out, persistent-grid occupancy).  Entry points do this
 * lazily on first use, but attribute calls made inside a CUDA-graph capture
 * invalidate the capture: call this once per device before capturing.       */
HS_API int hs_configure_device(void);

/* A non-blocking stream of the given priority on the current device (and its
 * destruction): the streams a frame graph forks onto and is captured on. */
HS_API int hs_stream_create(void** stream, int priority);
HS_API int hs_stream_destroy(void* stream);

/* ------------------------------------------------------------------------ */
/* Per-bucket constants (replaces the BucketTable array views,
 * reference spectrum.py:233-257).                                           */
typedef struct {
    double omega;      /* representative frequency (rad/s) */
    double width;      /* bucket width delta_omega */
    double radius;     /* pi g / omega^2 */
    double speed;      /* g / omega */
    double s1d;        /* S_J(omega) (spectrum.py:108-121), fp64 */
    double spread_s;   /* cos-2s exponent s at omega */
    double spread_c;   /* C(s) normalisation */
    double pad;
} HsBucket;

/* Axis-aligned patch rectangle + its pool / grid / layer bookkeeping
 * (replaces PatchRegion, particles.py:43-74, and PatchState, harness.py:49-62). */
typedef struct {
    double x0, y0;       /* min corner (world, m) */
    double x1, y1;       /* max corner = min + (l1, l2) */
    double l1, l2;       /* side lengths */
    double margin;       /* blend band width */
    double texel;        /* l1 / (res - 1) */
    long long pool_base; /* element offset of this patch's pool region */
    long long stage_base;/* element offset of this patch's staging region */
    long long grid_base; /* element offset of this patch's (res x ny) grids */
    int pool_capacity;
    int stage_capacity;
    int res, ny;         /* node grid: res along x, ny along y */
    int layer_base;      /* first HsLayer of this patch */
    int track;           /* source this patch follows (harness.py:115-123), -1: static */
    double sx0, sy0;     /* synthesis origin: where this frame's layers, heights and blend
                            sit.  Equal to (x0, y0) except for a tracking patch, whose region
                            moves onto its source AFTER injection, advection and emission
                            (hs_track / hs_emit); x0..y1 is the region those stages use */
} HsPatch;

/* One per (patch, bucket) synthesis layer (LayerPlan, patch_synthesis.py:227-258). */
typedef struct {
    long long raw_off;   /* float offset of the padded raw layer (wx rows of raw_pitch), multiple of 4 */
    long long sm_off;    /* float offset of the smoothed crop (ncx*ncy) */
    int f;               /* decimation factor */
    int H;               /* kernel half width (taps 2H+1) */
    int pad;             /* H + 1 */
    int ncx, ncy;        /* coarse node grid (crop) */
    int wx, wy;          /* padded layer dims ncx+2pad, ncy+2pad */
    int taps_off;        /* offset into the taps array */
    float gain;          /* output gain */
    int mid_off;         /* float offset into HsSmoothArgs.mid (wide kernels), -1 otherwise */
    int raw_pitch;       /* raw row pitch in floats: >= wy, multiple of 4 (16-byte rows for
                            the splat's vector reductions); columns >= wy stay zero */
    int group;           /* layer groups (consecutive fused layers with one factor f > 1, hence
                            one coarse grid): n > 1 on the first layer of a group of n, -k on
                            the k-th following member, 0 or 1 on a lone layer.  hs_smooth
                            folds a group's smoothed crops into the FIRST layer's crop as
                            sum_m gain_m smooth_m (fixed member order); hs_compose then reads
                            that crop with gain 1 and skips the members */
    int ticket;          /* group layers: first of the group's per-tile completion tickets in
                            HsSmoothArgs.tickets (one per 32x64 smooth tile); -1 otherwise */
    int pad2;
} HsLayer;

/* Structure-of-arrays particle pool.  Pools of all patches live in one set of
 * arrays; patch p owns [pool_base, pool_base + pool_capacity).  Within a patch
 * particles are bucket-segmented: bucket b occupies count[p*nb + b] elements
 * starting after buckets < b, each segment in stable birth order (the
 * reference's order restricted to that bucket, particles.py:167-178).        */
typedef struct {
    double* x;  double* y;     /* world position (fp64: keeps cull decisions exact) */
    double* ux; double* uy;    /* unit direction (fp64) */
    float* amp;                /* signed amplitude */
    double* birth;             /* optional birth time t = frame * dt (ParticleSet.birth_times,
                                  particles.py:128-129); NULL: not kept */
} HsPool;

/* ------------------------------------------------------------------------ */
/* FFT background at time t.  Replaces evolve_and_synthesize
 * (fft_background.py:181-208) incl. spectral_at (:155-159) and periodic
 * grid_normals (:162-178).                                                  */
typedef struct {
    int n;                    /* power of two, 4..4096 */
    int emit_normals;         /* write `normal` (n*n*3) */
    double g, t, choppiness;  /* t is used when frame_ptr is NULL */
    const long long* frame_ptr; /* optional device frame counter: t = frame * dt
                                 (reference harness.py:134), graph-replay safe */
    double dt;
    double spacing;           /* domain / n */
    const double* kf;         /* [n] 2*pi*fftfreq(n, d=domain/n) */
    const float* h0;          /* [n*n] complex64 (re,im) */
    const float* twiddle;     /* [n] complex64 exp(+2 pi i k/n), fp64-accurate */
    float* work_a;            /* [n*n] complex64 scratch */
    float* work_b;            /* [(n/2+1)*n] complex64 scratch */
    float* height;            /* [n*n] */
    float* dx;                /* [n*n] */
    float* dy;                /* [n*n] */
    float* normal;            /* [n*n*3] or NULL */
    double* sumsq;            /* scalar, set to sum(height^2) (zeroed by this call), or NULL */
    long long* frame_advance; /* optional: device frame counter, += 1 after the transform */
    const double* omega;      /* optional [(n/2+1)^2] dispersion sqrt(g |k|) at (|i|, |j|) =
                                 (min(i, n-i), min(j, n-j)); NULL: formed per bin each call */
    int fixed_point;          /* 1: deterministic mode (HS_FIXED_*): float sums go through
                                 int64 fixed point, see hs_fixed_to_float */
} HsFftArgs;
/* height, dx, dy, work_a and work_b must be 16-byte aligned (rows move as float4). */
HS_API int hs_fft_evolve(const HsFftArgs* a, void* stream);

/* ------------------------------------------------------------------------ */
/* Device init of the background tile's spectral amplitudes: replaces
 * init_fft (fft_background.py:102-146) -- band mask, directional variance
 * (fft_background.py:77-87, spectrum.py:108-121,124-132) and the Gaussian
 * pairs of np.random.default_rng(seed).standard_normal((n, n, 2))
 * (fft_background.py:136-137), drawn on the device from the same PCG64
 * stream through the 256-strip ziggurat (tables from the host,
 * normal_draws.py).  Draws are parsed from the raw stream in parallel: every
 * raw position is classified as an attempt, chunks of HS_ZIG_CHUNK positions
 * summarise "entry offset -> (exit offset, draws)" and a warp scan stitches
 * the chain from position 0.                                                */
#define HS_ZIG_CHUNK 128      /* raw positions per chunk */
#define HS_ZIG_ENTRIES 32     /* entry offsets tracked per chunk */
#define HS_ZIG_GROUP 64       /* chunks per composition group */
typedef struct {
    int n;                    /* power of two, 4..4096 */
    int spread_const;         /* 1: cos-2s exponent = spread_s; 0: Mitsuyasu s(omega) */
    double g, dk;             /* dk = 2 pi / domain */
    const double* kf;         /* [n] 2*pi*fftfreq(n, d=domain/n) (HsFftArgs.kf) */
    double alpha, omega_p, gamma, sigma_low, sigma_high, spread_s, mean_direction;
    double k_lo, k_hi;        /* live iff k_lo <= |k| <= k_hi (host applies the 1e-12 slack) */
    double kb_lo, kb_hi;      /* and, if kb_hi > 0, kb_lo <= |k| < kb_hi (cascade band) */
    unsigned long long pcg_state[2], pcg_inc[2]; /* (hi, lo) before the first draw */
    const unsigned long long* zig_k;  /* [256] */
    const double* zig_w;      /* [256] */
    const double* zig_f;      /* [256] */
    double zig_r;
    void* work;               /* hs_init_workspace_bytes(n) */
    double* xi;               /* [n*n*2] the draws, or NULL (kept in `work`) */
    double* h0;               /* [n*n] complex128 (re, im), or NULL */
    float* h0_f32;            /* [n*n] complex64 (HsFftArgs.h0), or NULL */
    int* status;              /* device int: 0 ok, 1 attempt ran past the chunk window,
                                 2 raw stream too short for 2 n^2 draws */
} HsInitArgs;
HS_API long long hs_init_workspace_bytes(int n);
HS_API int hs_init_h0(const HsInitArgs* a, void* stream);

/* ------------------------------------------------------------------------ */
/* Resident pool (the Simulation frame path), see hs_advect_resident below.  */
typedef struct {
    int n_patches, nb;
    const HsBucket* buckets;
    const HsPatch* patches;
    double dt, rho, g;
    HsPool pool;                   /* the current buffer */
    const int* seg_base;           /* [n_patches*nb] absolute element offset */
    const int* seg_cap;            /* [n_patches*nb] */
    const int* tile_map;           /* [max_tiles*4], 16-byte aligned: (segment, tile within
                                      segment, absolute first slot, 0); unused tiles (-1, 0, 0, 0) */
    int max_tiles;                 /* tile-map entries */
    const int* len_in;             /* [n_patches*nb] slots in use at frame start */
    int* len_out;                  /* [n_patches*nb] written by hs_append_resident */
    int* live;                     /* [n_patches*nb] live particles (atomic updates) */
    HsPool stage; const int* stage_count;   /* hs_append_resident: this frame's injected set */
    double* e_out;                 /* [n_patches*nb] despawn ledger */
    float* raw_layers;             /* must be zero at frame start (not cleared here) */
    const HsLayer* layers;
    int* clamped;                  /* [n_patches] */
    int* status;
    int fixed_point;          /* 1: deterministic mode (HS_FIXED_*): float sums go through
                                 int64 fixed point, see hs_fixed_to_float */
} HsResidentArgs;

/* ------------------------------------------------------------------------ */
/* Boundary injection for all patches (one CTA per patch).  Replaces inject
 * (particles.py:219-300).  Random draws follow numpy's Philox4x64-10 stream:
 * rng[8*p + 0..1] = key, [2..5] = counter0 (256-bit LE), [6] = draw index.   */
typedef struct {
    int n_patches, nb, n_theta;
    const HsBucket* buckets;       /* [nb] */
    const HsPatch* patches;        /* [n_patches] */
    const double* half_rate;       /* [n_patches*nb*4] */
    double mean_dir, beta, rho, g;
    double* acc;                   /* [n_patches*nb*4] ledger accumulators */
    long long* groups;             /* [n_patches*nb] */
    double* e_in;                  /* [n_patches*nb] */
    unsigned long long* rng;       /* [n_patches*8] */
    HsPool stage;                  /* staging arrays (per-patch regions) */
    int* stage_count;              /* [n_patches*nb] out */
    double* scratch;               /* [n_patches*member_capacity*6]: per-member records */
    int member_capacity;           /* per patch: >= max groups * n_theta */
    int* status;
    int* zero_words;               /* optional: 4-byte words zeroed by this launch (per-frame */
    int n_zero_words;              /*   stat accumulators read by later kernels)             */
    int append;                    /* 1: the new particles skip the stage -- they are advected,
                                      culled and splatted here and appended to the resident
                                      segments (what hs_append_resident does with a stage) */
    HsResidentArgs res;            /* resident pool for append (its stage fields are unused) */
    double birth_t;                /* birth time of this step's particles (particles.py:296-299) ... */
    const long long* birth_frame;  /* ... or, if set, *birth_frame * birth_dt (graph replays) */
    double birth_dt;
} HsInjectArgs;
HS_API int hs_inject(const HsInjectArgs* a, void* stream);

/* ------------------------------------------------------------------------ */
/* Advect + cull + stable bucket-segmented compaction (+ fused splat) for all
 * patches.  Replaces advect (particles.py:303-328), ParticleSet.compact
 * (:167-178) and the per-bucket _splat of synthesize
 * (patch_synthesis.py:165-186, 298-310).                                    */
typedef struct {
    int n_patches, nb;
    const HsBucket* buckets;
    const HsPatch* patches;
    double dt, rho, g;
    HsPool in;  const int* in_count;       /* [n_patches*nb] */
    HsPool stage; const int* stage_count;  /* [n_patches*nb]; may be NULL */
    HsPool out; int* out_count;            /* [n_patches*nb]; zeroed here */
    HsPool dropped; int* dropped_count;    /* optional (x == NULL to skip): despawned
                                              particles, same segmented layout */
    double* e_out;                         /* [n_patches*nb] despawn ledger */
    int splat;                             /* fuse the layer splat */
    float* raw_layers;                     /* zeroed here when splat */
    long long raw_layers_len;              /* floats */
    const HsLayer* layers;                 /* [n_patches*nb] */
    int* clamped;                          /* [n_patches] += clamp counts */
    unsigned long long* tile_state;        /* [max_tiles] look-back state / per-tile counts */
    int max_tiles;                         /* >= sum over patches of ceil((pool+stage capacity)/1024) */
    int* tile_counter;                     /* scalar */
    int* status;
    unsigned* keep_words;                  /* optional [max_tiles*32]: selects the count + scatter
                                              two-kernel compaction (no serial look-back chain) */
    /* resident-pool compaction (HsResidentArgs below); all optional */
    const int* in_seg_base;                /* [n_patches*nb]: input bucket b of patch p occupies the
                                              absolute slots [in_seg_base, +in_count) of `in`, and
                                              slots whose x is NaN are holes (skipped, not despawned) */
    const int* out_slack_prefix;           /* [n_patches*nb]: survivor of bucket b with patch rank r
                                              goes to pool_base + r + out_slack_prefix (gaps between
                                              segments for later in-place appends) */
    int raw_is_clear;                      /* 1: raw layers are already zero (skip the clear) */
    int fixed_point;          /* 1: deterministic mode (HS_FIXED_*): float sums go through
                                 int64 fixed point, see hs_fixed_to_float */
} HsAdvectArgs;
HS_API int hs_advect(const HsAdvectArgs* a, void* stream);

/* ------------------------------------------------------------------------ */
/* Resident pool (the Simulation frame path).  Between compactions every
 * (patch, bucket) segment keeps fixed storage [seg_base, seg_base + seg_cap)
 * with len slots in use; a despawned particle leaves a hole (x = NaN) in
 * place, so the live particles of a segment, read in slot order, are exactly
 * the reference's stable compaction of that bucket (particles.py:167-178).
 * Per frame:
 *   hs_advect_resident  advect + cull + splat every used slot IN PLACE
 *                       (reads x,y,ux,uy,amp; writes x,y -- or the hole mark)
 *   hs_append_resident  advect + cull + splat this frame's injected particles
 *                       and append them at the segment tails (len_out = len_in
 *                       + staged); independent of hs_advect_resident, so the
 *                       two run concurrently
 * Every K frames hs_advect (count + scatter, in_seg_base/out_slack_prefix)
 * squeezes the holes out into the other buffer and hs_resident_layout
 * re-derives the segment table.                                             */

HS_API int hs_advect_resident(const HsResidentArgs* a, void* stream);
HS_API int hs_append_resident(const HsResidentArgs* a, void* stream);

/* One further tile of a summed-cascade background (fft.cascades): periodic,
 * origin 0, its own spacing.  Samplers add its bilinear height and combine
 * normals through slopes, n = normalize(sum_c n_c.xy / n_c.z, 1), n_c the
 * renormalised bilinear of the tile's periodic node normals.               */
#define HS_MAX_CASCADES 4
typedef struct {
    const float* height;      /* [n*n] */
    int n;                    /* power of two */
    int pad;
    double spacing;
} HsBgTile;

/* ------------------------------------------------------------------------ */
/* Kinematic emitting bodies: the reference's per-frame
 * buoyancy_step + emit_from_motion + _retrack_patches (interaction.py:140,
 * 175-231; harness.py:115-123,155-167) for bodies moving at a constant
 * velocity with a fixed displaced-volume change per frame.  Everything that
 * is constant per source (energy split, fan directions, amplitudes, buckets)
 * is formed on the host with the reference's own numpy expressions; the device
 * moves the sources, finds each one's owning patch, appends the fans to the
 * resident segments (after this frame's injected particles), splats them,
 * books the energy and moves tracking patches.                              */
typedef struct {
    double vx, vy;            /* horizontal velocity: position += v dt each frame (interaction.py:140) */
    double hull_extent;       /* fan radius around the source (m) */
    double e_ring, e_wake;    /* energy booked per frame per branch, 0 = branch silent */
    double amp_ring, amp_wake;/* signed crest amplitude of each branch (fp64) */
    int n_ring, n_wake;       /* fan sizes */
    int ring_bucket, wake_bucket;
    int dir_off;              /* ring directions, then wake directions, in HsEmitArgs.dirs */
    int body;                 /* >= 0: a floating body (HsEmitArgs.bodies[body]): position, energy
                                 split, amplitudes and the wake's direction come from its state every
                                 frame; the wake entries at dir_off + n_ring hold the fan's angle
                                 offsets (np.linspace(-h, h, n_wake), x component) */
} HsSource;

/* A floating body (FloatingBody / box_body, interaction.py:36-102), state
 * updated in place by hs_bodies.                                            */
#define HS_MAX_PROBES 8
typedef struct {
    double pos[3], vel[3];
    double yaw, yaw_rate;
    double submerged, prev_submerged, mean_submersion;
    double mass, hull_extent, draft, drag_linear, drag_yaw;
    double thrust_force;      /* thrust * max_thrust (N) */
    double yaw_torque;        /* rudder * max_yaw_torque (N m) */
    double displaced;         /* sum of probe volumes, in probe order */
    double probe_off[HS_MAX_PROBES][3];
    double probe_vol[HS_MAX_PROBES];
    int n_probes, pad;
} HsBody;

/* buoyancy_step (interaction.py:105-149) of every body against the blended
 * surface of the previous frame (SurfaceSampler._raw, coupling.py:120-141):
 * the periodic background (+ cascades) and the patch heights at their
 * synthesis rectangles, normals from their finite differences.  Call before
 * the frame's transform and hs_track overwrite them; `flat` = 1 before the
 * first synthesised frame (the reference's initial SurfaceSampler(None, [])). */
typedef struct {
    int n_bodies;
    HsBody* bodies;
    double dt, rho, g;
    int flat;
    const float* bg_height; int bg_n; double bg_spacing;
    int n_extra_bg; HsBgTile extra_bg[HS_MAX_CASCADES - 1];
    int n_patches;
    const HsPatch* patches;
    const float* patch_height;
    const long long* frame;   /* optional device frame counter: if set, the surface is flat
                                 while *frame == 0 (read on the device, so a captured graph
                                 replayed from frame 0 on still sees the live value) */
} HsBodyArgs;
HS_API int hs_bodies(const HsBodyArgs* a, void* stream);

#define HS_MAX_SOURCES 1024
typedef struct {
    int n_sources, n_patches, nb;
    const HsSource* sources;
    const double* dirs;       /* [total fan size * 2] unit directions (ux, uy) */
    const double* pos_in;     /* [n_sources*2] positions after the previous frame */
    double* pos_out;          /* [n_sources*2] positions after this frame (written by hs_emit) */
    HsPatch* patches;         /* hs_track moves tracking patches */
    const HsBucket* buckets;
    double dt, beta, rho, g;
    HsPool pool; const int* seg_base; const int* seg_cap;
    int* len;                 /* [n_patches*nb] slots in use; emitted particles are appended */
    int* live;
    double* e_in;
    float* raw_layers; const HsLayer* layers; int* clamped;
    int* status;
    const HsBody* bodies;     /* for sources with body >= 0 */
    int n_theta;              /* ring fan of bodies (interaction.py:220-222) */
    int fixed_point;          /* 1: deterministic mode (HS_FIXED_*): float sums go through
                                 int64 fixed point, see hs_fixed_to_float */
} HsEmitArgs;
/* Frame start: tracking patches adopt last frame's synthesis origin as their
 * region, and take this frame's synthesis origin from their source's new
 * position, _snap(p - l/2, texel) (harness.py:65-66,115-123).               */
HS_API int hs_track(const HsEmitArgs* a, void* stream);
/* After advection and this frame's appends: move every source, emit into its
 * owning patch (first patch whose region contains it, particles.py:71-74),
 * splat at the synthesis origin, book e_in (harness.py:155-163).            */
HS_API int hs_emit(const HsEmitArgs* a, void* stream);

/* Segment table after a compaction (or at start, count = NULL): segment
 * (p, b) gets base = pool_base + sum_{b'<b} count + slack_prefix, cap = count
 * + slack, len = live = count, and tiles of 1024 slots in tile_map.          */
typedef struct {
    int n_patches, nb;
    const HsPatch* patches;
    const int* count;              /* [n_patches*nb] packed counts, or NULL (empty pool) */
    const int* slack;              /* [n_patches*nb] */
    const int* slack_prefix;       /* [n_patches*nb] exclusive prefix of slack within the patch */
    int* seg_base; int* seg_cap; int* len; int* live;
    int* tile_map;                 /* [max_tiles*4] */
    int max_tiles;
    int* status;
} HsLayoutArgs;
HS_API int hs_resident_layout(const HsLayoutArgs* a, void* stream);

/* Splat-only pass over a bucket-segmented pool (synthesize on a pool that was
 * not just advected).                                                       */
typedef struct {
    int n_patches, nb;
    const HsPatch* patches;
    HsPool pool; const int* count;         /* [n_patches*nb] */
    float* raw_layers; long long raw_layers_len;
    const HsLayer* layers;
    int* clamped;
    int max_count;                         /* host upper bound of any patch count */
} HsSplatArgs;
HS_API int hs_splat(const HsSplatArgs* a, void* stream);

/* ------------------------------------------------------------------------ */
/* Separable raised-cosine smoothing of every layer (all patches, all
 * buckets) from the raw padded layers into the cropped smoothed layers.
 * Replaces smooth_layer/convolve1d_zero (patch_synthesis.py:105-130,206-209). */
/* Layers with H <= HS_SMOOTH_FUSED_MAX_H run one fused 2-D tile pass; wider
 * kernels (texel-exact plans) run two 1-D passes through `mid`
 * (HsLayer.mid_off, ncx*wy floats per wide layer).                          */
#define HS_SMOOTH_FUSED_MAX_H 40
typedef struct {
    int n_layers;
    const HsLayer* layers;
    const float* taps;
    const float* raw_layers;
    float* smooth_layers;
    const int* tile_info;     /* [total_tiles*3] fused 32x32 tiles: layer, cx0, cy0 */
    int total_tiles;
    int max_H;                /* max H over fused layers */
    float* mid;               /* wide-layer intermediate, or NULL */
    const int* xtile_prefix;  /* [n_layers+1] x-pass tiles of wide layers (ncx x wy) */
    int total_xtiles;
    const int* ytile_prefix;  /* [n_layers+1] y-pass tiles of wide layers (ncx x ncy) */
    int total_ytiles;
    int max_H_wide;           /* max H over wide layers (<= 780) */
    int* tickets;             /* zeroed per-tile group tickets (HsLayer.ticket); the kernel
                                 re-arms them, so one zeroing serves every frame.  Required
                                 when any layer has group != 0/1 */
} HsSmoothArgs;
HS_API int hs_smooth(const HsSmoothArgs* a, void* stream);



/* ------------------------------------------------------------------------ */
/* Compose: gain-sum of the bilinearly upsampled layers (synthesize,
 * patch_synthesis.py:301-313), clamped-border normals (finish_field,
 * :323-340) and the smoothstep blend against the periodic background at the
 * patch nodes (SurfaceSampler._raw, coupling.py:120-141).                   */
typedef struct {
    int n_patches, nb;
    const HsPatch* patches;
    const HsLayer* layers;
    const float* smooth_layers;
    const int* tile_info;       /* [total_tiles*3] 30x30 output tiles: patch, i0, j0 */
    int total_tiles;
    /* background (may be NULL: flat water) */
    const float* bg_height; const float* bg_normal; int bg_n; double bg_spacing;
    /* outputs, per patch at grid_base (res*ny), NULL to skip */
    float* patch_height;        /* pre-blend patch heights */
    float* patch_normal;        /* (res*ny*3) patch FD normals */
    float* blend_height;        /* blended heights */
    float* blend_normal;        /* (res*ny*3) blended normals */
    int blend_mode;             /* 0: no blend, 1: blend */
    double* interior_sumsq;     /* [n_patches] += sum h^2 over the interior inset, or NULL */
    long long* interior_count;  /* [n_patches] matching counts, or NULL */
    long long* frame_advance;   /* optional: device frame counter, += 1 by this launch */
    int n_extra_bg;             /* further cascades added to the background (0..3) */
    HsBgTile extra_bg[HS_MAX_CASCADES - 1];
    int fixed_point;          /* 1: deterministic mode (HS_FIXED_*): float sums go through
                                 int64 fixed point, see hs_fixed_to_float */
    float* composite;           /* optional [bg_n*bg_n] FFT-resolution composite (stitched_heights,
                                   harness.py:219-241) that already holds the background: every
                                   composite node strictly inside a patch is blended in place from
                                   the tile that covers it (needs bg_height) */
} HsComposeArgs;
HS_API int hs_compose(const HsComposeArgs* a, void* stream);

/* ------------------------------------------------------------------------ */
/* Surface queries at arbitrary world points: periodic background plus
 * clamped patch sampling with smoothstep weights.  Replaces
 * SurfaceSampler.sample (coupling.py:143-161, normal_mode "blend"),
 * sample_periodic (fft_background.py:222-249), sample_clamped (coupling.py:63-82). */
typedef struct {
    int n_points;
    const double* points;       /* [n_points*2] world x,y */
    const float* bg_height; const float* bg_normal; int bg_n; double bg_spacing;
    double bg_x0, bg_y0;
    int n_patches;
    const HsPatch* patches;
    const float* patch_height;  /* per patch at grid_base */
    const float* patch_normal;
    float* out_height;
    float* out_normal;          /* [n_points*3] or NULL */
    int clamped_only;           /* 1: sample_clamped of patch 0 only, no weights */
    int n_extra_bg;             /* further background cascades (bg_* is cascade 0) */
    HsBgTile extra_bg[HS_MAX_CASCADES - 1];
    int from_heights;           /* 1: normals from finite differences of the height grids (periodic
                                   background, clamped patches), bg_normal / patch_normal unused;
                                   patches at their synthesis rectangles, bg origin 0 -- the
                                   sampler hs_bodies uses */
} HsSampleArgs;
HS_API int hs_sample(const HsSampleArgs* a, void* stream);

/* Global FFT-resolution composite: copy the background and resample the
 * patch boxes (Simulation.stitched_heights, harness.py:219-241).            */
typedef struct {
    int n; double spacing;
    const float* bg_height; const float* bg_normal;
    int n_patches;
    const HsPatch* patches;
    const float* patch_height; const float* patch_normal;
    const int* box;             /* [n_patches*4] i0, i1, j0, j1 (half-open) */
    const int* box_prefix;      /* [n_patches+1] cumulative box sizes */
    int total_box;
    float* out;                 /* [n*n] */
    int n_extra_bg;             /* further background cascades, summed at the grid nodes */
    HsBgTile extra_bg[HS_MAX_CASCADES - 1];
} HsCompositeArgs;
HS_API int hs_composite(const HsCompositeArgs* a, void* stream);

/* Multi-GPU composite exchange (the reference composite is
 * Simulation.stitched_heights, harness.py:219-241).  Every rank packs the
 * FFT-resolution box of each of its patches -- rows/columns
 * [floor(min/spacing), ceil(max/spacing)+1) clipped to the grid, computed on
 * the device from the patch's current synthesis rectangle, so boxes follow
 * tracking patches -- out of its frame composite (which hs_compose already
 * blended) into its slots of `payload`; one NCCL all-gather of `payload`
 * (in place) follows; hs_box_paste then writes every other rank's boxes into
 * this rank's composite, the later patch (global order = slot order) winning
 * where boxes overlap, as the reference loop does.
 * Slot layout: 4 header words (i0, i1, j0, j1 as int bits; i0 == i1: empty)
 * then bw x bh values, row-major with stride bh.                           */
typedef struct {
    int n; double spacing;      /* composite grid side and node spacing */
    float* composite;           /* [n*n] this rank's frame composite */
    int n_local;                /* patches of this rank (pack) */
    const HsPatch* patches;     /* [n_local] */
    int bw, bh;                 /* box capacity (nodes); a larger box is cut and sets
                                   HS_STATUS_BOX_OVERFLOW in status */
    float* payload;             /* [world * slots * (4 + bw*bh)] */
    int slots, world, rank;     /* slots per rank; paste skips this rank's own */
    int* status;
} HsBoxArgs;
HS_API int hs_box_pack(const HsBoxArgs* a, void* stream);
HS_API int hs_box_paste(const HsBoxArgs* a, void* stream);

/* fp64 helpers of the function-level API (not on the frame path):
 * spectral_at (fft_background.py:155-159): hh = h0 e^{-i w t} + conj(h0(-k)) e^{+i w t}
 * over the n x n grid, h0 complex128 [n*n*2], omega on the (|i|, |j|) quarter
 * grid [(n/2+1)^2] as FftState.omega_dev, out complex128 [n*n*2];
 * convolve1d_zero (patch_synthesis.py:105-130): same-size zero-padded
 * convolution of an [outer, n, inner] fp64 array along its middle axis with
 * 2H+1 taps (direct taps: the reference's cumsum window sums are the same
 * convolution).                                                            */
HS_API int hs_spectral_at(const double* h0, const double* omega, int n, double t, double* out, void* stream);
HS_API int hs_conv1d_zero(const double* in, double* out, long long outer, int n, long long inner,
                          const double* taps, int H, void* stream);

/* Non-periodic (clamped-border) normals and optional choppy displacement of
 * patch grids (finish_field, patch_synthesis.py:323-340).                   */
typedef struct {
    int nx, ny; double spacing; double chop_scale;  /* -chi*displacement_scale */
    const float* height; float* normal; float* disp; /* disp may be NULL */
} HsFinishArgs;
/* dst[i] = (float)(src[i] * 2^-bits) for i < n (deterministic-mode raw layers). */
HS_API int hs_fixed_to_float(const long long* src, float* dst, long long n, int bits, void* stream);

HS_API int hs_finish(const HsFinishArgs* a, void* stream);

/* Reductions used by FrameStats (harness.py:171-206). */
HS_API int hs_sumsq(const float* x, long long n, double* out, void* stream);

/* Periodic central-difference normals of an n x n height grid (the
 * grid_normals(periodic=True) part of evolve_and_synthesize,
 * fft_background.py:162-178), for lazily materialised background normals. */
HS_API int hs_periodic_normals(const float* height, float* normal, int n, double spacing, void* stream);

/* frame += 1 on the device (end of a captured frame). */
HS_API int hs_advance_frame(long long* frame, void* stream);
/* Zero `bytes` bytes at `p` (the consumed raw layers at the end of a frame):
 * a memset node when captured, cheaper than a fill kernel. */
HS_API int hs_clear(void* p, long long bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HYBRIDSEA_B200_H */
