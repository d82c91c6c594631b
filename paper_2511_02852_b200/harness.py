"""Frame pipeline on the B200: the hybrid ocean step as one CUDA graph.

Mirror of `hybridsea.harness.Simulation` (`pkg/src/hybridsea/harness.py:69-241`)
for the hot path.  Per frame (stage order of harness.py:131-209):

    hs_fft_evolve   t = frame*dt read on the device; rotation + IFFT2 +
                    normals + fft variance (fused)
    hs_inject       all patches, one CTA each, Philox streams on the device
    hs_advect       all patches: advect + cull + stable bucket compaction of
                    [survivors | new crests | new troughs] + layer splat
    hs_smooth       every (patch, bucket) layer
    hs_compose      gain-sum + FD normals + smoothstep blend + interior
                    variance, all patches
    hs_advance_frame

Everything lives in preallocated device buffers (two ping-pong pools); the
frame is captured once per pool parity into a CUDA graph and replayed, so a
step is one graph launch with no host synchronisation.  Stats are read from
device buffers only when asked for.

Bodies / buoyancy / emission (harness.py:155-167) are outside the B200 hot
path and rejected here.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from ._layout import (COMPOSE_TILE, bucket_structs, half_rates, max_groups_per_step, patch_struct, stream_ptr,
                      structs_to_device)
from .config import SimConfig, cascade_bands
from .coupling import PatchSurface, SurfaceSampler, validate_patches
from .errors import CapacityError, ConfigError
from .fft_background import FftWorkspace, HeightField, fft_args, init_fft
from .particles import PatchRegion, PhiloxStream, ParticleSet
from .patch_synthesis import SynthWorkspace, plan_layers
from .interaction import body_structs, source_structs
from .spectrum import DirectionalSpectrum, build_buckets, derive_params, log_buckets

STAGES = ("fft", "inject", "advect", "interact", "synth", "blend", "output")
ADV_TILE = 1024
RES_TILE = 1024          # hs_advect_resident tile (slots of one bucket segment)
RESIDENT_PERIOD = 64    # frames between resident-pool compactions (64 vs 32: -0.6 us/frame at C3)


def build_table(cfg: SimConfig, params):
    if cfg.bucket_spacing == "log":
        return log_buckets(params, cfg.omega_lo, cfg.omega_hi, cfg.n_omega, cfg.n_theta)
    return build_buckets(params, cfg.n_omega, cfg.n_theta)


def estimate_population(table, region: PatchRegion, trough_fraction: float) -> float:
    """Steady-state particles of one patch: inflow rate x residence time per
    bucket.  Groups/s through all four sides = 4 (l1 + l2) w^3/(pi^3 g)
    (particles.py:210-216); residence ~ (mean side + 2 r)/c."""
    per_group = table.n_theta * (2 if trough_fraction != 0.0 else 1)
    g = table.buckets[0].speed * table.buckets[0].omega
    side = 0.5 * (region.l1 + region.l2)
    tot = 0.0
    for b in table.buckets:
        rate = 4.0 * (region.l1 + region.l2) * b.omega ** 3 / (math.pi ** 3 * g)
        tot += rate * per_group * (side + 2.0 * b.radius) / b.speed
    return tot


def fixed_to_double(a: np.ndarray, bits: int) -> np.ndarray:
    """Deterministic-mode accumulator (int64 fixed point in fp64 slots) -> fp64."""
    return np.asarray(a).view(np.int64).astype(np.float64) * (2.0 ** -bits)


@dataclass
class FrameStats:
    """Per-frame statistics (harness.py:32-46).  Device-resident values are
    materialised lazily, so stepping never synchronises."""
    frame: int
    t: float
    stage_ms: dict
    _snap: dict = field(default=None, repr=False)
    _nb: int = 0
    _n_patches: int = 0
    _fft_n: int = 0
    body_states: list = field(default_factory=list)
    _cache: dict = field(default_factory=dict, repr=False)
    _fixed: bool = False        # deterministic mode: e_out / isum / fsum hold int64 fixed point

    def _get(self):
        if not self._cache:
            s = {k: v.cpu().numpy() for k, v in self._snap.items()}
            if self._fixed:
                for k, bits in (("e_out", N.HS_FIXED_ENERGY_BITS), ("isum", N.HS_FIXED_SUMSQ_BITS),
                                ("fsum", N.HS_FIXED_SUMSQ_BITS)):
                    if k in s:
                        s[k] = fixed_to_double(s[k], bits)
            counts = s["counts"].reshape(self._n_patches, self._nb).sum(0) if self._n_patches else np.zeros(self._nb, np.int64)
            e_in = s["e_in"].reshape(self._n_patches, self._nb).sum(0) if self._n_patches else np.zeros(self._nb)
            e_out = s["e_out"].reshape(self._n_patches, self._nb).sum(0) if self._n_patches else np.zeros(self._nb)
            pv = 0.0
            if self._n_patches:
                cnt = np.maximum(s["icount"], 1)
                pv = float(np.mean(s["isum"] / cnt))
            fv = float(s["fsum"][0]) / float(self._fft_n * self._fft_n) if self._fft_n else 0.0
            self._cache.update(particle_counts=counts.astype(np.int64), injected_energy=e_in,
                               despawned_energy=e_out, patch_variance=pv, fft_band_variance=fv)
            if "bodies" in s:
                raw, sz = s["bodies"].tobytes(), C.sizeof(N.HsBody)
                self.body_states = [(b.pos[0], b.pos[1], b.pos[2], b.yaw) for b in
                                    (N.HsBody.from_buffer_copy(raw[k * sz:(k + 1) * sz]) for k in range(len(raw) // sz))]
        return self._cache

    @property
    def particle_counts(self) -> np.ndarray:
        return self._get()["particle_counts"]

    @property
    def injected_energy(self) -> np.ndarray:
        return self._get()["injected_energy"]

    @property
    def despawned_energy(self) -> np.ndarray:
        return self._get()["despawned_energy"]

    @property
    def patch_variance(self) -> float:
        return self._get()["patch_variance"]

    @property
    def fft_band_variance(self) -> float:
        return self._get()["fft_band_variance"]

    @property
    def total_ms(self) -> float:
        return sum(self.stage_ms.values())


class Simulation:
    """Owns all device state of one hybrid scene; `step()` advances a frame."""

    def __init__(self, config: SimConfig, device=None, *, pool_capacity: int | None = None,
                 rng_seed_keys: list | None = None, compact_period: int | None = None):
        cfg = config.validate()
        self.config = cfg
        self.det = bool(cfg.deterministic)
        # The frame ends with the FFT-resolution composite (stitched_heights,
        # harness.py:219-241, part of the north_star step) written to
        # composite_out.  `post_frame`, if set, replaces it: an optional callable
        # enqueued at the end of every frame (captured into the frame graphs),
        # e.g. the multi-GPU composite exchange (bench.py, sharding.py).
        self.composite_each_frame = True
        self.post_frame = None
        self._cshard = None               # sharding.CascadeShard (multi-GPU C4), see shard_cascades
        # frame schedule knobs (tools/ab_sched.py): FFT branch fork point, stream priorities
        self.fft_fork_at_start = False
        self.sched_priorities = False
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        dev = self.device
        self.params = derive_params(cfg.u10, cfg.fetch, cfg.g, gamma=cfg.gamma, spread_s=cfg.spread_s)
        self.spectrum = DirectionalSpectrum(self.params, cfg.mean_direction)
        self.table = build_table(cfg, self.params)
        self.nb = self.table.n_omega
        self.frame = 0
        self.t = 0.0
        self._parity = 0
        self._graphs = {}
        self._stats = []

        pcs = cfg.active_patches()
        self.regions = [PatchRegion(tuple(pc.origin), pc.size[0], pc.size[1], pc.margin) for pc in pcs]
        validate_patches(self.regions)
        self.res = [pc.res for pc in pcs]
        self.n_patches = len(self.regions)
        if self.n_patches > N.HS_MAX_PATCHES:
            raise ConfigError(f"at most {N.HS_MAX_PATCHES} patches per device")
        self.plans = [plan_layers(self.table, r.l1 / (res - 1), res, convention=cfg.amplitude_convention,
                                  trough_fraction=cfg.trough_fraction) for r, res in zip(self.regions, self.res)]

        # ---- background ------------------------------------------------
        self.fft_state = None
        self.fft_ws = None
        self.cascades = []                # [(FftState, FftWorkspace)], cascade 0 = fft_state / fft_ws
        if cfg.mode != "wp-only":
            band = None
            if cfg.fft_band_lo is not None or cfg.fft_band_hi is not None:
                band = (cfg.fft_band_lo, cfg.fft_band_hi)
            # one tile, or summed tiles with disjoint |k| bands, seeds seed + c (config.cascade_bands)
            tiles = cascade_bands(cfg.fft_cascades, cfg.fft_n) if cfg.fft_cascades else [(cfg.fft_domain, None, None)]
            for c, (L, klo, khi) in enumerate(tiles):
                st = init_fft(self.spectrum, cfg.fft_n, L, cfg.seed + c, choppiness=cfg.fft_choppiness, band=band,
                              kband=None if klo is None else (klo, khi), device=dev)
                self.cascades.append((st, FftWorkspace(cfg.fft_n, dev, normals=cfg.fft_normals or self.n_patches > 0)))
            self.fft_state, self.fft_ws = self.cascades[0]
        self.frame_dev = torch.zeros(1, dtype=torch.int64, device=dev)

        # ---- constants ---------------------------------------------------
        self.buckets_dev = structs_to_device(bucket_structs(self.table, self.params), dev)
        self._hr_cache = {}
        self.pool_caps, self.stage_caps, self.member_cap = [], [], 1
        per_member = 2 if cfg.trough_fraction != 0.0 else 1
        max_new = []                     # per patch, per bucket: particles one frame can append
        explicit = pool_capacity is not None or bool(cfg.pool_capacity)
        # emitting bodies (interaction.py): floating bodies first
        # (the reference's order), then kinematic sources; patch track indices
        # point into that combined list
        self.bodies = tuple(cfg.bodies) if self.n_patches else ()
        self.n_bodies = len(self.bodies)
        self.sources = tuple(cfg.sources) if self.n_patches else ()
        body_st, body_dirs, self._body_init = body_structs(self.bodies, self.table, 0)
        src_structs, src_dirs, src_plans = source_structs(self.sources, self.table, cfg.rho, cfg.g,
                                                          offset=len(body_dirs))
        self.n_sources = self.n_bodies + len(self.sources)
        if self.n_sources > N.HS_MAX_SOURCES:
            raise ConfigError(f"at most {N.HS_MAX_SOURCES} sources and bodies per device")
        src_structs = body_st + src_structs
        src_dirs = np.concatenate([body_dirs.reshape(-1, 2), src_dirs.reshape(-1, 2)])
        self._track_idx = [pc.track_body if pc.track_body >= 0 else
                           (self.n_bodies + pc.track_source if pc.track_source >= 0 else -1) for pc in pcs]
        self._tracking = any(t >= 0 for t in self._track_idx)
        emit_new = np.zeros((self.n_patches, self.nb), np.int64)     # per frame
        emit_pop = np.zeros(self.n_patches)
        tracker = {t: k for k, t in enumerate(self._track_idx) if t >= 0}
        plans = []
        for j, b in enumerate(self.bodies):       # a body may fire both fans every frame
            st_ = body_st[j]
            plans.append(({"e_ring": 1.0, "ring_dirs": np.zeros((st_.n_ring, 2)), "ring_bucket": st_.ring_bucket,
                           "e_wake": 1.0, "wake_dirs": np.zeros((st_.n_wake, 2)), "wake_bucket": st_.wake_bucket},
                          0.0))
        plans += [(pl, float(np.hypot(*src.velocity[:2]))) for src, pl in zip(self.sources, src_plans)]
        for j, (pl, speed) in enumerate(plans):
            # a tracked source only ever emits into its patch; others may enter any patch
            cand = [tracker[j]] if j in tracker else range(self.n_patches)
            vt = speed if j in tracker else 0.0
            for key_e, key_d, key_b in (("e_ring", "ring_dirs", "ring_bucket"), ("e_wake", "wake_dirs", "wake_bucket")):
                if pl[key_e] <= 0.0:
                    continue
                n, b = per_member * len(pl[key_d]), pl[key_b]
                bk = self.table.buckets[b]
                for k in cand:
                    emit_new[k, b] += n
                    side = 0.5 * (self.regions[k].l1 + self.regions[k].l2)
                    stay = (side + 2.0 * bk.radius) / (bk.speed + vt) / cfg.dt
                    if j not in tracker and speed > 0:
                        stay = min(stay, 2.0 * side / speed / cfg.dt)
                    emit_pop[k] += n * stay
        for k, r in enumerate(self.regions):
            hr_max = half_rates(r, self.table.omegas, 0.1, cfg.g)       # dt <= 0.1 (config.py validate)
            mg = max_groups_per_step(hr_max)
            self.member_cap = max(self.member_cap, mg * self.table.n_theta)
            max_new.append((np.floor(hr_max) + 1.0).sum(axis=1).astype(np.int64) * self.table.n_theta * per_member
                           + emit_new[k])
            if pool_capacity is not None:
                cap = int(pool_capacity)
            elif cfg.pool_capacity:
                cap = cfg.pool_capacity
            else:
                cap = max(4096, int(1.6 * (estimate_population(self.table, r, cfg.trough_fraction) + emit_pop[k])))
                cap += (RESIDENT_PERIOD if compact_period is None else max(1, int(compact_period))) \
                    * int(max_new[-1].sum())
                cap = -(-cap // 1024) * 1024
            self.pool_caps.append(cap)
            self.stage_caps.append(2 * mg * self.table.n_theta)
        # resident pool: compaction every K frames; every bucket segment keeps
        # room for K frames of its largest possible inflow
        K = RESIDENT_PERIOD if compact_period is None else max(1, int(compact_period))
        if explicit:
            while K > 1 and any(K * int(m.sum()) > c // 2 for m, c in zip(max_new, self.pool_caps)):
                K //= 2
        self.compact_period = K
        self._slack_np = (np.stack(max_new) * K).astype(np.int32) if max_new else np.zeros((0, self.nb), np.int32)
        self.pool_base = np.concatenate([[0], np.cumsum(self.pool_caps)]).astype(np.int64)
        self.stage_base = np.concatenate([[0], np.cumsum(self.stage_caps)]).astype(np.int64)
        total_pool = int(self.pool_base[-1])
        total_stage = int(self.stage_base[-1])

        if self.n_patches:
            self.synth = SynthWorkspace(self.regions, self.res, self.plans, dev)
            self._order_compose_tiles()
            if self.det:
                self.raw_fixed = torch.zeros(self.synth.raw.numel(), dtype=torch.int64, device=dev)
            structs = []
            for k, (r, res) in enumerate(zip(self.regions, self.res)):
                structs.append(patch_struct(r, res, pool_base=self.pool_base[k], pool_capacity=self.pool_caps[k],
                                            stage_base=self.stage_base[k], stage_capacity=self.stage_caps[k],
                                            grid_base=self.synth.grid_base[k], layer_base=k * self.nb,
                                            track=self._track_idx[k]))
            self.patches_dev = structs_to_device(structs, dev)
            if self.n_sources:
                self.sources_dev = structs_to_device(src_structs, dev)
                self.src_dirs = torch.from_numpy(src_dirs.reshape(-1).copy()).to(dev) if src_dirs.size else \
                    torch.zeros(2, dtype=torch.float64, device=dev)
                pos = [(b.position[0], b.position[1]) for b in self.bodies] + [tuple(c.position) for c in self.sources]
                p0 = torch.tensor(np.array(pos, dtype=np.float64).reshape(-1), device=dev)
                self.src_pos = [p0, p0.clone()]
                self.bodies_dev = structs_to_device(self._body_init, dev) if self.n_bodies else None
            f64 = lambda n: torch.zeros(max(1, n), dtype=torch.float64, device=dev)  # noqa: E731
            f32 = lambda n: torch.zeros(max(1, n), dtype=torch.float32, device=dev)  # noqa: E731
            # one tile of padding: hs_advect_resident issues a tile's slot loads
            # before it knows the segment length, so the last tile of the last
            # segment may read up to RES_TILE - 1 slots past pool_base[-1]
            # (explicit capacities are not rounded to the tile)
            padded = total_pool + RES_TILE
            # x, y, ux, uy, amp and the birth times (read only by the pool accessor)
            self.pools = [[f64(padded), f64(padded), f64(padded), f64(padded), f32(padded), f64(padded)]
                          for _ in range(2)]
            PB = self.n_patches * self.nb
            i32 = lambda n: torch.zeros(max(1, n), dtype=torch.int32, device=dev)  # noqa: E731
            # resident segment table (hs_resident_layout)
            self.seg_base, self.seg_cap, self.live = i32(PB), i32(PB), i32(PB)
            self.seg_len = [i32(PB), i32(PB)]
            self.compact_count = i32(PB)
            self.slack = torch.from_numpy(self._slack_np.ravel().copy()).to(dev)
            sp = np.concatenate([np.zeros((self.n_patches, 1), np.int64), np.cumsum(self._slack_np, axis=1)[:, :-1]],
                                axis=1)
            self.slack_prefix = torch.from_numpy(sp.astype(np.int32).ravel().copy()).to(dev)
            self.res_tiles = int(sum(-(-c // RES_TILE) for c in self.pool_caps)) + PB
            self.tile_map = i32(4 * self.res_tiles)
            self._buf, self._lp, self._since = 0, 0, 0
            self.stage = [f64(total_stage), f64(total_stage), f64(total_stage), f64(total_stage), f32(total_stage),
                          f64(total_stage)]
            self.stage_count = torch.zeros(self.n_patches * self.nb, dtype=torch.int32, device=dev)
            self.scratch = f64(6 * self.member_cap * self.n_patches)   # member records (HsInjectArgs.scratch)
            self.acc = torch.zeros(self.n_patches * self.nb * 4, dtype=torch.float64, device=dev)
            self.groups = torch.zeros(self.n_patches * self.nb, dtype=torch.int64, device=dev)
            self.e_in = torch.zeros(self.n_patches * self.nb, dtype=torch.float64, device=dev)
            self.e_out = torch.zeros(self.n_patches * self.nb, dtype=torch.float64, device=dev)
            keys = rng_seed_keys if rng_seed_keys is not None else [(cfg.seed, k) for k in range(self.n_patches)]
            self.rng = torch.cat([PhiloxStream(keys[k], dev).state for k in range(self.n_patches)])
            n_grid = int(self.synth.grid_base[-1])
            if 3 * n_grid >= 2 ** 31:            # hs_compose indexes the (texel, 3) normals in 32 bits
                raise ConfigError(f"patch grids hold {n_grid} texels; at most {(2 ** 31 - 1) // 3} per GPU")
            self.patch_h = f32(n_grid)
            self.patch_n = f32(3 * n_grid)
            # blended heights per length parity (which flips every frame): frame
            # f writes one buffer while the other still holds frame f - 1, so a
            # host copy of a finished frame (HostFramePipe) reads it in place;
            # `blend_h` is the latest frame's
            self._blend_h2 = (f32(n_grid), f32(n_grid))
            self.blend_h = self._blend_h2[0]
            # the live counts as of each frame's end, per length parity likewise
            # (copied beside the raw-layer clear, off the critical path)
            self._live_snap2 = (torch.zeros_like(self.live), torch.zeros_like(self.live))
            self.blend_n = f32(3 * n_grid)
            # per-frame accumulators in one block of 4-byte words per frame parity:
            # frame f accumulates into set f & 1 while its hs_inject zeroes the other
            # set (frame f + 1's), so no clear sits between concurrent producers
            P = self.n_patches
            nw = 5 * P + (P & 1)
            self.stat_words2 = torch.zeros(2 * nw, dtype=torch.int32, device=dev)
            self._stat_sets = []
            for q in range(2):
                w = self.stat_words2[q * nw:(q + 1) * nw]
                self._stat_sets.append((w, w[0:2 * P].view(torch.float64), w[2 * P:4 * P].view(torch.int64),
                                        w[4 * P:5 * P]))
            self.max_tiles = int(sum(-(-(pc + sc) // ADV_TILE) for pc, sc in zip(self.pool_caps, self.stage_caps)))
            self.tile_state = torch.zeros(self.max_tiles, dtype=torch.int64, device=dev)
            self.keep_words = torch.zeros(self.max_tiles * 32, dtype=torch.int32, device=dev)
            self.tile_counter = torch.zeros(1, dtype=torch.int32, device=dev)
            self._init_boxes()
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        if self.n_patches:
            self._layout(None, self.seg_len[0])

    # ------------------------------------------------------------ helpers --
    def _hr(self, dt: float) -> torch.Tensor:
        if dt not in self._hr_cache:
            hr = np.concatenate([half_rates(r, self.table.omegas, dt, self.config.g).ravel() for r in self.regions])
            self._hr_cache[dt] = torch.from_numpy(hr).to(self.device)
        return self._hr_cache[dt]

    def current_regions(self) -> list:
        """The patch rectangles the last frame synthesised (tracking patches
        move with their source: the device-side synthesis origin, synchronises)."""
        if not (self.n_sources and self._tracking):
            return self.regions
        raw = self.patches_dev.cpu().numpy().tobytes()
        sz = C.sizeof(N.HsPatch)
        out = []
        for k, r in enumerate(self.regions):
            st = N.HsPatch.from_buffer_copy(raw[k * sz:(k + 1) * sz])
            out.append(PatchRegion((st.sx0, st.sy0), r.l1, r.l2, r.margin))
        return out

    def _init_boxes(self) -> None:
        cfg = self.config
        if self.fft_state is None:
            self.box_prefix_np = np.zeros(self.n_patches + 1, np.int32)
            return
        n, spacing = cfg.fft_n, cfg.fft_domain / cfg.fft_n
        boxes, pre = [], [0]
        for r in self.current_regions():       # harness.py:230-233
            lo = np.clip(np.floor(r.min_corner / spacing).astype(int), 0, n)
            hi = np.clip(np.ceil(r.max_corner / spacing).astype(int) + 1, 0, n)
            boxes += [lo[0], hi[0], lo[1], hi[1]]
            pre.append(pre[-1] + max(0, hi[0] - lo[0]) * max(0, hi[1] - lo[1]))
        self.box_np = np.array(boxes, np.int32)
        self.box_prefix_np = np.array(pre, np.int32)
        self.box_dev = torch.from_numpy(self.box_np).to(self.device)
        self.box_prefix_dev = torch.from_numpy(self.box_prefix_np).to(self.device)
        if not hasattr(self, "composite_out"):
            self.composite_out = torch.zeros((n, n), dtype=torch.float32, device=self.device)
        if not hasattr(self, "composite_frame"):
            # every frame's composite (written inside the captured graphs: the
            # background copy on the FFT branch, the patch nodes by hs_compose,
            # which follows tracking patches on the device)
            self.composite_frame = torch.zeros((n, n), dtype=torch.float32, device=self.device)

    def _order_compose_tiles(self) -> None:
        """Launch the compose tiles that touch a patch's blend band first: they
        carry the background work, and in the kernel's single wave the warp
        schedulers favour the older (lower-index) CTAs, so the heavy tiles no
        longer finish last.  (Host geometry only; the kernel decides per tile.)"""
        info = self.synth.compose_info_np
        T = COMPOSE_TILE
        band = np.zeros(len(info), bool)
        for k, (p, i0, j0) in enumerate(info):
            r = self.regions[p]
            res, ny = self.synth.grids[p]
            texel = r.l1 / (res - 1)
            rl, cl = min(T, res - i0) - 1, min(T, ny - j0) - 1
            d = min(min(i0, res - 1 - (i0 + rl)), min(j0, ny - 1 - (j0 + cl))) * texel
            band[k] = d < r.margin + texel
        order = np.concatenate([np.nonzero(band)[0], np.nonzero(~band)[0]])
        self.synth.compose_info_np = np.ascontiguousarray(info[order])
        self.synth.compose_info = torch.from_numpy(self.synth.compose_info_np).to(self.device)

    def _raw_target(self) -> int:
        """Where the splats accumulate: the float raw layers, or (deterministic
        mode) their int64 fixed-point twin."""
        return N.ptr(self.raw_fixed) if self.det else N.ptr(self.synth.raw)

    def _pool(self, k: int) -> N.HsPool:
        return N.pool_struct(*self.pools[k])

    # per-frame stat words of the frame that ran last (see __init__)
    @property
    def stat_words(self):
        return self._stat_sets[self._lp ^ 1][0]

    @property
    def isum(self):
        return self._stat_sets[self._lp ^ 1][1]

    @property
    def icount(self):
        return self._stat_sets[self._lp ^ 1][2]

    @property
    def clamped(self):
        return self._stat_sets[self._lp ^ 1][3]

    def _layout(self, count, len_out) -> None:
        N.call("hs_resident_layout", N.HsLayoutArgs(
            n_patches=self.n_patches, nb=self.nb, patches=N.ptr(self.patches_dev), count=N.ptr(count),
            slack=N.ptr(self.slack), slack_prefix=N.ptr(self.slack_prefix), seg_base=N.ptr(self.seg_base),
            seg_cap=N.ptr(self.seg_cap), len=N.ptr(len_out), live=N.ptr(self.live), tile_map=N.ptr(self.tile_map),
            max_tiles=self.res_tiles, status=N.ptr(self.status)), stream_ptr())

    def _emit_args(self, buf: int, lp: int, dt: float, stats) -> N.HsEmitArgs:
        cfg = self.config
        return N.HsEmitArgs(
            n_sources=self.n_sources, n_patches=self.n_patches, nb=self.nb, sources=N.ptr(self.sources_dev),
            dirs=N.ptr(self.src_dirs), pos_in=N.ptr(self.src_pos[lp]), pos_out=N.ptr(self.src_pos[lp ^ 1]),
            patches=N.ptr(self.patches_dev), buckets=N.ptr(self.buckets_dev), dt=float(dt),
            beta=float(cfg.trough_fraction), rho=float(cfg.rho), g=float(cfg.g), pool=self._pool(buf),
            seg_base=N.ptr(self.seg_base), seg_cap=N.ptr(self.seg_cap), len=N.ptr(self.seg_len[lp ^ 1]),
            live=N.ptr(self.live), e_in=N.ptr(self.e_in), raw_layers=self._raw_target(),
            layers=N.ptr(self.synth.layers), clamped=N.ptr(stats[3]), status=N.ptr(self.status),
            bodies=N.ptr(self.bodies_dev), n_theta=self.table.n_theta, fixed_point=int(self.det))

    def _bodies_args(self, dt: float) -> N.HsBodyArgs:
        cfg = self.config
        bg = self.fft_ws
        a = N.HsBodyArgs(n_bodies=self.n_bodies, bodies=N.ptr(self.bodies_dev), dt=float(dt), rho=float(cfg.rho),
                         g=float(cfg.g), flat=0, frame=N.ptr(self.frame_dev),
                         bg_height=N.ptr(bg.height) if bg is not None else 0,
                         bg_n=cfg.fft_n if bg is not None else 0,
                         bg_spacing=self.fft_state.spacing if bg is not None else 1.0,
                         n_patches=self.n_patches, patches=N.ptr(self.patches_dev), patch_height=N.ptr(self.patch_h))
        ex = self._extra_bg()
        if ex:
            a.n_extra_bg = ex["n_extra_bg"]
            a.extra_bg = ex["extra_bg"]
        return a

    def _resident_args(self, buf: int, lp: int, dt: float, stats) -> N.HsResidentArgs:
        return N.HsResidentArgs(
            n_patches=self.n_patches, nb=self.nb, buckets=N.ptr(self.buckets_dev), patches=N.ptr(self.patches_dev),
            dt=float(dt), rho=float(self.config.rho), g=float(self.config.g), pool=self._pool(buf),
            seg_base=N.ptr(self.seg_base), seg_cap=N.ptr(self.seg_cap), tile_map=N.ptr(self.tile_map),
            max_tiles=self.res_tiles, len_in=N.ptr(self.seg_len[lp]), len_out=N.ptr(self.seg_len[lp ^ 1]),
            live=N.ptr(self.live), stage=N.pool_struct(*self.stage), stage_count=N.ptr(self.stage_count),
            e_out=N.ptr(self.e_out), raw_layers=self._raw_target(), layers=N.ptr(self.synth.layers),
            clamped=N.ptr(stats[3]), status=N.ptr(self.status), fixed_point=int(self.det))

    # --------------------------------------------------------- the frame --
    def _enqueue_frame(self, state: tuple, dt: float, mark=None) -> None:
        """Enqueue one frame (graph-capturable) for resident-pool state
        `state` = (buffer, length parity, compaction frame?).

        In-place frames (K - 1 of every K):
            side  :               └► hs_fft_evolve (rows, cols) ........┐
            inj   : hs_inject (+append) ─┴► hs_emit ──┐                 │
            main  : hs_advect_resident ──────────────┴► hs_smooth ─► join ─► hs_compose
            clr   :                                      └► raw-layer clear ─┘ (end of frame)
        The FFT branch forks after the (one CTA per patch) inject kernel, so
        the resident advect -- the head of the critical chain -- takes the SMs
        first and the transforms fill in behind it (every kernel here fills the
        register file, so the two do not co-reside; forking at frame start cost
        ~8 us of C3 frame).  Compaction frames replace the advect pair by
        hs_inject -> hs_advect (count + scatter into the other buffer,
        squeezing the holes out) -> hs_resident_layout.  `mark(stage)` (optional) is called after each
        stage's launches on the stream that ran it (CUDA events for stage
        timing)."""
        buf, lp, compact = state
        mark = mark or (lambda _name: None)
        main = torch.cuda.current_stream(self.device)
        if self.n_patches and self.n_bodies:
            # buoyancy against the previous frame's surface, before this frame's
            # transform and compose overwrite it (harness.py:155-157)
            N.call("hs_bodies", self._bodies_args(dt), stream_ptr())
        fork = self.fft_state is not None and self.n_patches > 0
        frame_composite = fork and (self.composite_each_frame or self.post_frame is not None)
        def fft_branch(after):
            side = self._side_stream("fft") if fork else main
            if fork:
                side.wait_stream(after)
            with torch.cuda.stream(side):
                mark("fft_start")
                for c, (st_c, ws_c) in enumerate(self.cascades):
                    if self._cshard is not None and not self._cshard.owned(c):
                        continue                    # another rank transforms it (CascadeShard)
                    fa = fft_args(st_c, ws_c, frame_ptr=self.frame_dev, dt=dt)
                    fa.emit_normals = 0      # normals are derived lazily (background) / in hs_compose
                    fa.normal = 0
                    fa.fixed_point = int(self.det)
                    if not self.n_patches and c == len(self.cascades) - 1:
                        fa.frame_advance = N.ptr(self.frame_dev)
                    N.call("hs_fft_evolve", fa, stream_ptr())
                if self._cshard is not None:
                    self._cshard.gather()           # every rank gets every cascade's heights
                if frame_composite:             # the composite starts as the background; hs_compose
                    self._composite(self.composite_frame, (None, None, 0))   # blends the patch nodes in
                mark("fft")
        if self.fft_state is not None and not fork:
            fft_branch(main)
        if self.n_patches:
            stats, nxt = self._stat_sets[lp], self._stat_sets[lp ^ 1]
            cfg = self.config
            if self.n_sources and self._tracking:       # before every stage that reads the patch rectangles
                N.call("hs_track", self._emit_args(buf, lp, dt, stats), stream_ptr())
            inj_args = N.HsInjectArgs(
                n_patches=self.n_patches, nb=self.nb, n_theta=self.table.n_theta, buckets=N.ptr(self.buckets_dev),
                patches=N.ptr(self.patches_dev), half_rate=N.ptr(self._hr(dt)),
                mean_dir=float(cfg.mean_direction), beta=float(cfg.trough_fraction),
                rho=float(cfg.rho), g=float(cfg.g), acc=N.ptr(self.acc), groups=N.ptr(self.groups),
                e_in=N.ptr(self.e_in), rng=N.ptr(self.rng), stage=N.pool_struct(*self.stage),
                stage_count=N.ptr(self.stage_count), scratch=N.ptr(self.scratch), member_capacity=self.member_cap,
                status=N.ptr(self.status), zero_words=N.ptr(nxt[0]), n_zero_words=nxt[0].numel(),
                birth_frame=N.ptr(self.frame_dev), birth_dt=float(dt))    # t = frame * dt (harness.py:134)
            if compact:
                mark("particles_start")
                N.call("hs_inject", inj_args, stream_ptr())
                mark("inject")
                if fork:
                    fft_branch(main)
                N.call("hs_advect", N.HsAdvectArgs(
                    n_patches=self.n_patches, nb=self.nb, buckets=N.ptr(self.buckets_dev),
                    patches=N.ptr(self.patches_dev), dt=float(dt), rho=float(cfg.rho), g=float(cfg.g),
                    in_=self._pool(buf), in_count=N.ptr(self.seg_len[lp]), stage=N.pool_struct(*self.stage),
                    stage_count=N.ptr(self.stage_count), out=self._pool(buf ^ 1),
                    out_count=N.ptr(self.compact_count), dropped=N.pool_struct(), dropped_count=0,
                    e_out=N.ptr(self.e_out), splat=1, raw_layers=self._raw_target(),
                    raw_layers_len=self.synth.pack.raw_len * (2 if self.det else 1), layers=N.ptr(self.synth.layers),
                    clamped=N.ptr(stats[3]), tile_state=N.ptr(self.tile_state), max_tiles=self.max_tiles,
                    tile_counter=N.ptr(self.tile_counter), status=N.ptr(self.status),
                    keep_words=N.ptr(self.keep_words), in_seg_base=N.ptr(self.seg_base),
                    out_slack_prefix=N.ptr(self.slack_prefix), raw_is_clear=1, fixed_point=int(self.det)), stream_ptr())
                self._layout(self.compact_count, self.seg_len[lp ^ 1])
                if self.n_sources:
                    N.call("hs_emit", self._emit_args(buf ^ 1, lp, dt, stats), stream_ptr())
                mark("advect")
            else:
                ra = self._resident_args(buf, lp, dt, stats)
                inj_args.append = 1                 # new particles go straight to the segment tails
                inj_args.res = ra
                inj = self._side_stream("inject")
                inj.wait_stream(main)
                with torch.cuda.stream(inj):
                    mark("inject_start")
                    N.call("hs_inject", inj_args, stream_ptr())
                    mark("inject")
                if fork:                            # FFT branch forks after the 1-CTA-per-patch inject:
                    fft_branch(main if self.fft_fork_at_start else inj)   # the resident advect fills the SMs first
                with torch.cuda.stream(inj):
                    if self.n_sources:
                        N.call("hs_emit", self._emit_args(buf, lp, dt, stats), stream_ptr())
                        mark("emit")
                mark("particles_start")
                N.call("hs_advect_resident", ra, stream_ptr())
                mark("advect")
                main.wait_stream(inj)
                mark("join_inject")
            if self.det:                        # fixed-point raw layers -> the float ones hs_smooth reads
                N.call_raw("hs_fixed_to_float", N.vp(N.ptr(self.raw_fixed)), N.vp(N.ptr(self.synth.raw)),
                           N.i64(self.raw_fixed.numel()), N.i32(N.HS_FIXED_SPLAT_BITS), N.vp(stream_ptr()))
            N.call("hs_smooth", self.synth.smooth_args(), stream_ptr())
            mark("smooth")
            clr = self._side_stream("clear")
            clr.wait_stream(main)
            with torch.cuda.stream(clr):        # raw layers are consumed: clear them for the next splat
                self._live_snap2[lp].copy_(self.live)
                raw = self.raw_fixed if self.det else self.synth.raw
                N.call_raw("hs_clear", N.vp(N.ptr(raw)), N.i64(raw.numel() * raw.element_size()), N.vp(stream_ptr()))
            if fork:
                main.wait_stream(self._side_stream("fft"))
                mark("join")
            bg = self.fft_ws
            N.call("hs_compose", N.HsComposeArgs(
                n_patches=self.n_patches, nb=self.nb, patches=N.ptr(self.patches_dev), layers=N.ptr(self.synth.layers),
                smooth_layers=N.ptr(self.synth.smooth), tile_info=N.ptr(self.synth.compose_info),
                total_tiles=self.synth.compose_tiles,
                bg_height=N.ptr(bg.height) if bg is not None else 0,
                bg_normal=0,                  # hs_compose derives them from the staged heights
                bg_n=self.config.fft_n if bg is not None else 0,
                bg_spacing=self.config.fft_domain / self.config.fft_n if bg is not None else 1.0,
                patch_height=N.ptr(self.patch_h), patch_normal=0,
                blend_height=N.ptr(self._blend_h2[state[1]]), blend_normal=N.ptr(self.blend_n), blend_mode=1,
                interior_sumsq=N.ptr(stats[1]), interior_count=N.ptr(stats[2]),
                frame_advance=N.ptr(self.frame_dev), fixed_point=int(self.det),
                composite=N.ptr(self.composite_frame) if frame_composite else 0, **self._extra_bg()), stream_ptr())
            mark("compose")
            main.wait_stream(clr)
            self._patch_n_frame = -1          # patch normals are derived lazily (patch_field)
        self._bg_n_frame = -1                 # so are the background normals (background)
        if self.fft_state is None and not self.n_patches:
            N.call_raw("hs_advance_frame", N.vp(N.ptr(self.frame_dev)), N.vp(stream_ptr()))
        if self.post_frame is not None:
            self.post_frame()
            mark("post_frame")

    def _extra_bg(self) -> dict:
        """n_extra_bg / extra_bg args for cascades 1.. (HsBgTile)."""
        if len(self.cascades) < 2:
            return {}
        arr = (N.HsBgTile * (N.HS_MAX_CASCADES - 1))()
        for c, (st_c, ws_c) in enumerate(self.cascades[1:]):
            arr[c] = N.HsBgTile(N.ptr(ws_c.height), st_c.n, 0, float(st_c.spacing))
        return {"n_extra_bg": len(self.cascades) - 1, "extra_bg": arr}

    def cascade_fields(self) -> list:
        """HeightFields of every background cascade (cascade 0 = `background`)."""
        return [ws.field(st) for st, ws in self.cascades]

    def _state(self) -> tuple:
        if not self.n_patches:
            return (0, 0, False)
        return (self._buf, self._lp, self._since == self.compact_period - 1)

    def _advance_state(self, state: tuple) -> None:
        """After the frame of `state` ran (never during a capture)."""
        if not self.n_patches:
            return
        buf, lp, compact = state
        self.blend_h = self._blend_h2[lp]
        self._lp = lp ^ 1
        if compact:
            self._buf = buf ^ 1
            self._since = 0
        else:
            self._since += 1

    # stream priorities of the frame's branches (lower = more urgent): the
    # particle / synthesis chain is the critical path, the FFT fills idle SMs
    # (tools/ab_sched.py: no measurable effect at C3, off by default)
    STREAM_PRIORITY = {"fft": 0}
    CRITICAL_PRIORITY = -5

    def _side_stream(self, name: str = "fft"):
        if not hasattr(self, "_sides"):
            self._sides = {}
        if name not in self._sides:
            prio = self.STREAM_PRIORITY.get(name, self.CRITICAL_PRIORITY) if self.sched_priorities else 0
            # streams of this Simulation alone (not torch's shared round-robin pool,
            # whose streams a collective library may also be handed)
            self._sides[name] = N.OwnedStream(self.device, prio)
        return self._sides[name].stream

    def _capture_stream(self):
        if not hasattr(self, "_capture_owned"):
            self._capture_owned = N.OwnedStream(self.device, self.CRITICAL_PRIORITY if self.sched_priorities else 0)
        return self._capture_owned.stream

    def _graph(self, state: tuple):
        g = self._graphs.get(state)
        if g is None:
            if self.n_patches:
                self._hr(self.config.dt)        # host->device uploads must precede capture
            N.configure_device(self.device)     # so must the kernels' attribute calls
            g = torch.cuda.CUDAGraph()
            s = self._capture_stream()
            s.wait_stream(torch.cuda.current_stream(self.device))
            # thread_local: CUDA calls other threads make meanwhile (the NCCL
            # watchdog of a multi-GPU run) must not invalidate this capture
            with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
                self._enqueue_frame(state, self.config.dt)
            torch.cuda.current_stream(self.device).wait_stream(s)
            self._graphs[state] = g
        return g

    def prepare_graphs(self) -> None:
        """Capture the frame graph of every resident-pool state up front
        (buffer x length parity x compaction), so no capture happens while
        stepping (capture enqueues nothing; it only records)."""
        if not self.config.graph:
            return
        states = [(b, l, c) for b in (0, 1) for l in (0, 1) for c in (False, True)] if self.n_patches else [(0, 0, False)]
        for st in states:
            self._graph(st)

    def kernel_launches_per_frame(self) -> float:
        """Library kernels one frame launches on average (csrc/*.cu): fft rows
        + cols; inject; in-place frames advect_resident + append_resident,
        compaction frames (1 in K) advect count + scatter + layout; smooth
        (1 or 3); compose.  (The raw-layer clear is a memset node.)"""
        k = 0.0
        if self.fft_state is not None:
            k += 2                            # rows + columns (normals are lazy)
        if self.n_patches:
            pk = self.synth.pack
            K = self.compact_period
            k += 1 + (1.0 * (K - 1) + 3.0) / K       # inject (+append fused); advect or count+scatter+layout
            if self.n_sources:
                k += 2 + (1 if self._tracking else 0)      # emit + commit (+ track)
            k += (1 if pk.smooth_tile_info.shape[0] > 0 else 0) + (2 if pk.xtile_prefix[-1] > 0 else 0)
            k += 1 if self.det else 0                 # fixed-point raw layers -> float
            k += 1                                    # compose
            if self.fft_state is not None and (self.composite_each_frame or self.post_frame is not None):
                k += 1 if len(self.cascades) > 1 else 0   # composite background (cascade sum; else a copy)
        return max(k, 1.0)

    def timed_frame(self) -> dict:
        """Replay one frame from a CUDA graph that carries timing-event record
        nodes after every stage; returns {stage: ms} (synchronises).  Each
        stage is timed against the previous event on its own stream, so the
        concurrently running branches are each per-kernel device times
        without host launch gaps.  Used by bench.py for the per-kernel
        roofline.  Returns the stages of an in-place frame (the K - 1 in K
        common case); compaction frames are timed by `timed_compaction`."""
        state = self._state()
        key = ("timed",) + state
        if key not in self._graphs:
            if self.n_patches:
                self._hr(self.config.dt)
            N.configure_device(self.device)
            evs = []

            def mark(name):
                e = torch.cuda.Event(enable_timing=True, external=True)
                strm = torch.cuda.current_stream(self.device)
                e.record(strm)
                evs.append((name, e, strm.cuda_stream))
            g = torch.cuda.CUDAGraph()
            s = self._capture_stream()
            s.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
                self._enqueue_frame(state, self.config.dt, mark)
            torch.cuda.current_stream(self.device).wait_stream(s)
            self._graphs[key] = (g, evs)
        g, evs = self._graphs[key]
        g.replay()
        self._advance_state(state)
        self.frame += 1
        torch.cuda.synchronize(self.device)
        out, last = {}, {}
        for name, e, sid in evs:
            if sid in last and not name.endswith("_start") and not name.startswith("join"):
                out[name] = out.get(name, 0.0) + last[sid].elapsed_time(e)
            last[sid] = e
        names = [n for n, _, _ in evs]
        if "compose" in out:
            first = next(e for n, e, _ in evs if n in ("fft_start", "particles_start", "inject_start"))
            end = next(e for n, e, _ in evs if n == "compose")
            out["frame"] = first.elapsed_time(end)
        out["compaction"] = 1.0 if state[2] else 0.0
        del names
        return out

    def step(self, dt: float | None = None, *, stats: bool = True):
        """Advance one frame.  With the configured dt and `config.graph` the
        frame is a single CUDA graph replay (the first frame runs eagerly to
        load modules).  Returns lazy FrameStats (or None if stats=False)."""
        cfg = self.config
        use_dt = cfg.dt if dt is None else float(dt)
        self.t = self.frame * use_dt
        state = self._state()
        if cfg.graph and use_dt == cfg.dt and self.frame > 0:
            self._graph(state).replay()
        else:
            self._enqueue_frame(state, use_dt)
        self._advance_state(state)
        out = None
        if stats:
            out = self._snapshot()
            self._stats.append(out)
        self.frame += 1
        return out

    def run_frames(self, k: int, dt: float | None = None) -> None:
        for _ in range(k):
            self.step(dt, stats=False)

    def _snapshot(self) -> FrameStats:
        # summed cascades: band variances add (disjoint |k| bands)
        snap = {"fsum": sum(ws.sumsq for _, ws in self.cascades).clone() if self.cascades
                else torch.zeros(1, dtype=torch.float64)}
        if self.n_patches:
            snap.update(counts=self.live.clone(), e_in=self.e_in.clone(), e_out=self.e_out.clone(),
                        isum=self.isum.clone(), icount=self.icount.clone())
            if self.n_bodies:
                snap["bodies"] = self.bodies_dev.clone()
        return FrameStats(frame=self.frame, t=self.t, stage_ms={s: 0.0 for s in STAGES}, _snap=snap, _nb=self.nb,
                          _n_patches=self.n_patches, _fft_n=self.config.fft_n if self.fft_ws is not None else 0,
                          _fixed=self.det)

    def check(self) -> None:
        """Raise if a device capacity flag was set (synchronises)."""
        s = int(self.status.item())
        if s & N.HS_STATUS_POOL_OVERFLOW:
            raise CapacityError(f"particle pool overflow (capacity {self.pool_caps}); raise device.pool_capacity")
        if s & N.HS_STATUS_STAGE_OVERFLOW:
            raise CapacityError("injection staging overflow")
        if s & N.HS_STATUS_BOX_OVERFLOW:
            raise CapacityError("composite exchange box larger than its slot")

    # ----------------------------------------------------------- outputs --
    @property
    def background(self) -> HeightField | None:
        """The frame's background HeightField; its normals (grid_normals,
        fft_background.py:205) are materialised on first access per frame."""
        if self.fft_ws is None:
            return None
        if getattr(self, "_bg_n_frame", -1) != self.frame and self.fft_ws.normal is not None:
            N.call_raw("hs_periodic_normals", N.vp(N.ptr(self.fft_ws.height)), N.vp(N.ptr(self.fft_ws.normal)),
                       self.config.fft_n, self.config.fft_domain / self.config.fft_n, N.vp(stream_ptr()))
            self._bg_n_frame = self.frame
        return self.fft_ws.field(self.fft_state)

    @property
    def counts(self) -> torch.Tensor:
        """(n_patches * nb) live particles per (patch, bucket), on the device."""
        return self.live

    def counts_host(self) -> np.ndarray:
        """(n_patches, nb) live particles per bucket (synchronises)."""
        return self.live.cpu().numpy().reshape(self.n_patches, self.nb).astype(np.int64)

    def live_particles(self) -> int:
        return int(self.live.sum().item()) if self.n_patches else 0

    def pool(self, k: int) -> ParticleSet:
        """Patch k's current pool as a ParticleSet, bucket-segmented in the
        reference's stable order: the live slots of each resident segment,
        holes dropped (the compaction the device defers, particles.py:167-178)."""
        nb = self.nb
        base = self.seg_base.cpu().numpy()[k * nb:(k + 1) * nb]
        ln = self.seg_len[self._lp].cpu().numpy()[k * nb:(k + 1) * nb]
        arrs = self.pools[self._buf]
        parts = [[] for _ in range(6)]
        counts = np.zeros(nb, np.int64)
        for b in range(nb):
            lo, n = int(base[b]), int(ln[b])
            x = arrs[0][lo:lo + n]
            keep = ~torch.isnan(x)
            for q in range(6):
                parts[q].append(arrs[q][lo:lo + n][keep])
            counts[b] = int(keep.sum().item())
        cat = [torch.cat(p_) if p_ else arrs[q][:0] for q, p_ in enumerate(parts)]
        return ParticleSet.from_segments(*cat[:5], counts, self.device, birth=cat[5])

    def _grid(self, buf: torch.Tensor, k: int, comps: int = 1) -> torch.Tensor:
        res, ny = self.synth.grids[k]
        b = int(self.synth.grid_base[k])
        if comps == 1:
            return buf[b:b + res * ny].view(res, ny)
        return buf[3 * b:3 * (b + res * ny)].view(res, ny, 3)

    def patch_heights(self, k: int) -> torch.Tensor:
        return self._grid(self.patch_h, k)

    def patch_field(self, k: int) -> HeightField:
        """Patch k's finished field (finish_field): heights from the last
        frame, clamped-border normals derived on demand (hs_finish)."""
        res, ny = self.synth.grids[k]
        r = self.current_regions()[k]
        if getattr(self, "_patch_n_frame", -1) != self.frame:
            for q, (rq, nyq) in enumerate(self.synth.grids):
                N.call("hs_finish", N.HsFinishArgs(nx=rq, ny=nyq, spacing=self.regions[q].l1 / (rq - 1),
                                                   chop_scale=0.0, height=N.ptr(self._grid(self.patch_h, q)),
                                                   normal=N.ptr(self._grid(self.patch_n, q, 3)), disp=0),
                       stream_ptr())
            self._patch_n_frame = self.frame
        return HeightField(resolution=res, origin=r.min_corner.copy(), spacing=r.l1 / (res - 1),
                           height=self._grid(self.patch_h, k), normal=self._grid(self.patch_n, k, 3),
                           displacement=torch.zeros((res, ny, 2), dtype=torch.float32, device=self.device),
                           periodic=False)

    def blended_tile(self, k: int) -> tuple[torch.Tensor, torch.Tensor]:
        """Blended (height, normal) at patch k's nodes (SurfaceSampler at the
        patch grid, coupling.py:120-141)."""
        return self._grid(self.blend_h, k), self._grid(self.blend_n, k, 3)

    @property
    def sampler(self) -> SurfaceSampler:
        surfaces = [PatchSurface(r, self.patch_field(k)) for k, r in enumerate(self.current_regions())]
        return SurfaceSampler(self.background, surfaces, self.config.normal_mode,
                              cascades=self.cascade_fields()[1:])

    def surface_from_heights(self, points) -> tuple:
        """(heights, normals) of the last frame's blended surface at world
        points, normals from finite differences of the height grids -- the
        sampler the bodies step against (hs_sample, from_heights)."""
        cfg = self.config
        pts = torch.as_tensor(np.asarray(points, dtype=np.float64).reshape(-1, 2), device=self.device).contiguous()
        n = pts.shape[0]
        out_h = torch.empty(n, dtype=torch.float32, device=self.device)
        out_n = torch.empty((n, 3), dtype=torch.float32, device=self.device)
        bg = self.fft_ws
        a = N.HsSampleArgs(n_points=n, points=N.ptr(pts), bg_height=N.ptr(bg.height) if bg is not None else 0,
                           bg_normal=0, bg_n=cfg.fft_n if bg is not None else 0,
                           bg_spacing=self.fft_state.spacing if bg is not None else 1.0, bg_x0=0.0, bg_y0=0.0,
                           n_patches=self.n_patches, patches=N.ptr(self.patches_dev) if self.n_patches else 0,
                           patch_height=N.ptr(self.patch_h) if self.n_patches else 0, patch_normal=0,
                           out_height=N.ptr(out_h), out_normal=N.ptr(out_n), clamped_only=0, from_heights=1)
        ex = self._extra_bg()
        if ex:
            a.n_extra_bg = ex["n_extra_bg"]
            a.extra_bg = ex["extra_bg"]
        N.call("hs_sample", a, stream_ptr())
        return out_h, out_n

    def _composite(self, out: torch.Tensor, boxes=None) -> None:
        """Enqueue the FFT-resolution composite into `out` (graph-capturable);
        boxes = (box, box_prefix, total) device geometry, default the current."""
        cfg = self.config
        n = cfg.fft_n
        bg = self.fft_ws
        if boxes is None:
            boxes = (self.box_dev, self.box_prefix_dev, int(self.box_prefix_np[-1])) if self.n_patches else (None, None, 0)
        N.call("hs_composite", N.HsCompositeArgs(
            n=n, spacing=cfg.fft_domain / n, bg_height=N.ptr(bg.height), bg_normal=0,
            n_patches=self.n_patches, patches=N.ptr(self.patches_dev) if self.n_patches else 0,
            patch_height=N.ptr(self.patch_h) if self.n_patches else 0, patch_normal=0,
            box=N.ptr(boxes[0]), box_prefix=N.ptr(boxes[1]), total_box=boxes[2], out=N.ptr(out),
            **self._extra_bg()), stream_ptr())

    def stitched_heights(self) -> torch.Tensor:
        """FFT-resolution composite with patch boxes resampled (harness.py:219-241).
        Every frame already ends with it (composite_out); this re-forms it on
        demand (tracking patches: with the boxes moved to their current rectangles)."""
        cfg = self.config
        n = cfg.fft_n
        if self.fft_state is None:
            raise ConfigError("stitched_heights needs the FFT background (mode != wp-only)")
        if self.n_sources and self._tracking:
            self._init_boxes()                    # the composited boxes follow the tracking patches
        if not self.n_patches:
            out = torch.empty((n, n), dtype=torch.float32, device=self.device)
            self._composite(out)
            return out
        self._composite(self.composite_out)
        return self.composite_out

    def shard_cascades(self, shard) -> None:
        """Transform only this rank's FFT cascades (sharding.CascadeShard) and
        all-gather their heights every frame.  Call before the frame graphs are
        captured; the cascades' height grids become views of the shard buffer.
        Displacement grids and FFT-band variances of other ranks' cascades are
        not exchanged (neither enters the blend or the composite)."""
        if len(self.cascades) < 2 or shard.n_cascades != len(self.cascades) or shard.n != self.config.fft_n:
            raise ConfigError("shard_cascades needs a summed-cascade background matching the shard")
        for c, (_, ws) in enumerate(self.cascades):
            v = shard.view(c)
            v.copy_(ws.height)
            ws.height = v
        self._cshard = shard
        self._graphs = {}

    def background_sum(self, out: torch.Tensor) -> torch.Tensor:
        """The background height grid the composite starts from (the summed
        cascades on cascade 0's grid, or the single FFT tile)."""
        cfg = self.config
        n = cfg.fft_n
        bg = self.fft_ws
        N.call("hs_composite", N.HsCompositeArgs(
            n=n, spacing=cfg.fft_domain / n, bg_height=N.ptr(bg.height), bg_normal=0, n_patches=0,
            total_box=0, out=N.ptr(out), **self._extra_bg()), stream_ptr())
        return out

    def source_positions(self) -> np.ndarray:
        """(n_bodies + n_sources, 2) emitter positions after the last frame
        (bodies first, then kinematic sources; synchronises)."""
        if not self.n_sources:
            return np.zeros((0, 2))
        return self.src_pos[self._lp].cpu().numpy().reshape(-1, 2).copy()

    def ledger_host(self) -> dict:
        P, nb = self.n_patches, self.nb
        e_out = self.e_out.cpu().numpy()
        if self.det:
            e_out = fixed_to_double(e_out, N.HS_FIXED_ENERGY_BITS)
        return {"acc": self.acc.cpu().numpy().reshape(P, nb, 4), "groups": self.groups.cpu().numpy().reshape(P, nb),
                "e_in": self.e_in.cpu().numpy().reshape(P, nb), "e_out": e_out.reshape(P, nb)}


class HostFramePipe:
    """Streams every frame's blended patch tiles and live counts to pinned host
    memory while the next frame computes.  Both are copied straight from the
    frame's own buffers (blended heights and a live-count snapshot, one of
    each per length parity, so frame k + 1 writes the other ones): no device
    copy sits between frames.  A frame waits only for the host copy that last
    read its buffers (frame k - 2) and for the host slot it reuses, so
    end-to-end throughput is max(frame time, transfer time) instead of their
    sum.  `step()` returns the slot whose host buffers
    `result(slot)` fills."""

    def __init__(self, sim: "Simulation", depth: int = 2):
        self.sim = sim
        self.depth = depth
        self.n = int(sim.synth.grid_base[-1])
        dev = sim.device
        self.host = [torch.empty(self.n, dtype=torch.float32, pin_memory=True) for _ in range(depth)]
        self.host_cnt = [torch.empty(sim.live.numel(), dtype=torch.int32, pin_memory=True) for _ in range(depth)]
        self.copy = torch.cuda.Stream(device=dev)
        self.done = [torch.cuda.Event() for _ in range(depth)]
        self.buf_read = [torch.cuda.Event(), torch.cuda.Event()]     # last host copy out of parity p's buffers
        self.k = 0

    @property
    def bytes_per_frame(self) -> int:
        return 4 * self.n + 4 * self.sim.live.numel()

    def step(self, dt: float | None = None) -> int:
        i = self.k % self.depth
        sim = self.sim
        main = torch.cuda.current_stream(sim.device)
        lp = sim._state()[1]                      # the blend buffer this frame writes
        main.wait_event(self.done[i])            # slot i's previous host copy has landed
        main.wait_event(self.buf_read[lp])       # and so has the last copy out of parity lp's buffers
        sim.step(dt, stats=False)
        ready = torch.cuda.Event()
        ready.record(main)
        with torch.cuda.stream(self.copy):
            self.copy.wait_event(ready)
            self.host[i].copy_(sim.blend_h[: self.n], non_blocking=True)
            self.host_cnt[i].copy_(sim._live_snap2[lp], non_blocking=True)
            self.buf_read[lp].record(self.copy)
            self.done[i].record(self.copy)
        self.k += 1
        return i

    def result(self, slot: int) -> tuple:
        """(blended tiles of every patch, flat f32; live counts) of the frame in `slot`."""
        self.done[slot].synchronize()
        return self.host[slot], self.host_cnt[slot]


@dataclass
class BenchRow:
    """One cell of the throughput sweep (harness.py:324-343)."""
    label: str
    mode: str
    n_omega: int
    n_theta: int
    u10: float
    res: int
    fps: float
    median_frame_ms: float
    particles: int
    particle_rate: float


def wp_only_config(base: SimConfig) -> SimConfig:
    """Single patch covering the whole domain at the same texel density (harness.py:332-342)."""
    from dataclasses import replace
    from .config import PatchConfig
    density_res = base.patches[0].res if base.patches else 512
    patch_size = base.patches[0].size[0] if base.patches else 100.0
    scale = base.fft_domain / patch_size
    big = PatchConfig(origin=(0.0, 0.0), size=(base.fft_domain, base.fft_domain),
                      res=int(round((density_res - 1) * scale)) + 1,
                      margin=base.patches[0].margin if base.patches else 10.0)
    return replace(base, mode="wp-only", patches=(big,), bodies=())


def benchmark_cell(cfg: SimConfig, warmup: int | None = None, measure: int | None = None,
                   label: str = "") -> BenchRow:
    """Steady-state throughput of one cell (harness.py:345-369): median of the
    per-frame device times (CUDA events), particle rate over the wall clock."""
    warmup = cfg.bench_warmup if warmup is None else warmup
    measure = cfg.bench_measure if measure is None else measure
    sim = Simulation(cfg)
    sim.run_frames(warmup)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(measure)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for a, b in ev:
        a.record()
        sim.step(stats=False)
        b.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = float(np.median([a.elapsed_time(b) for a, b in ev])) if ev else float("nan")
    live = sim.live_particles()
    res = cfg.patches[0].res if cfg.patches else 0
    return BenchRow(label=label or cfg.mode, mode=cfg.mode, n_omega=cfg.n_omega, n_theta=cfg.n_theta, u10=cfg.u10,
                    res=res, fps=1e3 / ms if ms > 0 else float("inf"), median_frame_ms=ms, particles=live,
                    particle_rate=live * measure / wall if wall > 0 else 0.0)


def trend_matrix(base: SimConfig) -> list:
    """The performance-sweep cells (harness.py:372-396): method, sampling
    counts, wind, resolution."""
    from dataclasses import replace

    def with_counts(n):
        return replace(base, n_omega=n, n_theta=n)

    def with_res(r):
        return replace(base, patches=tuple(replace(p, res=r) for p in base.patches))

    return [
        ("fft-only", replace(base, mode="fft-only")),
        ("wp-only", wp_only_config(base)),
        ("hybrid-16x16", with_counts(16)),
        ("hybrid-12x12", with_counts(12)),
        ("hybrid-8x8", with_counts(8)),
        ("res-256", with_res(256)),
        ("res-1024", with_res(1024)),
        ("u10-3", replace(base, u10=3.0)),
        ("u10-10", replace(base, u10=10.0)),
        ("u10-15", replace(base, u10=15.0)),
    ]


def benchmark(cells: list, warmup: int | None = None, measure: int | None = None, progress=None) -> list:
    """benchmark_cell over the cells (harness.py:399-413); the full-domain
    wp-only cell keeps its sample short, as the reference does."""
    rows = []
    for label, cfg in cells:
        w, m = warmup, measure
        if cfg.mode == "wp-only":
            w = min(w if w is not None else cfg.bench_warmup, 4)
            m = min(m if m is not None else cfg.bench_measure, 3)
        row = benchmark_cell(cfg, w, m, label)
        rows.append(row)
        if progress is not None:
            progress(row)
    return rows


def bench_table(rows: list) -> str:
    """CSV of benchmark rows, the reference's columns (harness.py:416-423)."""
    header = "label,mode,n_omega,n_theta,u10,res,fps,median_frame_ms,particles,particle_rate"
    lines = [header]
    for r in rows:
        lines.append(f"{r.label},{r.mode},{r.n_omega},{r.n_theta},{r.u10},{r.res},"
                     f"{r.fps:.3f},{r.median_frame_ms:.3f},{r.particles},"
                     f"{r.particle_rate:.1f}")
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------------------
# headless run with file outputs (harness.py:248-329)
# ---------------------------------------------------------------------------

def _format_float(x: float) -> str:
    return repr(float(x))


def stats_header(cfg: SimConfig) -> str:
    """stats.csv header (harness.py:252-260)."""
    cols = ["frame", "t", "particles_total"]
    cols += [f"particles_b{i:02d}" for i in range(cfg.n_omega)]
    cols += [f"injected_J_b{i:02d}" for i in range(cfg.n_omega)]
    cols += [f"despawned_J_b{i:02d}" for i in range(cfg.n_omega)]
    cols += ["patch_variance", "fft_band_variance"]
    for j in range(len(cfg.bodies)):
        cols += [f"body{j}_x", f"body{j}_y", f"body{j}_z", f"body{j}_yaw"]
    return ",".join(cols)


def stats_row(cfg: SimConfig, s: FrameStats) -> str:
    """One stats.csv row (harness.py:263-271); reads the frame's device snapshot."""
    parts = [str(s.frame), _format_float(s.t), str(int(s.particle_counts.sum()))]
    parts += [str(int(c)) for c in s.particle_counts]
    parts += [_format_float(x) for x in s.injected_energy]
    parts += [_format_float(x) for x in s.despawned_energy]
    parts += [_format_float(s.patch_variance), _format_float(s.fft_band_variance)]
    for b in s.body_states:
        parts += [_format_float(v) for v in b]
    return ",".join(parts)


def run(config: SimConfig, output_dir: str | None = None, progress=None) -> list:
    """Headless scenario (harness.py:274-329): config.echo, stats.csv,
    timings.csv and `frame_%06d.raw` (<f4, row-major, x-major) + `.meta`
    sidecars of the FFT-resolution composite every `output.stride` frames.
    Frames are stepped as CUDA-graph replays; the device->host copies of the
    stats snapshots and frames happen after each step, in frame order.
    timings.csv carries the device time of each frame (CUDA events) in
    total_ms; per-stage wall times do not exist for a single-graph frame and
    are written as 0."""
    import os
    from .config import dump_config

    cfg = config.validate()
    out_dir = output_dir if output_dir is not None else cfg.output_dir
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "config.echo"), "w", encoding="utf-8") as fh:
        fh.write(dump_config(cfg))
    sim = Simulation(cfg)
    n = cfg.fft_n
    spacing = cfg.fft_domain / n
    with open(os.path.join(out_dir, "stats.csv"), "w", encoding="utf-8") as sfh, \
            open(os.path.join(out_dir, "timings.csv"), "w", encoding="utf-8") as tfh:
        sfh.write(stats_header(cfg) + "\n")
        tfh.write("frame," + ",".join(f"{st}_ms" for st in STAGES) + ",total_ms\n")
        for k in range(cfg.frames):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s = sim.step()
            e1.record()
            if cfg.write_frames and k % cfg.output_stride == 0 and sim.fft_state is not None:
                grid = sim.stitched_heights().cpu().numpy()
                path = os.path.join(out_dir, f"frame_{k:06d}.raw")
                grid.astype("<f4").tofile(path)
                with open(path[:-4] + ".meta", "w", encoding="utf-8") as mfh:
                    mfh.write(f"res={n}x{n} spacing={spacing!r} origin=0.0,0.0 t={s.t!r}\n")
            sfh.write(stats_row(cfg, s) + "\n")
            e1.synchronize()
            tfh.write(",".join([str(s.frame)] + ["0.000" for _ in STAGES] + [f"{e0.elapsed_time(e1):.3f}"]) + "\n")
            if progress is not None:
                progress(s)
    return sim._stats
