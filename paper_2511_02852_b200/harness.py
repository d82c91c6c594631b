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

import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from ._layout import (bucket_structs, half_rates, max_groups_per_step, patch_struct, stream_ptr,
                      structs_to_device)
from .config import SimConfig
from .coupling import PatchSurface, SurfaceSampler, validate_patches
from .errors import CapacityError, ConfigError
from .fft_background import FftWorkspace, HeightField, fft_args, init_fft
from .particles import PatchRegion, PhiloxStream, ParticleSet
from .patch_synthesis import SynthWorkspace, plan_layers
from .spectrum import DirectionalSpectrum, build_buckets, derive_params, log_buckets

STAGES = ("fft", "inject", "advect", "interact", "synth", "blend", "output")
ADV_TILE = 1024


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

    def _get(self):
        if not self._cache:
            s = {k: v.cpu().numpy() for k, v in self._snap.items()}
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
                 rng_seed_keys: list | None = None):
        cfg = config.validate()
        if cfg.bodies:
            raise ConfigError("floating bodies are outside the B200 hybrid-step path (SURVEY 8(f))")
        self.config = cfg
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
        if cfg.mode != "wp-only":
            band = None
            if cfg.fft_band_lo is not None or cfg.fft_band_hi is not None:
                band = (cfg.fft_band_lo, cfg.fft_band_hi)
            self.fft_state = init_fft(self.spectrum, cfg.fft_n, cfg.fft_domain, cfg.seed,
                                      choppiness=cfg.fft_choppiness, band=band, device=dev)
            self.fft_ws = FftWorkspace(cfg.fft_n, dev, normals=cfg.fft_normals or self.n_patches > 0)
        self.frame_dev = torch.zeros(1, dtype=torch.int64, device=dev)

        # ---- constants ---------------------------------------------------
        self.buckets_dev = structs_to_device(bucket_structs(self.table, self.params), dev)
        self._hr_cache = {}
        self.pool_caps, self.stage_caps, self.member_cap = [], [], 1
        for k, r in enumerate(self.regions):
            if pool_capacity is not None:
                cap = int(pool_capacity)
            elif cfg.pool_capacity:
                cap = cfg.pool_capacity
            else:
                cap = max(4096, int(1.6 * estimate_population(self.table, r, cfg.trough_fraction)))
                cap = -(-cap // 1024) * 1024
            hr_max = half_rates(r, self.table.omegas, 0.1, cfg.g)       # dt <= 0.1 (config.py validate)
            mg = max_groups_per_step(hr_max)
            self.member_cap = max(self.member_cap, mg * self.table.n_theta)
            self.pool_caps.append(cap)
            self.stage_caps.append(2 * mg * self.table.n_theta)
        self.pool_base = np.concatenate([[0], np.cumsum(self.pool_caps)]).astype(np.int64)
        self.stage_base = np.concatenate([[0], np.cumsum(self.stage_caps)]).astype(np.int64)
        total_pool = int(self.pool_base[-1])
        total_stage = int(self.stage_base[-1])

        if self.n_patches:
            self.synth = SynthWorkspace(self.regions, self.res, self.plans, dev)
            structs = []
            for k, (r, res) in enumerate(zip(self.regions, self.res)):
                structs.append(patch_struct(r, res, pool_base=self.pool_base[k], pool_capacity=self.pool_caps[k],
                                            stage_base=self.stage_base[k], stage_capacity=self.stage_caps[k],
                                            grid_base=self.synth.grid_base[k], layer_base=k * self.nb))
            self.patches_dev = structs_to_device(structs, dev)
            f64 = lambda n: torch.zeros(max(1, n), dtype=torch.float64, device=dev)  # noqa: E731
            f32 = lambda n: torch.zeros(max(1, n), dtype=torch.float32, device=dev)  # noqa: E731
            self.pools = [[f64(total_pool), f64(total_pool), f64(total_pool), f64(total_pool), f32(total_pool)]
                          for _ in range(2)]
            self.counts = [torch.zeros(self.n_patches * self.nb, dtype=torch.int32, device=dev) for _ in range(2)]
            self.stage = [f64(total_stage), f64(total_stage), f64(total_stage), f64(total_stage), f32(total_stage)]
            self.stage_count = torch.zeros(self.n_patches * self.nb, dtype=torch.int32, device=dev)
            self.scratch = f64(2 * self.member_cap * self.n_patches)
            self.acc = torch.zeros(self.n_patches * self.nb * 4, dtype=torch.float64, device=dev)
            self.groups = torch.zeros(self.n_patches * self.nb, dtype=torch.int64, device=dev)
            self.e_in = torch.zeros(self.n_patches * self.nb, dtype=torch.float64, device=dev)
            self.e_out = torch.zeros(self.n_patches * self.nb, dtype=torch.float64, device=dev)
            keys = rng_seed_keys if rng_seed_keys is not None else [(cfg.seed, k) for k in range(self.n_patches)]
            self.rng = torch.cat([PhiloxStream(keys[k], dev).state for k in range(self.n_patches)])
            n_grid = int(self.synth.grid_base[-1])
            self.patch_h = f32(n_grid)
            self.patch_n = f32(3 * n_grid)
            self.blend_h = f32(n_grid)
            self.blend_n = f32(3 * n_grid)
            # per-frame accumulators in one block of 4-byte words, zeroed by hs_inject
            P = self.n_patches
            self.stat_words = torch.zeros(5 * P + (P & 1), dtype=torch.int32, device=dev)
            self.isum = self.stat_words[0:2 * P].view(torch.float64)
            self.icount = self.stat_words[2 * P:4 * P].view(torch.int64)
            self.clamped = self.stat_words[4 * P:5 * P]
            self.max_tiles = int(sum(-(-(pc + sc) // ADV_TILE) for pc, sc in zip(self.pool_caps, self.stage_caps)))
            self.tile_state = torch.zeros(self.max_tiles, dtype=torch.int64, device=dev)
            self.keep_words = torch.zeros(self.max_tiles * 32, dtype=torch.int32, device=dev)
            self.tile_counter = torch.zeros(1, dtype=torch.int32, device=dev)
            self._init_boxes()
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)

    # ------------------------------------------------------------ helpers --
    def _hr(self, dt: float) -> torch.Tensor:
        if dt not in self._hr_cache:
            hr = np.concatenate([half_rates(r, self.table.omegas, dt, self.config.g).ravel() for r in self.regions])
            self._hr_cache[dt] = torch.from_numpy(hr).to(self.device)
        return self._hr_cache[dt]

    def _init_boxes(self) -> None:
        cfg = self.config
        if self.fft_state is None:
            self.box_prefix_np = np.zeros(self.n_patches + 1, np.int32)
            return
        n, spacing = cfg.fft_n, cfg.fft_domain / cfg.fft_n
        boxes, pre = [], [0]
        for r in self.regions:       # harness.py:230-233
            lo = np.clip(np.floor(r.min_corner / spacing).astype(int), 0, n)
            hi = np.clip(np.ceil(r.max_corner / spacing).astype(int) + 1, 0, n)
            boxes += [lo[0], hi[0], lo[1], hi[1]]
            pre.append(pre[-1] + max(0, hi[0] - lo[0]) * max(0, hi[1] - lo[1]))
        self.box_np = np.array(boxes, np.int32)
        self.box_prefix_np = np.array(pre, np.int32)
        self.box_dev = torch.from_numpy(self.box_np).to(self.device)
        self.box_prefix_dev = torch.from_numpy(self.box_prefix_np).to(self.device)
        self.composite_out = torch.zeros((n, n), dtype=torch.float32, device=self.device)

    def _pool(self, k: int) -> N.HsPool:
        return N.pool_struct(*self.pools[k])

    # --------------------------------------------------------- the frame --
    def _enqueue_frame(self, parity: int, dt: float, mark=None) -> None:
        """Enqueue one frame (graph-capturable).  The background transform
        only feeds the blend, so it runs on a side stream concurrently with
        the particle chain inject -> advect -> smooth; the streams join before
        hs_compose.  `mark(stage)` (optional) is called after each stage's
        launches on the stream that ran it (CUDA events for stage timing)."""
        mark = mark or (lambda _name: None)
        main = torch.cuda.current_stream(self.device)
        fork = self.fft_state is not None and self.n_patches > 0
        if self.fft_state is not None:
            side = self._side_stream() if fork else main
            if fork:
                side.wait_stream(main)
            with torch.cuda.stream(side):
                mark("fft_start")
                fa = fft_args(self.fft_state, self.fft_ws, frame_ptr=self.frame_dev, dt=dt)
                fa.emit_normals = 0          # normals are derived lazily (background) / in hs_compose
                fa.normal = 0
                if not self.n_patches:
                    fa.frame_advance = N.ptr(self.frame_dev)
                N.call("hs_fft_evolve", fa, stream_ptr())
                mark("fft")
        st = stream_ptr()
        if self.n_patches:
            mark("particles_start")
            src, dst = parity, parity ^ 1
            N.call("hs_inject", N.HsInjectArgs(
                n_patches=self.n_patches, nb=self.nb, n_theta=self.table.n_theta, buckets=N.ptr(self.buckets_dev),
                patches=N.ptr(self.patches_dev), half_rate=N.ptr(self._hr(dt)),
                mean_dir=float(self.config.mean_direction), beta=float(self.config.trough_fraction),
                rho=float(self.config.rho), g=float(self.config.g), acc=N.ptr(self.acc), groups=N.ptr(self.groups),
                e_in=N.ptr(self.e_in), rng=N.ptr(self.rng), stage=N.pool_struct(*self.stage),
                stage_count=N.ptr(self.stage_count), scratch=N.ptr(self.scratch), member_capacity=self.member_cap,
                status=N.ptr(self.status), zero_words=N.ptr(self.stat_words),
                n_zero_words=self.stat_words.numel()), st)
            mark("inject")
            N.call("hs_advect", N.HsAdvectArgs(
                n_patches=self.n_patches, nb=self.nb, buckets=N.ptr(self.buckets_dev), patches=N.ptr(self.patches_dev),
                dt=float(dt), rho=float(self.config.rho), g=float(self.config.g), in_=self._pool(src),
                in_count=N.ptr(self.counts[src]), stage=N.pool_struct(*self.stage), stage_count=N.ptr(self.stage_count),
                out=self._pool(dst), out_count=N.ptr(self.counts[dst]), dropped=N.pool_struct(), dropped_count=0,
                e_out=N.ptr(self.e_out), splat=1, raw_layers=N.ptr(self.synth.raw),
                raw_layers_len=self.synth.pack.raw_len, layers=N.ptr(self.synth.layers),
                clamped=N.ptr(self.clamped), tile_state=N.ptr(self.tile_state), max_tiles=self.max_tiles,
                tile_counter=N.ptr(self.tile_counter), status=N.ptr(self.status),
                keep_words=N.ptr(self.keep_words)), st)
            mark("advect")
            N.call("hs_smooth", self.synth.smooth_args(), st)
            mark("smooth")
            if fork:
                main.wait_stream(self._side_stream())
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
                blend_height=N.ptr(self.blend_h), blend_normal=N.ptr(self.blend_n), blend_mode=1,
                interior_sumsq=N.ptr(self.isum), interior_count=N.ptr(self.icount),
                frame_advance=N.ptr(self.frame_dev)), st)
            mark("compose")
            self._patch_n_frame = -1          # patch normals are derived lazily (patch_field)
        self._bg_n_frame = -1                 # so are the background normals (background)
        if self.fft_state is None and not self.n_patches:
            N.call_raw("hs_advance_frame", N.vp(N.ptr(self.frame_dev)), N.vp(st))

    def _side_stream(self):
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=self.device)
        return self._side

    def _graph(self, parity: int):
        g = self._graphs.get(parity)
        if g is None:
            if self.n_patches:
                self._hr(self.config.dt)        # host->device uploads must precede capture
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream(device=self.device)
            s.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.graph(g, stream=s):
                self._enqueue_frame(parity, self.config.dt)
            torch.cuda.current_stream(self.device).wait_stream(s)
            self._graphs[parity] = g
        return g

    def kernel_launches_per_frame(self) -> int:
        """Library kernels one frame launches (csrc/*.cu): fft rows + cols
        (+ periodic normals), inject, advect, smooth (1 or 3), compose,
        advance_frame."""
        k = 0
        if self.fft_state is not None:
            k += 2                            # rows + columns (normals are lazy)
        if self.n_patches:
            pk = self.synth.pack
            # inject, advect count + scatter, compose, smooth (fused + 2 wide passes)
            k += 4 + (1 if pk.smooth_tile_info.shape[0] > 0 else 0) + (2 if pk.xtile_prefix[-1] > 0 else 0)
        return max(k, 1)

    def timed_frame(self) -> dict:
        """Replay one frame from a CUDA graph that carries timing-event record
        nodes after every stage; returns {stage: ms} (synchronises).  Each
        stage is timed against the previous event on its own stream, so the
        concurrently running background transform and particle chain are
        both per-kernel device times without host launch gaps.  Used by
        bench.py for the per-kernel roofline."""
        key = ("timed", self._parity)
        if key not in self._graphs:
            if self.n_patches:
                self._hr(self.config.dt)
            evs = []

            def mark(name):
                e = torch.cuda.Event(enable_timing=True, external=True)
                strm = torch.cuda.current_stream(self.device)
                e.record(strm)
                evs.append((name, e, strm.cuda_stream))
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream(device=self.device)
            s.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.graph(g, stream=s):
                self._enqueue_frame(self._parity, self.config.dt, mark)
            torch.cuda.current_stream(self.device).wait_stream(s)
            self._graphs[key] = (g, evs)
        g, evs = self._graphs[key]
        g.replay()
        self._parity ^= 1
        self.frame += 1
        torch.cuda.synchronize(self.device)
        out, last = {}, {}
        for name, e, sid in evs:
            if sid in last and not name.endswith("_start") and name != "join":
                out[name] = out.get(name, 0.0) + last[sid].elapsed_time(e)
            last[sid] = e
        if "fft_start" in [n for n, _, _ in evs] and "compose" in out:
            first = next(e for n, e, _ in evs if n in ("fft_start", "particles_start"))
            end = next(e for n, e, _ in evs if n == "compose")
            out["frame"] = first.elapsed_time(end)
        return out

    def step(self, dt: float | None = None, *, stats: bool = True):
        """Advance one frame.  With the configured dt and `config.graph` the
        frame is a single CUDA graph replay (the first frame runs eagerly to
        load modules).  Returns lazy FrameStats (or None if stats=False)."""
        cfg = self.config
        use_dt = cfg.dt if dt is None else float(dt)
        self.t = self.frame * use_dt
        if cfg.graph and use_dt == cfg.dt and self.frame > 0:
            self._graph(self._parity).replay()
        else:
            self._enqueue_frame(self._parity, use_dt)
        self._parity ^= 1
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
        snap = {"fsum": self.fft_ws.sumsq.clone() if self.fft_ws is not None else torch.zeros(1, dtype=torch.float64)}
        if self.n_patches:
            snap.update(counts=self.counts[self._parity].clone(), e_in=self.e_in.clone(), e_out=self.e_out.clone(),
                        isum=self.isum.clone(), icount=self.icount.clone())
        return FrameStats(frame=self.frame, t=self.t, stage_ms={s: 0.0 for s in STAGES}, _snap=snap, _nb=self.nb,
                          _n_patches=self.n_patches, _fft_n=self.config.fft_n if self.fft_ws is not None else 0)

    def check(self) -> None:
        """Raise if a device capacity flag was set (synchronises)."""
        s = int(self.status.item())
        if s & N.HS_STATUS_POOL_OVERFLOW:
            raise CapacityError(f"particle pool overflow (capacity {self.pool_caps}); raise device.pool_capacity")
        if s & N.HS_STATUS_STAGE_OVERFLOW:
            raise CapacityError("injection staging overflow")

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

    def counts_host(self) -> np.ndarray:
        """(n_patches, nb) live particles per bucket (synchronises)."""
        return self.counts[self._parity].cpu().numpy().reshape(self.n_patches, self.nb).astype(np.int64)

    def live_particles(self) -> int:
        return int(self.counts[self._parity].sum().item()) if self.n_patches else 0

    def pool(self, k: int) -> ParticleSet:
        """Patch k's current pool as a ParticleSet (views into device memory)."""
        c = self.counts_host()[k]
        lo, n = int(self.pool_base[k]), int(c.sum())
        x, y, ux, uy, amp = self.pools[self._parity]
        return ParticleSet.from_segments(x[lo:lo + n], y[lo:lo + n], ux[lo:lo + n], uy[lo:lo + n],
                                         amp[lo:lo + n], c, self.device)

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
        r = self.regions[k]
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
        surfaces = [PatchSurface(r, self.patch_field(k)) for k, r in enumerate(self.regions)]
        return SurfaceSampler(self.background, surfaces, self.config.normal_mode)

    def stitched_heights(self) -> torch.Tensor:
        """FFT-resolution composite with patch boxes resampled (harness.py:219-241)."""
        cfg = self.config
        n = cfg.fft_n
        if self.fft_state is None:
            raise ConfigError("stitched_heights needs the FFT background (mode != wp-only)")
        bg = self.fft_ws
        args = N.HsCompositeArgs(
            n=n, spacing=cfg.fft_domain / n, bg_height=N.ptr(bg.height), bg_normal=0,
            n_patches=self.n_patches, patches=N.ptr(self.patches_dev) if self.n_patches else 0,
            patch_height=N.ptr(self.patch_h) if self.n_patches else 0, patch_normal=0,
            box=N.ptr(self.box_dev) if self.n_patches else 0,
            box_prefix=N.ptr(self.box_prefix_dev) if self.n_patches else 0,
            total_box=int(self.box_prefix_np[-1]), out=N.ptr(self.composite_out if self.n_patches else None))
        if not self.n_patches:
            out = torch.empty((n, n), dtype=torch.float32, device=self.device)
            args.out = N.ptr(out)
            N.call("hs_composite", args, stream_ptr())
            return out
        N.call("hs_composite", args, stream_ptr())
        return self.composite_out

    def ledger_host(self) -> dict:
        P, nb = self.n_patches, self.nb
        return {"acc": self.acc.cpu().numpy().reshape(P, nb, 4), "groups": self.groups.cpu().numpy().reshape(P, nb),
                "e_in": self.e_in.cpu().numpy().reshape(P, nb), "e_out": self.e_out.cpu().numpy().reshape(P, nb)}


def benchmark_cell(cfg: SimConfig, warmup: int | None = None, measure: int | None = None, label: str = ""):
    """Steady-state throughput of one cell (harness.py:345-369), device-timed."""
    warmup = cfg.bench_warmup if warmup is None else warmup
    measure = cfg.bench_measure if measure is None else measure
    sim = Simulation(cfg)
    sim.run_frames(warmup)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    start.record()
    sim.run_frames(measure)
    end.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = start.elapsed_time(end) / max(measure, 1)
    live = sim.live_particles()
    return {"label": label or cfg.mode, "fps": 1e3 / ms if ms > 0 else float("inf"), "median_frame_ms": ms,
            "particles": live, "particle_rate": live * measure / wall if wall > 0 else 0.0}
