"""The per-frame hybrid step over a scene -- TEST INFRASTRUCTURE ONLY.

Follows `Simulation.__init__` / `Simulation.step` (reference
`pkg/src/hybridsea/harness.py:72-111,131-209`) stage order: t = frame*dt,
background synthesis, per-patch injection, per-patch advection, per-patch
synthesis + finish, blend (evaluated at patch nodes, the tile the stream and
buoyancy probes read), optional FFT-resolution composite (:219-241).

Differences from the reference harness, all SURVEY App. A knobs:
  * each patch owns a `Generator(Philox(key=[seed, patch_id]))` instead of a
    shared PCG64 (harness.py:79) -- the counter-based stream the GPU twins;
  * bucket tables may be log-spaced, gamma/spread may be pinned;
  * bodies are not part of the hot path.

A scene is a plain dict (see `paper_2511_02852_b200.config.SimConfig.scene_dict`).
"""
from __future__ import annotations

import math

import numpy as np

from . import blend_ref, body_ref, emit_ref, ocean_ref, particles_ref, spectrum_ref, synth_ref


def build_params(sc: dict) -> spectrum_ref.Params:
    return spectrum_ref.jonswap(sc["u10"], sc["fetch"], sc["g"], gamma=sc.get("gamma"),
                                spread_s=sc.get("spread_s"))


def build_buckets(sc: dict, p: spectrum_ref.Params) -> spectrum_ref.Buckets:
    if sc.get("bucket_spacing", "equal-energy") == "log":
        return spectrum_ref.log_buckets(p, sc["omega_lo"], sc["omega_hi"], sc["n_omega"], sc["n_theta"])
    return spectrum_ref.equal_energy_buckets(p, sc["n_omega"], sc["n_theta"])


def cascade_bands(cascades, n: int) -> list:
    """[(L, k_lo, k_hi)] largest tile first; boundaries at half the larger
    tile's Nyquist wavenumber pi n / (2 L) (the scene definition of C4,
    DESIGN.md; no reference semantics)."""
    tiles = sorted((float(c) for c in cascades), reverse=True)
    out, k_lo = [], 0.0
    for i, L in enumerate(tiles):
        k_hi = math.pi * n / (2.0 * L) if i + 1 < len(tiles) else math.inf
        out.append((L, k_lo, k_hi))
        k_lo = k_hi
    return out


class OracleScene:
    """CPU twin of one hybrid scene."""

    def __init__(self, sc: dict, h0: np.ndarray | None = None):
        self.sc = sc
        self.p = build_params(sc)
        self.bk = build_buckets(sc, self.p)
        self.frame = 0
        self.patches = [particles_ref.Patch(o[0], o[1], s[0], s[1], m)
                        for o, s, m in zip(sc["patch_origins"], sc["patch_sizes"], sc["patch_margins"])]
        self.res = list(sc["patch_res"])
        self.pools = [particles_ref.Pool() for _ in self.patches]
        self.ledgers = [particles_ref.Ledger(self.bk.n, rho=sc["rho"]) for _ in self.patches]
        # key = (seed, global patch id): a patch's stream is the same whichever
        # rank owns it (sharded runs pass their block's ids as "patch_ids")
        ids = sc.get("patch_ids") or list(range(len(self.patches)))
        self.rngs = [np.random.Generator(np.random.Philox(key=[sc["seed"], i])) for i in ids]
        self.plans = [synth_ref.plan(self.bk, pc.l1 / (r - 1), r, sc["amplitude_convention"],
                                     sc["trough_fraction"])
                      for pc, r in zip(self.patches, self.res)]
        self.fft = sc["mode"] != "wp-only"
        if self.fft:
            self.h0 = h0 if h0 is not None else ocean_ref.initial_amplitudes(
                self.p, sc["mean_direction"], sc["fft_n"], sc["fft_domain"], sc["seed"],
                band=sc.get("fft_band"))
        # summed FFT cascades: tile c of size L_c keeps its
        # disjoint |k| band and its own seed (seed + c)
        self.cascades = []
        if self.fft and sc.get("fft_cascades"):
            for c, (L, klo, khi) in enumerate(cascade_bands(sc["fft_cascades"], sc["fft_n"])):
                self.cascades.append((L, ocean_ref.initial_amplitudes(
                    self.p, sc["mean_direction"], sc["fft_n"], L, sc["seed"] + c, band=sc.get("fft_band"),
                    kband=(klo, khi))))
        self.background = None
        self.fields = []
        # kinematic emitting bodies + patch tracking (emit_ref; harness.py:115-123,155-167)
        self.sources = [emit_ref.Source(np.array(d["position"], dtype=float), np.array(d["velocity"], dtype=float),
                                        d["hull_extent"], d["volume_rate"], d["submersion"],
                                        d.get("wake_count", 0), d.get("energy_scale", 1.0))
                        for d in sc.get("sources", [])]
        self.track = list(sc.get("patch_track") or [-1] * len(self.patches))
        # floating bodies (interaction.py:79-149; harness.py:102-107,155-167): buoyancy
        # against the previous frame's blended surface, then emission; patches
        # with track_body follow them
        self.bodies = [body_ref.box_body(d["position"], d["size"], d.get("density", 500.0), d.get("yaw", 0.0),
                                         d.get("max_thrust", 0.0), d.get("max_yaw_torque", 0.0))
                       for d in sc.get("bodies", [])]
        self.track_body = list(sc.get("patch_track_body") or [-1] * len(self.patches))
        self.prev_surface = None          # (background, [(patch, field)]) of the last synthesised frame

    def step(self, dt: float | None = None, synth: bool = True, fft: bool = True) -> dict:
        sc = self.sc
        dt = sc["dt"] if dt is None else dt
        t = self.frame * dt
        out = {"t": t}
        if self.fft and fft and self.cascades:
            n = sc["fft_n"]
            self.background = []
            for L, h0c in self.cascades:
                h, dx, dy, nrm = ocean_ref.evolve(h0c, L, self.p.g, t, sc["fft_choppiness"])
                self.background.append(blend_ref.Field(h, nrm, np.zeros(2), L / n))
                out.setdefault("cascade_heights", []).append(h)
            out.update(height=self.background[0].height, normal=self.background[0].normal)
        elif self.fft and fft:
            h, dx, dy, nrm = ocean_ref.evolve(self.h0, sc["fft_domain"], self.p.g, t, sc["fft_choppiness"])
            n = sc["fft_n"]
            self.background = blend_ref.Field(h, nrm, np.zeros(2), sc["fft_domain"] / n)
            out.update(height=h, dx=dx, dy=dy, normal=nrm)
        for pc, pool, led, rng in zip(self.patches, self.pools, self.ledgers, self.rngs):
            pool.append(particles_ref.inject(pc, self.bk, self.p, sc["mean_direction"], led, dt, rng,
                                             t=t, beta=sc["trough_fraction"]))
        for pc, pool, led in zip(self.patches, self.pools, self.ledgers):
            particles_ref.advect(pool, self.bk, dt, pc, led, self.p.g)
        # interaction stage (harness.py:155-167): bodies first (buoyancy against the
        # previous frame's sampler -- flat water before the first synthesis -- then
        # emit_from_motion into the owning patch), then the kinematic sources
        for body in self.bodies:
            prev = self.prev_surface

            def query(pts, prev=prev):
                pts = np.asarray(pts, dtype=float)
                if prev is None:
                    n = np.zeros(pts.shape[:-1] + (3,))
                    n[..., 2] = 1.0
                    return np.zeros(pts.shape[:-1]), n
                return blend_ref.sample(prev[0], prev[1], pts)
            body_ref.buoyancy_step(body, query, dt, sc["rho"], self.p.g)
            owner = next((k for k, pc in enumerate(self.patches) if emit_ref.contains(pc, body.position[:2])), None)
            if owner is None:
                continue
            src = emit_ref.Source(body.position[:2].copy(), body.velocity.copy(), body.hull_extent,
                                  body.submerged_volume - body.prev_submerged_volume, body.mean_submersion)
            events, emitted = emit_ref.emit(src, self.bk.radius, self.bk.n_theta, sc["rho"], self.p.g,
                                            sc["trough_fraction"])
            self.pools[owner].append(emitted)
            for ev in events:
                self.ledgers[owner].e_in[ev.bucket] += ev.energy
        for src in self.sources:
            src.position = src.position + src.velocity[:2] * dt
            owner = next((k for k, pc in enumerate(self.patches) if emit_ref.contains(pc, src.position)), None)
            if owner is None:
                continue
            events, emitted = emit_ref.emit(src, self.bk.radius, self.bk.n_theta, sc["rho"], self.p.g,
                                            sc["trough_fraction"])
            self.pools[owner].append(emitted)
            for ev in events:
                self.ledgers[owner].e_in[ev.bucket] += ev.energy
        for k, j in enumerate(self.track):
            if 0 <= j < len(self.sources):
                self.patches[k] = emit_ref.retrack(self.patches[k], self.res[k], self.sources[j])
        for k, j in enumerate(self.track_body):
            if 0 <= j < len(self.bodies):
                self.patches[k] = emit_ref.retrack(self.patches[k], self.res[k], self.bodies[j])
        if synth:
            self.fields = []
            for pc, pool, r, pl in zip(self.patches, self.pools, self.res, self.plans):
                hp, clamped = synth_ref.synthesize(pool, pc, r, pl)
                nrm, _ = synth_ref.finish(hp, pc)
                self.fields.append(blend_ref.Field(hp, nrm, pc.lo.copy(), pc.l1 / (r - 1)))
            pairs = list(zip(self.patches, self.fields))
            out["patch_heights"] = [f.height for f in self.fields]
            out["patch_normals"] = [f.normal for f in self.fields]
            tiles = [blend_ref.sample(self.background, pairs, blend_ref.patch_nodes(pc, r))
                     for pc, r in zip(self.patches, self.res)]
            out["blend_heights"] = [tl[0] for tl in tiles]
            out["blend_normals"] = [tl[1] for tl in tiles]
            self.prev_surface = (self.background, pairs)
        out["bodies"] = [(b.position.copy(), b.yaw, b.velocity.copy(), b.submerged_volume) for b in self.bodies]
        out["counts"] = np.stack([pool.counts(self.bk.n) for pool in self.pools]) if self.pools else None
        self.frame += 1
        return out

    def composite(self) -> np.ndarray:
        sc = self.sc
        return blend_ref.stitched(self.background, sc["fft_n"], sc["fft_domain"],
                                  list(zip(self.patches, self.fields)))


def ledger_arrays(led: particles_ref.Ledger) -> dict:
    return {"acc": led.acc.copy(), "groups": led.groups.copy(), "e_in": led.e_in.copy(),
            "e_out": led.e_out.copy()}


__all__ = ["OracleScene", "build_params", "build_buckets", "ledger_arrays"]
