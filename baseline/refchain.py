"""The UNMODIFIED reference package as the CPU baseline -- BENCH
INFRASTRUCTURE ONLY (bench.py's reference arm and `cpu_baseline` leg; never
imported by the product).

`baseline/_ref` holds `hybridsea` 0.1.0 pip-installed from /root/reference
(`python -m pip install --no-index --no-build-isolation --no-deps --target
baseline/_ref <copy of /root/reference/pkg>`; git-ignored, travels to the GPU
box with the snapshot).  This module drives the reference's own
`harness.Simulation.step` + `Simulation.stitched_heights`
(`pkg/src/hybridsea/harness.py:131-241`) -- the stock code path, numpy on one
host core -- on a BASELINE scene expressed through the reference's public
types:

  * log-spaced buckets (PR1, C3): a `BucketTable` of reference
    `FrequencyBucket`s with the scene's fields, set on the Simulation after
    construction, and the patch `LayerPlan`s rebuilt from it with the
    reference's `plan_layers` (the reference tests build tables the same way,
    `test_particles.py:53-60`);
  * per-patch Philox streams: `sim.rng` is the scene's
    `Generator(Philox(key=[seed, 0]))` (single-patch scenes only: the
    reference shares one generator across patches, harness.py:79).

Scenes the reference cannot express (FFT cascades, kinematic wake sources,
gamma / spreading overrides, several patches with independent streams) are
reported as unavailable here; bench.py then times the oracle port instead
(`kind: "port"`).
"""
from __future__ import annotations

import os
import sys
from dataclasses import asdict

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")


def load():
    """The installed reference package, or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "hybridsea")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import hybridsea
    return hybridsea


def expressible(cfg) -> str | None:
    """None if `cfg` runs through the reference Simulation, else why not."""
    if cfg.fft_cascades:
        return "FFT cascades are a reference non-goal (SPEC.md:166)"
    if cfg.sources or cfg.bodies:
        return "kinematic wake sources have no reference config"
    if cfg.gamma is not None or cfg.spread_s is not None:
        return "gamma / spreading overrides have no reference config"
    if len(cfg.patches) != 1:
        return "several patches share one generator in the reference (harness.py:79)"
    if cfg.fft_band_lo is not None or cfg.fft_band_hi is not None:
        return "FFT band overrides have no reference config"
    return None


def build(cfg, ref=None):
    """A reference `Simulation` for scene `cfg` (see module docstring)."""
    ref = ref or load()
    if ref is None:
        raise RuntimeError("reference package not installed in baseline/_ref")
    why = expressible(cfg)
    if why:
        raise ValueError(why)
    from hybridsea import config as rconfig
    from hybridsea import harness as rharness
    from hybridsea import patch_synthesis as rsynth
    from hybridsea import spectrum as rspectrum
    pc = cfg.patches[0]
    rc = rconfig.SimConfig(
        u10=cfg.u10, fetch=cfg.fetch, g=cfg.g, mean_direction=cfg.mean_direction, n_omega=cfg.n_omega,
        n_theta=cfg.n_theta, rho=cfg.rho, dt=cfg.dt, frames=cfg.frames, mode=cfg.mode, seed=cfg.seed,
        trough_fraction=cfg.trough_fraction, amplitude_convention=cfg.amplitude_convention,
        normal_mode=cfg.normal_mode, fft_n=cfg.fft_n, fft_domain=cfg.fft_domain,
        fft_choppiness=cfg.fft_choppiness,
        patches=(rconfig.PatchConfig(origin=tuple(pc.origin), size=tuple(pc.size), res=pc.res, margin=pc.margin),),
        write_frames=False)
    sim = rharness.Simulation(rc)
    if cfg.bucket_spacing == "log":
        from paper_2511_02852_b200.spectrum import derive_params, log_buckets
        ours = log_buckets(derive_params(cfg.u10, cfg.fetch, cfg.g), cfg.omega_lo, cfg.omega_hi, cfg.n_omega,
                           cfg.n_theta)
        fields = set(rspectrum.FrequencyBucket.__dataclass_fields__)
        buckets = tuple(rspectrum.FrequencyBucket(**{k: v for k, v in asdict(b).items() if k in fields})
                        for b in ours.buckets)
        sim.table = rspectrum.BucketTable(buckets=buckets, n_omega=ours.n_omega, n_theta=ours.n_theta,
                                          total_energy=ours.total_energy)
        for ps in sim.patches:
            ps.plan = rsynth.plan_layers(sim.table, ps.texel, ps.resolution, convention=rc.amplitude_convention,
                                         trough_fraction=rc.trough_fraction)
    sim.rng = np.random.Generator(np.random.Philox(key=[cfg.seed, 0]))
    return sim


def warm(sim, frames: int, dt: float, budget_s: float | None = None) -> int:
    """Steady state with the reference's own inject + advect (the pool's
    population dynamics; synthesis does not feed back), as SURVEY App. C
    warmed its C3 pools.  Stops early after `budget_s` seconds; returns the
    frames run."""
    import time
    from hybridsea.particles import advect, inject
    cfg = sim.config
    t0 = time.perf_counter()
    for k in range(frames):
        if budget_s is not None and time.perf_counter() - t0 > budget_s:
            return k
        t = sim.frame * dt
        for ps in sim.patches:
            ps.pool.extend(inject(ps.region, sim.table, sim.spectrum, ps.ledger, dt, sim.rng, t=t,
                                  trough_fraction=cfg.trough_fraction))
        for ps in sim.patches:
            advect(ps.pool, sim.table, dt, ps.region, ps.ledger, g=cfg.g)
        sim.frame += 1
    return frames


def load_state(sim, pools, ledgers, rng_words, frame: int) -> None:
    """Put a cloned state (GPU steady state: per-patch (pos, dir, amp, bucket)
    in per-bucket reference order, ledgers, Philox stream words) into the
    reference Simulation, so its frames time the same workload."""
    from hybridsea.particles import ParticleSet
    from oracle.clone import philox_generator
    for ps, (pos, d, a, b), led in zip(sim.patches, pools, ledgers):
        pool = ParticleSet(max(1024, len(a)))
        pool.append_arrays(pos, d, a, b, np.zeros(len(a)))
        ps.pool = pool
        ps.ledger.accumulators[...] = led["acc"]
        ps.ledger.injected_groups[...] = led["groups"]
        ps.ledger.injected_energy[...] = led["e_in"]
        ps.ledger.despawned_energy[...] = led["e_out"]
    sim.rng = philox_generator(rng_words)
    sim.frame = frame


def frame(sim) -> None:
    """One reference frame of the north_star step: Simulation.step +
    stitched_heights (harness.py:131-241)."""
    sim.step()
    sim.stitched_heights()
