"""Generate golden vectors by running the REFERENCE package (hybridsea 0.1.0).

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes small .npz fixtures next to this file.  Every fixture is the output of
the reference's own public functions (`hybridsea.spectrum`, `.fft_background`,
`.particles`, `.patch_synthesis`, `.coupling`, `.harness`) on seeded inputs;
the oracle (`oracle/`) and the CUDA path are both checked against them.
Random streams use numpy's Philox (key=[seed, patch]) through the reference's
`rng` parameter (`particles.py:220`).
"""
from __future__ import annotations

import math
import os
import sys
from dataclasses import replace
from types import SimpleNamespace

import numpy as np

import hybridsea
from hybridsea import coupling, fft_background, particles, patch_synthesis, spectrum
from hybridsea.config import BodyConfig, PatchConfig, SimConfig
from hybridsea.harness import Simulation

HERE = os.path.dirname(os.path.abspath(__file__))
G = 9.81


def save(name: str, **arrays) -> None:
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name}: {os.path.getsize(path) / 1024:.1f} KiB")


def table_arrays(t: spectrum.BucketTable, prefix: str) -> dict:
    s, c = t.spread_params
    return {f"{prefix}_omega": t.omegas, f"{prefix}_width": t.widths, f"{prefix}_radius": t.radii,
            f"{prefix}_speed": t.speeds, f"{prefix}_energy": t.energies, f"{prefix}_s": s,
            f"{prefix}_c": c, f"{prefix}_lo": np.array([b.omega_lo for b in t.buckets]),
            f"{prefix}_hi": np.array([b.omega_hi for b in t.buckets])}


def log_table(params, lo, hi, n_omega, n_theta, spread_s=None) -> spectrum.BucketTable:
    """Log-spaced table expressed through the reference's public types."""
    edges = np.geomspace(lo, hi, n_omega + 1)
    reps = np.sqrt(edges[:-1] * edges[1:])
    bks = []
    for i, w in enumerate(reps):
        s = spread_s if spread_s is not None else spectrum.spreading_exponent(params, float(w))
        bks.append(spectrum.FrequencyBucket(
            index=i, omega=float(w), delta_omega=float(edges[i + 1] - edges[i]),
            omega_lo=float(edges[i]), omega_hi=float(edges[i + 1]),
            radius=math.pi * params.g / float(w) ** 2, speed=params.g / float(w),
            energy_density=spectrum.trapezoid_energy(params, float(edges[i]), float(edges[i + 1]), base=2048),
            spread_s=float(s), spread_norm=spectrum.spreading_norm(float(s))))
    return spectrum.BucketTable(buckets=tuple(bks), n_omega=n_omega, n_theta=n_theta,
                                total_energy=float(sum(b.energy_density for b in bks)))


def gen_spectrum() -> None:
    out = {}
    for tag, (u, f) in {"a": (5.0, 1e4), "b": (10.0, 1e5), "c": (15.0, 1e5)}.items():
        p = spectrum.derive_params(u, f, G)
        out[f"{tag}_params"] = np.array([p.alpha, p.omega_p, p.gamma])
        w = np.linspace(0.3, 6.0, 97)
        out[f"{tag}_s1d_w"] = w
        out[f"{tag}_s1d"] = spectrum.evaluate_1d(p, w)
        out[f"{tag}_band"] = np.array([spectrum.band_energy(p)])
        for n in (8, 12, 16):
            out.update(table_arrays(spectrum.build_buckets(p, n, 16), f"{tag}_eq{n}"))
    pb = replace(spectrum.derive_params(10.0, 1e5, G), gamma=3.3)
    out.update(table_arrays(log_table(pb, 0.5, 4.0, 8, 16, spread_s=8.0), "pr1_log8"))
    pc = spectrum.derive_params(10.0, 1e5, G)
    out.update(table_arrays(log_table(pc, 0.3, 6.0, 16, 2), "c3_log16"))
    s_vals = np.array([0.05, 0.5, 1.0, 4.0, 8.0, 16.0, 60.0])
    out["spread_s_vals"] = s_vals
    out["spread_norm_vals"] = np.array([spectrum.spreading_norm(float(s)) for s in s_vals])
    save("spectrum.npz", **out)


def gen_fft() -> None:
    out = {}
    sp = spectrum.DirectionalSpectrum(spectrum.derive_params(5.0, 1e4, G), 0.0)
    st = fft_background.init_fft(sp, 16, 500.0, seed=7, choppiness=1.0)
    out["n16_h0"] = st.h0
    for k, t in enumerate((0.0, 12.75)):
        f = fft_background.evolve_and_synthesize(st, t)
        out[f"n16_t{k}_h"], out[f"n16_t{k}_d"], out[f"n16_t{k}_n"] = f.height, f.displacement, f.normal
    out["n16_times"] = np.array([0.0, 12.75])

    sp2 = spectrum.DirectionalSpectrum(spectrum.derive_params(10.0, 1e5, G), 0.3)
    st2 = fft_background.init_fft(sp2, 64, 1000.0, seed=3, choppiness=1.2)
    out["n64_h0"] = st2.h0
    for k, t in enumerate((1.5, 123.4)):
        f = fft_background.evolve_and_synthesize(st2, t)
        out[f"n64_t{k}_h"], out[f"n64_t{k}_d"], out[f"n64_t{k}_n"] = f.height, f.displacement, f.normal
    out["n64_times"] = np.array([1.5, 123.4])
    pts = np.random.default_rng(1).uniform(-1200.0, 2200.0, size=(200, 2))
    hv, nv = fft_background.sample_periodic(f, pts)
    out["n64_sample_pts"], out["n64_sample_h"], out["n64_sample_n"] = pts, hv, nv
    save("fft.npz", **out)


def pool_arrays(pool: particles.ParticleSet, prefix: str) -> dict:
    return {f"{prefix}_pos": pool.positions.copy(), f"{prefix}_dir": pool.directions.copy(),
            f"{prefix}_amp": pool.amplitudes.copy(), f"{prefix}_bucket": pool.buckets.copy()}


def gen_particles() -> dict:
    """PR1-like inject+advect chain and a high-rate single injection."""
    out = {}
    pb = replace(spectrum.derive_params(10.0, 1e5, G), gamma=3.3)
    sp = spectrum.DirectionalSpectrum(pb, 0.0)
    tbl = log_table(pb, 0.5, 4.0, 8, 16, spread_s=8.0)
    patch = particles.PatchRegion((100.0, 200.0), 64.0, 64.0, 8.0)
    ledger = particles.InjectionLedger(8)
    rng = np.random.Generator(np.random.Philox(key=[0, 0]))
    pool = particles.ParticleSet(1 << 12)
    dt = 1.0 / 60.0
    counts, ninj = [], []
    for k in range(120):
        new = particles.inject(patch, tbl, sp, ledger, dt, rng, t=k * dt)
        ninj.append(len(new))
        if k == 30:
            out.update(pool_arrays(pool, "pre30"))
            out["pre30_acc"] = ledger.accumulators.copy()
            out.update(pool_arrays(new, "inj30"))
        pool.extend(new)
        particles.advect(pool, tbl, dt, patch, ledger, g=G)
        counts.append(pool.counts_per_bucket(8))
    out["chain_counts"] = np.array(counts)
    out["chain_ninj"] = np.array(ninj)
    out.update(pool_arrays(pool, "chain_final"))
    out["chain_acc"] = ledger.accumulators
    out["chain_groups"] = ledger.injected_groups
    out["chain_e_in"] = ledger.injected_energy
    out["chain_e_out"] = ledger.despawned_energy
    # one more advect of the final pool: moved positions + keep mask
    moved = particles.ParticleSet(len(pool) + 1)
    moved.extend(pool)
    led2 = particles.InjectionLedger(8)
    dropped = particles.advect(moved, tbl, dt * 7.0, patch, led2, g=G)
    out.update(pool_arrays(moved, "adv7_kept"))
    out.update(pool_arrays(dropped, "adv7_dropped"))
    out["adv7_e_out"] = led2.despawned_energy

    # high-rate single injection from a fresh ledger (C3-like table, n_theta 2)
    pc = spectrum.derive_params(10.0, 1e5, G)
    spc = spectrum.DirectionalSpectrum(pc, 0.7)
    t3 = log_table(pc, 0.3, 6.0, 16, 2)
    patch3 = particles.PatchRegion((-50.0, 30.0), 256.0, 192.0, 10.0)
    led3 = particles.InjectionLedger(16)
    rng3 = np.random.Generator(np.random.Philox(key=[5, 1]))
    for k in range(3):
        new3 = particles.inject(patch3, t3, spc, led3, 0.1, rng3, t=k * 0.1, trough_fraction=0.8)
    out.update(pool_arrays(new3, "hr_inj"))
    out["hr_acc"] = led3.accumulators
    out["hr_groups"] = led3.injected_groups
    out["hr_e_in"] = led3.injected_energy
    save("particles.npz", **out)
    return {"pool": pool, "patch": patch, "table": tbl}


def gen_synth(ctx: dict) -> None:
    out = {}
    pool, patch, tbl = ctx["pool"], ctx["patch"], ctx["table"]
    res = 129
    texel = patch.l1 / (res - 1)
    plan = patch_synthesis.plan_layers(tbl, texel, res)
    out["plan_factors"] = np.array(plan.factors)
    out["plan_half"] = np.array([k.half_width for k in plan.kernels])
    out["plan_gain"] = np.array([k.gain for k in plan.kernels])
    h_plan, c_plan = patch_synthesis.synthesize(pool, patch, res, plan)
    kern = patch_synthesis.build_kernels(tbl, texel)
    h_exact, c_exact = patch_synthesis.synthesize(pool, patch, res, kern)
    out["h_plan"], out["clamped_plan"] = h_plan, np.array([c_plan])
    out["h_exact"], out["clamped_exact"] = h_exact, np.array([c_exact])
    kpeak = patch_synthesis.build_kernels(tbl, texel, convention="peak")
    out["gain_peak"] = np.array([k.gain for k in kpeak])
    f = patch_synthesis.finish_field(h_plan, patch)
    out["finish_n"] = f.normal
    fch = patch_synthesis.finish_field(h_plan, patch, choppiness=0.7, displacement_scale=2.0)
    out["finish_chop_d"] = fch.displacement
    # blend against a 64^2 / 1000 m background (mean direction 0.3, chop 1.2)
    sp2 = spectrum.DirectionalSpectrum(spectrum.derive_params(10.0, 1e5, G), 0.3)
    st2 = fft_background.init_fft(sp2, 64, 1000.0, seed=3, choppiness=1.2)
    bg = fft_background.evolve_and_synthesize(st2, 1.5)
    surf = coupling.PatchSurface(patch, f)
    sampler = coupling.SurfaceSampler(bg, [surf])
    xs = patch.min_corner[0] + np.arange(res) * texel
    ys = patch.min_corner[1] + np.arange(res) * texel
    nodes = np.stack(np.meshgrid(xs, ys, indexing="ij"), axis=-1)
    hb, nb = sampler.sample(nodes.reshape(-1, 2))
    out["blend_h"], out["blend_n"] = hb.reshape(res, res), nb.reshape(res, res, 3)
    pts = np.random.default_rng(2).uniform(60.0, 300.0, size=(300, 2))
    hs, ns = sampler.sample(pts)
    out["sample_pts"], out["sample_h"], out["sample_n"] = pts, hs, ns
    fake = SimpleNamespace(config=SimpleNamespace(fft_n=64, fft_domain=1000.0), background=bg,
                           patches=[SimpleNamespace(surface=surf, region=patch)], sampler=sampler)
    out["stitched"] = Simulation.stitched_heights(fake)
    save("synth.npz", **out)


def gen_sim() -> None:
    """Whole reference Simulation.step chain with a Philox stream."""
    cfg = SimConfig(fft_n=64, fft_domain=500.0, dt=0.05, frames=6, n_omega=8, n_theta=8,
                    seed=11, patches=(PatchConfig(origin=(200.0, 180.0), size=(100.0, 80.0),
                                                  res=65, margin=10.0),), write_frames=False)
    sim = Simulation(cfg)
    sim.rng = np.random.Generator(np.random.Philox(key=[cfg.seed, 0]))
    stats = [sim.step() for _ in range(cfg.frames)]
    out = {
        "counts": np.array([s.particle_counts for s in stats]),
        "e_in": np.array([s.injected_energy for s in stats]),
        "e_out": np.array([s.despawned_energy for s in stats]),
        "patch_var": np.array([s.patch_variance for s in stats]),
        "fft_var": np.array([s.fft_band_variance for s in stats]),
        "stitched": sim.stitched_heights(),
        "bg_h": sim.background.height,
        "patch_h": sim.patches[0].surface.field.height,
    }
    out.update(pool_arrays(sim.patches[0].pool, "pool"))
    save("sim.npz", **out)


def gen_emit() -> None:
    """Emission (interaction.py:175-231) and a Simulation with kinematic
    bodies + a tracking patch (harness.py:115-123,155-167).  Kinematic bodies:
    `buoyancy_step` is replaced by position += velocity * dt (its own update,
    interaction.py:140) with a fixed displaced-volume change and submersion
    per frame, the SURVEY 8(f) form of the BASELINE wake sources."""
    from hybridsea import harness as H
    from hybridsea import interaction as I
    out = {}
    pb = replace(spectrum.derive_params(15.0, 1e5, G), gamma=3.3)
    patch = particles.PatchRegion((100.0, 200.0), 128.0, 128.0, 10.0)
    cases = [  # (count, velocity, d_v, h_c, hull size, trough fraction)
        (3, (2.0, 0.0, 0.0), 0.02, 0.5, (2.0, 2.0, 1.0), 1.0),
        (8, (1.2, 0.8, 0.0), 0.01, 0.4, (6.0, 3.0, 1.0), 1.0),
        (256, (-5.0, 3.0, 0.0), 0.05, 0.5, (12.0, 4.0, 2.0), 1.0),
        (16, (1.0, 0.0, 1.0), 0.02, 0.5, (2.0, 2.0, 1.0), 0.5),     # ring + wake split
        (8, (0.0, 0.0, 0.7), -0.02, 0.5, (3.0, 3.0, 1.0), 1.0),     # suction ring only
        (4, (0.0, 0.0, 0.0), 0.03, 0.2, (2.0, 2.0, 1.0), 1.0),      # static: ring
    ]
    for k, (count, vel, dv, hc, size, beta) in enumerate(cases):
        tbl = log_table(pb, 0.4, 3.0, 12, 2 * count)
        body = I.box_body([150.0, 260.0, 0.0], size)
        body.velocity = np.array(vel)
        body.prev_submerged_volume = 0.0          # d_v = submerged - prev == dv exactly
        body.submerged_volume = dv
        body.mean_submersion = hc
        events, ps = I.emit_from_motion(body, patch, tbl, 1 / 60, 1000.0, G, trough_fraction=beta)
        out[f"c{k}_params"] = np.array([count, *vel, dv, hc, body.hull_extent, beta, *size])
        out[f"c{k}_events"] = np.array([[0 if e.mode == "ring" else 1, e.energy, e.bucket] for e in events]).reshape(-1, 3)
        out.update(pool_arrays(ps, f"c{k}"))
        out[f"c{k}_radii"] = tbl.radii
    save("emit.npz", **out)

    # whole Simulation: body 0 (surge) is tracked by the patch, body 1 heaves + drifts
    cfg = SimConfig(fft_n=64, fft_domain=500.0, dt=0.05, frames=10, n_omega=8, n_theta=8, seed=21,
                    patches=(PatchConfig(origin=(200.0, 180.0), size=(100.0, 80.0), res=65, margin=10.0,
                                         track_body=0),),
                    bodies=(BodyConfig(position=(250.0, 220.0, 0.0), size=(4.0, 2.0, 1.0)),
                            BodyConfig(position=(230.0, 200.0, 0.0), size=(2.0, 2.0, 1.0))),
                    write_frames=False)
    kin = {0: ((3.0, 1.0, 0.0), 0.02, 0.5), 1: ((1.0, -0.5, 0.8), -0.01, 0.3)}

    def kinematic_step(body, query_surface, dt, rho=1000.0, g=9.81):
        vel, dv, hc = kin[body.body_id]
        body.velocity = np.array(vel)
        body.position += body.velocity * dt
        body.prev_submerged_volume = 0.0         # a fixed d_v per frame (exactly dv)
        body.submerged_volume = dv
        body.mean_submersion = hc
        return body

    orig = H.buoyancy_step
    H.buoyancy_step = kinematic_step
    try:
        sim = Simulation(cfg)
        sim.rng = np.random.Generator(np.random.Philox(key=[cfg.seed, 0]))
        stats, origins = [], []
        for _ in range(cfg.frames):
            stats.append(sim.step())
            origins.append(sim.patches[0].region.min_corner.copy())
    finally:
        H.buoyancy_step = orig
    sout = {
        "counts": np.array([st.particle_counts for st in stats]),
        "e_in": np.array([st.injected_energy for st in stats]),
        "e_out": np.array([st.despawned_energy for st in stats]),
        "origins": np.array(origins),
        "body_pos": np.array([b.position for b in sim.bodies]),
        "hulls": np.array([b.hull_extent for b in sim.bodies]),
        "patch_h": sim.patches[0].surface.field.height,
        "stitched": sim.stitched_heights(),
    }
    sout.update(pool_arrays(sim.patches[0].pool, "pool"))
    save("emit_sim.npz", **sout)


def gen_bodies() -> None:
    """A reference Simulation with two floating bodies (buoyancy against the
    previous frame's blended surface, interaction.py:105-149, and emission,
    :175-231) and a patch tracking body 0 (harness.py:115-123)."""
    cfg = SimConfig(u10=8.0, fetch=5e4, fft_n=64, fft_domain=400.0, dt=0.05, frames=16, n_omega=8, n_theta=8,
                    seed=31, patches=(PatchConfig(origin=(150.0, 150.0), size=(80.0, 80.0), res=81, margin=8.0,
                                                  track_body=0),),
                    bodies=(BodyConfig(position=(190.0, 188.0, 0.4), size=(4.0, 2.0, 1.0), density=450.0,
                                       yaw=0.3),
                            BodyConfig(position=(175.0, 200.0, -0.2), size=(2.0, 2.0, 1.0), density=600.0)),
                    write_frames=False)
    sim = Simulation(cfg)
    sim.rng = np.random.Generator(np.random.Philox(key=[cfg.seed, 0]))
    stats, origins, bstate = [], [], []
    for _ in range(cfg.frames):
        stats.append(sim.step())
        origins.append(sim.patches[0].region.min_corner.copy())
        bstate.append([np.concatenate([b.position, [b.yaw], b.velocity, [b.yaw_rate, b.submerged_volume,
                                                                       b.prev_submerged_volume, b.mean_submersion]])
                       for b in sim.bodies])
    out = {
        "counts": np.array([s.particle_counts for s in stats]),
        "e_in": np.array([s.injected_energy for s in stats]),
        "e_out": np.array([s.despawned_energy for s in stats]),
        "origins": np.array(origins),
        "bodies": np.array(bstate),
        "patch_h": sim.patches[0].surface.field.height,
    }
    out.update(pool_arrays(sim.patches[0].pool, "pool"))
    save("bodies_sim.npz", **out)


def main() -> int:
    print("reference hybridsea", hybridsea.__version__, "numpy", np.__version__)
    gen_spectrum()
    gen_fft()
    ctx = gen_particles()
    gen_synth(ctx)
    gen_sim()
    gen_emit()
    gen_bodies()
    return 0


if __name__ == "__main__":
    sys.exit(main())
