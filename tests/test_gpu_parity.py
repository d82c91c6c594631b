"""CUDA path vs the CPU oracle and the reference golden vectors (B200).

Tolerances (north_star): integer work -- group counts, buckets, compaction
order, keep decisions -- bit-exact; fp32 heights and displacements within
max-abs 1e-4*Hs and relative L2 1e-5 of the fp64 oracle.
"""
import math

import numpy as np
import pytest
import torch

from oracle import blend_ref, ocean_ref, particles_ref, scene_ref, spectrum_ref, synth_ref

pytestmark = pytest.mark.gpu
G = 9.81


def hs_of(h):
    return 4.0 * float(np.sqrt(np.mean(np.asarray(h) ** 2)))


def assert_field_close(got, ref, hs, rel_l2=1e-5, what=""):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.abs(got - ref).max()
    assert err <= 1e-4 * hs, f"{what}: max-abs {err:.3e} > 1e-4*Hs = {1e-4 * hs:.3e}"
    nrm = np.sqrt(np.sum(ref ** 2))
    if nrm > 0:
        rl2 = np.sqrt(np.sum((got - ref) ** 2)) / nrm
        assert rl2 <= rel_l2, f"{what}: rel-L2 {rl2:.3e} > {rel_l2:.1e}"


# ---------------------------------------------------------------- FFT ----

def _np(t):
    return t.double().cpu().numpy()


@pytest.mark.parametrize("key,domain,chop,times", [("n16", 500.0, 1.0, (0.0, 12.75)),
                                                    ("n64", 1000.0, 1.2, (1.5, 123.4))])
def test_fft_golden(cuda, golden, key, domain, chop, times):
    from paper_2511_02852_b200.fft_background import FftState, _upload, evolve_and_synthesize
    gd = golden("fft.npz")
    h0 = gd[f"{key}_h0"]
    st = _upload(FftState(n=h0.shape[0], domain_size=domain, g=G, rng_seed=0, choppiness=chop, h0=h0), cuda)
    for k, t in enumerate(times):
        f = evolve_and_synthesize(st, t)
        ref_h = gd[f"{key}_t{k}_h"]
        hs = hs_of(ref_h)
        assert_field_close(_np(f.height), ref_h, hs, what=f"{key} height t={t}")
        assert_field_close(_np(f.displacement), gd[f"{key}_t{k}_d"], hs, what=f"{key} disp t={t}")
        np.testing.assert_allclose(_np(f.normal), gd[f"{key}_t{k}_n"], atol=2e-5)


@pytest.mark.parametrize("n,domain,u10,chop,t", [(256, 1000.0, 10.0, 1.0, 2.0), (1024, 4000.0, 10.0, 1.2, 10.0),
                                                  (1024, 4000.0, 10.0, 1.2, 1000.0), (2048, 8000.0, 10.0, 1.0, 37.0),
                                                  (512, 2000.0, 15.0, 0.0, 5.0), (4, 100.0, 5.0, 1.0, 1.0)])
def test_fft_vs_oracle(cuda, n, domain, u10, chop, t):
    from paper_2511_02852_b200 import DirectionalSpectrum, derive_params, evolve_and_synthesize, init_fft
    p = derive_params(u10, 1e5, G)
    st = init_fft(DirectionalSpectrum(p, 0.4), n, domain, seed=n, choppiness=chop, device=cuda)
    f = evolve_and_synthesize(st, t)
    h, dx, dy, nrm = ocean_ref.evolve(st.h0, domain, G, t, chop)
    hs = max(hs_of(h), 1e-12)
    if np.abs(h).max() == 0:
        assert float(f.height.abs().max()) == 0.0
        return
    assert_field_close(_np(f.height), h, hs, what="height")
    assert_field_close(_np(f.displacement[..., 0]), dx, hs, what="dx")
    assert_field_close(_np(f.displacement[..., 1]), dy, hs, what="dy")
    np.testing.assert_allclose(_np(f.normal), nrm, atol=5e-5)
    if chop == 0.0:
        assert float(f.displacement.abs().max()) == 0.0


def test_fft_self_conjugate_bins(cuda):
    """Band widened to Nyquist with mean direction pi: the self-conjugate
    bins carry energy."""
    from paper_2511_02852_b200 import DirectionalSpectrum, derive_params, evolve_and_synthesize, init_fft
    p = derive_params(10.0, 1e5, G)
    st = init_fft(DirectionalSpectrum(p, math.pi), 256, 1000.0, seed=0, choppiness=1.0, band=(0.4, 4.0),
                  device=cuda)
    assert np.abs(st.h0[128, 0]) > 0 or np.abs(st.h0[0, 128]) > 0
    f = evolve_and_synthesize(st, 3.0)
    h, dx, dy, _ = ocean_ref.evolve(st.h0, 1000.0, G, 3.0, 1.0)
    hs = hs_of(h)
    assert_field_close(_np(f.height), h, hs, what="height")
    assert_field_close(_np(f.displacement[..., 0]), dx, hs, what="dx")
    assert_field_close(_np(f.displacement[..., 1]), dy, hs, what="dy")


def test_sample_periodic_golden(cuda, golden):
    from paper_2511_02852_b200.fft_background import FftState, _upload, evolve_and_synthesize, sample_periodic
    gd = golden("fft.npz")
    st = _upload(FftState(n=64, domain_size=1000.0, g=G, rng_seed=0, choppiness=1.2, h0=gd["n64_h0"]), cuda)
    f = evolve_and_synthesize(st, 123.4)
    h, n = sample_periodic(f, gd["n64_sample_pts"])
    hs = hs_of(gd["n64_t1_h"])
    assert np.abs(_np(h) - gd["n64_sample_h"]).max() <= 1e-4 * hs
    np.testing.assert_allclose(_np(n), gd["n64_sample_n"], atol=5e-5)


# ---------------------------------------------------------- particles ----

def _pr1_host():
    from paper_2511_02852_b200 import DirectionalSpectrum, PatchRegion, derive_params, log_buckets
    p = derive_params(10.0, 1e5, G, gamma=3.3, spread_s=8.0)
    table = log_buckets(p, 0.5, 4.0, 8, 16)
    return DirectionalSpectrum(p, 0.0), table, PatchRegion((100.0, 200.0), 64.0, 64.0, 8.0)


def _segments(pos, d, amp, bucket, nb):
    return [(pos[bucket == b], d[bucket == b], amp[bucket == b]) for b in range(nb)]


def _compare_segments(ps, gd, prefix, nb, pos_atol=0.0, dir_atol=0.0):
    ref = _segments(gd[f"{prefix}_pos"], gd[f"{prefix}_dir"], gd[f"{prefix}_amp"], gd[f"{prefix}_bucket"], nb)
    np.testing.assert_array_equal(ps.counts, [len(r[2]) for r in ref])
    for b in range(nb):
        seg = ps.segment(b)
        rp, rd, ra = ref[b]
        if pos_atol == 0.0:
            np.testing.assert_array_equal(seg["pos"], rp, err_msg=f"bucket {b} positions")
        else:
            np.testing.assert_allclose(seg["pos"], rp, rtol=0, atol=pos_atol, err_msg=f"bucket {b}")
        np.testing.assert_allclose(seg["dir"], rd, rtol=0, atol=dir_atol)
        np.testing.assert_allclose(seg["amp"], ra.astype(np.float32), rtol=1e-6, atol=0)


def test_inject_single_call_matches_reference(cuda, golden):
    from paper_2511_02852_b200 import InjectionLedger, inject
    gd = golden("particles.npz")
    sp, table, patch = _pr1_host()
    led = InjectionLedger(8, device=cuda)
    rng = np.random.Generator(np.random.Philox(key=[0, 0]))
    ref_led = particles_ref.Ledger(8)
    ref_rng = np.random.Generator(np.random.Philox(key=[0, 0]))
    p = spectrum_ref.jonswap(10.0, 1e5, G, gamma=3.3, spread_s=8.0)
    bk = spectrum_ref.log_buckets(p, 0.5, 4.0, 8, 16)
    pr = particles_ref.Patch(100.0, 200.0, 64.0, 64.0, 8.0)
    dt = 1.0 / 60.0
    for k in range(40):
        new = inject(patch, table, sp, led, dt, rng, t=k * dt)
        ref = particles_ref.inject(pr, bk, p, 0.0, ref_led, dt, ref_rng, t=k * dt)
        assert len(new) == len(ref), f"frame {k}"
        if len(ref):
            gdx = {"x_pos": ref.pos, "x_dir": ref.dir, "x_amp": ref.amp, "x_bucket": ref.bucket}
            _compare_segments(new, gdx, "x", 8, pos_atol=1e-12, dir_atol=1e-15)
    np.testing.assert_array_equal(led.accumulators, ref_led.acc)
    np.testing.assert_array_equal(led.injected_groups, ref_led.groups)
    np.testing.assert_allclose(led.injected_energy, ref_led.e_in, rtol=1e-13)
    # the host generator was advanced exactly like the reference's
    np.testing.assert_array_equal(rng.bit_generator.random_raw(3), ref_rng.bit_generator.random_raw(3))


def test_inject_high_rate_golden(cuda, golden):
    from paper_2511_02852_b200 import DirectionalSpectrum, InjectionLedger, PatchRegion, derive_params, inject, log_buckets
    gd = golden("particles.npz")
    p = derive_params(10.0, 1e5, G)
    table = log_buckets(p, 0.3, 6.0, 16, 2)
    sp = DirectionalSpectrum(p, 0.7)
    patch = PatchRegion((-50.0, 30.0), 256.0, 192.0, 10.0)
    led = InjectionLedger(16, device=cuda)
    rng = np.random.Generator(np.random.Philox(key=[5, 1]))
    for k in range(3):
        new = inject(patch, table, sp, led, 0.1, rng, t=k * 0.1, trough_fraction=0.8)
    _compare_segments(new, gd, "hr_inj", 16, pos_atol=1e-11, dir_atol=1e-15)
    np.testing.assert_array_equal(led.accumulators, gd["hr_acc"])
    np.testing.assert_array_equal(led.injected_groups, gd["hr_groups"])
    np.testing.assert_allclose(led.injected_energy, gd["hr_e_in"], rtol=1e-13)


def test_advect_bit_exact_on_reference_pool(cuda, golden):
    from paper_2511_02852_b200 import InjectionLedger, ParticleSet, advect
    gd = golden("particles.npz")
    sp, table, patch = _pr1_host()
    pool = ParticleSet.from_arrays(gd["chain_final_pos"], gd["chain_final_dir"], gd["chain_final_amp"],
                                   gd["chain_final_bucket"], 8, device=cuda)
    led = InjectionLedger(8, device=cuda)
    dropped = advect(pool, table, 7.0 / 60.0, patch, led, g=G)
    _compare_segments(pool, gd, "adv7_kept", 8)
    _compare_segments(dropped, gd, "adv7_dropped", 8)
    np.testing.assert_allclose(led.despawned_energy, gd["adv7_e_out"], rtol=2e-7)


def test_inject_advect_chain_matches_reference(cuda, golden):
    """120 PR1 frames of inject + advect: counts bit-exact every frame."""
    from paper_2511_02852_b200 import InjectionLedger, ParticleSet, advect, inject
    gd = golden("particles.npz")
    sp, table, patch = _pr1_host()
    led = InjectionLedger(8, device=cuda)
    rng = np.random.Generator(np.random.Philox(key=[0, 0]))
    pool = ParticleSet(n_buckets=8, device=cuda)
    dt = 1.0 / 60.0
    for k in range(120):
        pool.extend(inject(patch, table, sp, led, dt, rng, t=k * dt))
        advect(pool, table, dt, patch, led, g=G)
        np.testing.assert_array_equal(pool.counts, gd["chain_counts"][k], err_msg=f"frame {k}")
    _compare_segments(pool, gd, "chain_final", 8, pos_atol=1e-9, dir_atol=1e-15)
    np.testing.assert_array_equal(led.accumulators, gd["chain_acc"])
    np.testing.assert_array_equal(led.injected_groups, gd["chain_groups"])


# ------------------------------------------------------------ synthesis --

def test_synthesize_golden(cuda, golden):
    from paper_2511_02852_b200 import ParticleSet, build_kernels, plan_layers, synthesize
    gp = golden("particles.npz")
    gd = golden("synth.npz")
    sp, table, patch = _pr1_host()
    pool = ParticleSet.from_arrays(gp["chain_final_pos"], gp["chain_final_dir"], gp["chain_final_amp"],
                                   gp["chain_final_bucket"], 8, device=cuda)
    res = 129
    texel = patch.l1 / (res - 1)
    plan = plan_layers(table, texel, res)
    assert tuple(plan.factors) == tuple(gd["plan_factors"])
    h, c = synthesize(pool, patch, res, plan)
    hs = hs_of(gd["h_plan"])
    assert_field_close(_np(h), gd["h_plan"], hs, what="synth plan")
    assert c == gd["clamped_plan"][0]
    h2, c2 = synthesize(pool, patch, res, build_kernels(table, texel))
    assert_field_close(_np(h2), gd["h_exact"], hs, what="synth exact")
    assert c2 == gd["clamped_exact"][0]


def test_synthesize_random_pool_vs_oracle(cuda):
    """C3-geometry patch (1024^2 over 256 m), 16 log buckets, 200k random
    particles including ones in the grace band and beyond the pad."""
    from paper_2511_02852_b200 import DirectionalSpectrum, ParticleSet, PatchRegion, derive_params, log_buckets
    from paper_2511_02852_b200 import plan_layers, synthesize
    p = derive_params(10.0, 1e5, G)
    table = log_buckets(p, 0.3, 6.0, 16, 2)
    patch = PatchRegion((1872.0, 1872.0), 256.0, 256.0, 10.0)
    rng = np.random.default_rng(7)
    n = 200_000
    pos = rng.uniform(1872.0 - 40.0, 1872.0 + 296.0, size=(n, 2))
    pos[:20] = rng.uniform(-5000, 5000, size=(20, 2))
    ang = rng.uniform(-np.pi, np.pi, n)
    d = np.stack([np.cos(ang), np.sin(ang)], 1)
    amp = rng.normal(0, 0.05, n)
    b = rng.integers(0, 16, n)
    ps = ParticleSet.from_arrays(pos, d, amp, b, 16, device=cuda)
    res = 1024
    plan = plan_layers(table, 256.0 / 1023, res)
    h, c = synthesize(ps, patch, res, plan)
    bk = spectrum_ref.log_buckets(spectrum_ref.jonswap(10.0, 1e5, G), 0.3, 6.0, 16, 2)
    pl = synth_ref.plan(bk, 256.0 / 1023, res)
    rp = particles_ref.Pool(pos, d, amp.astype(np.float32).astype(np.float64), b.astype(np.int32), np.zeros(n))
    href, cref = synth_ref.synthesize(rp, particles_ref.Patch(1872.0, 1872.0, 256.0, 256.0, 10.0), res, pl)
    assert c == cref
    assert_field_close(_np(h), href, hs_of(href), what="C3 synth")


def test_finish_and_sampler_golden(cuda, golden):
    from paper_2511_02852_b200 import PatchSurface, SurfaceSampler, finish_field
    from paper_2511_02852_b200.fft_background import FftState, _upload, evolve_and_synthesize
    gd = golden("synth.npz")
    gf = golden("fft.npz")
    sp, table, patch = _pr1_host()
    f = finish_field(torch.from_numpy(gd["h_plan"]), patch)
    np.testing.assert_allclose(_np(f.normal), gd["finish_n"], atol=2e-6)
    fc = finish_field(torch.from_numpy(gd["h_plan"]), patch, choppiness=0.7, displacement_scale=2.0)
    np.testing.assert_allclose(_np(fc.displacement), gd["finish_chop_d"], atol=1e-6)
    st = _upload(FftState(n=64, domain_size=1000.0, g=G, rng_seed=0, choppiness=1.2, h0=gf["n64_h0"]), cuda)
    bg = evolve_and_synthesize(st, 1.5)
    sampler = SurfaceSampler(bg, [PatchSurface(patch, f)])
    res = 129
    texel = patch.l1 / (res - 1)
    xs = patch.min_corner[0] + np.arange(res) * texel
    ys = patch.min_corner[1] + np.arange(res) * texel
    nodes = np.stack(np.meshgrid(xs, ys, indexing="ij"), -1)
    hb, nb = sampler.sample(nodes.reshape(-1, 2))
    hs = hs_of(gf["n64_t0_h"])
    assert np.abs(_np(hb).reshape(res, res) - gd["blend_h"]).max() <= 1e-4 * hs
    np.testing.assert_allclose(_np(nb).reshape(res, res, 3), gd["blend_n"], atol=5e-5)
    hs2, ns2 = sampler.sample(gd["sample_pts"])
    assert np.abs(_np(hs2) - gd["sample_h"]).max() <= 1e-4 * hs
    np.testing.assert_allclose(_np(ns2), gd["sample_n"], atol=5e-5)
    # far field is exactly the background sample (coupling.py:6-8)
    far = np.array([[10.0, 10.0], [900.0, 40.0]])
    hf, _ = sampler.sample(far)
    from paper_2511_02852_b200 import sample_periodic
    hb0, _ = sample_periodic(bg, far)
    assert torch.equal(hf, hb0)


# ---------------------------------------------------------- simulation --

def _sim_cfg():
    from paper_2511_02852_b200 import PatchConfig, SimConfig
    return SimConfig(fft_n=64, fft_domain=500.0, dt=0.05, frames=6, n_omega=8, n_theta=8, seed=11,
                     patches=(PatchConfig(origin=(200.0, 180.0), size=(100.0, 80.0), res=65, margin=10.0),),
                     write_frames=False)


def test_simulation_matches_reference_simulation(cuda, golden):
    """The whole reference Simulation.step chain (Philox stream) vs the
    graph-captured B200 step."""
    from paper_2511_02852_b200 import Simulation
    gd = golden("sim.npz")
    sim = Simulation(_sim_cfg(), device=cuda)
    for k in range(6):
        s = sim.step()
        np.testing.assert_array_equal(s.particle_counts, gd["counts"][k], err_msg=f"frame {k}")
        np.testing.assert_allclose(s.injected_energy, gd["e_in"][k], rtol=1e-12)
        np.testing.assert_allclose(s.despawned_energy, gd["e_out"][k], rtol=1e-6, atol=1e-9)
        assert s.fft_band_variance == pytest.approx(gd["fft_var"][k], rel=1e-5)
        assert s.patch_variance == pytest.approx(gd["patch_var"][k], rel=1e-4, abs=1e-12)
    sim.check()
    hs = hs_of(gd["bg_h"])
    assert_field_close(_np(sim.background.height), gd["bg_h"], hs, what="bg")
    assert_field_close(_np(sim.patch_heights(0)), gd["patch_h"], hs, what="patch")
    assert_field_close(_np(sim.stitched_heights()), gd["stitched"], hs, what="stitched")
    # pool per bucket equals the reference pool's per-bucket subsequence
    pool = sim.pool(0)
    _compare_segments(pool, gd, "pool", 8, pos_atol=1e-9, dir_atol=1e-15)


@pytest.mark.parametrize("preset", ["PR1", "C2"])
def test_preset_scene_vs_oracle(cuda, preset):
    """Scene-level parity on BASELINE presets (shortened runs)."""
    from paper_2511_02852_b200 import Simulation, scenes
    cfg = scenes.PRESETS[preset](frames=30)
    sim = Simulation(cfg, device=cuda)
    ref = scene_ref.OracleScene(cfg.scene_dict())
    for k in range(30):
        sim.step(stats=False)
        out = ref.step(synth=(k == 29))
        np.testing.assert_array_equal(sim.counts_host(), out["counts"], err_msg=f"frame {k}")
    sim.check()
    hs = hs_of(out["height"])
    assert_field_close(_np(sim.background.height), out["height"], hs, what="bg")
    for p in range(sim.n_patches):
        assert_field_close(_np(sim.patch_heights(p)), out["patch_heights"][p], hs, what=f"patch {p}")
        bh, bn = sim.blended_tile(p)
        assert_field_close(_np(bh), out["blend_heights"][p], hs, what=f"blend {p}")
        np.testing.assert_allclose(_np(bn), out["blend_normals"][p], atol=1e-4)
    assert_field_close(_np(sim.stitched_heights()), ref.composite(), hs, what="composite")
