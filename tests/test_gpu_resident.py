"""Resident particle pool (in-place advect, holes, compaction every K frames)
against the CPU oracle, across compactions (B200).

The reference compacts its pool every frame (particles.py:167-178,
advect :303-328).  The B200 frame defers that compaction: a despawn leaves a
hole, injected particles are appended at their bucket segment's tail, and
every K frames hs_advect squeezes the holes out.  The live particles of each
bucket read in slot order must equal the reference's pool restricted to that
bucket at EVERY frame, whatever K is -- bit-exact counts, positions and
order.
"""
import numpy as np
import pytest
import torch

from oracle import scene_ref

pytestmark = pytest.mark.gpu


def hs_of(h):
    return 4.0 * float(np.sqrt(np.mean(np.asarray(h) ** 2)))


def assert_field_close(got, ref, hs, rel_l2=1e-5, what=""):
    err = np.abs(got - ref).max()
    assert err <= 1e-4 * hs, f"{what}: max-abs {err:.3e} > 1e-4*Hs"
    rl2 = np.sqrt(np.sum((got - ref) ** 2) / np.sum(ref ** 2))
    assert rl2 <= rel_l2, f"{what}: rel-L2 {rl2:.3e}"


def _run_vs_oracle(cfg, frames, compact_period, pool_every=7, device=None):
    from paper_2511_02852_b200 import Simulation
    sim = Simulation(cfg, device=device, compact_period=compact_period)
    ref = scene_ref.OracleScene(cfg.scene_dict())
    for k in range(frames):
        sim.step(stats=False)
        out = ref.step(synth=False, fft=False)
        np.testing.assert_array_equal(sim.counts_host(), out["counts"], err_msg=f"K={compact_period} frame {k}")
        if k % pool_every == pool_every - 1 or k == frames - 1:
            for p in range(sim.n_patches):
                ps = sim.pool(p)
                rp = ref.pools[p]
                for b in range(sim.nb):
                    seg = ps.segment(b)
                    sel = rp.bucket == b
                    # directions come from the device's cos/sin (ulp-level vs numpy)
                    np.testing.assert_allclose(seg["pos"], rp.pos[sel], rtol=0, atol=1e-9,
                                               err_msg=f"frame {k} patch {p} b {b}")
                    np.testing.assert_allclose(seg["dir"], rp.dir[sel], rtol=0, atol=1e-15)
                    np.testing.assert_allclose(seg["amp"], rp.amp[sel].astype(np.float32), rtol=1e-6, atol=0)
    sim.check()
    return sim, ref


@pytest.mark.parametrize("K", [1, 3, 8])
def test_pr1_pool_bit_exact_across_compactions(cuda, K):
    from paper_2511_02852_b200 import scenes
    _run_vs_oracle(scenes.pr1(frames=40), 40, K, device=cuda)


def test_c2_multi_patch_default_period(cuda):
    """4 patches, the default compaction period (64): frames 0..139 cross two
    compactions; per-patch Philox streams keep every patch bit-exact."""
    from paper_2511_02852_b200 import scenes
    _run_vs_oracle(scenes.c2(frames=140), 140, None, pool_every=47, device=cuda)


def test_high_rate_warmup_dt(cuda):
    """dt = 0.1 (the bench warm-up step) maximises per-frame inflow; the
    segment slack must absorb K frames of it without overflow."""
    from paper_2511_02852_b200 import Simulation, scenes
    cfg = scenes.pr1(frames=10, dt=0.1)
    sim, ref = _run_vs_oracle(cfg, 50, 16, pool_every=10, device=cuda)
    assert sim.live_particles() > 1000


def test_holes_are_invisible_to_synthesis(cuda):
    """Patch heights with holes in the pool (mid-period) equal those of the
    oracle, i.e. holes are never splatted."""
    from paper_2511_02852_b200 import Simulation, scenes
    cfg = scenes.pr1(frames=20, dt=0.1)
    sim = Simulation(cfg, device=cuda, compact_period=64)
    ref = scene_ref.OracleScene(cfg.scene_dict())
    for k in range(60):
        sim.step(stats=False)
        out = ref.step(synth=(k == 59), fft=(k == 59))
    holes = int((sim.seg_len[sim._lp] - sim.live).sum().item())
    assert holes > 0, "the scene should have despawned particles by frame 20"
    hs = hs_of(out["height"])
    assert_field_close(sim.patch_heights(0).double().cpu().numpy(), out["patch_heights"][0], hs, what="patch")


def test_compaction_period_is_invisible_bitwise(cuda):
    """K = 1 (compact every frame, the reference's per-frame compaction) and
    K = 5 / 32 give bit-identical pools, counts and ledgers: deferring the
    compaction changes where particles sit in memory, never a value or the
    order of a bucket's live particles."""
    from paper_2511_02852_b200 import Simulation, scenes
    cfg = scenes.c2(frames=10)
    sims = [Simulation(cfg, device=cuda, compact_period=K) for K in (1, 5, 32)]
    for k in range(45):
        for s in sims:
            s.step(stats=False, dt=0.1 if k < 20 else None)
    base = sims[0]
    for s in sims[1:]:
        np.testing.assert_array_equal(s.counts_host(), base.counts_host())
        la, lb = s.ledger_host(), base.ledger_host()
        np.testing.assert_array_equal(la["acc"], lb["acc"])
        np.testing.assert_array_equal(la["groups"], lb["groups"])
        np.testing.assert_array_equal(la["e_in"], lb["e_in"])
        for p in range(base.n_patches):
            pa, pb = s.pool(p), base.pool(p)
            for b in range(base.nb):
                sa, sb = pa.segment(b), pb.segment(b)
                np.testing.assert_array_equal(sa["pos"], sb["pos"])
                np.testing.assert_array_equal(sa["dir"], sb["dir"])
                np.testing.assert_array_equal(sa["amp"], sb["amp"])
