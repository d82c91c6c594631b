"""Scene-level parity at the BASELINE configs (B200 vs the CPU oracle).

The north_star correctness bar applies to the BASELINE scenes themselves
(reference `harness.py:131-241`): bucket assignment, compaction order and
particle counts bit-exact; fp32 heights within max-abs 1e-4*Hs and relative
L2 1e-5 of the fp64 oracle.

* Steady state (C3 headline, C4, a 4-ship C5 slice): the GPU warms the scene
  with the pipeline itself (dt = 0.1 for 200 s), its whole
  state is cloned into the oracle (`oracle/clone.py`), then both step 60
  frames at the config's dt = 1/60.  Every frame: per-(patch, bucket) counts
  bit-exact.  Last frame: per-bucket pool order and positions (particles that
  existed at the clone bit for bit; ones injected after it within 1e-9 m, the
  ulp-level device cos/sin of SURVEY App. B.5), ledgers, and background,
  patch, blend and composite fields within the north_star tolerance.
* From t = 0 (PR1 for its 120 frames, C2 for its 300): counts every frame,
  fields at the end.
"""
import numpy as np
import pytest

from oracle.clone import CLONED, oracle_from_sim

pytestmark = pytest.mark.gpu

WARM_FRAMES = 2000          # 200 s at dt = 0.1 (bench.py)
STEADY_FRAMES = 60


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


def _np(t):
    return t.double().cpu().numpy()


def compare_pools(sim, ref, nb):
    """Per patch and bucket: same count, same stable order.  Cloned particles
    (advected by both sides from identical fp64 state) must agree bit for
    bit; injected ones to 1e-9 m / 1e-15 in direction.  Returns
    (particles compared, bitwise fraction of the injected ones)."""
    n_new = n_new_bitwise = n_all = 0
    for k in range(sim.n_patches):
        ps = sim.pool(k)
        off = np.concatenate([[0], np.cumsum(ps.counts)])
        pos, dirs, amp, birth = ps.positions, ps.directions, ps.amplitudes, ps.birth_times
        rp = ref.pools[k]
        for b in range(nb):
            m = rp.bucket == b
            lo, hi = int(off[b]), int(off[b + 1])
            assert hi - lo == int(m.sum()), f"patch {k} bucket {b}: {hi - lo} vs {int(m.sum())}"
            gp, gd, ga, gb = pos[lo:hi], dirs[lo:hi], amp[lo:hi], birth[lo:hi]
            rpos, rdir, ramp, rbirth = rp.pos[m], rp.dir[m], rp.amp[m], rp.birth[m]
            old = rbirth == CLONED
            np.testing.assert_array_equal(gp[old], rpos[old], err_msg=f"patch {k} bucket {b} cloned positions")
            np.testing.assert_array_equal(gd[old], rdir[old], err_msg=f"patch {k} bucket {b} cloned directions")
            new = ~old
            # birth times t = frame * dt (particles.py:296-299; emitted ones 0, interaction.py:210)
            np.testing.assert_array_equal(gb[new], rbirth[new], err_msg=f"patch {k} bucket {b} births")
            if new.any():
                np.testing.assert_allclose(gp[new], rpos[new], rtol=0, atol=1e-9,
                                           err_msg=f"patch {k} bucket {b} injected positions")
                np.testing.assert_allclose(gd[new], rdir[new], rtol=0, atol=1e-15)
                n_new += int(new.sum())
                n_new_bitwise += int(np.all(gp[new] == rpos[new], axis=1).sum())
            np.testing.assert_allclose(ga, ramp.astype(np.float32).astype(np.float64), rtol=1e-6, atol=1e-12)
            n_all += hi - lo
    return n_all, (n_new_bitwise / n_new if n_new else 1.0)


def compare_fields(sim, ref, out, what):
    hs = hs_of(out["height"])
    assert_field_close(_np(sim.background.height), out["height"], hs, what=f"{what} background")
    for p in range(sim.n_patches):
        assert_field_close(_np(sim.patch_heights(p)), out["patch_heights"][p], hs, what=f"{what} patch {p}")
        bh, bn = sim.blended_tile(p)
        assert_field_close(_np(bh), out["blend_heights"][p], hs, what=f"{what} blend {p}")
        np.testing.assert_allclose(_np(bn), out["blend_normals"][p], atol=1e-4, err_msg=f"{what} normals {p}")
    assert_field_close(_np(sim.stitched_heights()), ref.composite(), hs, what=f"{what} composite")


def compare_ledgers(sim, ref):
    led = sim.ledger_host()
    for k in range(sim.n_patches):
        np.testing.assert_array_equal(led["acc"][k], ref.ledgers[k].acc)
        np.testing.assert_array_equal(led["groups"][k], ref.ledgers[k].groups)
        np.testing.assert_allclose(led["e_in"][k], ref.ledgers[k].e_in, rtol=1e-12, atol=0)
        # despawn energy from the pool's fp32 amplitudes (36 B/particle layout),
        # summed by atomics: ~1e-7 relative
        np.testing.assert_allclose(led["e_out"][k], ref.ledgers[k].e_out, rtol=1e-6, atol=1e-9)


def _steady_cfg(name):
    from paper_2511_02852_b200 import scenes
    if name == "C5-4":
        return scenes.c5(n_patches=4)
    return scenes.PRESETS[name]()


@pytest.mark.parametrize("name,min_live", [("C3", 800_000), ("C4", 3_500_000), ("C5-4", 300_000)])
def test_steady_state_scene_vs_oracle(cuda, name, min_live):
    from paper_2511_02852_b200 import Simulation
    cfg = _steady_cfg(name)
    sim = Simulation(cfg, device=cuda)
    sim.run_frames(WARM_FRAMES, dt=0.1)
    sim.check()
    live0 = sim.live_particles()
    assert live0 >= min_live, f"{name}: only {live0} live particles at steady state"
    ref = oracle_from_sim(sim, cfg)
    np.testing.assert_array_equal(sim.counts_host(), np.stack([p.counts(sim.nb) for p in ref.pools]))
    for k in range(STEADY_FRAMES):
        sim.step(stats=False)
        last = k == STEADY_FRAMES - 1
        out = ref.step(synth=last, fft=last)
        np.testing.assert_array_equal(sim.counts_host(), out["counts"], err_msg=f"{name} frame {k}")
    sim.check()
    n, frac = compare_pools(sim, ref, sim.nb)
    assert n == sim.live_particles()
    print(f"{name}: {n} live particles compared; injected after the clone bitwise: {frac:.4f}")
    compare_ledgers(sim, ref)
    compare_fields(sim, ref, out, name)


@pytest.mark.parametrize("preset", ["PR1", "C2"])
def test_preset_full_run_vs_oracle(cuda, preset):
    """The whole BASELINE run length from t = 0: PR1 120 frames, C2 300
    frames (with its four moving wake sources)."""
    from paper_2511_02852_b200 import Simulation, scenes
    from oracle import scene_ref
    cfg = scenes.PRESETS[preset]()
    frames = cfg.frames
    sim = Simulation(cfg, device=cuda)
    ref = scene_ref.OracleScene(cfg.scene_dict())
    for k in range(frames):
        sim.step(stats=False)
        last = k == frames - 1
        out = ref.step(synth=last, fft=last)
        np.testing.assert_array_equal(sim.counts_host(), out["counts"], err_msg=f"{preset} frame {k}")
    sim.check()
    # every particle was injected or emitted on the device: order exact, positions to 1e-9
    n, frac = compare_pools(sim, ref, sim.nb)
    print(f"{preset}: {n} live particles after {frames} frames; bitwise positions {frac:.4f}")
    compare_ledgers(sim, ref)
    compare_fields(sim, ref, out, preset)
