"""Deterministic mode (`device.deterministic = true`): the reference's
determinism contract (pkg/tests/test_acceptance.py:293-311, two `run`s of
one config give byte-identical stats.csv and frame files) on the B200.

Float sums whose order depends on scheduling -- the splat into the raw
layers, the despawn-energy ledger, the interior and FFT-band variances --
go through int64 fixed point (hybridsea_b200.h HS_FIXED_*), so reruns are
byte-identical; the default mode uses float atomics and is checked here to
stay within the north_star tolerances of the deterministic one."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cfg(deterministic, frames=20, body=True, **kw):
    from paper_2511_02852_b200 import BodyConfig, PatchConfig, SimConfig
    bodies = (BodyConfig(position=(250.0, 250.0, 0.0), size=(2.0, 2.0, 1.0), density=500.0),) if body else ()
    return SimConfig(fft_n=128, dt=0.05, frames=frames, n_omega=8, n_theta=8,
                     patches=(PatchConfig(origin=(200.0, 200.0), size=(100.0, 100.0), res=129, margin=10.0),),
                     bodies=bodies, write_frames=True, deterministic=deterministic, **kw).validate()


def _read(d):
    stats = open(os.path.join(d, "stats.csv"), "rb").read()
    frames = {f: open(os.path.join(d, f), "rb").read() for f in sorted(os.listdir(d)) if f.endswith(".raw")}
    return stats, frames


def test_byte_identical_runs(cuda, tmp_path):
    from paper_2511_02852_b200 import run
    cfg = _cfg(True)
    run(cfg, str(tmp_path / "a"))
    run(cfg, str(tmp_path / "b"))
    sa, fa = _read(tmp_path / "a")
    sb, fb = _read(tmp_path / "b")
    assert len(fa) == 20
    assert sa == sb, "stats.csv differs between reruns"
    assert fa.keys() == fb.keys() and all(fa[k] == fb[k] for k in fa), "frames differ between reruns"


def test_byte_identical_with_compaction_and_sources(cuda):
    """Past resident-pool compactions (K = 16 frames), with wake sources and
    their tracking patches: blended tiles, pools' live counts and the ledger."""
    from paper_2511_02852_b200 import Simulation, scenes
    outs = []
    for _ in range(2):
        cfg = scenes.c5(2, frames=40, fft_n=512, deterministic=True)
        sim = Simulation(cfg, device=cuda, compact_period=16)
        rows = [sim.step() for _ in range(cfg.frames)]
        sim.check()
        outs.append((sim.blend_h.cpu().numpy().tobytes(), sim.patch_h.cpu().numpy().tobytes(),
                     [(r.despawned_energy.tobytes(), r.patch_variance, r.fft_band_variance,
                       r.particle_counts.tobytes()) for r in rows]))
    assert outs[0][0] == outs[1][0] and outs[0][1] == outs[1][1]
    assert outs[0][2] == outs[1][2]


def test_deterministic_matches_default_mode(cuda):
    """Same scene, both modes: fixed point vs float atomics agree to the
    north_star tolerances (max-abs 1e-4 Hs, rel-L2 1e-5) and the ledger to
    1e-9 relative.  No floating body here: its wake firing amplifies any
    last-bit difference of the surface into a whole ring."""
    from paper_2511_02852_b200 import Simulation
    res = []
    for det in (False, True):
        cfg = _cfg(det, frames=60, body=False)
        sim = Simulation(cfg, device=cuda)
        for _ in range(cfg.frames):
            st = sim.step()
        res.append((sim.blend_h.double().cpu().numpy(), st.despawned_energy, st.patch_variance,
                    st.fft_band_variance, st.particle_counts))
    (h0, e0, pv0, fv0, c0), (h1, e1, pv1, fv1, c1) = res
    hs = 4.0 * np.sqrt(np.mean(h0 ** 2))
    assert np.abs(h1 - h0).max() <= 1e-4 * hs
    assert np.sqrt(np.sum((h1 - h0) ** 2) / np.sum(h0 ** 2)) <= 1e-5
    np.testing.assert_array_equal(c0, c1)
    np.testing.assert_allclose(e1, e0, rtol=1e-9, atol=1e-6)
    assert abs(pv1 - pv0) <= 1e-5 * abs(pv0) and abs(fv1 - fv0) <= 1e-9 * abs(fv0)
