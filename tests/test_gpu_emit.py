"""Kinematic emitting bodies and patch tracking on the B200
against the reference Simulation (golden vectors) and the CPU oracle.

Bar: integer work (counts per bucket, pool order, patch origins) bit-exact;
positions to 1e-9 m (directions of injected particles come from the
device's cos/sin; emitted fans are host numpy, exact);
fp32 heights within max-abs 1e-4*Hs and rel-L2 1e-5.
"""
import math

import numpy as np
import pytest

from oracle import scene_ref

pytestmark = pytest.mark.gpu


def hs_of(h):
    return 4.0 * float(np.sqrt(np.mean(np.asarray(h) ** 2)))


def assert_field_close(got, ref, hs, rel_l2=1e-5, what=""):
    got = np.asarray(got, dtype=np.float64)
    err = np.abs(got - ref).max()
    assert err <= 1e-4 * hs, f"{what}: max-abs {err:.3e} > 1e-4*Hs"
    rl2 = np.sqrt(np.sum((got - ref) ** 2) / np.sum(ref ** 2))
    assert rl2 <= rel_l2, f"{what}: rel-L2 {rl2:.3e}"


def _emit_sim_cfg():
    from paper_2511_02852_b200 import PatchConfig, SimConfig, SourceConfig
    hull0, hull1 = 0.5 * math.hypot(4.0, 2.0), 0.5 * math.hypot(2.0, 2.0)   # box_body (interaction.py:90)
    return SimConfig(fft_n=64, fft_domain=500.0, dt=0.05, frames=10, n_omega=8, n_theta=8, seed=21,
                     patches=(PatchConfig(origin=(200.0, 180.0), size=(100.0, 80.0), res=65, margin=10.0,
                                          track_source=0),),
                     sources=(SourceConfig(position=(250.0, 220.0), velocity=(3.0, 1.0, 0.0), hull_extent=hull0,
                                           volume_rate=0.02, submersion=0.5),
                              SourceConfig(position=(230.0, 200.0), velocity=(1.0, -0.5, 0.8), hull_extent=hull1,
                                           volume_rate=-0.01, submersion=0.3)),
                     write_frames=False)


def _segments_equal(ps, pos, d, amp, bucket, nb, pos_atol=1e-9):
    np.testing.assert_array_equal(ps.counts, np.bincount(bucket, minlength=nb))
    for b in range(nb):
        seg = ps.segment(b)
        sel = bucket == b
        np.testing.assert_allclose(seg["pos"], pos[sel], rtol=0, atol=pos_atol, err_msg=f"bucket {b}")
        np.testing.assert_allclose(seg["dir"], d[sel], rtol=0, atol=1e-15)
        np.testing.assert_allclose(seg["amp"], amp[sel].astype(np.float32), rtol=1e-6, atol=0)


@pytest.mark.parametrize("K", [None, 3])
def test_sources_and_tracking_match_reference_simulation(cuda, golden, K):
    """The reference Simulation with two kinematic bodies (one tracked by the
    patch, one heaving: ring + wake, suction) vs the graph-captured B200 step,
    with the default compaction period and with compactions every 3 frames."""
    from paper_2511_02852_b200 import Simulation
    gd = golden("emit_sim.npz")
    cfg = _emit_sim_cfg()
    sim = Simulation(cfg, device=cuda, compact_period=K)
    for k in range(cfg.frames):
        st = sim.step()
        np.testing.assert_array_equal(st.particle_counts, gd["counts"][k], err_msg=f"frame {k}")
        np.testing.assert_allclose(st.injected_energy, gd["e_in"][k], rtol=1e-12)
        np.testing.assert_allclose(st.despawned_energy, gd["e_out"][k], rtol=1e-6, atol=1e-9)
        np.testing.assert_array_equal(sim.current_regions()[0].min_corner, gd["origins"][k], err_msg=f"frame {k}")
    sim.check()
    _segments_equal(sim.pool(0), gd["pool_pos"], gd["pool_dir"], gd["pool_amp"], gd["pool_bucket"], 8)
    hs = hs_of(gd["patch_h"])
    assert_field_close(sim.patch_heights(0).double().cpu().numpy(), gd["patch_h"], hs, what="patch heights")
    assert_field_close(sim.stitched_heights().double().cpu().numpy(), gd["stitched"], hs, what="stitched")


def test_sources_crossing_patches_vs_oracle(cuda):
    """Untracked sources that leave one patch and enter another (ownership =
    first patch containing the source), several sources per patch and
    bucket (fans appended in source order), K = 4 compactions."""
    from paper_2511_02852_b200 import PatchConfig, SimConfig, Simulation, SourceConfig
    cfg = SimConfig(fft_n=64, fft_domain=1000.0, dt=0.1, frames=40, n_omega=8, n_theta=8, seed=5,
                    patches=(PatchConfig(origin=(100.0, 100.0), size=(60.0, 60.0), res=61, margin=8.0),
                             PatchConfig(origin=(160.0, 100.0), size=(60.0, 60.0), res=61, margin=8.0)),
                    sources=(SourceConfig(position=(140.0, 130.0), velocity=(8.0, 0.5, 0.0), hull_extent=1.5,
                                          volume_rate=0.02, submersion=0.5, wake_count=64),
                             SourceConfig(position=(150.0, 120.0), velocity=(6.0, 1.0, 0.0), hull_extent=1.5,
                                          volume_rate=0.01, submersion=0.4, wake_count=32),
                             SourceConfig(position=(120.0, 110.0), velocity=(0.0, 0.0, 0.5), hull_extent=3.0,
                                          volume_rate=-0.01, submersion=0.3)),
                    write_frames=False)
    sim = Simulation(cfg, device=cuda, compact_period=4)
    ref = scene_ref.OracleScene(cfg.scene_dict())
    for k in range(cfg.frames):
        sim.step(stats=False)
        out = ref.step(synth=(k == cfg.frames - 1))
        np.testing.assert_array_equal(sim.counts_host(), out["counts"], err_msg=f"frame {k}")
    sim.check()
    led = sim.ledger_host()
    for p in range(2):
        np.testing.assert_allclose(led["e_in"][p], ref.ledgers[p].e_in, rtol=1e-12)
        rp = ref.pools[p]
        _segments_equal(sim.pool(p), rp.pos, rp.dir, rp.amp, rp.bucket, 8)
        hs = hs_of(out["patch_heights"][p])
        assert_field_close(sim.patch_heights(p).double().cpu().numpy(), out["patch_heights"][p], hs,
                           what=f"patch {p}")
