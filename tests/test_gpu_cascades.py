"""Summed FFT cascades (C4: tiles with disjoint |k| bands) on the B200 vs the
CPU oracle: every cascade's heights, the blended patch tiles (heights add,
normals combine through slopes), the FFT-resolution composite and the band
variance.  Tolerances: max-abs 1e-4*Hs, rel-L2 1e-5 (fp32 vs fp64)."""
import numpy as np
import pytest

from oracle import scene_ref

pytestmark = pytest.mark.gpu


def hs_of(h):
    return 4.0 * float(np.sqrt(np.mean(np.asarray(h) ** 2)))


def close(got, ref, hs, what, rel_l2=1e-5):
    got = np.asarray(got, dtype=np.float64)
    err = np.abs(got - ref).max()
    assert err <= 1e-4 * hs, f"{what}: max-abs {err:.3e} > 1e-4*Hs ({hs:.3e})"
    rl2 = np.sqrt(np.sum((got - ref) ** 2) / np.sum(ref ** 2))
    assert rl2 <= rel_l2, f"{what}: rel-L2 {rl2:.3e}"


def test_cascaded_scene_vs_oracle(cuda):
    from paper_2511_02852_b200 import PatchConfig, SimConfig, Simulation
    cfg = SimConfig(u10=12.0, fetch=1e5, n_omega=8, n_theta=8, dt=0.1, frames=40, seed=9,
                    fft_n=128, fft_domain=1000.0, fft_cascades=(1000.0, 250.0, 60.0), fft_band_hi=8.0,
                    patches=(PatchConfig(origin=(400.0, 380.0), size=(64.0, 64.0), res=129, margin=8.0),
                             PatchConfig(origin=(480.0, 470.0), size=(48.0, 64.0), res=97, margin=6.0)),
                    write_frames=False)
    sim = Simulation(cfg, device=cuda)
    ref = scene_ref.OracleScene(cfg.scene_dict())
    for k in range(cfg.frames):
        st = sim.step()
        out = ref.step(synth=(k == cfg.frames - 1))
        np.testing.assert_array_equal(sim.counts_host(), out["counts"], err_msg=f"frame {k}")
    sim.check()
    fields = sim.cascade_fields()
    assert len(fields) == 3
    hs = hs_of(sum(np.mean(h ** 2) for h in out["cascade_heights"]) ** 0.5 * np.ones(1))
    for c, (f, hr) in enumerate(zip(fields, out["cascade_heights"])):
        assert np.abs(hr).max() > 0, f"cascade {c} carries no energy"
        assert np.abs(out["patch_heights"][0]).max() > 0
        close(f.height.double().cpu().numpy(), hr, hs_of(hr), f"cascade {c}")
    var = sum(float(np.mean(h ** 2)) for h in out["cascade_heights"])
    assert st.fft_band_variance == pytest.approx(var, rel=1e-5)
    for p in range(2):
        close(sim.patch_heights(p).double().cpu().numpy(), out["patch_heights"][p], hs, f"patch {p}")
        bh, bn = sim.blended_tile(p)
        close(bh.double().cpu().numpy(), out["blend_heights"][p], hs, f"blend {p}")
        np.testing.assert_allclose(bn.double().cpu().numpy(), out["blend_normals"][p], atol=2e-4)
    close(sim.stitched_heights().double().cpu().numpy(), ref.composite(), hs, "composite")
    # the public sampler sees the summed background too
    pts = np.array([[10.0, 20.0], [512.3, 700.9], [420.0, 400.0]])
    h, n = sim.sampler.sample(pts)
    from oracle import blend_ref
    pairs = list(zip(ref.patches, ref.fields))
    rh, rn = blend_ref.sample(ref.background, pairs, pts)
    np.testing.assert_allclose(h.double().cpu().numpy(), rh, atol=1e-4 * hs)
    np.testing.assert_allclose(n.double().cpu().numpy(), rn, atol=2e-4)
