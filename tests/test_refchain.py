"""The reference-arm driver (baseline/refchain.py) runs the unmodified
reference package on a BASELINE scene; this pins that its expression of the
scene (log bucket table, per-patch Philox stream) is the oracle's scene: same
counts every frame, fields equal to fp64 rounding.  Skipped where the
reference is not installed in baseline/_ref."""
import numpy as np
import pytest

from baseline import refchain

pytestmark = pytest.mark.skipif(refchain.load() is None, reason="reference not installed in baseline/_ref")


def test_refchain_scene_is_the_oracle_scene():
    from oracle import scene_ref
    from paper_2511_02852_b200 import scenes
    cfg = scenes.pr1(fft_n=64, gamma=None, spread_s=None, patches=(scenes.PatchConfig(origin=(468.0, 468.0), size=(64.0, 64.0), res=65,
                                                           margin=8.0),))
    sim = refchain.build(cfg)
    ref = scene_ref.OracleScene(cfg.scene_dict())
    for k in range(12):
        st = sim.step()
        out = ref.step()
        np.testing.assert_array_equal(st.particle_counts, out["counts"][0], err_msg=f"frame {k}")
    np.testing.assert_allclose(sim.background.height, out["height"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(sim.patches[0].surface.field.height, out["patch_heights"][0], rtol=0, atol=1e-12)
    np.testing.assert_allclose(sim.stitched_heights(), ref.composite(), rtol=0, atol=1e-12)


def test_refchain_rejects_what_the_reference_cannot_express():
    from paper_2511_02852_b200 import scenes
    assert refchain.expressible(scenes.c3()) is None
    assert refchain.expressible(scenes.pr1()) is not None          # gamma / spreading overrides
    assert refchain.expressible(scenes.c4()) is not None          # cascades
    assert refchain.expressible(scenes.c2()) is not None          # wake sources
