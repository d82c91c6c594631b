"""The function-level API as a drop-in (B200): the numpy face
(`paper_2511_02852_b200.host`), the texel-exact LayerStack path
(patch_synthesis.py:133-224), injection from the reference's own generator
(default_rng / PCG64, harness.py:79), birth times (particles.py:128-129,
296-299), the fp64 helpers spectral_at / convolve1d_zero, and the ctypes
stub INTEGRATION.md shows a maintainer -- executed as written."""
import ctypes
import math
import os
import re
import sys

import numpy as np
import pytest

from oracle import ocean_ref, particles_ref, spectrum_ref, synth_ref

pytestmark = pytest.mark.gpu
G = 9.81
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _pr1_objects():
    from paper_2511_02852_b200 import DirectionalSpectrum, PatchRegion, derive_params, log_buckets
    p = derive_params(10.0, 1e5, G, gamma=3.3, spread_s=8.0)
    return DirectionalSpectrum(p, 0.3), log_buckets(p, 0.5, 4.0, 8, 16), PatchRegion((100.0, 200.0), 64.0, 64.0, 8.0)


def _pr1_oracle():
    p = spectrum_ref.jonswap(10.0, 1e5, G, gamma=3.3, spread_s=8.0)
    return p, spectrum_ref.log_buckets(p, 0.5, 4.0, 8, 16), particles_ref.Patch(100.0, 200.0, 64.0, 64.0, 8.0)


def test_inject_from_default_rng_pcg64_matches_the_oracle(cuda):
    """The reference's generator (default_rng, PCG64) drives the device
    injection: the kernel jumps the 128-bit LCG per draw.  Counts, buckets and
    order exact, positions to 1e-9 m, and the host generator left exactly
    where the reference's calls leave it."""
    from paper_2511_02852_b200 import InjectionLedger, inject
    sp, table, patch = _pr1_objects()
    p, bk, pr = _pr1_oracle()
    led, ref_led = InjectionLedger(8, device=cuda), particles_ref.Ledger(8)
    rng, ref_rng = np.random.default_rng(42), np.random.default_rng(42)
    total = 0
    for k in range(40):
        new = inject(patch, table, sp, led, 1.0 / 60.0, rng, t=k / 60.0)
        ref = particles_ref.inject(pr, bk, p, 0.3, ref_led, 1.0 / 60.0, ref_rng, t=k / 60.0)
        assert len(new) == len(ref)
        np.testing.assert_array_equal(new.counts, ref.counts(8))
        for b in range(8):
            m = ref.bucket == b
            seg = new.segment(b)
            np.testing.assert_allclose(seg["pos"], ref.pos[m], rtol=0, atol=1e-9)
            np.testing.assert_array_equal(seg["birth"], ref.birth[m])
        total += len(new)
    assert total > 100
    np.testing.assert_array_equal(led.accumulators, ref_led.acc)
    np.testing.assert_array_equal(rng.bit_generator.random_raw(3), ref_rng.bit_generator.random_raw(3))


def test_birth_times_through_inject_and_advect(cuda):
    from paper_2511_02852_b200 import InjectionLedger, ParticleSet, WaveParticle, advect, inject
    sp, table, patch = _pr1_objects()
    led = InjectionLedger(8, device=cuda)
    rng = np.random.Generator(np.random.Philox(key=[7, 0]))
    pool = ParticleSet(n_buckets=8, device=cuda)
    for k in range(30):
        pool.extend(inject(patch, table, sp, led, 0.05, rng, t=0.05 * k))
        advect(pool, table, 0.05, patch, led, g=G)
    bt = pool.birth_times
    assert len(bt) == len(pool) > 0 and np.all(np.isin(bt, 0.05 * np.arange(30)))
    # a host-built set round-trips its values exactly (test_particles.py:270-275)
    host = ParticleSet(2)
    host.append(WaveParticle(np.array([1.0, 2.0]), np.array([0.0, 1.0]), -0.3, 7, 1.5))
    q = next(iter(host))
    assert q.amplitude == -0.3 and q.bucket == 7 and q.birth_time == 1.5


def test_layer_stack_accumulate_and_smooth_and_sum(cuda):
    """Texel-exact path: splat layers readable as numpy (a particle on a texel
    centre lands on that texel only), and smooth_and_sum equals synthesize
    with an all-factor-1 plan and the fp64 oracle within the north_star bar."""
    from paper_2511_02852_b200 import LayerStack, ParticleSet, accumulate, build_kernels, smooth_and_sum, synthesize
    sp, table, patch = _pr1_objects()
    kernels = build_kernels(table, 64.0 / 128)
    stack = LayerStack(patch, 129, kernels)
    one = ParticleSet(1)
    one.append_arrays(np.array([[100.0 + 25 * 0.5, 200.0 + 75 * 0.5]]), np.array([[1.0, 0.0]]), [0.375], [5])
    accumulate(one, patch, stack)
    v = stack.layer_view(5)
    assert v[25, 75] == 0.375 and np.count_nonzero(v) == 1 and stack.clamped_splats == 0
    stack.clear()
    rng = np.random.default_rng(3)
    n = 3000
    pos = rng.uniform([90.0, 190.0], [174.0, 274.0], size=(n, 2))
    ang = rng.uniform(0, 2 * np.pi, n)
    d = np.stack([np.cos(ang), np.sin(ang)], 1)
    amp, b = rng.normal(0, 0.1, n), rng.integers(0, 8, n)
    ps = ParticleSet.from_arrays(pos, d, amp, b, 8, device=cuda)
    accumulate(ps, patch, stack)
    h = smooth_and_sum(stack).double().cpu().numpy()
    h2, c2 = synthesize(ps, patch, 129, list(kernels))
    assert stack.clamped_splats == c2
    np.testing.assert_allclose(h, h2.double().cpu().numpy(), rtol=0, atol=1e-6 * np.abs(h).max())
    p, bk, pr = _pr1_oracle()
    pool = particles_ref.Pool(pos, d, amp, b.astype(np.int32), np.zeros(n))
    ref, _ = synth_ref.synthesize(pool, pr, 129, synth_ref.plan(bk, 64.0 / 128, 129, adaptive=False))
    hs = 4.0 * np.sqrt(np.mean(ref ** 2))
    assert np.abs(h - ref).max() <= 1e-4 * hs
    assert np.sqrt(np.sum((h - ref) ** 2) / np.sum(ref ** 2)) <= 1e-5


def test_fp64_helpers(cuda):
    from paper_2511_02852_b200 import DirectionalSpectrum, derive_params, init_fft
    from paper_2511_02852_b200.fft_background import spectral_at
    from paper_2511_02852_b200.patch_synthesis import convolve1d_zero, raised_cosine_taps, smooth_layer
    st = init_fft(DirectionalSpectrum(derive_params(10.0, 1e5, G), 0.4), 64, 500.0, seed=5, device=cuda)
    for t in (0.0, 12.75, 1000.0):
        want = ocean_ref.rotated_spectrum(st.h0, 500.0, G, t)
        np.testing.assert_allclose(spectral_at(st, t), want, rtol=0, atol=1e-12 * np.abs(want).max())
    a = np.random.default_rng(1).normal(size=(5, 33, 7))
    taps = raised_cosine_taps(6)
    for ax in range(3):
        if a.shape[ax] >= 13:
            np.testing.assert_allclose(convolve1d_zero(a, taps, ax), synth_ref.smooth_axis_direct(a, taps, ax),
                                       rtol=0, atol=1e-13)
    from paper_2511_02852_b200 import SmoothingKernel
    k = SmoothingKernel(taps=taps, half_width=6, gain=1.0)
    layer = a[0, :, :]
    layer = np.random.default_rng(2).normal(size=(40, 30))
    np.testing.assert_allclose(smooth_layer(layer, k),
                               synth_ref.smooth_axis_direct(synth_ref.smooth_axis_direct(layer, taps, 0), taps, 1),
                               rtol=0, atol=1e-13)


def test_host_face_returns_the_reference_types(cuda):
    """`paper_2511_02852_b200.host`: numpy HeightField / samples / heights,
    values within the north_star bar of the fp64 oracle."""
    import paper_2511_02852_b200.host as hybridsea
    sp = hybridsea.DirectionalSpectrum(hybridsea.derive_params(10.0, 1e5, G), 0.2)
    st = hybridsea.init_fft(sp, 128, 1000.0, seed=3, choppiness=1.2)
    f = hybridsea.evolve_and_synthesize(st, 37.5)
    assert isinstance(f.height, np.ndarray) and f.height.dtype == np.float64
    h, dx, dy, nrm = ocean_ref.evolve(st.h0, 1000.0, G, 37.5, 1.2)
    hs = 4.0 * np.sqrt(np.mean(h ** 2))
    assert np.abs(f.height - h).max() <= 1e-4 * hs
    np.testing.assert_allclose(f.normal, nrm, atol=5e-5)
    f.validate()
    pts = np.array([[10.0, 20.0], [999.0, 3.0]])
    sh, sn = hybridsea.SurfaceSampler(f, []).sample(pts)
    assert isinstance(sh, np.ndarray) and sh.shape == (2,) and sn.shape == (2, 3)
    rh, _ = ocean_ref.sample_periodic(h, nrm, np.zeros(2), 1000.0 / 128, pts)
    np.testing.assert_allclose(sh, rh, atol=1e-4 * hs)


def test_integration_stub_runs_as_written(cuda):
    """The ctypes binding INTEGRATION.md shows a reference maintainer,
    extracted from the document and executed: it must match the oracle."""
    from paper_2511_02852_b200 import DirectionalSpectrum, derive_params, init_fft
    from paper_2511_02852_b200 import _native as N
    import paper_2511_02852_b200.host as face
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    m = re.search(r"```python\n(# hybridsea/_b200\.py.*?)```", doc, re.S)
    assert m, "stub not found in INTEGRATION.md"
    code = m.group(1).replace("/path/to/paper_2511_02852_b200/_lib/libhybridsea_b200.so", N.LIB_PATH)
    saved = {k: sys.modules.get(k) for k in ("hybridsea", "hybridsea.fft_background")}
    sys.modules["hybridsea"], sys.modules["hybridsea.fft_background"] = face, face.fft_background
    try:
        ns = {}
        exec(compile(code, "INTEGRATION.md", "exec"), ns)
        assert ctypes.sizeof(ns["HsFftArgs"]) == ctypes.sizeof(N.HsFftArgs), "stub struct out of date"
        st = init_fft(DirectionalSpectrum(derive_params(10.0, 1e5, G), 0.0), 64, 500.0, seed=0, choppiness=1.0,
                      device=cuda)
        f = ns["evolve_and_synthesize"](st, 12.75)
    finally:
        for k, v in saved.items():
            if v is None:
                sys.modules.pop(k, None)
            else:
                sys.modules[k] = v
    h, dx, dy, nrm = ocean_ref.evolve(st.h0, 500.0, G, 12.75, 1.0)
    hs = 4.0 * np.sqrt(np.mean(h ** 2))
    assert np.abs(f.height - h).max() <= 1e-4 * hs
    assert np.abs(f.displacement[..., 0] - dx).max() <= 1e-4 * hs
    assert not math.isnan(float(f.normal.sum()))


def test_layer_groups_fold_equal_factor_layers(cuda, monkeypatch):
    """C3's plan has five f=63 layers: hs_smooth folds them into one crop
    (HsLayer.group, tickets) that the compose upsamples once.  Heights equal
    the ungrouped path to fp32 reordering, repeat runs are bitwise identical
    (the tickets re-arm), and the oracle bar holds."""
    import torch
    from bench import scene_config
    from paper_2511_02852_b200 import ParticleSet, PatchRegion, _layout, synthesize
    from paper_2511_02852_b200 import _native as N
    from paper_2511_02852_b200 import harness as Hm
    from paper_2511_02852_b200._layout import stream_ptr
    from paper_2511_02852_b200.patch_synthesis import SynthWorkspace, plan_layers
    cfg, _, _, _ = scene_config("C3", 0, 1)
    params = Hm.derive_params(cfg.u10, cfg.fetch, cfg.g, gamma=cfg.gamma, spread_s=cfg.spread_s)
    table = Hm.build_table(cfg, params)
    res = 257
    patch = PatchRegion((0.0, 0.0), 256.0, 256.0, 10.0)
    plan = plan_layers(table, 256.0 / (res - 1), res, convention=cfg.amplitude_convention,
                       trough_fraction=cfg.trough_fraction)
    assert len(set(plan.factors)) < len(plan.factors)
    rng = np.random.default_rng(11)
    n = 100000
    pos = rng.uniform(-5.0, 261.0, size=(n, 2))
    ang = rng.uniform(0, 2 * np.pi, n)
    d = np.stack([np.cos(ang), np.sin(ang)], 1)
    amp, b = rng.normal(0, 0.05, n), rng.integers(0, table.n_omega, n)
    ps = ParticleSet.from_arrays(pos, d, amp, b, table.n_omega, device=cuda)
    ws = SynthWorkspace([patch], [res], [plan], cuda)
    assert any(L.group > 1 for L in ws.pack.layers) and ws.pack.n_tickets > 0
    for _ in range(2):                            # the kernel re-arms its tickets
        ws.raw.zero_()
        N.call("hs_smooth", ws.smooth_args(), stream_ptr())
        torch.cuda.synchronize()
        assert int(ws.tickets.count_nonzero()) == 0
    h1, _ = synthesize(ps, patch, res, plan)
    monkeypatch.setattr(_layout, "GROUP_LAYERS", False)
    h0, _ = synthesize(ps, patch, res, plan)
    h0, h1 = h0.double().cpu().numpy(), h1.double().cpu().numpy()
    np.testing.assert_allclose(h1, h0, rtol=0, atol=2e-6 * np.abs(h0).max())
    pool = particles_ref.Pool(pos, d, amp, b.astype(np.int32), np.zeros(n))
    opl = synth_ref.Plan(tuple(synth_ref.Kernel(np.asarray(k.taps, np.float64), k.half_width, float(k.gain))
                               for k in plan.kernels), tuple(plan.factors))
    ref, _ = synth_ref.synthesize(pool, particles_ref.Patch(0.0, 0.0, 256.0, 256.0, 10.0), res, opl)
    hs = 4.0 * np.sqrt(np.mean(ref ** 2))
    assert np.abs(h1 - ref).max() <= 1e-4 * hs
