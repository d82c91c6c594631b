"""CPU-only checks: the C-ABI library loads and exports every declared
symbol, the host-side mirrors (config, spectrum, layer plans) match the
reference, and the oracle-free host logic behaves."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

G = 9.81


def test_library_exports_every_header_symbol():
    from paper_2511_02852_b200 import _native
    header = open(os.path.join(ROOT, "include", "hybridsea_b200.h")).read()
    declared = set(re.findall(r"HS_API\s+[\w\s\*]+?\b(hs_\w+)\s*\(", header))
    assert declared == set(_native.EXPORTS), declared ^ set(_native.EXPORTS)
    L = _native.lib()          # also verifies every struct size against the C side
    for name in declared:
        assert hasattr(L, name)
    assert L.hs_abi_version() == 1


def test_config_roundtrip_and_errors():
    from paper_2511_02852_b200 import ConfigError, dump_config, parse_config
    text = """
    # comment
    spectrum.u10 = 10
    spectrum.gamma = 3.3
    spectrum.bucket_spacing = log
    spectrum.omega_lo = 0.5
    spectrum.omega_hi = 4
    fft.n = 256
    patch.0.origin = 10,20
    patch.0.size = 64,64
    patch.0.res = 256
    patch.0.margin = 8
    """
    cfg = parse_config(text)
    assert cfg.u10 == 10.0 and cfg.gamma == 3.3 and cfg.bucket_spacing == "log"
    assert cfg.patches[0].origin == (10.0, 20.0)
    again = parse_config(dump_config(cfg))
    assert again == cfg
    with pytest.raises(ConfigError, match="line 1"):
        parse_config("spectrum.u11 = 3")
    with pytest.raises(ConfigError):
        parse_config("fft.n = 100")
    with pytest.raises(ConfigError):
        parse_config("patch.0.margin = 80")
    with pytest.raises(ConfigError):
        parse_config("spectrum.n_omega = 40")


def test_spectrum_mirror_matches_golden(golden):
    from paper_2511_02852_b200 import build_buckets, derive_params, log_buckets
    gd = golden("spectrum.npz")
    p = derive_params(5.0, 1e4, G)
    np.testing.assert_array_equal([p.alpha, p.omega_p, p.gamma], gd["a_params"])
    for n in (8, 12, 16):
        t = build_buckets(p, n, 16)
        np.testing.assert_allclose(t.omegas, gd[f"a_eq{n}_omega"], rtol=1e-13)
        np.testing.assert_allclose(t.energies, gd[f"a_eq{n}_energy"], rtol=1e-10)
    pb = derive_params(10.0, 1e5, G, gamma=3.3, spread_s=8.0)
    t = log_buckets(pb, 0.5, 4.0, 8, 16)
    np.testing.assert_allclose(t.omegas, gd["pr1_log8_omega"], rtol=1e-14)
    np.testing.assert_allclose(t.spread_params[0], gd["pr1_log8_s"], rtol=1e-14)
    np.testing.assert_allclose(t.spread_params[1], gd["pr1_log8_c"], rtol=1e-14)
    np.testing.assert_allclose(t.energies, gd["pr1_log8_energy"], rtol=1e-10)


def test_layer_plan_mirror_matches_golden(golden):
    from paper_2511_02852_b200 import PatchRegion, derive_params, log_buckets, plan_layers
    from paper_2511_02852_b200._layout import pack_layers
    gd = golden("synth.npz")
    t = log_buckets(derive_params(10.0, 1e5, G, gamma=3.3, spread_s=8.0), 0.5, 4.0, 8, 16)
    patch = PatchRegion((100.0, 200.0), 64.0, 64.0, 8.0)
    plan = plan_layers(t, patch.l1 / 128, 129)
    np.testing.assert_array_equal(plan.factors, gd["plan_factors"])
    np.testing.assert_array_equal([k.half_width for k in plan.kernels], gd["plan_half"])
    np.testing.assert_allclose([k.gain for k in plan.kernels], gd["plan_gain"], rtol=1e-14)
    pack = pack_layers([plan], [(129, 129)])
    for L, f, k in zip(pack.layers, plan.factors, plan.kernels):
        ncx = -((128) // -f) + 1
        assert (L.f, L.H, L.pad, L.ncx, L.wx) == (f, k.half_width, k.half_width + 1, ncx, ncx + 2 * L.pad)
    # raw rows are padded to 16-byte pitches (vector splat reductions), offsets stay 16-byte aligned
    assert all(L.raw_pitch >= L.wy and L.raw_pitch % 4 == 0 and L.raw_off % 4 == 0 for L in pack.layers)
    assert pack.raw_len == sum(L.wx * L.raw_pitch for L in pack.layers)


def test_half_rates_bit_exact_with_oracle():
    from oracle import particles_ref, spectrum_ref
    from paper_2511_02852_b200 import PatchRegion, derive_params, log_buckets
    from paper_2511_02852_b200._layout import half_rates, max_groups_per_step
    p = derive_params(10.0, 1e5, G)
    t = log_buckets(p, 0.3, 6.0, 16, 2)
    patch = PatchRegion((0.0, 0.0), 256.0, 192.0, 10.0)
    hr = half_rates(patch, t.omegas, 1 / 60, G)
    bk = spectrum_ref.log_buckets(spectrum_ref.jonswap(10.0, 1e5, G), 0.3, 6.0, 16, 2)
    ref = particles_ref.half_rates(particles_ref.Patch(0.0, 0.0, 256.0, 192.0, 10.0), bk, 1 / 60, G)
    np.testing.assert_array_equal(hr, ref)
    # the staging bound holds for any accumulator state
    acc = np.nextafter(np.ones_like(hr), 0)
    assert np.floor(acc + hr).sum() <= max_groups_per_step(hr)


def test_presets_validate():
    from paper_2511_02852_b200 import scenes
    from paper_2511_02852_b200.coupling import validate_patches
    from paper_2511_02852_b200.particles import PatchRegion
    for name, mk in scenes.PRESETS.items():
        cfg = mk()
        regs = [PatchRegion(p.origin, p.size[0], p.size[1], p.margin) for p in cfg.patches]
        validate_patches(regs)
        for r in regs:
            assert 0 <= r.min_corner.min() and r.max_corner.max() <= cfg.fft_domain


def test_population_estimate_brackets_c3():
    """The pool-capacity estimate must cover the measured C3 steady state
    (858k live at n_theta 2) with the 1.6x headroom."""
    from paper_2511_02852_b200 import scenes
    from paper_2511_02852_b200.harness import build_table, estimate_population
    from paper_2511_02852_b200.particles import PatchRegion
    from paper_2511_02852_b200.spectrum import derive_params
    cfg = scenes.c3()
    t = build_table(cfg, derive_params(cfg.u10, cfg.fetch, cfg.g))
    est = estimate_population(t, PatchRegion(cfg.patches[0].origin, 256.0, 256.0, 10.0), 1.0)
    assert 858_000 < 1.6 * est < 4_000_000


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2511_02852_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f


def test_cascade_bands_partition_k():
    """fft.cascades: disjoint, contiguous |k| bands, largest tile first,
    boundaries at half the larger tile's Nyquist (config.cascade_bands),
    identical to the oracle's scene definition."""
    import math
    from oracle.scene_ref import cascade_bands as ref_bands
    from paper_2511_02852_b200.config import cascade_bands
    b = cascade_bands((250.0, 4000.0, 1000.0), 512)
    assert [t[0] for t in b] == [4000.0, 1000.0, 250.0]
    assert b[0][1] == 0.0 and math.isinf(b[-1][2])
    for (_, _, hi), (_, lo, _) in zip(b, b[1:]):
        assert hi == lo
    assert b[0][2] == math.pi * 512 / (2 * 4000.0)
    assert b == ref_bands((250.0, 4000.0, 1000.0), 512)


def test_single_cascade_scene_equals_plain_scene():
    """A one-tile cascade list is the plain background (oracle)."""
    import numpy as np
    from dataclasses import replace
    from oracle import scene_ref
    from paper_2511_02852_b200 import scenes
    cfg = scenes.pr1(fft_n=64)
    a = scene_ref.OracleScene(cfg.scene_dict())
    b = scene_ref.OracleScene(replace(cfg, fft_cascades=(cfg.fft_domain,)).scene_dict())
    oa, ob = a.step(), b.step()
    np.testing.assert_array_equal(oa["height"], ob["height"])
    np.testing.assert_array_equal(oa["blend_heights"][0], ob["blend_heights"][0])


def test_deterministic_mode_config_and_fixed_point_decoding():
    """device.deterministic parses / round-trips, and the host decodes the
    int64 fixed-point accumulators (HS_FIXED_* in the header) exactly."""
    from paper_2511_02852_b200 import _native as N
    from paper_2511_02852_b200 import dump_config, parse_config
    from paper_2511_02852_b200.harness import fixed_to_double
    cfg = parse_config("device.deterministic = true\nfft.n = 64\n")
    assert cfg.deterministic and parse_config(dump_config(cfg)) == cfg
    assert not parse_config("fft.n = 64\n").deterministic
    header = open(os.path.join(ROOT, "include", "hybridsea_b200.h")).read()
    for name in ("HS_FIXED_SPLAT_BITS", "HS_FIXED_ENERGY_BITS", "HS_FIXED_SUMSQ_BITS"):
        assert int(re.search(rf"#define {name} (\d+)", header).group(1)) == getattr(N, name)
    e = np.array([1234.5, 0.0, 3.0e6])
    fx = np.rint(e * 2.0 ** N.HS_FIXED_ENERGY_BITS).astype(np.int64)
    np.testing.assert_array_equal(fixed_to_double(fx.view(np.float64), N.HS_FIXED_ENERGY_BITS), e)


def test_device_init_workspace_sizes():
    """hs_init_workspace_bytes: positive and growing with n for the supported
    sizes, -1 outside them (no device work)."""
    from paper_2511_02852_b200 import _native as N
    L = N.lib()
    sizes = [L.hs_init_workspace_bytes(n) for n in (4, 64, 1024, 4096)]
    assert all(b > 0 for b in sizes) and sizes == sorted(sizes)
    assert L.hs_init_workspace_bytes(100) == -1 and L.hs_init_workspace_bytes(8192) == -1


def test_abi_rejects_bad_arguments_without_a_device():
    """Every entry point validates its arguments on the host before touching
    the device: bad calls return nonzero with a message in hs_last_error()
    (the ABI's error convention, include/hybridsea_b200.h), here on a CPU-only
    host."""
    import ctypes as C
    from paper_2511_02852_b200 import _native as N
    L = N.lib()

    def rejected(rc, *words):
        msg = L.hs_last_error().decode()
        assert rc != 0, msg
        assert all(w in msg for w in words), msg

    for name in ("hs_fft_evolve", "hs_inject", "hs_advect", "hs_splat", "hs_smooth", "hs_compose", "hs_sample",
                 "hs_composite", "hs_finish", "hs_advect_resident", "hs_append_resident", "hs_resident_layout",
                 "hs_track", "hs_emit", "hs_bodies", "hs_init_h0"):
        rejected(getattr(L, name)(None, None), name)
    rejected(L.hs_fft_evolve(C.byref(N.HsFftArgs(n=100)), None), "power of two")
    rejected(L.hs_init_h0(C.byref(N.HsInitArgs(n=100)), None), "power of two")
    rejected(L.hs_compose(C.byref(N.HsComposeArgs(nb=0)), None), "nb")
    rejected(L.hs_clear(None, N.i64(-1), None), "hs_clear")
    rejected(L.hs_fixed_to_float(None, None, N.i64(16), N.i32(0), None), "hs_fixed_to_float")
