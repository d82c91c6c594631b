"""The device init's Gaussian stream model, on the CPU: numpy's
default_rng(seed).standard_normal is PCG64 XSL-RR 128/64 feeding a 52-bit
256-strip ziggurat (reference fft_background.py:136-137 draws h0 with it).
`oracle.normal_ref` restates both with the constructed strip tables of
`normal_draws.py`; this pins the restatement against numpy itself: the raw
stream bit-exact, the attempt chain identical (same accept decisions, same
consumption) and every draw within 2e-14 relative (the tables are
constructed, not numpy's own, and agree to a few ulp)."""
import numpy as np
import pytest

from oracle import normal_ref
from paper_2511_02852_b200.normal_draws import pcg64_seed_state, ziggurat_r, ziggurat_tables


@pytest.mark.parametrize("seed", [0, 3, 2**40 + 17])
def test_pcg64_raw_stream_bit_exact(seed):
    np.testing.assert_array_equal(normal_ref.pcg64_raw(seed, 2000), np.random.PCG64(seed).random_raw(2000))


def test_seed_state_is_default_rng():
    s, inc = pcg64_seed_state(5)
    st = np.random.default_rng(5).bit_generator.state["state"]
    assert (s, inc) == (st["state"], st["inc"])
    assert inc & 1 == 1


def test_ziggurat_tables_shape():
    k, w, f = ziggurat_tables()
    assert k.dtype == np.uint64 and w.dtype == np.float64 and f.dtype == np.float64
    r = ziggurat_r()
    # x_i = w_i 2^52 increases to r; f_i = exp(-x_i^2 / 2) decreases from 1
    x = w[1:] * 2.0 ** 52
    assert np.all(np.diff(x) > 0) and abs(x[-1] - r) < 1e-15 * r
    assert f[0] == 1.0 and np.all(np.diff(f[1:]) < 0)
    np.testing.assert_allclose(f[1:], np.exp(-0.5 * x * x), rtol=1e-14)
    assert int(k[1]) == 0 and np.all(k[2:] < np.uint64(2 ** 52))
    # equal-area strips: x_i (f(x_{i-1}) - f(x_i)) = v for the inner strips
    v = x[1:] * (f[1:-1] - f[2:])
    np.testing.assert_allclose(v, v[0], rtol=1e-12)


@pytest.mark.parametrize("seed", [0, 7, 123456789])
def test_standard_normal_stream_matches_numpy(seed):
    n = 120_000
    got = normal_ref.standard_normal(seed, n)
    ref = np.random.default_rng(seed).standard_normal(n)
    rel = np.abs(got - ref) / np.abs(ref)
    assert rel.max() <= 2e-14, f"max rel {rel.max():.3e}"
    assert np.all(np.sign(got) == np.sign(ref))


def test_stream_covers_tail_and_wedge():
    """The sample above exercises the slow paths: count them on one stream."""
    raws = np.random.PCG64(11).random_raw(60_000)
    kinds = {1: 0, 2: 0, "tail": 0}
    p = 0
    while p < 50_000:
        c, ok, v = normal_ref.attempt(raws, p)
        if c == 1:
            kinds[1] += 1
        elif abs(v) > ziggurat_r():
            kinds["tail"] += 1
        else:
            kinds[2] += 1
        p += c
    assert kinds[2] > 50 and kinds["tail"] > 3
