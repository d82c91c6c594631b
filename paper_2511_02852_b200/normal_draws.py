"""Constants for drawing the reference's Gaussian amplitudes on the device.

The reference draws h0's Gaussian pairs with `np.random.default_rng(seed)
.standard_normal((n, n, 2))` (`pkg/src/hybridsea/fft_background.py:136-137`).
numpy (un-vendored dependency, >= 2.0, `pkg/pyproject.toml:10-12`) builds
that from two published pieces which `hs_init_h0` restates on the GPU:

  * PCG64 (O'Neill 2014, "XSL-RR 128/64"): a 128-bit LCG
    s <- s * PCG_MULT + inc, output rotr64(hi(s) ^ lo(s), hi(s) >> 58) taken
    from the stepped state.  The seed -> (state, inc) map is numpy's
    SeedSequence; it runs once on the host (`pcg64_seed_state`).
  * the 256-strip Marsaglia-Tsang ziggurat in numpy's 52-bit variant: one
    uint64 per attempt, low 8 bits = strip, next bit = sign, next 52 bits =
    magnitude; fast accept if magnitude < k[strip], else a wedge test with one
    more uniform, or (strip 0) the exponential tail with two uniforms per try.

The strip tables are *constructed* here from r and the strip area v (60
digit decimal arithmetic), not copied: the x[i] recursion is Marsaglia &
Tsang's x[i-1] = sqrt(-2 ln(v / x[i] + f(x[i]))).  numpy's own tables were
generated with a slightly different precision, so the magnitudes agree to a
few ulp (relative <= 2e-14) and accept decisions to within a few counts in
2^52 -- the device draws equal the reference's to ~1e-14 relative, which
`tests/test_normal_draws.py` (CPU) and `tests/test_gpu_init.py` pin.
"""
from __future__ import annotations

from decimal import Decimal, getcontext
from functools import lru_cache

import numpy as np

PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
ZIG_R = "3.6541528853610087963519472518"      # right edge of the base strip


def pcg64_seed_state(seed: int) -> tuple[int, int]:
    """(state, inc) of `np.random.default_rng(seed)`'s PCG64 before its
    first draw (numpy's SeedSequence, host-side, once)."""
    st = np.random.PCG64(seed).state["state"]
    return int(st["state"]), int(st["inc"])


def _tail_area(x: Decimal) -> Decimal:
    """int_x^inf exp(-t^2/2) dt by the Laplace continued fraction."""
    cf = x
    for k in range(400, 0, -1):
        cf = x + Decimal(k) / cf
    return (-(x * x) / 2).exp() / cf


@lru_cache(maxsize=1)
def ziggurat_tables() -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(k uint64[256], w float64[256], f float64[256]) for the 52-bit,
    256-strip half-normal ziggurat."""
    getcontext().prec = 60
    two52 = Decimal(2) ** 52
    f = lambda x: (-(x * x) / 2).exp()  # noqa: E731
    r = Decimal(ZIG_R)
    v = r * f(r) + _tail_area(r)          # common strip area
    x = [Decimal(0)] * 256
    x[255] = r
    for i in range(255, 1, -1):
        x[i - 1] = (-2 * (v / x[i] + f(x[i])).ln()).sqrt()
    k = np.zeros(256, np.uint64)
    w = np.zeros(256, np.float64)
    fv = np.zeros(256, np.float64)
    k[0] = int(r * f(r) / v * two52)
    w[0] = float(v / f(r) / two52)
    fv[0] = 1.0
    for i in range(1, 256):
        k[i] = int(x[i - 1] / x[i] * two52) if i > 1 else 0
        w[i] = float(x[i] / two52)
        fv[i] = float(f(x[i]))
    return k, w, fv


def ziggurat_r() -> float:
    return float(Decimal(ZIG_R))


__all__ = ["PCG_MULT", "pcg64_seed_state", "ziggurat_tables", "ziggurat_r"]
