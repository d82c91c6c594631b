"""numpy's `standard_normal` on PCG64, restated -- TEST INFRASTRUCTURE ONLY.

The reference's h0 draws are `np.random.default_rng(seed).standard_normal(
(n, n, 2))` (`pkg/src/hybridsea/fft_background.py:136-137`).  numpy (>= 2.0,
un-vendored dependency of the reference, `pkg/pyproject.toml:10-12`)
implements it as PCG64 XSL-RR 128/64 (O'Neill 2014) feeding the 52-bit
256-strip Marsaglia-Tsang ziggurat.  This module restates both, with the
strip tables of `paper_2511_02852_b200.normal_draws` (constructed, not
copied), in the attempt-per-position form the GPU kernel uses:

  attempt(p) = (consumed raws, accepted?, value) for an attempt starting at
  raw position p; the draws are the accepted attempts along the chain
  p_0 = 0, p_{j+1} = p_j + consumed(p_j).

`standard_normal` is the checker of `hs_init_h0`'s draw stage and is itself
pinned against numpy (tests/test_oracle_golden.py).
"""
from __future__ import annotations

import math

import numpy as np

from paper_2511_02852_b200.normal_draws import PCG_MULT, pcg64_seed_state, ziggurat_r, ziggurat_tables

M128 = (1 << 128) - 1
M64 = (1 << 64) - 1


def pcg64_raw(seed: int, count: int) -> np.ndarray:
    """First `count` raw uint64 outputs (state stepped, then XSL-RR)."""
    s, inc = pcg64_seed_state(seed)
    out = np.empty(count, np.uint64)
    for i in range(count):
        s = (s * PCG_MULT + inc) & M128
        hi, lo = s >> 64, s & M64
        rot = hi >> 58
        x = hi ^ lo
        out[i] = ((x >> rot) | (x << ((64 - rot) & 63))) & M64
    return out


def _unit(raw) -> float:
    return (int(raw) >> 11) * (1.0 / 9007199254740992.0)


def attempt(raws: np.ndarray, p: int) -> tuple[int, bool, float]:
    """One ziggurat attempt starting at raw position p."""
    k, w, f = ziggurat_tables()
    r = int(raws[p])
    idx = r & 0xFF
    r >>= 8
    sign = r & 1
    rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
    x = rabs * float(w[idx])
    if sign:
        x = -x
    if rabs < int(k[idx]):
        return 1, True, x
    if idx == 0:                                   # exponential tail beyond r
        zr = ziggurat_r()
        q = p + 1
        while True:
            xx = -(1.0 / zr) * math.log1p(-_unit(raws[q]))
            yy = -math.log1p(-_unit(raws[q + 1]))
            q += 2
            if yy + yy > xx * xx:
                v = zr + xx
                return q - p, True, (-v if (rabs >> 8) & 1 else v)
    u = _unit(raws[p + 1])                         # wedge test
    if (float(f[idx - 1]) - float(f[idx])) * u + float(f[idx]) < math.exp(-0.5 * x * x):
        return 2, True, x
    return 2, False, 0.0


def standard_normal(seed: int, count: int) -> np.ndarray:
    raws = np.random.PCG64(seed).random_raw(int(count * 1.1) + 64)
    out = np.empty(count)
    p = j = 0
    while j < count:
        c, ok, v = attempt(raws, p)
        if ok:
            out[j] = v
            j += 1
        p += c
    return out


__all__ = ["pcg64_raw", "attempt", "standard_normal"]
