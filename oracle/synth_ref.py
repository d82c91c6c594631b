"""Per-bucket layered synthesis of a patch height grid -- TEST INFRASTRUCTURE ONLY.

Restates `pkg/src/hybridsea/patch_synthesis.py` (reference): raised-cosine
kernels with energy/peak gains (:50-90), decimation plan (:242-258), bilinear
splat into padded layers (:165-186), zero-padded separable smoothing (:93-130,
206-209), bilinear upsampling (:261-274), the streaming synthesize loop
(:277-314) and finish_field (:323-340).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .ocean_ref import normals
from .particles_ref import Patch, Pool
from .spectrum_ref import Buckets


def raised_cosine(h: int) -> np.ndarray:
    """Taps proportional to 1 + cos(pi m/(h+1)), m = -h..h, summing to 1."""
    m = np.arange(-h, h + 1)
    t = 1.0 + np.cos(math.pi * m / (h + 1))
    return t / t.sum()


def pair_energy_sum(taps: np.ndarray, shift: int, beta: float) -> float:
    """Sum of squares of a unit crest+trough bump pair, trough `shift` texels
    behind (patch_synthesis.py:57-66)."""
    w = len(taps)
    bump = np.outer(taps, taps)
    canvas = np.zeros((w + shift, w))
    canvas[:w] += bump
    if beta != 0.0:
        canvas[shift:] -= beta * bump
    return float(np.sum(canvas ** 2))


@dataclass(frozen=True)
class Kernel:
    taps: np.ndarray
    half: int
    gain: float


def kernel_for(radius: float, texel: float, convention: str = "energy", beta: float = 1.0) -> Kernel:
    """Support matched to the particle radius at this texel (:69-82)."""
    if convention not in ("energy", "peak"):
        raise ValueError(f"unknown amplitude convention {convention!r}")
    h = max(1, int(round(radius / texel)))
    taps = raised_cosine(h)
    if convention == "peak":
        gain = 1.0 / float(taps[h] ** 2)
    else:
        gain = math.sqrt((math.pi * radius ** 2 / 8.0) / (pair_energy_sum(taps, h, beta) * texel ** 2))
    return Kernel(taps, h, gain)


@dataclass(frozen=True)
class Plan:
    kernels: tuple
    factors: tuple


def plan(bk: Buckets, texel: float, res: int, convention: str = "energy", beta: float = 1.0,
         min_taps: int = 4, adaptive: bool = True) -> Plan:
    """Per-bucket decimation factor f and kernel at texel*f (:242-258)."""
    fs = []
    for r in bk.radius:
        f = max(1, int((r / texel) / min_taps)) if adaptive else 1
        if adaptive:
            f = min(f, max(1, (res - 1) // (4 * min_taps)))
        fs.append(f)
    ks = tuple(kernel_for(float(r), texel * f, convention, beta) for r, f in zip(bk.radius, fs))
    return Plan(ks, tuple(fs))


def splat(layer: np.ndarray, pad: int, gx: np.ndarray, gy: np.ndarray, amp: np.ndarray) -> int:
    """Bilinear scatter-add with border clamping; returns clamp count (:165-186)."""
    nx, ny = layer.shape
    u, v = gx + pad, gy + pad
    n_clamped = int(np.count_nonzero((u < 0) | (u > nx - 1) | (v < 0) | (v > ny - 1)))
    u = np.clip(u, 0.0, nx - 1 - 1e-9)
    v = np.clip(v, 0.0, ny - 1 - 1e-9)
    i, j = u.astype(np.int64), v.astype(np.int64)
    fu, fv = u - i, v - j
    for di, dj, w in ((0, 0, (1 - fu) * (1 - fv)), (1, 0, fu * (1 - fv)),
                      (0, 1, (1 - fu) * fv), (1, 1, fu * fv)):
        np.add.at(layer, (i + di, j + dj), amp * w)
    return n_clamped


def _window(x: np.ndarray, r: int) -> np.ndarray:
    """Zero-padded sliding sum over [i-r, i+r] along the last axis."""
    n = x.shape[-1]
    cs = np.concatenate([np.zeros(x.shape[:-1] + (1,)), np.cumsum(x, axis=-1)], axis=-1)
    idx = np.arange(n)
    return cs[..., np.minimum(idx + r + 1, n)] - cs[..., np.maximum(idx - r, 0)]


def smooth_axis(arr: np.ndarray, taps: np.ndarray, axis: int) -> np.ndarray:
    """Same-size zero-padded convolution with raised-cosine taps, O(n) via
    three demodulated window sums (:105-130): taps[m] = c (1 + cos(w0 m))."""
    n = arr.shape[axis]
    r = (len(taps) - 1) // 2
    if len(taps) > n:
        raise ValueError(f"kernel of {len(taps)} taps wider than grid axis of {n}")
    a = np.moveaxis(arr, axis, -1)
    c = float(taps[r]) / 2.0
    ph = (math.pi / (r + 1)) * np.arange(n)
    co, si = np.cos(ph), np.sin(ph)
    out = c * (_window(a, r) + co * _window(a * co, r) + si * _window(a * si, r))
    return np.moveaxis(out, -1, axis)


def smooth_axis_direct(arr: np.ndarray, taps: np.ndarray, axis: int) -> np.ndarray:
    """Direct-tap version of smooth_axis (cross-check)."""
    r = (len(taps) - 1) // 2
    a = np.moveaxis(arr, axis, -1)
    n = a.shape[-1]
    padded = np.concatenate([np.zeros(a.shape[:-1] + (r,)), a, np.zeros(a.shape[:-1] + (r,))], -1)
    out = np.zeros_like(a)
    for m in range(-r, r + 1):
        out += taps[m + r] * padded[..., r - m:r - m + n]
    return np.moveaxis(out, -1, axis)


def smooth(layer: np.ndarray, k: Kernel) -> np.ndarray:
    return smooth_axis(smooth_axis(layer, k.taps, 0), k.taps, 1)


def upsample(coarse: np.ndarray, f: int, nx: int, ny: int) -> np.ndarray:
    """Node-grid bilinear upsampling: fine i <-> coarse i/f (:261-274)."""
    if f == 1:
        return coarse[:nx, :ny]

    def lerp_axis0(a: np.ndarray, n_out: int) -> np.ndarray:
        i = np.arange(n_out)
        c, k = i // f, i % f
        w = (k / f)[:, None]
        nxt = np.minimum(c + 1, a.shape[0] - 1)
        out = a[c] * (1.0 - w) + a[nxt] * w
        return out

    ux = lerp_axis0(coarse, nx)
    return lerp_axis0(ux.T, ny).T


def grid_shape(patch: Patch, res: int) -> tuple[float, int]:
    texel = patch.l1 / (res - 1)
    return texel, int(round(patch.l2 / texel)) + 1


def synthesize(pool: Pool, patch: Patch, res: int, pl: Plan) -> tuple[np.ndarray, int]:
    """Streaming per-bucket splat + smooth + upsample + gain-sum (:277-314)."""
    if res < 2:
        raise ValueError("patch resolution must be >= 2")
    texel, ny = grid_shape(patch, res)
    heights = np.zeros((res, ny))
    clamped = 0
    if len(pool) == 0:
        return heights, clamped
    gx = (pool.pos[:, 0] - patch.x0) / texel
    gy = (pool.pos[:, 1] - patch.y0) / texel
    for b, (k, f) in enumerate(zip(pl.kernels, pl.factors)):
        sel = pool.bucket == b
        if not np.any(sel):
            continue
        pad = k.half + 1
        ncx = -((res - 1) // -f) + 1
        ncy = -((ny - 1) // -f) + 1
        layer = np.zeros((ncx + 2 * pad, ncy + 2 * pad))
        clamped += splat(layer, pad, gx[sel] / f, gy[sel] / f, pool.amp[sel])
        crop = smooth(layer, k)[pad:pad + ncx, pad:pad + ncy]
        heights += k.gain * upsample(crop, f, res, ny)
    return heights, clamped


def finish(heights: np.ndarray, patch: Patch, choppiness: float = 0.0, scale: float = 1.0):
    """Clamped-border FD normals and optional displacement -chi*scale*grad h (:323-340)."""
    if not np.all(np.isfinite(heights)):
        raise ValueError("patch heights contain non-finite values")
    spacing = patch.l1 / (heights.shape[0] - 1)
    nrm = normals(heights, spacing, periodic=False)
    if choppiness != 0.0:
        gx, gy = np.gradient(heights, spacing)
        disp = -choppiness * scale * np.stack([gx, gy], axis=-1)
    else:
        disp = np.zeros(heights.shape + (2,))
    return nrm, disp
