"""Periodic FFT background -- TEST INFRASTRUCTURE ONLY.

Restates `pkg/src/hybridsea/fft_background.py` (reference): initial amplitudes
(:102-146), the per-frame Hermitian rotation (:155-159), the three inverse
transforms (:181-208), periodic/clamped central-difference normals (:162-178)
and periodic bilinear sampling (:222-249).  All fp64; numpy's pocketfft is the
transform, as in the reference.
"""
from __future__ import annotations

import math

import numpy as np

from .spectrum_ref import BAND, Params, dir_density


def wavenumbers(n: int, domain: float) -> np.ndarray:
    """2 pi fftfreq(n, d = L/n) -- axis 0 is x, axis 1 is y (indexing 'ij')."""
    return 2.0 * math.pi * np.fft.fftfreq(n, d=domain / n)


def resolved_band(p: Params, n: int, domain: float, band=None) -> tuple[float, float]:
    """Sampled band clipped to the fundamental and the inscribed Nyquist
    circle (fft_background.py:90-99).  `band` overrides [0.5, 2.5] omega_p."""
    lo, hi = band if band is not None else (None, None)
    lo = BAND[0] * p.omega_p if lo is None else lo
    hi = BAND[1] * p.omega_p if hi is None else hi
    w_min = math.sqrt(p.g * (2.0 * math.pi / domain))
    w_max = math.sqrt(p.g * (math.pi * n / domain))
    return max(lo, w_min), min(hi, w_max)


def initial_amplitudes(p: Params, mean_dir: float, n: int, domain: float, seed: int,
                       band=None, kband=None) -> np.ndarray:
    """Complex Gaussian h0 with one-sided variance S (g/2w)/|k| dk^2/2 per bin
    inside the resolved band, zero elsewhere (fft_background.py:102-146).
    `kband` = (k_lo, k_hi) further keeps k_lo <= |k| < k_hi only: one cascade
    of a summed-tile background (zero h0 outside the cascade's
    band; the mirrored conjugate follows from the masked h0)."""
    if n < 2 or n & (n - 1):
        raise ValueError("n must be a power of two")
    kv = wavenumbers(n, domain)
    kx, ky = np.meshgrid(kv, kv, indexing="ij")
    kmag = np.hypot(kx, ky)
    dk = 2.0 * math.pi / domain
    w_lo, w_hi = resolved_band(p, n, domain, band)
    inside = (kmag >= (w_lo ** 2 / p.g) * (1.0 - 1e-12)) & (kmag <= (w_hi ** 2 / p.g) * (1.0 + 1e-12))
    inside[0, 0] = False
    if kband is not None:
        inside &= (kmag >= kband[0]) & (kmag < kband[1])
    ks = kmag[inside]
    om = np.sqrt(p.g * ks)
    th = np.arctan2(ky[inside], kx[inside]) - mean_dir
    var = np.zeros((n, n))
    var[inside] = dir_density(p, om, th) * (p.g / (2.0 * om)) / ks * dk * dk / 2.0
    xi = np.random.default_rng(seed).standard_normal((n, n, 2))
    h0 = np.sqrt(var / 2.0) * (xi[..., 0] + 1j * xi[..., 1])
    h0[~inside] = 0.0
    return h0


def mirror_conj(h0: np.ndarray) -> np.ndarray:
    """conj(h0(-k)) on the periodic index grid."""
    n = h0.shape[0]
    idx = (n - np.arange(n)) % n
    return np.conj(h0[idx][:, idx])


def rotated_spectrum(h0: np.ndarray, domain: float, g: float, t: float) -> np.ndarray:
    """hh = h0 e^{-i w t} + conj(h0(-k)) e^{+i w t} (fft_background.py:155-159)."""
    n = h0.shape[0]
    kv = wavenumbers(n, domain)
    kx, ky = np.meshgrid(kv, kv, indexing="ij")
    ph = np.sqrt(g * np.hypot(kx, ky)) * t
    e = np.cos(ph) - 1j * np.sin(ph)
    return h0 * e + mirror_conj(h0) * np.conj(e)


def normals(height: np.ndarray, spacing: float, periodic: bool) -> np.ndarray:
    """normalize(-dh/dx, -dh/dy, 1) by central differences; wrap-around or
    one-sided borders (fft_background.py:162-178)."""
    h = height
    if periodic:
        gx = (np.roll(h, -1, 0) - np.roll(h, 1, 0)) / (2.0 * spacing)
        gy = (np.roll(h, -1, 1) - np.roll(h, 1, 1)) / (2.0 * spacing)
    else:
        gx = np.empty_like(h)
        gy = np.empty_like(h)
        gx[1:-1] = (h[2:] - h[:-2]) / (2.0 * spacing)
        gy[:, 1:-1] = (h[:, 2:] - h[:, :-2]) / (2.0 * spacing)
        gx[0] = (h[1] - h[0]) / spacing
        gx[-1] = (h[-1] - h[-2]) / spacing
        gy[:, 0] = (h[:, 1] - h[:, 0]) / spacing
        gy[:, -1] = (h[:, -1] - h[:, -2]) / spacing
    nv = np.stack([-gx, -gy, np.ones_like(h)], axis=-1)
    return nv / np.linalg.norm(nv, axis=-1, keepdims=True)


def evolve(h0: np.ndarray, domain: float, g: float, t: float, choppiness: float):
    """(height, dx, dy, normal) of the background tile at t
    (fft_background.py:181-208): unnormalised inverse DFT (numpy ifft2 * n^2)."""
    n = h0.shape[0]
    hh = rotated_spectrum(h0, domain, g, t)
    scale = float(n * n)
    height = np.fft.ifft2(hh).real * scale
    if choppiness != 0.0:
        kv = wavenumbers(n, domain)
        kx, ky = np.meshgrid(kv, kv, indexing="ij")
        kk = np.hypot(kx, ky)
        kk[0, 0] = 1.0
        dx = np.fft.ifft2(-1j * (kx / kk) * hh).real * scale * choppiness
        dy = np.fft.ifft2(-1j * (ky / kk) * hh).real * scale * choppiness
    else:
        dx = np.zeros((n, n))
        dy = np.zeros((n, n))
    return height, dx, dy, normals(height, domain / n, periodic=True)


def sample_periodic(height: np.ndarray, normal: np.ndarray | None, origin, spacing: float,
                    pts: np.ndarray):
    """Bilinear height/normal with wrap-around (fft_background.py:222-249)."""
    n = height.shape[0]
    u = (pts[..., 0] - origin[0]) / spacing
    v = (pts[..., 1] - origin[1]) / spacing
    i0 = np.floor(u).astype(int)
    j0 = np.floor(v).astype(int)
    fu, fv = u - i0, v - j0
    i0 %= n
    j0 %= n
    i1, j1 = (i0 + 1) % n, (j0 + 1) % n
    w00, w10, w01, w11 = (1 - fu) * (1 - fv), fu * (1 - fv), (1 - fu) * fv, fu * fv
    hv = height[i0, j0] * w00 + height[i1, j0] * w10 + height[i0, j1] * w01 + height[i1, j1] * w11
    if normal is None:
        return hv, None
    nv = (normal[i0, j0] * w00[..., None] + normal[i1, j0] * w10[..., None]
          + normal[i0, j1] * w01[..., None] + normal[i1, j1] * w11[..., None])
    return hv, nv / np.linalg.norm(nv, axis=-1, keepdims=True)
