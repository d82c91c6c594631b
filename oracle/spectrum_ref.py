"""JONSWAP x cos-2s spectrum and bucket tables -- TEST INFRASTRUCTURE ONLY.

Restates `pkg/src/hybridsea/spectrum.py` (reference) as plain functions over a
small parameter record.  Everything is fp64.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# sampled band as multiples of omega_p  (spectrum.py:40-41)
BAND = (0.5, 2.5)
PARTITION_INTERVALS = 8192          # spectrum.py:197


@dataclass(frozen=True)
class Params:
    u10: float
    fetch: float
    g: float
    alpha: float
    omega_p: float
    gamma: float
    sigma_low: float = 0.07
    sigma_high: float = 0.09
    # optional constant spreading exponent (App. A knob; None = Mitsuyasu)
    spread_s: float | None = None


def jonswap(u10: float, fetch: float, g: float = 9.81, gamma: float | None = None,
            spread_s: float | None = None) -> Params:
    """Wind/fetch parameterisation (spectrum.py:88-105); gamma may be pinned."""
    if u10 <= 0 or fetch <= 0 or g <= 0:
        raise ValueError("u10, fetch and g must be positive")
    a = 0.076 * (u10 ** 2 / (fetch * g)) ** 0.22
    wp = 22.0 * (g ** 2 / (u10 * fetch)) ** (1.0 / 3.0)
    gm = 7.0 * (g * fetch / u10 ** 2) ** (-0.142) if gamma is None else float(gamma)
    return Params(u10, fetch, g, a, wp, gm, spread_s=spread_s)


def s1d(p: Params, w):
    """S_J(omega) (spectrum.py:108-121)."""
    w = np.asarray(w, dtype=float)
    if np.any(w <= 0.0):
        raise ValueError("omega must be positive")
    wp = p.omega_p
    sig = np.where(w <= wp, p.sigma_low, p.sigma_high)
    peak = np.exp(-((w - wp) ** 2) / (2.0 * sig ** 2 * wp ** 2))
    val = p.alpha * p.g ** 2 * w ** -5.0 * np.exp(-1.25 * (wp / w) ** 4) * p.gamma ** peak
    return val if val.ndim else float(val)


def spread_exponent(p: Params, w: float) -> float:
    """s(omega) = 16 (omega/omega_p)^mu (spectrum.py:124-127), or the pinned s."""
    if p.spread_s is not None:
        return float(p.spread_s)
    mu = 5.0 if w <= p.omega_p else -2.5
    return 16.0 * (w / p.omega_p) ** mu


def spread_norm(s: float) -> float:
    """C(s) = Gamma(s+1)/Gamma(s+1/2)/(2 sqrt(pi)) (spectrum.py:130-132)."""
    return math.exp(math.lgamma(s + 1.0) - math.lgamma(s + 0.5)) / (2.0 * math.sqrt(math.pi))


def dir_density(p: Params, w, theta):
    """Vectorised S(omega) C(s) |cos(theta/2)|^{2s} (fft_background.py:77-87,
    spectrum.py:141-154); theta relative to the mean direction."""
    w = np.asarray(w, dtype=float)
    th = np.arctan2(np.sin(theta), np.cos(theta))
    if p.spread_s is None:
        s = 16.0 * (w / p.omega_p) ** np.where(w <= p.omega_p, 5.0, -2.5)
    else:
        s = np.full(w.shape, float(p.spread_s))
    lg = np.vectorize(math.lgamma, otypes=[float])
    c = np.exp(lg(s + 1.0) - lg(s + 0.5)) / (2.0 * math.sqrt(math.pi))
    return s1d(p, w) * c * np.abs(np.cos(0.5 * th)) ** (2.0 * s)


def band_integral(p: Params, lo: float, hi: float, base: int = 4096, rtol: float = 1e-8) -> float:
    """Grid-doubling trapezoid of S_J (spectrum.py:162-184)."""
    if hi <= lo:
        return 0.0
    n, prev = base, None
    for _ in range(8):
        w = np.linspace(lo, hi, n + 1)
        est = float(np.trapezoid(s1d(p, w), w))
        if prev is not None and abs(est - prev) <= rtol * max(abs(est), 1e-300):
            return est
        prev, n = est, 2 * n
    return prev


@dataclass(frozen=True)
class Buckets:
    """Per-bucket constants as arrays (spectrum.py:200-257)."""
    omega: np.ndarray
    width: np.ndarray
    lo: np.ndarray
    hi: np.ndarray
    radius: np.ndarray
    speed: np.ndarray
    energy: np.ndarray
    spread_s: np.ndarray
    spread_c: np.ndarray
    n_theta: int

    @property
    def n(self) -> int:
        return len(self.omega)


def _bucket_record(p: Params, edges: np.ndarray, reps: np.ndarray, n_theta: int,
                   energies: np.ndarray) -> Buckets:
    s = np.array([spread_exponent(p, float(w)) for w in reps])
    return Buckets(omega=reps.astype(float), width=np.diff(edges), lo=edges[:-1].copy(),
                   hi=edges[1:].copy(), radius=np.array([math.pi * p.g / w ** 2 for w in reps]),
                   speed=np.array([p.g / w for w in reps]), energy=energies,
                   spread_s=s, spread_c=np.array([spread_norm(float(x)) for x in s]),
                   n_theta=int(n_theta))


def equal_energy_buckets(p: Params, n_omega: int, n_theta: int) -> Buckets:
    """Equal-energy partition of [0.5, 2.5] omega_p with energy centroids
    (spectrum.py:260-307)."""
    lo, hi = BAND[0] * p.omega_p, BAND[1] * p.omega_p
    w = np.linspace(lo, hi, PARTITION_INTERVALS + 1)
    sv = s1d(p, w)
    cum = np.concatenate([[0.0], np.cumsum(0.5 * (sv[1:] + sv[:-1]) * np.diff(w))])
    edges = np.interp(np.linspace(0.0, float(cum[-1]), n_omega + 1), cum, w)
    edges[0], edges[-1] = lo, hi
    reps, ens = [], []
    for a, b in zip(edges[:-1], edges[1:]):
        wi = np.linspace(a, b, 2049)
        si = s1d(p, wi)
        den = float(np.trapezoid(si, wi))
        reps.append(float(np.trapezoid(wi * si, wi)) / den if den > 0 else 0.5 * (a + b))
        ens.append(band_integral(p, float(a), float(b), base=2048))
    return _bucket_record(p, edges, np.array(reps), n_theta, np.array(ens))


def log_buckets(p: Params, w_lo: float, w_hi: float, n_omega: int, n_theta: int) -> Buckets:
    """Log-spaced buckets over an explicit [w_lo, w_hi] (BASELINE knob, SURVEY
    App. A): edges geomspace, representative = geometric mid, energy = band
    integral of each interval."""
    edges = np.geomspace(w_lo, w_hi, n_omega + 1)
    reps = np.sqrt(edges[:-1] * edges[1:])
    ens = np.array([band_integral(p, float(a), float(b), base=2048)
                    for a, b in zip(edges[:-1], edges[1:])])
    return _bucket_record(p, edges, reps, n_theta, ens)
