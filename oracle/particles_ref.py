"""Wave-particle pool, boundary injection and advection -- TEST INFRASTRUCTURE ONLY.

Restates `pkg/src/hybridsea/particles.py` (reference).  The pool is kept in
the reference's order (stable birth order, `particles.py:167-178`): survivors,
then each frame's new crests (bucket-major, side-minor, group, member), then
the new troughs in the same order (`particles.py:251-253,296-299`).

Integer-exact pieces are written with the reference's fp64 operation order
so counts, keep decisions and positions are bit-identical:
  ledger  acc += half_rate; n = floor(acc); acc -= n        (:243-245)
  advect  pos += dir * (c * dt); keep = dx^2 + dy^2 <= r^2   (:312-320)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .spectrum_ref import Buckets, Params, s1d

INWARD = np.array([[1.0, 0.0], [-1.0, 0.0], [0.0, 1.0], [0.0, -1.0]])  # W E S N (:38-40)


@dataclass(frozen=True)
class Patch:
    """Axis-aligned patch rectangle (particles.py:43-74)."""
    x0: float
    y0: float
    l1: float
    l2: float
    margin: float

    @property
    def lo(self) -> np.ndarray:
        return np.array([self.x0, self.y0], dtype=float)

    @property
    def hi(self) -> np.ndarray:
        return self.lo + np.array([self.l1, self.l2])

    def side(self, s: int) -> float:
        return self.l2 if s < 2 else self.l1


@dataclass
class Pool:
    """SoA particle pool in reference order."""
    pos: np.ndarray = field(default_factory=lambda: np.zeros((0, 2)))
    dir: np.ndarray = field(default_factory=lambda: np.zeros((0, 2)))
    amp: np.ndarray = field(default_factory=lambda: np.zeros(0))
    bucket: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int32))
    birth: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def __len__(self) -> int:
        return len(self.amp)

    def append(self, other: "Pool") -> None:
        self.pos = np.concatenate([self.pos, other.pos])
        self.dir = np.concatenate([self.dir, other.dir])
        self.amp = np.concatenate([self.amp, other.amp])
        self.bucket = np.concatenate([self.bucket, other.bucket]).astype(np.int32)
        self.birth = np.concatenate([self.birth, other.birth])

    def take(self, mask: np.ndarray) -> "Pool":
        return Pool(self.pos[mask], self.dir[mask], self.amp[mask], self.bucket[mask],
                    self.birth[mask])

    def bucket_segments(self, n_buckets: int) -> list["Pool"]:
        """Per-bucket subsequences in pool order (the GPU pool layout)."""
        return [self.take(self.bucket == b) for b in range(n_buckets)]

    def counts(self, n_buckets: int) -> np.ndarray:
        return np.bincount(self.bucket, minlength=n_buckets)


@dataclass
class Ledger:
    """Quota accumulators + energy books (particles.py:187-202)."""
    n: int
    rho: float = 1000.0
    acc: np.ndarray = None
    groups: np.ndarray = None
    e_in: np.ndarray = None
    e_out: np.ndarray = None

    def __post_init__(self):
        self.acc = np.zeros((self.n, 4))
        self.groups = np.zeros(self.n, dtype=np.int64)
        self.e_in = np.zeros(self.n)
        self.e_out = np.zeros(self.n)


def energy(rho: float, g: float, amp, radius):
    """rho g A^2 pi r^2 / 8 (particles.py:205-207)."""
    return 0.125 * rho * g * np.asarray(amp) ** 2 * math.pi * np.asarray(radius) ** 2


def half_rates(patch: Patch, bk: Buckets, dt: float, g: float) -> np.ndarray:
    """Per (bucket, side) group quota per step: half of 4 L dt w^3/(pi^3 g)
    (particles.py:237-241)."""
    hr = np.empty((bk.n, 4))
    for s in range(4):
        hr[:, s] = 0.5 * (4.0 * patch.side(s) * dt * bk.omega ** 3 / (math.pi ** 3 * g))
    return hr


def inject(patch: Patch, bk: Buckets, p: Params, mean_dir: float, led: Ledger, dt: float,
           rng: np.random.Generator, t: float = 0.0, beta: float = 1.0) -> Pool:
    """Advance quotas and emit due groups (particles.py:219-300)."""
    if dt <= 0:
        raise ValueError("dt must be positive")
    nb, nth = bk.n, bk.n_theta
    dth = 2.0 * math.pi / nth
    led.acc += half_rates(patch, bk, dt, p.g)
    n_emit = np.floor(led.acc).astype(np.int64)
    led.acc -= n_emit
    g_tot = int(n_emit.sum())
    if g_tot == 0:
        return Pool()
    cell = np.arange(nb * 4)
    gb = np.repeat(cell // 4, n_emit.ravel())
    gs = np.repeat(cell % 4, n_emit.ravel())
    led.groups += np.bincount(gb, minlength=nb)

    th0 = -math.pi + (np.arange(nth) + 0.5) * dth
    jit = rng.uniform(-0.5 * dth, 0.5 * dth, size=g_tot)
    th = th0[None, :] + jit[:, None]
    sdir = bk.spread_c[gb][:, None] * np.abs(np.cos(0.5 * th)) ** (2.0 * bk.spread_s[gb][:, None])
    amp = np.sqrt(2.0 * s1d(p, bk.omega)[gb][:, None] * sdir * bk.width[gb][:, None] * dth)
    thw = th + mean_dir
    dx, dy = np.cos(thw), np.sin(thw)
    inw = INWARD[gs]
    flow_in = dx * inw[:, 0][:, None] + dy * inw[:, 1][:, None] > 0.0
    side = np.where(flow_in, gs[:, None], gs[:, None] ^ 1).ravel()

    u = rng.uniform(0.0, 1.0, size=(g_tot, nth)).ravel()
    px = np.where(side == 0, patch.x0, np.where(side == 1, patch.x0 + patch.l1, 0.0))
    py = np.where(side == 2, patch.y0, np.where(side == 3, patch.y0 + patch.l2, 0.0))
    along_y = side < 2
    py = np.where(along_y, patch.y0 + u * patch.l2, py)
    px = np.where(along_y, px, patch.x0 + u * patch.l1)

    pos = np.stack([px, py], axis=1)
    d2 = np.stack([dx.ravel(), dy.ravel()], axis=1)
    a2 = amp.ravel()
    b2 = np.repeat(gb, nth).astype(np.int32)
    r2 = bk.radius[b2]
    led.e_in += np.bincount(b2, weights=energy(led.rho, p.g, a2, r2), minlength=nb)

    live = a2 > 0.0
    out = Pool(pos[live], d2[live], a2[live], b2[live], np.full(int(live.sum()), t))
    if beta != 0.0:
        out.append(Pool(pos[live] - r2[live, None] * d2[live], d2[live], -beta * a2[live],
                        b2[live], np.full(int(live.sum()), t)))
    return out


def advect(pool: Pool, bk: Buckets, dt: float, patch: Patch, led: Ledger | None, g: float) -> Pool:
    """Move at c_b, cull by support-disk distance, stable compaction; returns
    the dropped set and books crest despawn energy (particles.py:303-328)."""
    if dt < 0:
        raise ValueError("dt must be nonnegative")
    if len(pool) == 0:
        return Pool()
    step = bk.speed[pool.bucket] * dt
    pos = pool.pos + pool.dir * step[:, None]
    r = bk.radius[pool.bucket]
    lo, hi = patch.lo, patch.hi
    ox = np.maximum(np.maximum(lo[0] - pos[:, 0], pos[:, 0] - hi[0]), 0.0)
    oy = np.maximum(np.maximum(lo[1] - pos[:, 1], pos[:, 1] - hi[1]), 0.0)
    keep = ox * ox + oy * oy <= r * r
    pool.pos = pos
    dropped = pool.take(~keep)
    kept = pool.take(keep)
    pool.pos, pool.dir, pool.amp, pool.bucket, pool.birth = (
        kept.pos, kept.dir, kept.amp, kept.bucket, kept.birth)
    if led is not None and len(dropped):
        e = energy(led.rho, g, np.abs(dropped.amp), bk.radius[dropped.bucket])
        crest = dropped.amp > 0.0
        led.e_out += np.bincount(dropped.bucket[crest], weights=e[crest], minlength=bk.n)
    return dropped
