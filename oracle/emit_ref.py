"""Body -> water emission and patch tracking -- TEST INFRASTRUCTURE ONLY.

Restates `pkg/src/hybridsea/interaction.py:161-231` (nearest_bucket, _fan,
emit_from_motion) and `harness.py:65-66,115-123,155-167` (_snap,
_retrack_patches, the per-frame emission loop) for KINEMATIC sources: bodies
moving at a constant velocity whose displaced-volume change per frame and
mean submersion are fixed, so the energy budget rho g |dV| h_c is the same
every frame.  This is the SURVEY App. A / 8(f) form of the BASELINE wake
sources (C2 point sources, C5 ships): with a constant velocity the reference's
`buoyancy_step` reduces to `position += velocity * dt` (interaction.py:140),
and `emit_from_motion` yields ring and wake fans of fixed size.

The reference fans a wake over max(n_theta // 2, 3) directions; a source's
`wake_count` overrides that (the fixed-count emitters of C2/C5), which is
what the reference produces for a table with n_theta = 2 * count.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .particles_ref import Patch, Pool

KELVIN_HALF_ANGLE = math.radians(19.47)          # interaction.py:26


def nearest_bucket(radii: np.ndarray, radius: float) -> int:
    """interaction.py:161-163."""
    return int(np.argmin(np.abs(radii - radius)))


def fan(center_angle: float, half_angle: float, count: int) -> np.ndarray:
    """interaction.py:166-172: `count` unit directions across +-half_angle."""
    if count == 1:
        angles = np.array([center_angle])
    else:
        angles = center_angle + np.linspace(-half_angle, half_angle, count)
    return np.stack([np.cos(angles), np.sin(angles)], axis=1)


@dataclass
class Source:
    """A kinematic emitting body (FloatingBody with fixed velocity / volume rate)."""
    position: np.ndarray          # world (2,), advanced by velocity * dt every frame
    velocity: np.ndarray          # (3,) constant
    hull_extent: float
    volume_rate: float            # dV per frame (m^3), sign selects crest / trough rings
    submersion: float             # h_c (m)
    wake_count: int = 0           # 0: the reference's max(n_theta // 2, 3)
    energy_scale: float = 1.0

    def budget(self, rho: float, g: float) -> float:
        # interaction.py:187: energy_scale * rho * g * abs(d_v) * h_c
        return self.energy_scale * rho * g * abs(self.volume_rate) * self.submersion


@dataclass
class Event:
    mode: str
    energy: float
    bucket: int


def emit(src: Source, radii: np.ndarray, n_theta: int, rho: float, g: float,
         trough_fraction: float = 1.0) -> tuple[list, Pool]:
    """emit_from_motion (interaction.py:175-231) at the source's position."""
    out = Pool()
    budget = src.budget(rho, g)
    if budget <= 0.0:
        return [], out
    v_z = abs(float(src.velocity[2]))
    v_h = float(np.hypot(src.velocity[0], src.velocity[1]))
    ring_weight = 1.0 if v_z + v_h == 0.0 else v_z / (v_z + v_h)
    sign = 1.0 if src.volume_rate >= 0.0 else -1.0
    center = np.asarray(src.position, dtype=float)[:2]
    events = []

    def spawn(energy, b, dirs, mode):
        r_b = float(radii[b])
        per = energy / len(dirs)
        amp = math.sqrt(8.0 * per / (rho * g * math.pi * r_b ** 2))
        pos = center[None, :] + src.hull_extent * dirs
        amps = np.full(len(dirs), sign * amp)
        bk = np.full(len(dirs), b, dtype=np.int32)
        out.append(Pool(pos, dirs, amps, bk, np.zeros(len(dirs))))
        if trough_fraction != 0.0:
            out.append(Pool(pos - r_b * dirs, dirs, -trough_fraction * amps, bk, np.zeros(len(dirs))))
        events.append(Event(mode, energy, b))

    e_ring = ring_weight * budget
    if e_ring > 0.0:
        b = nearest_bucket(radii, src.hull_extent)
        spawn(e_ring, b, fan(0.0, math.pi * (1.0 - 1.0 / n_theta), n_theta), "ring")
    e_wake = (1.0 - ring_weight) * budget
    if e_wake > 0.0 and v_h > 0.0:
        b = nearest_bucket(radii, src.hull_extent / 2.0)
        back = math.atan2(-src.velocity[1], -src.velocity[0])
        count = src.wake_count if src.wake_count > 0 else max(n_theta // 2, 3)
        spawn(e_wake, b, fan(back, KELVIN_HALF_ANGLE, count), "wake")
    return events, out


def contains(patch: Patch, p: np.ndarray) -> bool:
    """PatchRegion.contains, inclusive (particles.py:71-74)."""
    return bool(np.all((p >= patch.lo) & (p <= patch.hi)))


def snap(value: float, step: float) -> float:
    """harness.py:65-66."""
    return round(value / step) * step


def retrack(patch: Patch, res: int, src: Source) -> Patch:
    """_retrack_patches for one patch following `src` (harness.py:115-123)."""
    texel = patch.l1 / (res - 1)
    cx = snap(src.position[0] - patch.l1 / 2.0, texel)
    cy = snap(src.position[1] - patch.l2 / 2.0, texel)
    return Patch(cx, cy, patch.l1, patch.l2, patch.margin)


__all__ = ["KELVIN_HALF_ANGLE", "Source", "Event", "nearest_bucket", "fan", "emit", "contains", "snap", "retrack"]
