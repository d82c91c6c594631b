"""Body -> water emission for kinematic sources.

Mirror of the emission half of `hybridsea.interaction`
(`pkg/src/hybridsea/interaction.py:26,161-231`): `KELVIN_HALF_ANGLE`,
`nearest_bucket`, `_fan` and the energy split / amplitude rule of
`emit_from_motion`.  A *source* is a body moving at constant velocity with a
fixed displaced-volume change per frame (the BASELINE C2 point sources and C5
ships); everything that is constant for it -- ring / wake energy, fan
directions, amplitudes, buckets -- is evaluated here once, with the
reference's own numpy expressions, and uploaded as `HsSource` records.  The
per-frame work (moving the sources, owning patch, appending, splatting,
booking, patch retracking) runs on the device in `hs_track` / `hs_emit`
(csrc/particles.cu).
"""
from __future__ import annotations

import math

import numpy as np

from . import _native as N

KELVIN_HALF_ANGLE = math.radians(19.47)          # interaction.py:26


def nearest_bucket(table, radius: float) -> int:
    """Index of the bucket whose particle radius is closest to `radius` (interaction.py:161-163)."""
    radii = table.radii if hasattr(table, "radii") else np.asarray(table)
    return int(np.argmin(np.abs(radii - radius)))


def _fan(center_angle: float, half_angle: float, count: int) -> np.ndarray:
    """`count` unit directions spread evenly across +-half_angle (interaction.py:166-172)."""
    if count == 1:
        angles = np.array([center_angle])
    else:
        angles = center_angle + np.linspace(-half_angle, half_angle, count)
    return np.stack([np.cos(angles), np.sin(angles)], axis=1)


def source_plan(src, table, rho: float, g: float) -> dict:
    """Per-frame constants of one kinematic source: the branch energies
    (interaction.py:185-195,218-225), fans and signed crest amplitudes
    (:203-208) exactly as emit_from_motion forms them."""
    budget = src.energy_scale * rho * g * abs(src.volume_rate) * src.submersion
    vel = np.asarray(src.velocity, dtype=float)
    v_z = abs(float(vel[2]))
    v_h = float(np.hypot(vel[0], vel[1]))
    ring_weight = 1.0 if v_z + v_h == 0.0 else v_z / (v_z + v_h)
    sign = 1.0 if src.volume_rate >= 0.0 else -1.0
    n_th = table.n_theta
    plan = {"e_ring": 0.0, "e_wake": 0.0, "ring_dirs": np.zeros((0, 2)), "wake_dirs": np.zeros((0, 2)),
            "amp_ring": 0.0, "amp_wake": 0.0, "ring_bucket": 0, "wake_bucket": 0}
    if budget <= 0.0:
        return plan

    def amp_of(energy, b, n):
        r_b = table.buckets[b].radius
        per = energy / n
        return sign * math.sqrt(8.0 * per / (rho * g * math.pi * r_b ** 2))

    e_ring = ring_weight * budget
    if e_ring > 0.0:
        b = nearest_bucket(table, src.hull_extent)
        dirs = _fan(0.0, math.pi * (1.0 - 1.0 / n_th), n_th)
        plan.update(e_ring=e_ring, ring_dirs=dirs, ring_bucket=b, amp_ring=amp_of(e_ring, b, len(dirs)))
    e_wake = (1.0 - ring_weight) * budget
    if e_wake > 0.0 and v_h > 0.0:
        b = nearest_bucket(table, src.hull_extent / 2.0)
        back = math.atan2(-vel[1], -vel[0])
        count = src.wake_count if src.wake_count > 0 else max(n_th // 2, 3)
        dirs = _fan(back, KELVIN_HALF_ANGLE, count)
        plan.update(e_wake=e_wake, wake_dirs=dirs, wake_bucket=b, amp_wake=amp_of(e_wake, b, len(dirs)))
    return plan


def box_body(cfg) -> N.HsBody:
    """HsBody of a BodyConfig: box_body's mass, four bottom probes, hull extent
    and drags (interaction.py:79-102), at rest."""
    sx, sy, sz = cfg.size
    volume = sx * sy * sz
    mass = cfg.density * volume
    extent = 0.5 * math.hypot(sx, sy)
    b = N.HsBody()
    for k in range(3):
        b.pos[k] = float(cfg.position[k])
        b.vel[k] = 0.0
    b.yaw, b.yaw_rate = float(cfg.yaw), 0.0
    b.submerged = b.prev_submerged = b.mean_submersion = 0.0
    b.mass, b.hull_extent, b.draft = mass, extent, float(sz)
    b.drag_linear, b.drag_yaw = 2.0 * mass, 0.2 * mass * extent ** 2
    b.thrust_force = 0.0 * cfg.max_thrust          # thrust / rudder commands start at 0 (interaction.py:50-51)
    b.yaw_torque = 0.0 * cfg.max_yaw_torque
    half = (sx / 2.0, sy / 2.0)
    q = 0
    vols = []
    for dx in (-1.0, 1.0):
        for dy in (-1.0, 1.0):
            b.probe_off[q][0], b.probe_off[q][1], b.probe_off[q][2] = dx * half[0], dy * half[1], -sz / 2.0
            b.probe_vol[q] = volume / 4.0
            vols.append(volume / 4.0)
            q += 1
    b.displaced = sum(vols)                          # FloatingBody.displaced_volume (:66-67)
    b.n_probes = 4
    return b


def body_structs(bodies, table, offset: int) -> tuple[list, np.ndarray, list]:
    """HsSource records of floating bodies (body >= 0): ring fan directions
    fan(0, pi (1 - 1/n_theta), n_theta) and the wake fan's angle offsets
    linspace(-K, K, max(n_theta // 2, 3)) (interaction.py:218-230); bucket by
    nearest radius to the hull extent (ring) and half of it (wake)."""
    structs, dirs, hb = [], [], []
    n_th = table.n_theta
    for j, cfg in enumerate(bodies):
        b = box_body(cfg)
        ring = _fan(0.0, math.pi * (1.0 - 1.0 / n_th), n_th)
        n_w = max(n_th // 2, 3)
        lin = np.linspace(-KELVIN_HALF_ANGLE, KELVIN_HALF_ANGLE, n_w) if n_w > 1 else np.zeros(1)
        wake = np.stack([lin, np.zeros_like(lin)], axis=1)
        structs.append(N.HsSource(0.0, 0.0, b.hull_extent, 0.0, 0.0, 0.0, 0.0, n_th, n_w,
                                  nearest_bucket(table, b.hull_extent), nearest_bucket(table, b.hull_extent / 2.0),
                                  offset, j))
        dirs += [ring, wake]
        offset += n_th + n_w
        hb.append(b)
    d = np.concatenate(dirs) if dirs else np.zeros((0, 2))
    return structs, d, hb


def source_structs(sources, table, rho: float, g: float, offset: int = 0) -> tuple[list, np.ndarray, list]:
    """(HsSource records, concatenated fan directions [n, 2] f64, plans)."""
    structs, dirs, plans = [], [], []
    off = offset
    for src in sources:
        pl = source_plan(src, table, rho, g)
        nr, nw = len(pl["ring_dirs"]), len(pl["wake_dirs"])
        structs.append(N.HsSource(float(src.velocity[0]), float(src.velocity[1]), float(src.hull_extent),
                                  float(pl["e_ring"]), float(pl["e_wake"]), float(pl["amp_ring"]),
                                  float(pl["amp_wake"]), nr, nw, pl["ring_bucket"], pl["wake_bucket"], off, -1))
        dirs += [pl["ring_dirs"], pl["wake_dirs"]]
        off += nr + nw
        plans.append(pl)
    d = np.concatenate(dirs) if dirs else np.zeros((0, 2))
    return structs, np.ascontiguousarray(d, dtype=np.float64), plans


__all__ = ["KELVIN_HALF_ANGLE", "nearest_bucket", "_fan", "source_plan", "source_structs", "box_body",
           "body_structs"]
