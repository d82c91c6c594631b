"""Floating bodies: probe buoyancy against the blended surface -- TEST INFRASTRUCTURE ONLY.

Restates `pkg/src/hybridsea/interaction.py:29-149` (FloatingBody, box_body,
buoyancy_step) with the reference's operation order, so a scene driven by the
same surface samples reproduces the reference's body trajectories.  Emission
from a body's state goes through `emit_ref.emit` (interaction.py:175-231) with
the body's displaced-volume change and mean submersion of the step.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Body:
    """FloatingBody (interaction.py:36-77) with box_body's four bottom probes."""
    position: np.ndarray
    yaw: float
    velocity: np.ndarray
    yaw_rate: float
    mass: float
    probe_offsets: np.ndarray          # (4, 3) body frame
    probe_volumes: np.ndarray          # (4,)
    hull_extent: float
    draft_height: float
    drag_linear: float
    drag_yaw: float
    max_thrust: float = 0.0
    max_yaw_torque: float = 0.0
    thrust: float = 0.0
    rudder: float = 0.0
    submerged_volume: float = 0.0
    prev_submerged_volume: float = 0.0
    mean_submersion: float = 0.0

    @property
    def displaced_volume(self) -> float:
        return sum(float(v) for v in self.probe_volumes)          # interaction.py:66-67

    def probe_world_positions(self) -> np.ndarray:
        """interaction.py:69-77."""
        off = self.probe_offsets
        c, s = math.cos(self.yaw), math.sin(self.yaw)
        world = np.empty_like(off)
        world[:, 0] = self.position[0] + c * off[:, 0] - s * off[:, 1]
        world[:, 1] = self.position[1] + s * off[:, 0] + c * off[:, 1]
        world[:, 2] = self.position[2] + off[:, 2]
        return world


def box_body(position, size, density=500.0, yaw=0.0, max_thrust=0.0, max_yaw_torque=0.0) -> Body:
    """interaction.py:79-102: four corner probes at the bottom face."""
    sx, sy, sz = size
    volume = sx * sy * sz
    mass = density * volume
    half = np.array([sx, sy]) / 2.0
    offs, vols = [], []
    for dx in (-1.0, 1.0):
        for dy in (-1.0, 1.0):
            offs.append([dx * half[0], dy * half[1], -sz / 2.0])
            vols.append(volume / 4.0)
    extent = 0.5 * math.hypot(sx, sy)
    return Body(position=np.asarray(position, dtype=float).copy(), yaw=yaw, velocity=np.zeros(3), yaw_rate=0.0,
                mass=mass, probe_offsets=np.array(offs), probe_volumes=np.array(vols), hull_extent=extent,
                draft_height=sz, drag_linear=2.0 * mass, drag_yaw=0.2 * mass * extent ** 2,
                max_thrust=max_thrust, max_yaw_torque=max_yaw_torque)


def buoyancy_step(body: Body, query_surface, dt: float, rho: float = 1000.0, g: float = 9.81) -> Body:
    """interaction.py:105-149 (mutates body)."""
    if dt <= 0:
        raise ValueError("dt must be positive")
    world = body.probe_world_positions()
    heights, normals = query_surface(world[:, :2])
    heights = np.atleast_1d(np.asarray(heights, dtype=float))
    normals = np.atleast_2d(np.asarray(normals, dtype=float))
    depth = heights - world[:, 2]
    frac = np.clip(depth / body.draft_height, 0.0, 1.0)
    volumes = body.probe_volumes
    submerged = float(np.sum(volumes * frac))
    force = np.zeros(3)
    torque_z = 0.0
    for i_p in range(len(volumes)):
        f = rho * g * volumes[i_p] * frac[i_p] * normals[i_p]
        force += f
        r = world[i_p] - body.position
        torque_z += r[0] * f[1] - r[1] * f[0]
    wet = submerged / body.displaced_volume if body.displaced_volume > 0 else 0.0
    force -= body.drag_linear * wet * body.velocity
    heading = np.array([math.cos(body.yaw), math.sin(body.yaw), 0.0])
    force += body.thrust * body.max_thrust * heading
    torque_z += body.rudder * body.max_yaw_torque - body.drag_yaw * wet * body.yaw_rate
    inertia = 0.5 * body.mass * body.hull_extent ** 2
    body.velocity += (force / body.mass + np.array([0.0, 0.0, -g])) * dt
    body.position += body.velocity * dt
    body.yaw_rate += torque_z / inertia * dt
    body.yaw += body.yaw_rate * dt
    body.prev_submerged_volume = body.submerged_volume
    body.submerged_volume = submerged
    wet_depths = depth[depth > 0.0]
    body.mean_submersion = float(np.mean(np.minimum(wet_depths, body.draft_height))) if wet_depths.size else 0.0
    return body


__all__ = ["Body", "box_body", "buoyancy_step"]
