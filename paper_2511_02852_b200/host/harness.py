"""Host face of `harness` (reference harness.py): the same device
Simulation, with the reference's host-side views -- numpy background and
stitched grid, a numpy SurfaceSampler, per-patch state objects -- and the
reference's determinism contract (a run is a pure function of (config,
seed), harness.py:1-11): the face runs in the device's deterministic mode
(int64 fixed-point sums) unless told otherwise."""
from __future__ import annotations

from dataclasses import dataclass, replace

from .. import harness as _dev
from ..harness import *  # noqa: F401,F403
from ..harness import (STAGES, BenchRow, FrameStats, bench_table, benchmark_cell, stats_header,  # noqa: F401
                       stats_row, trend_matrix, wp_only_config)
from ._conv import field_to_host, to_numpy
from .coupling import PatchSurface, SurfaceSampler


class _LedgerView:
    """InjectionLedger-shaped numpy view of patch k's device ledger (particles.py:187-202)."""

    def __init__(self, sim, k: int):
        self._sim, self._k = sim, k

    def _get(self, key):
        return self._sim.ledger_host()[key][self._k]

    @property
    def accumulators(self):
        return self._get("acc")

    @property
    def injected_groups(self):
        return self._get("groups")

    @property
    def injected_energy(self):
        return self._get("e_in")

    @property
    def despawned_energy(self):
        return self._get("e_out")


@dataclass
class PatchState:
    """Per-patch run state as the reference exposes it (harness.py:49-62)."""
    region: object
    resolution: int
    pool: object
    ledger: object
    surface: object = None

    @property
    def texel(self) -> float:
        return self.region.l1 / (self.resolution - 1)


class BodyView:
    """FloatingBody-shaped view of body j's device state (interaction.py:35-76):
    pose, velocity and submerged volumes read back from hs_bodies' struct;
    the thrust / rudder commands write the force and torque it integrates."""

    def __init__(self, sim, j: int, cfg):
        self._sim, self._j, self._cfg = sim, j, cfg
        self._thrust = 0.0
        self._rudder = 0.0

    def _raw(self):
        import ctypes as C
        from .. import _native as N
        sz = C.sizeof(N.HsBody)
        return N.HsBody.from_buffer_copy(self._sim.bodies_dev[self._j * sz:(self._j + 1) * sz].cpu().numpy().tobytes())

    def _write(self, field: str, value: float) -> None:
        import ctypes as C
        import torch
        from .. import _native as N
        off = self._j * C.sizeof(N.HsBody) + getattr(N.HsBody, field).offset
        self._sim.bodies_dev[off:off + 8].view(torch.float64).fill_(float(value))

    @property
    def position(self):
        import numpy as np
        return np.array(self._raw().pos[:])

    @property
    def velocity(self):
        import numpy as np
        return np.array(self._raw().vel[:])

    @property
    def yaw(self) -> float:
        return self._raw().yaw

    @property
    def yaw_rate(self) -> float:
        return self._raw().yaw_rate

    @property
    def submerged_volume(self) -> float:
        return self._raw().submerged

    @property
    def prev_submerged_volume(self) -> float:
        return self._raw().prev_submerged

    @property
    def mean_submersion(self) -> float:
        return self._raw().mean_submersion

    @property
    def thrust(self) -> float:
        return self._thrust

    @thrust.setter
    def thrust(self, v: float) -> None:
        self._thrust = float(v)
        self._write("thrust_force", self._thrust * self._cfg.max_thrust)

    @property
    def rudder(self) -> float:
        return self._rudder

    @rudder.setter
    def rudder(self, v: float) -> None:
        self._rudder = float(v)
        self._write("yaw_torque", self._rudder * self._cfg.max_yaw_torque)


class Simulation(_dev.Simulation):
    def __init__(self, config, device=None, deterministic: bool = True, **kw):
        if deterministic and not config.deterministic:
            config = replace(config, deterministic=True)
        super().__init__(config, device, **kw)
        self._body_views = [BodyView(self, j, c) for j, c in enumerate(self.__dict__["_body_cfgs"])] \
            if getattr(self, "bodies_dev", None) is not None else None

    @property
    def bodies(self):
        """The floating bodies (FloatingBody views of the device state)."""
        views = self.__dict__.get("_body_views")
        return views if views is not None else self.__dict__.get("_body_cfgs", ())

    @bodies.setter
    def bodies(self, value) -> None:
        self.__dict__["_body_cfgs"] = value

    @property
    def background(self):
        return field_to_host(_dev.Simulation.background.fget(self))

    def stitched_heights(self):
        return to_numpy(super().stitched_heights())

    def _surfaces(self):
        return [PatchSurface(r, field_to_host(self.patch_field(k))) for k, r in enumerate(self.current_regions())]

    @property
    def sampler(self):
        return SurfaceSampler(self.background, self._surfaces(), self.config.normal_mode,
                              cascades=[field_to_host(f) for f in self.cascade_fields()[1:]])

    @property
    def patches(self) -> list:
        surf = self._surfaces() if self.frame > 0 else [None] * self.n_patches
        return [PatchState(r, res, self.pool(k), _LedgerView(self, k), surf[k])
                for k, (r, res) in enumerate(zip(self.current_regions(), self.res))]


def run(config, output_dir: str | None = None, progress=None, deterministic: bool = True) -> list:
    """harness.py:274-329 (stats.csv, timings.csv, frame files), byte-identical
    across reruns in the default deterministic mode."""
    if deterministic and not config.deterministic:
        config = replace(config, deterministic=True)
    return _dev.run(config, output_dir, progress)


def benchmark(cells: list, warmup=None, measure=None, progress=None) -> list:
    return _dev.benchmark(cells, warmup, measure, progress)
