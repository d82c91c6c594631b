"""Host face of `coupling` (reference coupling.py): samplers accept numpy
HeightFields and return numpy arrays; the blend runs on the device."""
from __future__ import annotations

import numpy as np

from .. import coupling as _dev
from ..coupling import *  # noqa: F401,F403
from ..coupling import BlendMask, blend_weight, boundary_depth, build_mask, smoothstep, validate_patches  # noqa: F401
from ._conv import field_to_device, to_numpy
from .fft_background import evolve_and_synthesize


class PatchSurface(_dev.PatchSurface):
    pass


def _dev_surfaces(patches):
    return [_dev.PatchSurface(p.patch, field_to_device(p.field)) for p in patches]


class SurfaceSampler(_dev.SurfaceSampler):
    """coupling.py:103-161 with numpy fields in and numpy samples out."""

    def __init__(self, background, patches: list, normal_mode: str = "blend", cascades=None):
        super().__init__(field_to_device(background), _dev_surfaces(patches), normal_mode,
                         cascades=[field_to_device(c) for c in (cascades or [])])
        self.host_background, self.host_patches = background, patches

    def sample(self, points):
        out = super().sample(np.asarray(points, dtype=float) if not np.isscalar(points) else points)
        if isinstance(out[0], float):
            return out
        return to_numpy(out[0]), to_numpy(out[1])


def sample_clamped(field, points):
    h, n = _dev.sample_clamped(field_to_device(field), np.asarray(points, dtype=float))
    return to_numpy(h), to_numpy(n)


def query_surface(world_pos, t: float, fft_state, patches: list, normal_mode: str = "blend"):
    background = evolve_and_synthesize(fft_state, t) if fft_state is not None else None
    return SurfaceSampler(background, patches, normal_mode).sample(world_pos)
