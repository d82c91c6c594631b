"""Host face of `patch_synthesis` (reference patch_synthesis.py): heights and
fields as numpy float64 arrays; splat, smoothing and upsampling run on the device."""
from __future__ import annotations

from .. import patch_synthesis as _dev
from ..patch_synthesis import *  # noqa: F401,F403
from ..patch_synthesis import (LayerPlan, LayerStack, SmoothingKernel, accumulate, build_kernels,  # noqa: F401
                               convolve1d_zero, plan_layers, raised_cosine_taps, smooth_layer)
from ._conv import field_to_host, to_device, to_numpy


def synthesize(particles, patch, resolution: int, plan):
    """(heights (res, ny) numpy, clamped splat count) (patch_synthesis.py:277-314)."""
    h, clamped = _dev.synthesize(particles, patch, resolution, plan)
    return to_numpy(h), clamped


def finish_field(heights, patch, choppiness: float = 0.0, displacement_scale: float = 1.0):
    """Clamped-border normals and optional displacement (patch_synthesis.py:323-340)."""
    return field_to_host(_dev.finish_field(to_device(heights), patch, choppiness, displacement_scale))


def smooth_and_sum(stack, kernels=None):
    return to_numpy(_dev.smooth_and_sum(stack, kernels))
