"""Host face of `fft_background` (reference fft_background.py): fields come
back as numpy float64 arrays; the transform runs on the device."""
from __future__ import annotations

import numpy as np

from .. import fft_background as _dev
from ..fft_background import *  # noqa: F401,F403
from ..fft_background import FftState, HeightField, init_fft, resolved_band, spectral_at, zeroed  # noqa: F401
from ._conv import field_to_device, field_to_host, to_numpy


def evolve_and_synthesize(state: FftState, t: float) -> HeightField:
    """Height, choppy displacement and periodic normals at time t
    (fft_background.py:181-208), as numpy arrays."""
    return field_to_host(_dev.evolve_and_synthesize(state, t))


def sample_periodic(field: HeightField, points):
    """Periodic bilinear height / renormalised normal (fft_background.py:222-249)."""
    h, n = _dev.sample_periodic(field_to_device(field), np.asarray(points, dtype=float))
    return to_numpy(h), to_numpy(n)
