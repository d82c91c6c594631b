"""Device <-> numpy conversions of the host face."""
from __future__ import annotations

import numpy as np
import torch


def to_numpy(x):
    """fp32/fp64 device tensor -> float64 numpy (the reference's dtype); other values unchanged."""
    if torch.is_tensor(x):
        return x.detach().double().cpu().numpy()
    return x


def to_device(x, device=None, dtype=torch.float32):
    if x is None:
        return None
    if torch.is_tensor(x):
        return x.to(device=device or x.device, dtype=dtype).contiguous()
    dev = device or torch.device("cuda", torch.cuda.current_device())
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to(dev, dtype).contiguous()


def field_to_host(f):
    """A HeightField with numpy (float64) arrays."""
    from ..fft_background import HeightField
    if f is None:
        return None
    return HeightField(resolution=f.resolution, origin=np.asarray(f.origin, dtype=float).copy(), spacing=f.spacing,
                       height=to_numpy(f.height), displacement=to_numpy(f.displacement),
                       normal=to_numpy(f.normal), periodic=f.periodic)


def field_to_device(f, device=None):
    """A HeightField with fp32 device tensors (numpy arrays uploaded)."""
    from ..fft_background import HeightField
    if f is None:
        return None
    if torch.is_tensor(f.height):
        return f
    return HeightField(resolution=f.resolution, origin=np.asarray(f.origin, dtype=float), spacing=f.spacing,
                       height=to_device(f.height, device), displacement=to_device(f.displacement, device),
                       normal=to_device(f.normal, device), periodic=f.periodic)
