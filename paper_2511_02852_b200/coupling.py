"""Blending of patch fields into the FFT background, and surface queries.

Mirror of `hybridsea.coupling` (`pkg/src/hybridsea/coupling.py`).  Weight
helpers are small host functions (used at init / by tests); sampling and
compositing are CUDA kernels (csrc/synth.cu: hs_sample, hs_compose).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._layout import patch_struct, stream_ptr, structs_to_device
from .errors import ConfigError
from .fft_background import FftState, HeightField, evolve_and_synthesize
from .particles import PatchRegion


def smoothstep(t):
    t = np.clip(t, 0.0, 1.0)
    return t * t * (3.0 - 2.0 * t)


def boundary_depth(patch: PatchRegion, points) -> np.ndarray:
    p = np.asarray(points, dtype=float)
    lo, hi = patch.min_corner, patch.max_corner
    return np.minimum(np.minimum(p[..., 0] - lo[0], hi[0] - p[..., 0]),
                      np.minimum(p[..., 1] - lo[1], hi[1] - p[..., 1]))


def blend_weight(patch: PatchRegion, points) -> np.ndarray:
    """0 at/outside the boundary, smoothstep(d/margin) inside (coupling.py:37-40)."""
    d = boundary_depth(patch, points)
    return np.where(d > 0.0, smoothstep(d / patch.margin), 0.0)


@dataclass(eq=False)
class BlendMask:
    weights: np.ndarray
    margin: float


def build_mask(patch: PatchRegion, resolution: int) -> BlendMask:
    if patch.margin <= 0:
        raise ConfigError("patch margin must be positive")
    texel = patch.l1 / (resolution - 1)
    ny = int(round(patch.l2 / texel)) + 1
    xs = patch.min_corner[0] + np.arange(resolution) * texel
    ys = patch.min_corner[1] + np.arange(ny) * texel
    pts = np.stack(np.meshgrid(xs, ys, indexing="ij"), axis=-1)
    return BlendMask(weights=blend_weight(patch, pts), margin=patch.margin)


def validate_patches(patches: list) -> None:
    """Open-interval overlap test; shared edges allowed (coupling.py:85-92)."""
    for i in range(len(patches)):
        for j in range(i + 1, len(patches)):
            a, b = patches[i], patches[j]
            if (a.min_corner[0] < b.max_corner[0] and b.min_corner[0] < a.max_corner[0]
                    and a.min_corner[1] < b.max_corner[1] and b.min_corner[1] < a.max_corner[1]):
                raise ConfigError(f"patches {i} and {j} overlap")


@dataclass(eq=False)
class PatchSurface:
    patch: PatchRegion
    field: HeightField


def _points(points, device) -> tuple:
    pts = points if torch.is_tensor(points) else torch.from_numpy(np.asarray(points, dtype=np.float64))
    pts = pts.to(device=device, dtype=torch.float64)
    return pts.reshape(-1, 2).contiguous(), pts.shape[:-1]


def sample_clamped(field: HeightField, points) -> tuple:
    """Bilinear height/normal on a non-periodic grid, clamped (coupling.py:63-82)."""
    dev = field.height.device
    flat, shape = _points(points, dev)
    nx, ny = field.height.shape
    region = PatchRegion(tuple(field.origin), field.spacing * (nx - 1), field.spacing * (ny - 1),
                         0.25 * field.spacing * min(nx - 1, ny - 1))
    pst = structs_to_device([patch_struct(region, nx)], dev)
    out_h = torch.empty(flat.shape[0], dtype=torch.float32, device=dev)
    out_n = torch.empty((flat.shape[0], 3), dtype=torch.float32, device=dev)
    args = N.HsSampleArgs(n_points=flat.shape[0], points=N.ptr(flat), bg_height=0, bg_normal=0, bg_n=0,
                          bg_spacing=1.0, bg_x0=0.0, bg_y0=0.0, n_patches=1, patches=N.ptr(pst),
                          patch_height=N.ptr(field.height.contiguous()),
                          patch_normal=N.ptr(field.normal.contiguous()), out_height=N.ptr(out_h),
                          out_normal=N.ptr(out_n), clamped_only=1)
    N.call("hs_sample", args, stream_ptr())
    return out_h.reshape(shape), out_n.reshape(tuple(shape) + (3,))


class SurfaceSampler:
    """World-space queries against one frame's fields (coupling.py:103-161).
    Pure reads; the patch fields are packed once into contiguous device
    buffers on construction."""

    def __init__(self, background: HeightField | None, patches: list, normal_mode: str = "blend",
                 cascades: list | None = None):
        if normal_mode not in ("blend", "recompute"):
            raise ConfigError(f"unknown normal mode {normal_mode!r}")
        validate_patches([p.patch for p in patches])
        self.background = background
        self.cascades = list(cascades or [])      # further summed background tiles (HeightField, origin 0)
        self.patches = patches
        self.normal_mode = normal_mode
        self._packed = None

    def _pack(self, device):
        if self._packed is None:
            structs, hs, ns, base = [], [], [], 0
            for ps in self.patches:
                nx, ny = ps.field.height.shape
                # keep the patch's own texel (l1/(res-1)) and grid
                structs.append(patch_struct(ps.patch, nx, grid_base=base))
                hs.append(ps.field.height.to(device, torch.float32).reshape(-1))
                ns.append(ps.field.normal.to(device, torch.float32).reshape(-1))
                base += nx * ny
            if structs:
                self._packed = (structs_to_device(structs, device), torch.cat(hs), torch.cat(ns), len(structs))
            else:
                self._packed = (None, None, None, 0)
        return self._packed

    def _device(self):
        if self.background is not None:
            return self.background.height.device
        if self.patches:
            return self.patches[0].field.height.device
        return torch.device("cuda", torch.cuda.current_device())

    def _raw(self, flat: torch.Tensor) -> tuple:
        dev = flat.device
        pst, ph, pn, npatch = self._pack(dev)
        bg = self.background
        out_h = torch.empty(flat.shape[0], dtype=torch.float32, device=dev)
        out_n = torch.empty((flat.shape[0], 3), dtype=torch.float32, device=dev)
        args = N.HsSampleArgs(
            n_points=flat.shape[0], points=N.ptr(flat),
            bg_height=N.ptr(bg.height.contiguous()) if bg is not None else 0,
            bg_normal=N.ptr(bg.normal.contiguous()) if bg is not None and bg.normal is not None else 0,
            bg_n=bg.resolution if bg is not None else 0, bg_spacing=bg.spacing if bg is not None else 1.0,
            bg_x0=float(bg.origin[0]) if bg is not None else 0.0, bg_y0=float(bg.origin[1]) if bg is not None else 0.0,
            n_patches=npatch, patches=N.ptr(pst), patch_height=N.ptr(ph), patch_normal=N.ptr(pn),
            out_height=N.ptr(out_h), out_normal=N.ptr(out_n), clamped_only=0)
        if bg is not None and self.cascades:
            args.n_extra_bg = len(self.cascades)
            for c, f in enumerate(self.cascades):
                args.extra_bg[c] = N.HsBgTile(N.ptr(f.height), f.resolution, 0, float(f.spacing))
        N.call("hs_sample", args, stream_ptr())
        return out_h, out_n

    def sample(self, points):
        dev = self._device()
        scalar = (not torch.is_tensor(points)) and np.ndim(points) == 1
        flat, shape = _points(points, dev)
        h, nrm = self._raw(flat)
        if self.normal_mode == "recompute":
            eps = 1e-2
            off = torch.tensor([[eps, 0.0]], dtype=torch.float64, device=dev)
            offy = torch.tensor([[0.0, eps]], dtype=torch.float64, device=dev)
            hx1, _ = self._raw((flat + off).contiguous())
            hx0, _ = self._raw((flat - off).contiguous())
            hy1, _ = self._raw((flat + offy).contiguous())
            hy0, _ = self._raw((flat - offy).contiguous())
            gx = (hx1.double() - hx0.double()) / (2 * eps)
            gy = (hy1.double() - hy0.double()) / (2 * eps)
            nv = torch.stack([-gx, -gy, torch.ones_like(gx)], -1)
            nrm = (nv / torch.linalg.vector_norm(nv, dim=-1, keepdim=True)).float()
        if scalar:
            return float(h[0].item()), nrm[0].cpu().numpy()
        return h.reshape(shape), nrm.reshape(tuple(shape) + (3,))


def query_surface(world_pos, t: float, fft_state: FftState | None, patches: list,
                  normal_mode: str = "blend"):
    background = evolve_and_synthesize(fft_state, t) if fft_state is not None else None
    return SurfaceSampler(background, patches, normal_mode).sample(world_pos)
