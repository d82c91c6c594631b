"""Smoothstep blend of patch fields into the background -- TEST INFRASTRUCTURE ONLY.

Restates `pkg/src/hybridsea/coupling.py` (reference) blend weights (:21-60),
clamped sampling (:63-82), the `SurfaceSampler._raw` compositing loop
(:120-141, normal_mode="blend"), and `Simulation.stitched_heights`
(`harness.py:219-241`).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .ocean_ref import sample_periodic
from .particles_ref import Patch


def smoothstep(t):
    t = np.clip(t, 0.0, 1.0)
    return t * t * (3.0 - 2.0 * t)


def depth(patch: Patch, pts: np.ndarray) -> np.ndarray:
    lo, hi = patch.lo, patch.hi
    return np.minimum(np.minimum(pts[..., 0] - lo[0], hi[0] - pts[..., 0]),
                      np.minimum(pts[..., 1] - lo[1], hi[1] - pts[..., 1]))


def weight(patch: Patch, pts: np.ndarray) -> np.ndarray:
    d = depth(patch, pts)
    return np.where(d > 0.0, smoothstep(d / patch.margin), 0.0)


def patch_nodes(patch: Patch, res: int) -> np.ndarray:
    """World positions of the node-centred patch grid (coupling.py:51-60)."""
    texel = patch.l1 / (res - 1)
    ny = int(round(patch.l2 / texel)) + 1
    xs = patch.x0 + np.arange(res) * texel
    ys = patch.y0 + np.arange(ny) * texel
    return np.stack(np.meshgrid(xs, ys, indexing="ij"), axis=-1)


def sample_clamped(height: np.ndarray, normal: np.ndarray | None, origin, spacing: float,
                   pts: np.ndarray):
    nx, ny = height.shape
    u = np.clip((pts[..., 0] - origin[0]) / spacing, 0.0, nx - 1.0)
    v = np.clip((pts[..., 1] - origin[1]) / spacing, 0.0, ny - 1.0)
    i = np.minimum(u.astype(int), nx - 2)
    j = np.minimum(v.astype(int), ny - 2)
    fu, fv = u - i, v - j
    w00, w10, w01, w11 = (1 - fu) * (1 - fv), fu * (1 - fv), (1 - fu) * fv, fu * fv
    hv = height[i, j] * w00 + height[i + 1, j] * w10 + height[i, j + 1] * w01 + height[i + 1, j + 1] * w11
    if normal is None:
        return hv, None
    nv = (normal[i, j] * w00[..., None] + normal[i + 1, j] * w10[..., None]
          + normal[i, j + 1] * w01[..., None] + normal[i + 1, j + 1] * w11[..., None])
    return hv, nv / np.linalg.norm(nv, axis=-1, keepdims=True)


@dataclass
class Field:
    """Height/normal grid with origin and spacing (HeightField subset)."""
    height: np.ndarray
    normal: np.ndarray
    origin: np.ndarray
    spacing: float


def sample_background(background, pts: np.ndarray):
    """sample_periodic of the background (fft_background.py:222-249).  A list
    of Fields is a summed-cascade background: heights add; normals combine
    through their slopes, n = normalize(sum_c n_c.xy / n_c.z, 1), which for
    one cascade is the renormalised bilinear normal itself."""
    if isinstance(background, (list, tuple)):
        if len(background) == 1:
            return sample_background(background[0], pts)
        h = np.zeros(pts.shape[:-1])
        sl = np.zeros(pts.shape[:-1] + (2,))
        for f in background:
            hc, nc = sample_periodic(f.height, f.normal, f.origin, f.spacing, pts)
            h = h + hc
            sl = sl + nc[..., :2] / nc[..., 2:3]
        nrm = np.concatenate([sl, np.ones(pts.shape[:-1] + (1,))], axis=-1)
        return h, nrm / np.linalg.norm(nrm, axis=-1, keepdims=True)
    h, nrm = sample_periodic(background.height, background.normal, background.origin, background.spacing, pts)
    return np.array(h, dtype=float), nrm


def sample(background, patches: list[tuple[Patch, Field]], pts: np.ndarray):
    """Blended (height, normal) at world points (coupling.py:120-141)."""
    pts = np.asarray(pts, dtype=float)
    if background is not None:
        h, nrm = sample_background(background, pts)
    else:
        h = np.zeros(pts.shape[:-1])
        nrm = np.zeros(pts.shape[:-1] + (3,))
        nrm[..., 2] = 1.0
    for patch, fld in patches:
        w = weight(patch, pts)
        m = w > 0.0
        if not np.any(m):
            continue
        ph, pn = sample_clamped(fld.height, fld.normal, fld.origin, fld.spacing, pts[m])
        wi = w[m]
        h[m] = wi * ph + (1.0 - wi) * h[m]
        mix = wi[:, None] * pn + (1.0 - wi)[:, None] * nrm[m]
        nrm[m] = mix / np.linalg.norm(mix, axis=-1, keepdims=True)
    return h, nrm


def stitched(background: Field | None, n: int, domain: float,
             patches: list[tuple[Patch, Field]]) -> np.ndarray:
    """Global FFT-resolution composite with patch boxes resampled (harness.py:219-241)."""
    spacing = domain / n
    if isinstance(background, (list, tuple)) and len(background) > 1:
        # summed cascades on the largest tile's grid (cascade 0)
        xs = np.arange(n) * spacing
        nodes = np.stack(np.meshgrid(xs, xs, indexing="ij"), axis=-1)
        grid = background[0].height.copy()
        for f in background[1:]:
            grid += sample_periodic(f.height, None, f.origin, f.spacing, nodes)[0]
    elif isinstance(background, (list, tuple)):
        grid = background[0].height.copy()
    else:
        grid = background.height.copy() if background is not None else np.zeros((n, n))
    for patch, _ in patches:
        lo = np.clip(np.floor(patch.lo / spacing).astype(int), 0, n)
        hi = np.clip(np.ceil(patch.hi / spacing).astype(int) + 1, 0, n)
        xs = np.arange(lo[0], hi[0]) * spacing
        ys = np.arange(lo[1], hi[1]) * spacing
        if len(xs) == 0 or len(ys) == 0:
            continue
        pts = np.stack(np.meshgrid(xs, ys, indexing="ij"), axis=-1).reshape(-1, 2)
        hv, _ = sample(background, patches, pts)
        grid[lo[0]:hi[0], lo[1]:hi[1]] = hv.reshape(len(xs), len(ys))
    return grid
