"""Patch height synthesis on the B200: per-bucket splat, separable
raised-cosine smoothing, bilinear upsampling, gain-sum, finish.

Mirror of `hybridsea.patch_synthesis` (`pkg/src/hybridsea/patch_synthesis.py`).
Kernel/plan construction is host fp64 (init time, :50-90, :242-258); the
per-frame work is three CUDA launches (hs_splat, hs_smooth, hs_compose) --
inside `Simulation.step` the splat is fused into the advect kernel.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._layout import (compose_tile_info, grid_dims, pack_layers, patch_struct, stream_ptr,
                      structs_to_device)
from .errors import ConfigError
from .fft_background import HeightField
from .particles import DEFAULT_TROUGH_FRACTION, ParticleSet, PatchRegion
from .spectrum import BucketTable

AMPLITUDE_CONVENTIONS = ("energy", "peak")


@dataclass(frozen=True)
class SmoothingKernel:
    """Normalised symmetric taps + output gain (patch_synthesis.py:37-47)."""
    taps: np.ndarray
    half_width: int
    gain: float

    def __post_init__(self):
        if len(self.taps) != 2 * self.half_width + 1:
            raise ValueError("taps length must be 2*half_width + 1")


def raised_cosine_taps(half_width: int) -> np.ndarray:
    """1 + cos(pi m/(R+1)) over m = -R..R, summing to 1 (:50-54)."""
    m = np.arange(-half_width, half_width + 1)
    taps = 1.0 + np.cos(math.pi * m / (half_width + 1))
    return taps / taps.sum()


def _pair_square_sum(taps: np.ndarray, shift: int, trough_fraction: float) -> float:
    """Sum of squares of a unit crest + trailing trough bump pair (:57-66)."""
    bump = np.outer(taps, taps)
    w = bump.shape[0]
    canvas = np.zeros((w + shift, w))
    canvas[:w] += bump
    if trough_fraction != 0.0:
        canvas[shift:] -= trough_fraction * bump
    return float(np.sum(canvas ** 2))


def _kernel_for(radius: float, texel_size: float, convention: str, trough_fraction: float) -> SmoothingKernel:
    if convention not in AMPLITUDE_CONVENTIONS:
        raise ConfigError(f"unknown amplitude convention {convention!r}")
    half = max(1, int(round(radius / texel_size)))
    taps = raised_cosine_taps(half)
    if convention == "peak":
        gain = 1.0 / float(taps[half] ** 2)
    else:
        ss = _pair_square_sum(taps, half, trough_fraction) * texel_size ** 2
        gain = math.sqrt((math.pi * radius ** 2 / 8.0) / ss)
    return SmoothingKernel(taps=taps, half_width=half, gain=gain)


def build_kernels(table: BucketTable, texel_size: float, convention: str = "energy",
                  trough_fraction: float = DEFAULT_TROUGH_FRACTION) -> list:
    return [_kernel_for(b.radius, texel_size, convention, trough_fraction) for b in table.buckets]


@dataclass(frozen=True)
class LayerPlan:
    """Per-bucket decimation factor + kernel at the coarse texel (:227-240)."""
    kernels: tuple
    factors: tuple


def plan_layers(table: BucketTable, texel_size: float, resolution: int, convention: str = "energy",
                trough_fraction: float = DEFAULT_TROUGH_FRACTION, min_taps: int = 4,
                adaptive: bool = True) -> LayerPlan:
    """Coarse grids at ~min_taps texels per radius (:242-258)."""
    factors = []
    for b in table.buckets:
        if not adaptive:
            factors.append(1)
            continue
        f = max(1, int((b.radius / texel_size) / min_taps))
        factors.append(min(f, max(1, (resolution - 1) // (4 * min_taps))))
    kernels = tuple(_kernel_for(b.radius, texel_size * f, convention, trough_fraction)
                    for b, f in zip(table.buckets, factors))
    return LayerPlan(kernels=kernels, factors=tuple(factors))


def as_plan(plan) -> LayerPlan:
    if isinstance(plan, LayerPlan):
        return plan
    return LayerPlan(kernels=tuple(plan), factors=(1,) * len(plan))


def mean_radius(table: BucketTable) -> float:
    e = table.energies
    return float(np.sum(e * table.radii) / np.sum(e))


class SynthWorkspace:
    """Device layers and descriptors for synthesising a set of patches."""

    def __init__(self, regions: list, resolutions: list, plans: list, device):
        self.device = device
        self.regions = list(regions)
        self.grids = [(res, grid_dims(r, res)[1]) for r, res in zip(regions, resolutions)]
        plans = [as_plan(p) for p in plans]
        self.nb = len(plans[0].kernels)
        if any(len(p.kernels) != self.nb for p in plans):
            raise ConfigError("all patches need one kernel per bucket")
        self.pack = pack_layers(plans, self.grids)
        self.layers = structs_to_device(self.pack.layers, device)
        self.taps = torch.from_numpy(self.pack.taps).to(device)
        self.raw = torch.zeros(max(1, self.pack.raw_len), dtype=torch.float32, device=device)
        self.smooth = torch.zeros(max(1, self.pack.smooth_len), dtype=torch.float32, device=device)
        self.smooth_info = torch.from_numpy(np.ascontiguousarray(self.pack.smooth_tile_info)).to(device)
        self.xtile_prefix = torch.from_numpy(self.pack.xtile_prefix).to(device)
        self.ytile_prefix = torch.from_numpy(self.pack.ytile_prefix).to(device)
        self.mid = torch.zeros(self.pack.mid_len, dtype=torch.float32, device=device) if self.pack.mid_len else None
        self.tickets = torch.zeros(max(1, self.pack.n_tickets), dtype=torch.int32, device=device)
        self.compose_info_np = compose_tile_info(self.grids)
        self.compose_info = torch.from_numpy(self.compose_info_np).to(device)
        self.compose_tiles = int(self.compose_info_np.shape[0])
        self.grid_base = np.concatenate([[0], np.cumsum([r * ny for r, ny in self.grids])]).astype(np.int64)
        self.clamped = torch.zeros(len(regions), dtype=torch.int32, device=device)

    def patch_structs(self, **kw) -> list:
        return [patch_struct(r, res, grid_base=int(self.grid_base[k]), layer_base=k * self.nb, **kw)
                for k, (r, (res, _)) in enumerate(zip(self.regions, self.grids))]

    def smooth_args(self) -> N.HsSmoothArgs:
        return N.HsSmoothArgs(n_layers=len(self.pack.layers), layers=N.ptr(self.layers), taps=N.ptr(self.taps),
                              raw_layers=N.ptr(self.raw), smooth_layers=N.ptr(self.smooth),
                              tile_info=N.ptr(self.smooth_info),
                              total_tiles=int(self.pack.smooth_tile_info.shape[0]), max_H=self.pack.max_H,
                              mid=N.ptr(self.mid), xtile_prefix=N.ptr(self.xtile_prefix),
                              total_xtiles=int(self.pack.xtile_prefix[-1]), ytile_prefix=N.ptr(self.ytile_prefix),
                              total_ytiles=int(self.pack.ytile_prefix[-1]), max_H_wide=self.pack.max_H_wide,
                              tickets=N.ptr(self.tickets))


def synthesize(particles: ParticleSet, patch: PatchRegion, resolution: int, plan) -> tuple:
    """Splat + smooth + upsample + gain-sum of one patch (:277-314).
    Returns (heights (res, ny) fp32 device tensor, clamped splat count)."""
    if resolution < 2:
        raise ConfigError(f"patch resolution must be >= 2, got {resolution}")
    plan = as_plan(plan)
    nb = len(plan.kernels)
    particles.materialize(nb)
    dev = particles.device
    ws = SynthWorkspace([patch], [resolution], [plan], dev)
    res, ny = ws.grids[0]
    heights = torch.zeros((res, ny), dtype=torch.float32, device=dev)
    if len(particles) == 0:
        return heights, 0
    pst = structs_to_device(ws.patch_structs(), dev)
    count = torch.from_numpy(particles.counts.astype(np.int32)).to(dev)
    st = stream_ptr()
    N.call("hs_splat", N.HsSplatArgs(n_patches=1, nb=nb, patches=N.ptr(pst), pool=particles.pool_struct(),
                                     count=N.ptr(count), raw_layers=N.ptr(ws.raw), raw_layers_len=ws.pack.raw_len,
                                     layers=N.ptr(ws.layers), clamped=N.ptr(ws.clamped),
                                     max_count=int(particles.counts.sum())), st)
    N.call("hs_smooth", ws.smooth_args(), st)
    N.call("hs_compose", N.HsComposeArgs(
        n_patches=1, nb=nb, patches=N.ptr(pst), layers=N.ptr(ws.layers), smooth_layers=N.ptr(ws.smooth),
        tile_info=N.ptr(ws.compose_info), total_tiles=ws.compose_tiles, bg_height=0,
        bg_normal=0, bg_n=0, bg_spacing=1.0, patch_height=N.ptr(heights), patch_normal=0, blend_height=0,
        blend_normal=0, blend_mode=0, interior_sumsq=0, interior_count=0), st)
    return heights, int(ws.clamped.item())


def convolve1d_zero(arr, taps, axis: int) -> np.ndarray:
    """Same-size 1-D convolution with zero-padded borders along an axis
    (patch_synthesis.py:105-130), fp64 on the device (hs_conv1d_zero) with
    direct taps.  ConfigError if the kernel is wider than the axis."""
    a = np.asarray(arr, dtype=np.float64)
    taps = np.asarray(taps, dtype=np.float64)
    axis = axis % a.ndim
    n = a.shape[axis]
    if len(taps) > n:
        raise ConfigError(f"kernel of {len(taps)} taps wider than grid axis of {n}")
    outer = int(np.prod(a.shape[:axis], dtype=np.int64))
    inner = int(np.prod(a.shape[axis + 1:], dtype=np.int64))
    dev = torch.device("cuda", torch.cuda.current_device())
    src = torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    tp = torch.from_numpy(np.ascontiguousarray(taps)).to(dev)
    out = torch.empty_like(src)
    N.call_raw("hs_conv1d_zero", N.vp(N.ptr(src)), N.vp(N.ptr(out)), N.i64(outer), N.i32(n), N.i64(inner),
               N.vp(N.ptr(tp)), N.i32((len(taps) - 1) // 2), N.vp(stream_ptr()))
    return out.cpu().numpy()


def smooth_layer(layer, kernel: SmoothingKernel) -> np.ndarray:
    """Two separable zero-padded passes along x then y (patch_synthesis.py:206-209)."""
    return convolve1d_zero(convolve1d_zero(layer, kernel.taps, axis=0), kernel.taps, axis=1)


def finish_field(heights, patch: PatchRegion, choppiness: float = 0.0,
                 displacement_scale: float = 1.0) -> HeightField:
    """Clamped-border FD normals and optional choppy displacement (:323-340)."""
    h = torch.as_tensor(heights)
    if not h.is_cuda:
        h = h.to(torch.device("cuda", torch.cuda.current_device()))
    h = h.to(torch.float32).contiguous()
    if not bool(torch.isfinite(h).all()):
        raise ValueError("patch heights contain non-finite values")
    nx, ny = h.shape
    spacing = patch.l1 / (nx - 1)
    normal = torch.empty((nx, ny, 3), dtype=torch.float32, device=h.device)
    disp = torch.zeros((nx, ny, 2), dtype=torch.float32, device=h.device)
    args = N.HsFinishArgs(nx=nx, ny=ny, spacing=spacing, chop_scale=-choppiness * displacement_scale,
                          height=N.ptr(h), normal=N.ptr(normal), disp=N.ptr(disp) if choppiness != 0.0 else 0)
    N.call("hs_finish", args, stream_ptr())
    return HeightField(resolution=nx, origin=patch.min_corner.copy(), spacing=spacing, height=h,
                       displacement=disp, normal=normal, periodic=False)


class LayerStack:
    """Texel-exact (factor 1) per-bucket accumulation grids over a patch
    (patch_synthesis.py:133-162): padded raw layers in device memory (the
    synthesis workspace's), splatted by `accumulate` (hs_splat), smoothed and
    summed by `smooth_and_sum` (hs_smooth + hs_compose).  `layers` /
    `layer_view` read them back as numpy (node-centred; the crop of layer i is
    [pad_i : pad_i + res, pad_i : pad_i + ny])."""

    def __init__(self, patch: PatchRegion, resolution: int, kernels: list):
        if resolution < 2:
            raise ConfigError(f"patch resolution must be >= 2, got {resolution}")
        self.patch = patch
        self.resolution = resolution
        self.texel_size = patch.l1 / (resolution - 1)
        self.ny = int(round(patch.l2 / self.texel_size)) + 1
        self.kernels = list(kernels)
        self.pads = [k.half_width + 1 for k in self.kernels]
        dev = torch.device("cuda", torch.cuda.current_device())
        self.ws = SynthWorkspace([patch], [resolution], [as_plan(self.kernels)], dev)
        self.clamped_splats = 0

    def _layer(self, i: int) -> torch.Tensor:
        L = self.ws.pack.layers[i]
        return self.ws.raw[L.raw_off:L.raw_off + L.wx * L.raw_pitch].view(L.wx, L.raw_pitch)[:, :L.wy]

    @property
    def layers(self) -> list:
        return [self._layer(i).double().cpu().numpy() for i in range(len(self.kernels))]

    def layer_view(self, i: int) -> np.ndarray:
        p = self.pads[i]
        return self._layer(i)[p:p + self.resolution, p:p + self.ny].double().cpu().numpy()

    def clear(self) -> None:
        self.ws.raw.zero_()
        self.clamped_splats = 0


def accumulate(particles: ParticleSet, patch: PatchRegion, stack: LayerStack) -> LayerStack:
    """Splat every particle's signed amplitude into its bucket's layer
    (patch_synthesis.py:189-203): one hs_splat launch."""
    nb = len(stack.kernels)
    particles.materialize(nb)
    if len(particles) == 0:
        return stack
    ws = stack.ws
    dev = ws.device
    pst = structs_to_device([patch_struct(patch, stack.resolution, grid_base=0, layer_base=0)], dev)
    count = torch.from_numpy(particles.counts.astype(np.int32)).to(dev)
    ws.clamped.zero_()
    N.call("hs_splat", N.HsSplatArgs(n_patches=1, nb=nb, patches=N.ptr(pst), pool=particles.pool_struct(),
                                     count=N.ptr(count), raw_layers=N.ptr(ws.raw), raw_layers_len=ws.pack.raw_len,
                                     layers=N.ptr(ws.layers), clamped=N.ptr(ws.clamped),
                                     max_count=int(particles.counts.sum())), stream_ptr())
    stack.clamped_splats += int(ws.clamped.item())
    return stack


def smooth_and_sum(stack: LayerStack, kernels: list | None = None) -> torch.Tensor:
    """Smooth each layer, apply the gain, sum to the (res, ny) grid
    (patch_synthesis.py:212-224) -- hs_smooth + hs_compose over the stack's
    layers.  Other `kernels` must keep each layer's half width (the padding
    the layers were laid out with)."""
    kernels = list(kernels) if kernels is not None else stack.kernels
    if len(kernels) != len(stack.kernels):
        raise ConfigError("need exactly one kernel per layer")
    ws = stack.ws
    if kernels is not stack.kernels:
        if any(k.half_width != s.half_width for k, s in zip(kernels, stack.kernels)):
            raise ConfigError("smooth_and_sum kernels must keep the stack's half widths")
        other = SynthWorkspace([stack.patch], [stack.resolution], [as_plan(kernels)], ws.device)
        other.raw.copy_(ws.raw)
        ws = other
    dev = ws.device
    heights = torch.zeros((stack.resolution, stack.ny), dtype=torch.float32, device=dev)
    pst = structs_to_device(ws.patch_structs(), dev)
    st = stream_ptr()
    N.call("hs_smooth", ws.smooth_args(), st)
    N.call("hs_compose", N.HsComposeArgs(
        n_patches=1, nb=len(kernels), patches=N.ptr(pst), layers=N.ptr(ws.layers), smooth_layers=N.ptr(ws.smooth),
        tile_info=N.ptr(ws.compose_info), total_tiles=ws.compose_tiles, bg_height=0, bg_normal=0, bg_n=0,
        bg_spacing=1.0, patch_height=N.ptr(heights), patch_normal=0, blend_height=0, blend_normal=0, blend_mode=0,
        interior_sumsq=0, interior_count=0), st)
    return heights
