"""Host-side packing of bucket / patch / layer descriptors into the C ABI
structs (include/hybridsea_b200.h) and their device copies.

Everything here runs once per configuration (init time); the per-frame path
only passes the resulting device pointers.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError

TILE = 32          # smooth wide-kernel tile edge (csrc/synth.cu SM_TILE)
TILE_X, TILE_Y = 32, 64   # fused smooth tile (csrc/synth.cu SM_TX, SM_TY)
COMPOSE_TILE = 30  # compose output tile edge (csrc/compose.cu: 32 x 32 haloed heights)


def stream_ptr() -> int:
    return int(torch.cuda.current_stream().cuda_stream)


def to_device_bytes(arr: np.ndarray, device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device)


def bucket_structs(table, params, s1d=None) -> list:
    """HsBucket per bucket: the array views the kernels read (spectrum.py:233-257)
    plus S_J(omega_b) in fp64 (particles.py:262)."""
    from .spectrum import evaluate_1d
    s_arr, c_arr = table.spread_params
    s1d = evaluate_1d(params, table.omegas) if s1d is None else np.asarray(s1d, dtype=float)
    out = []
    for k, b in enumerate(table.buckets):
        out.append(N.HsBucket(b.omega, b.delta_omega, b.radius, b.speed, float(s1d[k]),
                              float(s_arr[k]), float(c_arr[k]), 0.0))
    return out


def half_rates(patch, omegas: np.ndarray, dt: float, g: float) -> np.ndarray:
    """(nb, 4) per-side group quota per step (particles.py:237-241), computed
    with the reference's fp64 operation order so the device ledger is exact."""
    hr = np.empty((len(omegas), 4))
    for side in range(4):
        pair = 4.0 * patch.side_length(side) * dt * omegas ** 3 / (math.pi ** 3 * g)
        hr[:, side] = 0.5 * pair
    return hr


def max_groups_per_step(hr: np.ndarray) -> int:
    """Upper bound of groups emitted in one step: each (bucket, side) cell can
    emit floor(acc + hr) <= floor(hr) + 1 with acc in [0, 1)."""
    return int(np.sum(np.floor(hr) + 1.0))


def grid_dims(patch, res: int) -> tuple[float, int]:
    texel = patch.l1 / (res - 1)
    return texel, int(round(patch.l2 / texel)) + 1


@dataclass
class LayerPack:
    """Packed layers of several patches (one HsLayer per (patch, bucket))."""
    layers: list               # HsLayer structs
    taps: np.ndarray           # float32
    raw_len: int               # floats
    smooth_len: int            # floats
    smooth_tile_prefix: np.ndarray   # int32 [n_layers + 1] fused tiles
    max_H: int
    smooth_tile_info: np.ndarray = None   # int32 [tiles, 3]: layer, cx0, cy0 (fused path)
    mid_len: int = 0           # floats of the wide-kernel intermediate
    xtile_prefix: np.ndarray = None
    ytile_prefix: np.ndarray = None
    max_H_wide: int = 0
    n_tickets: int = 0         # layer-group tile tickets (HsSmoothArgs.tickets)


def _tiles(a: int, b: int) -> int:
    return (-(-a // TILE)) * (-(-b // TILE))


GROUP_LAYERS = os.environ.get("HS_GROUP_LAYERS", "1") != "0"


def _groups(factors: list, wide: list) -> list[int]:
    """HsLayer.group per layer: runs of consecutive fused coarse layers with
    one factor (hence one coarse grid): n on the first, -k on the k-th
    following member, 1 on lone layers.  Full-resolution (f = 1) layers stay
    apart: the compose reads them as plain coalesced rows anyway."""
    out = [1] * len(factors)
    if not GROUP_LAYERS:
        return out
    i = 0
    while i < len(factors):
        j = i + 1
        while j < len(factors) and factors[j] == factors[i] > 1 and not wide[i] and not wide[j]:
            j += 1
        if j - i > 1:
            out[i] = j - i
            out[i + 1:j] = [-k for k in range(1, j - i)]
        i = j
    return out


def pack_layers(plans: list, grids: list[tuple[int, int]]) -> LayerPack:
    """Lay out the per-bucket decimated layers of every patch (LayerPlan,
    patch_synthesis.py:227-258; layer dims :306-308).  Kernels wider than
    HS_SMOOTH_FUSED_MAX_H take the two-pass path through a scratch layer.
    Consecutive fused coarse layers with one factor form a group
    (HsLayer.group): hs_smooth folds them into the first layer's crop, which
    the compose upsamples once."""
    layers, taps, prefix, xpre, ypre = [], [], [0], [0], [0]
    raw_off = sm_off = tap_off = mid_off = tickets = 0
    max_h, max_hw = 1, 0
    for plan, (res, ny) in zip(plans, grids):
        factors = list(plan.factors)
        wides = [k.half_width > N.HS_SMOOTH_FUSED_MAX_H for k in plan.kernels]
        groups = _groups(factors, wides)
        ticket = -1
        for k, f, wide, grp in zip(plan.kernels, factors, wides, groups):
            pad = k.half_width + 1
            ncx = -((res - 1) // -f) + 1
            ncy = -((ny - 1) // -f) + 1
            wx, wy = ncx + 2 * pad, ncy + 2 * pad
            if len(k.taps) > min(wx, wy):
                raise ConfigError(f"kernel of {len(k.taps)} taps wider than grid axis of {min(wx, wy)}")
            if wide and k.half_width > 780:
                raise ConfigError(f"kernel half width {k.half_width} exceeds the device limit of 780 texels")
            pitch = -(-wy // 4) * 4                  # 16-byte rows (vector splat reductions)
            tiles = (-(-ncx // TILE_X)) * (-(-ncy // TILE_Y))
            if grp > 1:                               # a group's tickets: one per tile
                ticket, tickets = tickets, tickets + tiles
            elif grp == 1:
                ticket = -1
            layers.append(N.HsLayer(raw_off, sm_off, f, k.half_width, pad, ncx, ncy, wx, wy, tap_off,
                                    float(k.gain), mid_off if wide else -1, pitch, grp, ticket, 0))
            taps.append(np.asarray(k.taps, dtype=np.float32))
            raw_off += wx * pitch                     # stays a multiple of 4
            sm_off += -(-(ncx * ncy) // 4) * 4          # 16-byte aligned crops (vector stores)
            tap_off += len(k.taps)
            if wide:
                mid_off += ncx * wy
                max_hw = max(max_hw, k.half_width)
            else:
                max_h = max(max_h, k.half_width)
            prefix.append(prefix[-1] + (0 if wide else tiles))
            xpre.append(xpre[-1] + (_tiles(ncx, wy) if wide else 0))
            ypre.append(ypre[-1] + (_tiles(ncx, ncy) if wide else 0))
    info = [(l, tx * TILE_X, ty * TILE_Y) for l, L in enumerate(layers) if L.mid_off < 0
            for tx in range(-(-L.ncx // TILE_X)) for ty in range(-(-L.ncy // TILE_Y))]
    # group tiles first (their last member folds the group), then the largest
    # kernels: the long-tap tiles start earliest
    info.sort(key=lambda t: (layers[t[0]].group in (0, 1), -layers[t[0]].H))
    return LayerPack(layers, np.concatenate(taps) if taps else np.zeros(0, np.float32), raw_off, sm_off,
                     np.array(prefix, dtype=np.int32), max_h, np.array(info, dtype=np.int32).reshape(-1, 3),
                     mid_off, np.array(xpre, dtype=np.int32), np.array(ypre, dtype=np.int32), max_hw,
                     n_tickets=tickets)


def compose_tile_info(grids: list[tuple[int, int]]) -> np.ndarray:
    """[tiles, 3] int32: patch, i0, j0 of every compose output tile."""
    T = COMPOSE_TILE
    info = [(p, tx * T, ty * T) for p, (res, ny) in enumerate(grids)
            for tx in range(-(-res // T)) for ty in range(-(-ny // T))]
    return np.array(info, dtype=np.int32).reshape(-1, 3)


def patch_struct(region, res: int, *, pool_base=0, pool_capacity=0, stage_base=0, stage_capacity=0,
                 grid_base=0, layer_base=0, track=-1) -> N.HsPatch:
    texel, ny = grid_dims(region, res)
    lo = region.min_corner
    hi = region.max_corner
    return N.HsPatch(float(lo[0]), float(lo[1]), float(hi[0]), float(hi[1]), float(region.l1),
                     float(region.l2), float(region.margin), float(texel), int(pool_base), int(stage_base),
                     int(grid_base), int(pool_capacity), int(stage_capacity), int(res), int(ny),
                     int(layer_base), int(track), float(lo[0]), float(lo[1]))


def structs_to_device(items: list, device) -> torch.Tensor:
    return to_device_bytes(N.struct_array_bytes(items), device)
