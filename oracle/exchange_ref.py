"""The multi-GPU composite exchange protocol -- TEST INFRASTRUCTURE ONLY.

numpy restatement of hs_box_pack / hs_box_paste (csrc/synth.cu): a patch's
box of the FFT-resolution stitched grid is rows/columns
[floor(min / spacing), ceil(max / spacing) + 1) clipped to [0, n]
(`Simulation.stitched_heights`, reference harness.py:230-233); pasting the
boxes of all patches in global order over a composite, the later box
winning where two overlap, is the reference's loop (harness.py:234-240).
Payload slot: 4 header words (i0, i1, j0, j1 as int32 bits) + bw x bh values.
"""
from __future__ import annotations

import math

import numpy as np


def box_of(x0: float, y0: float, l1: float, l2: float, n: int, spacing: float) -> tuple:
    lo = np.clip(np.floor(np.array([x0, y0]) / spacing).astype(int), 0, n)
    hi = np.clip(np.ceil(np.array([x0 + l1, y0 + l2]) / spacing).astype(int) + 1, 0, n)
    return int(lo[0]), int(hi[0]), int(lo[1]), int(hi[1])


def pack_slot(slot: np.ndarray, composite: np.ndarray, box, bw: int, bh: int) -> None:
    """Write one slot (float32 view of 4 + bw*bh words) from `composite`."""
    i0, i1, j0, j1 = box
    slot[:4] = np.array([i0, i1, j0, j1], dtype=np.int32).view(np.float32)
    vals = slot[4:].reshape(bw, bh)
    vals[: i1 - i0, : j1 - j0] = composite[i0:i1, j0:j1]


def unpack_slot(slot: np.ndarray, bw: int, bh: int):
    i0, i1, j0, j1 = (int(v) for v in np.asarray(slot[:4], dtype=np.float32).view(np.int32))
    return (i0, i1, j0, j1), slot[4:].reshape(bw, bh)[: max(i1 - i0, 0), : max(j1 - j0, 0)]


def paste(composite: np.ndarray, payload: np.ndarray, slots: int, world: int, rank: int, bw: int, bh: int):
    """Every other rank's boxes into `composite` in slot order (later wins)."""
    stride = 4 + bw * bh
    rows = payload.reshape(world * slots, stride)
    boxes = [unpack_slot(r, bw, bh) for r in rows]
    out = composite.copy()
    for s, ((i0, i1, j0, j1), vals) in enumerate(boxes):
        if s // slots == rank or i1 <= i0 or j1 <= j0:
            continue
        keep = np.ones((i1 - i0, j1 - j0), bool)
        for (a0, a1, b0, b1), _ in boxes[s + 1:]:
            ii = np.arange(i0, i1)[:, None]
            jj = np.arange(j0, j1)[None, :]
            keep &= ~((ii >= a0) & (ii < a1) & (jj >= b0) & (jj < b1))
        out[i0:i1, j0:j1] = np.where(keep, vals, out[i0:i1, j0:j1])
    return out


def capacity(sizes, spacing: float) -> int:
    return max(int(math.ceil(float(l) / spacing)) + 3 for size in sizes for l in size)


__all__ = ["box_of", "pack_slot", "unpack_slot", "paste", "capacity"]
