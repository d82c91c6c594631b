"""Multi-GPU sharding of the hybrid step.

Patches are independent given the shared bucket table (no particle crosses
patches, reference SPEC.md:231), so a scene shards by patch: rank r owns a
contiguous block of patches, each with its own pool, ledger and Philox
stream (key = (seed, global patch id)).  FFT cascades (C4) are assigned
round-robin (`CascadeShard`: one all-gather of their height grids per frame);
a single background tile is replicated (it is needed at every rank's patch
nodes and costs less than its exchange).  The composite exchange is one
all-gather of every rank's FFT-resolution patch boxes (`BoxExchange`, packed
and pasted by hand-written kernels).

The host logic (partitioning, keys, payload layout, in-place gathers) is
covered by `gloo` world-size-2 tests on CPU; the kernels by GPU tests.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def partition(n_items: int, world: int) -> list[range]:
    """Contiguous blocks, sizes differing by at most one (C4: 8 patches over
    8 ranks -> one each; C5: 64 over 8 -> eight each)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    base, extra = divmod(n_items, world)
    out, start = [], 0
    for r in range(world):
        size = base + (1 if r < extra else 0)
        out.append(range(start, start + size))
        start += size
    return out


def shard_config(cfg, rank: int, world: int):
    """Rank `rank`'s share of a multi-patch scene: the config restricted to its
    contiguous patch block, the global ids of those patches and their Philox
    keys (seed, global id) -- pass the keys as `Simulation(rng_seed_keys=...)`
    so every patch draws the same stream as in a single-process run."""
    from dataclasses import replace
    pcs = tuple(cfg.patches)
    block = partition(len(pcs), world)[rank]
    # sources: those tracked by a local patch, plus every untracked one (it may
    # wander into any patch); track indices remapped to the local list
    tracked = {pc.track_source for pc in pcs if pc.track_source >= 0}
    keep = [j for j in range(len(cfg.sources))
            if j not in tracked or any(pcs[k].track_source == j for k in block)]
    remap = {j: i for i, j in enumerate(keep)}
    local_pcs = tuple(replace(pcs[k], track_source=remap.get(pcs[k].track_source, -1)) for k in block)
    local = replace(cfg, patches=local_pcs, sources=tuple(cfg.sources[j] for j in keep))
    ids = list(block)
    return local, ids, [(cfg.seed, k) for k in ids]


def cascade_owner(cascade: int, world: int) -> int:
    """Round-robin owner of an FFT cascade (C4: 3 cascades on ranks 0-2)."""
    return cascade % world


def box_capacity(patch_sizes, spacing: float) -> int:
    """Nodes per axis of the largest composite box a patch of these sizes can
    cover anywhere (harness.py:230-233: [floor(min/sp), ceil(max/sp) + 1))."""
    import math
    return max(int(math.ceil(float(l) / spacing)) + 3 for size in patch_sizes for l in size)


class BoxExchange:
    """Per-frame composite exchange at FFT resolution: each rank
    packs the stitched-grid box of each of its patches out of its own frame
    composite (hs_box_pack: boxes computed on the device from the patches'
    current synthesis rectangles, so tracking patches' boxes move with them),
    one in-place NCCL all-gather moves every rank's slots, and hs_box_paste
    writes the other ranks' boxes into this rank's composite, the later patch
    in global order winning where boxes overlap (the reference loop,
    harness.py:219-241).  C3 weak scaling: a 67 x 67 box per rank (18 KB)
    instead of a 4 MB native tile; C5: 64 boxes of 52 x 52.

    Payload: world x slots x (4 header words + bw*bh values); slot order is
    rank-major, i.e. global patch order (contiguous blocks, `partition`).
    Fixed buffers, no host synchronisation: `exchange` is captured into the
    frame graph (Simulation.post_frame)."""

    def __init__(self, n: int, spacing: float, slots: int, bw: int, bh: int, world: int, rank: int,
                 group=None, device=None):
        self.n, self.spacing, self.slots, self.bw, self.bh = int(n), float(spacing), int(slots), int(bw), int(bh)
        self.world, self.rank, self.group = int(world), int(rank), group
        self.stride = 4 + self.bw * self.bh
        self.chunk = self.slots * self.stride
        self.payload = torch.zeros(self.world * self.chunk, dtype=torch.float32, device=device)

    @classmethod
    def for_scene(cls, cfg, sim, world: int, rank: int, group=None):
        """The exchange of `sim` (this rank's shard of the global scene `cfg`)."""
        spacing = cfg.fft_domain / cfg.fft_n
        slots = max(len(b) for b in partition(len(cfg.patches), world))
        cap = box_capacity([pc.size for pc in cfg.patches], spacing)
        return cls(cfg.fft_n, spacing, slots, cap, cap, world, rank, group, device=sim.device)

    @property
    def own(self) -> torch.Tensor:
        return self.payload[self.rank * self.chunk:(self.rank + 1) * self.chunk]

    def _args(self, sim):
        from . import _native as N
        return N.HsBoxArgs(n=self.n, spacing=self.spacing, composite=N.ptr(sim.composite_frame),
                           n_local=sim.n_patches, patches=N.ptr(sim.patches_dev), bw=self.bw, bh=self.bh,
                           payload=N.ptr(self.payload), slots=self.slots, world=self.world, rank=self.rank,
                           status=N.ptr(sim.status))

    def pack(self, sim) -> None:
        from . import _native as N
        from ._layout import stream_ptr
        N.call("hs_box_pack", self._args(sim), stream_ptr())

    def gather(self) -> torch.Tensor:
        """In-place all-gather of every rank's slots (NCCL on the GPU, gloo in the CPU tests)."""
        if self.world > 1:
            dist.all_gather_into_tensor(self.payload, self.own, group=self.group)
        return self.payload

    def paste(self, sim) -> None:
        from . import _native as N
        from ._layout import stream_ptr
        N.call("hs_box_paste", self._args(sim), stream_ptr())

    def exchange(self, sim) -> None:
        self.pack(sim)
        self.gather()
        self.paste(sim)

    def slots_host(self) -> list:
        """[(i0, i1, j0, j1, values (i1-i0, j1-j0))] of every slot (synchronises)."""
        import numpy as np
        raw = self.payload.cpu().numpy().reshape(self.world * self.slots, self.stride)
        out = []
        for row in raw:
            i0, i1, j0, j1 = (int(v) for v in row[:4].view(np.int32))
            vals = row[4:].reshape(self.bw, self.bh)[: max(i1 - i0, 0), : max(j1 - j0, 0)]
            out.append((i0, i1, j0, j1, vals.copy()))
        return out


class CascadeShard:
    """Round-robin FFT cascades over the ranks (C4: 3 cascades on ranks 0-2):
    rank r transforms the cascades c with c % world == r; one in-place
    all-gather of their height grids per frame gives every rank the whole
    summed background its patch blend and composite read (displacements and
    FFT-band statistics stay with the owner).  Cascade c's heights live at
    `buffer[c % world, c // world]`."""

    def __init__(self, n: int, n_cascades: int, world: int, rank: int, group=None, device=None):
        self.n, self.n_cascades, self.world, self.rank, self.group = n, n_cascades, world, rank, group
        self.per_rank = max(1, -(-n_cascades // world))
        self.buffer = torch.zeros((world, self.per_rank, n, n), dtype=torch.float32, device=device)

    def owned(self, c: int) -> bool:
        return cascade_owner(c, self.world) == self.rank

    def view(self, c: int) -> torch.Tensor:
        return self.buffer[cascade_owner(c, self.world), c // self.world]

    def gather(self) -> None:
        if self.world > 1:
            flat = self.buffer.view(-1)
            dist.all_gather_into_tensor(flat, self.buffer[self.rank].view(-1), group=self.group)
