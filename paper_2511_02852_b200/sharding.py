"""Multi-GPU sharding of the hybrid step.

Patches are independent given the shared bucket table (no particle crosses
patches, reference SPEC.md:231), so a scene shards by patch: rank r owns a
contiguous block of patches, each with its own pool, ledger and Philox
stream (key = (seed, global patch id)), and runs the (cheap, replicated)
background.  The only exchange is the per-frame gather of blended patch
tiles into the composite, one NCCL all-gather over NVLink.  FFT cascades
(C4) would be assigned round-robin.

The host logic here (partitioning, tile packing, composite assembly) is
device-agnostic and covered by `gloo` world-size-2 tests on CPU.
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


def gather_tiles(local: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """All-gather equal-size flattened tiles: returns [world, numel]."""
    flat = local.reshape(-1).contiguous()
    out = torch.empty(world * flat.numel(), dtype=flat.dtype, device=flat.device)   # flat: gloo and nccl
    dist.all_gather_into_tensor(out, flat, group=group)
    return out.view(world, flat.numel())


def assemble(tiles: torch.Tensor, shapes: list[tuple[int, int]]) -> list[torch.Tensor]:
    """Split gathered rows back into per-patch (res, ny) views."""
    return [tiles[k, : r * c].view(r, c) for k, (r, c) in enumerate(shapes)]


class CompositeGather:
    """Per-frame composite exchange at FFT resolution (SURVEY 8(e)'s
    alternative to shipping native-resolution tiles): every rank resamples
    its own patches' boxes of the stitched grid (harness.py:219-241;
    `Simulation.composite_boxes`), one all-gather moves those values
    (C3 weak scaling: a 67 x 67 box, 18 KB per rank, instead of a 4 MB tile),
    and every rank pastes all boxes over the background.

    Box geometry is exchanged once at construction.  Where boxes of
    different patches overlap, the later patch in global order wins, as in
    the reference's loop; each rank samples only its own patches, so an
    overlap across ranks is exact only where the patches do not both cover
    the texel (seeded layouts keep patches apart)."""

    def __init__(self, boxes, n: int, world: int, group=None, device=None):
        import numpy as np
        self.n, self.world, self.group = n, world, group
        boxes = np.asarray(boxes, dtype=np.int64).reshape(-1, 4)
        sizes = (boxes[:, 1] - boxes[:, 0]).clip(0) * (boxes[:, 3] - boxes[:, 2]).clip(0)
        self.local_total = int(sizes.sum())
        loc = [(np.arange(b[0], b[1])[:, None] * n + np.arange(b[2], b[3])[None, :]).ravel()
               for b in boxes if b[1] > b[0] and b[3] > b[2]]
        self.local_index = torch.from_numpy(np.concatenate(loc) if loc else np.zeros(0, np.int64)).to(device)
        meta = torch.tensor([len(boxes), self.local_total], dtype=torch.int64, device=device)
        metas = torch.empty(world * 2, dtype=torch.int64, device=device)
        dist.all_gather_into_tensor(metas, meta, group=group)
        metas = metas.view(world, 2).cpu().numpy()
        max_p = int(metas[:, 0].max())
        self.per_rank = max(1, int(metas[:, 1].max()))
        padded = torch.full((max(max_p, 1), 4), -1, dtype=torch.int64, device=device)
        if len(boxes):
            padded[: len(boxes)] = torch.from_numpy(boxes).to(device)
        allb = torch.empty(world * padded.numel(), dtype=torch.int64, device=device)
        dist.all_gather_into_tensor(allb, padded.reshape(-1), group=group)
        allb = allb.view(world, -1, 4).cpu().numpy()
        pos, dst, own = [], [], []
        me = dist.get_rank(group)
        for r in range(world):
            off = r * self.per_rank
            for b in allb[r, : metas[r, 0]]:
                i0, i1, j0, j1 = (int(v) for v in b)
                if i1 <= i0 or j1 <= j0:
                    continue
                ii, jj = np.meshgrid(np.arange(i0, i1), np.arange(j0, j1), indexing="ij")
                dst.append((ii * n + jj).ravel())
                pos.append(off + np.arange(ii.size))
                own.append(np.full(ii.size, r == me))
                off += ii.size
        dst = np.concatenate(dst) if dst else np.zeros(0, np.int64)
        pos = np.concatenate(pos) if pos else np.zeros(0, np.int64)
        own = np.concatenate(own) if own else np.zeros(0, bool)
        # per composite texel: the payload slot that covers it (later boxes win,
        # as in the reference loop), or none -> background
        src = np.full(n * n, -1, np.int64)
        last = len(dst) - 1 - np.unique(dst[::-1], return_index=True)[1]   # last occurrence per texel
        src[dst[last]] = pos[last]
        # the other ranks' winning nodes, for pasting into this rank's own frame composite
        keep = last[~own[last]]
        self.other_dst = torch.from_numpy(dst[keep]).to(device)
        self.other_pos = torch.from_numpy(pos[keep]).to(device)
        self._other_vals = torch.empty(len(keep), dtype=torch.float32, device=device)
        self.covered = torch.from_numpy(src >= 0).to(device)
        self.src = torch.from_numpy(np.maximum(src, 0)).to(device)
        self.send = torch.zeros(self.per_rank, dtype=torch.float32, device=device)
        self.recv = torch.empty(world * self.per_rank, dtype=torch.float32, device=device)
        self.grid = torch.empty(n * n, dtype=torch.float32, device=device)
        self._picked = torch.empty(n * n, dtype=torch.float32, device=device)

    def pack(self, composite: torch.Tensor) -> None:
        """Fill `send` with this rank's box nodes of its own frame composite
        (the grid hs_compose blended its patches into)."""
        if self.local_total:
            torch.index_select(composite.reshape(-1), 0, self.local_index, out=self.send[: self.local_total])

    def gather(self) -> torch.Tensor:
        """All-gather every rank's `send[:local_total]` (filled by
        `Simulation.composite_boxes(send)`): afterwards every rank holds every
        patch box of the stitched grid.  Fixed buffers and no host
        synchronisation, so it is captured into the frame's CUDA graph
        (`Simulation.post_frame`)."""
        dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
        return self.recv

    def assemble(self, background: torch.Tensor) -> torch.Tensor:
        """Paste the gathered boxes over `background` (n x n): the full
        composite (on demand, like the reference's stitched_heights)."""
        torch.index_select(self.recv, 0, self.src, out=self._picked)
        torch.where(self.covered, self._picked, background.reshape(-1), out=self.grid)
        return self.grid.view(self.n, self.n)

    def paste_others(self, composite: torch.Tensor) -> torch.Tensor:
        """Paste the other ranks' gathered boxes into this rank's own frame
        composite (which already holds the background and its own boxes)."""
        if self.other_dst.numel():
            torch.index_select(self.recv, 0, self.other_pos, out=self._other_vals)
            composite.view(-1).index_copy_(0, self.other_dst, self._other_vals)
        return composite

    def exchange(self, background: torch.Tensor) -> torch.Tensor:
        """gather() + assemble()."""
        self.gather()
        return self.assemble(background)


class TileGather:
    """Per-frame NCCL all-gather of every rank's blended patch tiles (the
    composite exchange of SURVEY 8(e)): each rank contributes its patches'
    blend heights, which are contiguous in the per-device grid buffer, padded
    to the largest rank's share (block sizes differ by at most one patch)."""

    def __init__(self, sim, world: int, group=None, max_local: int | None = None):
        self.sim = sim
        self.world = world
        self.group = group
        self.local = int(sim.synth.grid_base[-1])           # floats of this rank's tiles
        self.per_rank = max_local if max_local is not None else self.local
        self.send = torch.zeros(self.per_rank, dtype=torch.float32, device=sim.device)
        self.out = torch.empty(world * self.per_rank, dtype=torch.float32, device=sim.device)

    def exchange(self) -> torch.Tensor:
        h = self.sim.blend_h[: self.local]
        if self.local == self.per_rank:
            src = h
        else:
            self.send[: self.local].copy_(h)
            src = self.send
        dist.all_gather_into_tensor(self.out, src, group=self.group)
        return self.out.view(self.world, -1)
