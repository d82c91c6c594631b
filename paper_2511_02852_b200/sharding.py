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
