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
    local = replace(cfg, patches=tuple(pcs[k] for k in block))
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
    """Per-frame all-gather of every rank's blended tile of its first patch
    (bench.py weak-scaling workload: one equal-size patch per rank)."""

    def __init__(self, sim, world: int, group=None):
        self.sim = sim
        self.world = world
        self.group = group
        res, ny = sim.synth.grids[0]
        self.shape = (res, ny)
        self.out = torch.empty(world * res * ny, dtype=torch.float32, device=sim.device)

    def exchange(self) -> torch.Tensor:
        h = self.sim.blended_tile(0)[0].reshape(-1)
        dist.all_gather_into_tensor(self.out, h, group=self.group)
        return self.out.view(self.world, -1)
