"""Multi-process (gloo, world size 2) tests of the patch sharding host logic
(SURVEY 8(e)): partitioning, per-patch Philox keys, the tile all-gather and
composite assembly, and that integer results (per-patch bucket counts) of a
sharded run equal the single-process run.  CPU only.
"""
from __future__ import annotations

import os
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2511_02852_b200 import scenes  # noqa: E402
from paper_2511_02852_b200.sharding import (CompositeGather, assemble, cascade_owner, gather_tiles,  # noqa: E402
                                            partition, shard_config)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank: int, world: int, port: int) -> None:
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _tile(pid: int, shape) -> torch.Tensor:
    """Deterministic stand-in for a blended patch tile of global patch pid."""
    g = torch.Generator().manual_seed(1000 + pid)
    return torch.randn(shape, generator=g)


def _small_scene(n_patches: int):
    """Small wp-only multi-patch scene: 48 m patches on 96^2 grids, 6 buckets."""
    cfg = scenes.c2(n_omega=6, n_theta=4, fft_n=64, mode="wp-only")
    from dataclasses import replace
    pcs = tuple(replace(p, size=(48.0, 48.0), res=96, margin=4.0) for p in cfg.patches[:n_patches])
    return replace(cfg, patches=pcs).validate()


# ----------------------------------------------------------------- workers --
def _gather_worker(rank: int, world: int, port: int, n_patches: int, out_dir: str) -> None:
    _init(rank, world, port)
    try:
        shape = (24, 24)
        blocks = partition(n_patches, world)
        width = max(len(b) for b in blocks)
        # each rank packs its block's tiles into a fixed-width slab (padding slots zero)
        slab = torch.zeros((width, shape[0] * shape[1]))
        for k, pid in enumerate(blocks[rank]):
            slab[k] = _tile(pid, shape).reshape(-1)
        got = gather_tiles(slab, world)                     # [world, width * numel]
        got = got.view(world, width, -1)
        tiles = torch.cat([got[r, : len(blocks[r])] for r in range(world)])
        views = assemble(tiles, [shape] * n_patches)
        for pid, v in enumerate(views):
            assert torch.equal(v, _tile(pid, shape)), f"rank {rank}: tile {pid} differs after the gather"
        open(os.path.join(out_dir, f"ok{rank}"), "w").close()
    finally:
        dist.destroy_process_group()


# boxes (i0, i1, j0, j1) of the global patch list on a 16 x 16 composite;
# patches 1 and 2 overlap in row 6-7 (the later one must win)
_BOXES = [(0, 4, 0, 5), (5, 8, 3, 9), (6, 10, 8, 12), (12, 16, 12, 16)]


def _box_values(pid: int) -> np.ndarray:
    i0, i1, j0, j1 = _BOXES[pid]
    return (100.0 * (pid + 1) + np.arange((i1 - i0) * (j1 - j0))).astype(np.float32)


def _composite_worker(rank: int, world: int, port: int, out_dir: str) -> None:
    _init(rank, world, port)
    try:
        block = partition(len(_BOXES), world)[rank]
        g = CompositeGather([_BOXES[k] for k in block], 16, world)
        vals = np.concatenate([_box_values(k) for k in block])
        g.send[: len(vals)] = torch.from_numpy(vals)
        bg = torch.full((16, 16), -1.0)
        grid = g.exchange(bg).numpy()
        np.save(os.path.join(out_dir, f"grid{rank}.npy"), grid)
        # the in-place route: own frame composite (background + own boxes) + others pasted
        own = torch.full((16, 16), -1.0)
        for k in block:
            i0, i1, j0, j1 = _BOXES[k]
            own[i0:i1, j0:j1] = torch.from_numpy(_box_values(k).reshape(i1 - i0, j1 - j0))
        np.save(os.path.join(out_dir, f"own{rank}.npy"), g.paste_others(own).numpy())
    finally:
        dist.destroy_process_group()


def _oracle_worker(rank: int, world: int, port: int, frames: int, out_dir: str) -> None:
    _init(rank, world, port)
    try:
        from oracle.scene_ref import OracleScene
        cfg = _small_scene(3)
        local, ids, keys = shard_config(cfg, rank, world)
        assert keys == [(cfg.seed, k) for k in ids]
        sc = local.scene_dict()
        sc["patch_ids"] = ids
        scene = OracleScene(sc)
        counts = None
        for _ in range(frames):
            counts = scene.step(dt=0.1, synth=False)["counts"]
        gathered = [None] * world
        dist.all_gather_object(gathered, (ids, counts.tolist()))
        if rank == 0:
            np.save(os.path.join(out_dir, "sharded.npy"),
                    np.array([row for _, c in gathered for row in c], dtype=np.int64))
            np.save(os.path.join(out_dir, "ids.npy"), np.array([i for ids_r, _ in gathered for i in ids_r]))
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------------- tests --
def test_partition_is_contiguous_and_balanced():
    for n in (0, 1, 3, 8, 64, 65):
        for w in (1, 2, 4, 8):
            blocks = partition(n, w)
            assert [i for b in blocks for i in b] == list(range(n))
            sizes = [len(b) for b in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        partition(4, 0)
    assert [cascade_owner(c, 2) for c in range(3)] == [0, 1, 0]


def test_shard_config_keeps_global_keys():
    cfg = scenes.c4()
    seen = []
    for r in range(4):
        local, ids, keys = shard_config(cfg, r, 4)
        assert len(local.patches) == len(ids) == 2
        assert keys == [(cfg.seed, k) for k in ids]
        assert tuple(local.patches) == tuple(cfg.patches[k] for k in ids)
        seen += ids
    assert seen == list(range(len(cfg.patches)))


def test_gloo_tile_gather_world2():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gather_worker, args=(2, _free_port(), 3, d), nprocs=2, join=True)
        assert os.path.exists(os.path.join(d, "ok0")) and os.path.exists(os.path.join(d, "ok1"))


def test_sharded_counts_equal_single_process_world2():
    """Per-patch bucket counts after a few frames: 2-rank sharded oracle run
    == single-process run (integer results must not depend on sharding)."""
    from oracle.scene_ref import OracleScene
    frames = 12
    cfg = _small_scene(3)
    single = OracleScene(cfg.scene_dict())
    for _ in range(frames):
        ref = single.step(dt=0.1, synth=False)["counts"]
    assert ref.sum() > 0
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_oracle_worker, args=(2, _free_port(), frames, d), nprocs=2, join=True)
        got = np.load(os.path.join(d, "sharded.npy"))
        ids = np.load(os.path.join(d, "ids.npy"))
    assert ids.tolist() == [0, 1, 2]
    np.testing.assert_array_equal(got, ref)


def test_gloo_composite_gather_world2():
    """The FFT-resolution box exchange: both ranks assemble the composite the
    reference's stitched_heights loop would (background, then every patch box
    in global order, later boxes overwriting earlier ones)."""
    want = np.full((16, 16), -1.0, np.float32)
    for pid, (i0, i1, j0, j1) in enumerate(_BOXES):
        want[i0:i1, j0:j1] = _box_values(pid).reshape(i1 - i0, j1 - j0)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_composite_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        for r in range(2):
            np.testing.assert_array_equal(np.load(os.path.join(d, f"grid{r}.npy")), want)
            np.testing.assert_array_equal(np.load(os.path.join(d, f"own{r}.npy")), want)
