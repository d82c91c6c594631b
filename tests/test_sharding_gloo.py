"""Multi-process (gloo, world size 2) tests of the sharding host logic
(SURVEY 8(e)): partitioning, per-patch Philox keys, the composite box
exchange (BoxExchange payload, in-place all-gather, the later-box-wins paste
of oracle/exchange_ref.py that hs_box_paste restates), FFT cascade sharding
(CascadeShard), and that integer results (per-patch bucket counts) of a
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
from paper_2511_02852_b200.sharding import (BoxExchange, CascadeShard, cascade_owner,  # noqa: E402
                                            partition, shard_config)
from oracle import exchange_ref  # noqa: E402


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank: int, world: int, port: int) -> None:
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _small_scene(n_patches: int):
    """Small wp-only multi-patch scene: 48 m patches on 96^2 grids, 6 buckets."""
    cfg = scenes.c2(n_omega=6, n_theta=4, fft_n=64, mode="wp-only")
    from dataclasses import replace
    pcs = tuple(replace(p, size=(48.0, 48.0), res=96, margin=4.0) for p in cfg.patches[:n_patches])
    return replace(cfg, patches=pcs).validate()


# ----------------------------------------------------------------- workers --
# patch rectangles (x0, y0, l1, l2) on a 16 x 16 composite of spacing 1 m;
# the boxes of patches 1 and 2 overlap (the later one must win)
_RECTS = [(0.2, 0.5, 3.0, 3.5), (5.3, 3.1, 2.0, 4.6), (6.6, 7.2, 3.0, 3.0), (12.4, 12.1, 2.9, 2.2)]
_N, _SP = 16, 1.0


def _stitched(pid: int) -> np.ndarray:
    """Stand-in for a rank's frame composite over patch pid's box."""
    return (100.0 * (pid + 1) + np.arange(_N * _N).reshape(_N, _N)).astype(np.float32)


def _box_worker(rank: int, world: int, port: int, out_dir: str) -> None:
    _init(rank, world, port)
    try:
        block = partition(len(_RECTS), world)[rank]
        cap = exchange_ref.capacity([(r[2], r[3]) for r in _RECTS], _SP)
        ex = BoxExchange(_N, _SP, max(len(b) for b in partition(len(_RECTS), world)), cap, cap, world, rank)
        own = np.full((_N, _N), -1.0, np.float32)          # background + this rank's boxes (hs_compose)
        slots = ex.own.numpy().reshape(ex.slots, ex.stride)
        for k, pid in enumerate(block):
            box = exchange_ref.box_of(*_RECTS[pid], _N, _SP)
            i0, i1, j0, j1 = box
            own[i0:i1, j0:j1] = _stitched(pid)[i0:i1, j0:j1]
            exchange_ref.pack_slot(slots[k], own, box, cap, cap)
        ex.gather()                                         # in-place all-gather of the slots
        got = exchange_ref.paste(own, ex.payload.numpy(), ex.slots, world, rank, cap, cap)
        np.save(os.path.join(out_dir, f"grid{rank}.npy"), got)
    finally:
        dist.destroy_process_group()


def _cascade_worker(rank: int, world: int, port: int, out_dir: str) -> None:
    _init(rank, world, port)
    try:
        sh = CascadeShard(8, 3, world, rank)
        for c in range(3):
            if sh.owned(c):
                sh.view(c).fill_(10.0 * (c + 1))
        sh.gather()
        np.save(os.path.join(out_dir, f"casc{rank}.npy"), np.stack([sh.view(c).numpy() for c in range(3)]))
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


def test_gloo_box_exchange_world2():
    """The FFT-resolution composite exchange: both ranks end with the
    composite the reference's stitched_heights loop builds (background, then
    every patch box in global order, later boxes overwriting earlier ones)."""
    want = np.full((_N, _N), -1.0, np.float32)
    for pid, rect in enumerate(_RECTS):
        i0, i1, j0, j1 = exchange_ref.box_of(*rect, _N, _SP)
        want[i0:i1, j0:j1] = _stitched(pid)[i0:i1, j0:j1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_box_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        for r in range(2):
            np.testing.assert_array_equal(np.load(os.path.join(d, f"grid{r}.npy")), want)


def test_gloo_cascade_shard_world2():
    """Round-robin cascades (0, 2 on rank 0; 1 on rank 1): after the in-place
    gather every rank holds every cascade's heights."""
    assert [cascade_owner(c, 2) for c in range(3)] == [0, 1, 0]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_cascade_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        for r in range(2):
            got = np.load(os.path.join(d, f"casc{r}.npy"))
            for c in range(3):
                assert np.all(got[c] == 10.0 * (c + 1)), (r, c)
