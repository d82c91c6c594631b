"""The multi-GPU composite exchange on one GPU.

* A 1-rank NCCL group runs the exact path bench.py uses for N > 1
  (sharding.BoxExchange: hs_box_pack -> in-place NCCL all-gather ->
  hs_box_paste), captured into the frame graphs through
  Simulation.post_frame, on the C5 fleet slice whose patches track their
  ships: every frame's payload slots must be the boxes of the patches'
  *current* rectangles (oracle/exchange_ref.py restates the protocol), and the
  composite must still equal the on-demand stitched_heights
  (harness.py:219-241).
* Two shards of C2 on one device (no collective: the test moves the payload
  chunks itself, as the all-gather would): both shards' composites after the
  paste equal the single-process scene's composite.
* C4's cascades through sharding.CascadeShard at one rank equal the
  unsharded scene bit for bit (deterministic mode).
"""
import os
import socket

import numpy as np
import pytest

from oracle import exchange_ref

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_box_exchange_one_rank_nccl_tracking_patches(cuda):
    import torch
    import torch.distributed as dist
    from paper_2511_02852_b200 import Simulation, scenes
    from paper_2511_02852_b200.sharding import BoxExchange
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    try:
        cfg = scenes.c5(n_patches=4, frames=40)
        sim = Simulation(cfg, device=cuda, compact_period=16)
        ex = BoxExchange.for_scene(cfg, sim, 1, 0)
        ex.exchange(sim)                            # communicator set up outside capture
        torch.cuda.synchronize()
        sim.post_frame = lambda: ex.exchange(sim)
        sim.prepare_graphs()
        first = None
        for k in range(cfg.frames):                 # graph replays past a compaction
            sim.step(stats=False)
            if k == 0:
                torch.cuda.synchronize()
                first = [s[:4] for s in ex.slots_host()]
        torch.cuda.synchronize()
        sim.check()
        comp = sim.composite_frame.clone().cpu().numpy()
        slots = ex.slots_host()
        spacing = cfg.fft_domain / cfg.fft_n
        for k, r in enumerate(sim.current_regions()):
            box = exchange_ref.box_of(r.origin[0], r.origin[1], r.l1, r.l2, cfg.fft_n, spacing)
            assert slots[k][:4] == box, (k, slots[k][:4], box)
            i0, i1, j0, j1 = box
            np.testing.assert_array_equal(slots[k][4], comp[i0:i1, j0:j1])
        assert [s[:4] for s in slots] != first, "the ships moved: their boxes must have moved"
        want = sim.stitched_heights().cpu().numpy()
        assert np.abs(comp - want).max() <= 1e-6 * np.abs(want).max()
    finally:
        dist.destroy_process_group()


def test_two_shards_paste_to_the_single_process_composite(cuda):
    from paper_2511_02852_b200 import Simulation, scenes
    from paper_2511_02852_b200.sharding import BoxExchange, shard_config
    cfg = scenes.c2(frames=20)
    whole = Simulation(cfg, device=cuda)
    shards = []
    for r in range(2):
        local, _, keys = shard_config(cfg, r, 2)
        sim = Simulation(local.validate(), device=cuda, rng_seed_keys=keys)
        shards.append((sim, BoxExchange.for_scene(cfg, sim, 2, r)))
    for _ in range(cfg.frames):
        whole.step(stats=False)
        for sim, _ in shards:
            sim.step(stats=False)
    for sim, ex in shards:
        ex.pack(sim)
    (s0, e0), (s1, e1) = shards
    e0.payload[e1.chunk:].copy_(e1.own)             # what the all-gather moves
    e1.payload[:e0.chunk].copy_(e0.own)
    for sim, ex in shards:
        ex.paste(sim)
        sim.check()
    want = whole.composite_frame.cpu().numpy()
    scale = np.abs(want).max()
    np.testing.assert_array_equal(np.concatenate([s0.counts_host(), s1.counts_host()]), whole.counts_host())
    for sim, _ in shards:
        got = sim.composite_frame.cpu().numpy()
        assert np.abs(got - want).max() <= 1e-5 * scale     # float splat atomics: order-free sums


def test_cascade_shard_one_rank_matches_the_unsharded_scene(cuda):
    """C4's summed cascades through sharding.CascadeShard (the N > 1 path:
    owned transforms into the shard buffer, the background read from its
    views) at one rank: the frame's background sum, blended tiles and
    composite equal the unsharded scene's bit for bit."""
    import torch
    from paper_2511_02852_b200 import Simulation, scenes
    from paper_2511_02852_b200.sharding import CascadeShard
    # deterministic mode: the splat's fixed-point sums make both runs bitwise comparable
    cfg = scenes.c4(frames=12, patches=scenes.c4().patches[:2], deterministic=True)
    sims = [Simulation(cfg, device=cuda) for _ in range(2)]
    sims[1].shard_cascades(CascadeShard(cfg.fft_n, len(sims[1].cascades), 1, 0, device=cuda))
    for sim in sims:
        sim.prepare_graphs()
        for _ in range(cfg.frames):
            sim.step(stats=False)
    torch.cuda.synchronize()
    a, b = sims
    assert torch.equal(a.composite_frame, b.composite_frame)
    for p in range(a.n_patches):
        ha, _ = a.blended_tile(p)
        hb, _ = b.blended_tile(p)
        assert torch.equal(ha, hb)
    np.testing.assert_array_equal(a.counts_host(), b.counts_host())
