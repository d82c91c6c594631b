"""The multi-GPU composite exchange on one GPU: a 1-rank NCCL group runs the
same code path bench.py uses for N > 1 (sharding.CompositeGather packed from
the frame composite, all-gathered, pasted), captured into the frame graphs
through Simulation.post_frame.  The gathered payload must be this rank's
patch boxes of the frame composite, and the composite must still equal the
on-demand stitched_heights (harness.py:219-241)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_composite_exchange_one_rank_nccl(cuda):
    import torch
    import torch.distributed as dist
    from paper_2511_02852_b200 import Simulation, scenes
    from paper_2511_02852_b200.sharding import CompositeGather
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    try:
        cfg = scenes.c2(frames=40)
        sim = Simulation(cfg, device=cuda, compact_period=16)
        gather = CompositeGather(sim.box_np.reshape(-1, 4), cfg.fft_n, 1, device=cuda)

        def exchange():
            gather.pack(sim.composite_frame)
            gather.gather()
            gather.paste_others(sim.composite_frame)
        exchange()                                  # communicator set up outside capture
        torch.cuda.synchronize()
        sim.post_frame = exchange
        sim.prepare_graphs()
        for _ in range(cfg.frames):                 # graph replays past a compaction
            sim.step(stats=False)
        torch.cuda.synchronize()
        comp = sim.composite_frame.clone().cpu().numpy()
        total = gather.local_total
        payload = gather.recv[:total].cpu().numpy()
        boxes, pre = sim.box_np.reshape(-1, 4), sim.box_prefix_np
        for p, (i0, i1, j0, j1) in enumerate(boxes):
            np.testing.assert_array_equal(payload[pre[p]:pre[p + 1]].reshape(i1 - i0, j1 - j0),
                                          comp[i0:i1, j0:j1])
        want = sim.stitched_heights().cpu().numpy()
        assert np.abs(comp - want).max() <= 1e-6 * np.abs(want).max()
        sim.check()
    finally:
        dist.destroy_process_group()
