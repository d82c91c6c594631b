"""Experiment: time hs_advect in isolation on the warmed C3 pool.

Calls the kernel repeatedly on the same input pool (outputs to the other
buffer, so the state is unchanged between calls) with L2 flushed before each
call; variants: fused splat on/off.  Select the tile shape with
HS_ADVECT_CHUNKS=1|4 (read once per process).
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    import torch
    from paper_2511_02852_b200 import Simulation, scenes
    from paper_2511_02852_b200 import _native as N
    from paper_2511_02852_b200._layout import stream_ptr
    sim = Simulation(scenes.c3(), device="cuda:0")
    sim.run_frames(2000, dt=0.1)
    sim.run_frames(3)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
    src = sim._parity
    dst = src ^ 1
    out_count = torch.zeros_like(sim.counts[dst])
    for splat in (1, 0):
        args = N.HsAdvectArgs(
            n_patches=sim.n_patches, nb=sim.nb, buckets=N.ptr(sim.buckets_dev), patches=N.ptr(sim.patches_dev),
            dt=float(sim.config.dt), rho=1000.0, g=9.81, in_=sim._pool(src), in_count=N.ptr(sim.counts[src]),
            stage=N.pool_struct(*sim.stage), stage_count=N.ptr(sim.stage_count), out=sim._pool(dst),
            out_count=N.ptr(out_count), dropped=N.pool_struct(), dropped_count=0, e_out=N.ptr(sim.e_out),
            splat=splat, raw_layers=N.ptr(sim.synth.raw), raw_layers_len=sim.synth.pack.raw_len,
            layers=N.ptr(sim.synth.layers), clamped=N.ptr(sim.clamped), tile_state=N.ptr(sim.tile_state),
            max_tiles=sim.max_tiles, tile_counter=N.ptr(sim.tile_counter), status=N.ptr(sim.status),
            keep_words=N.ptr(sim.keep_words) if os.environ.get("HS_TWO_PASS", "1") == "1" else 0)
        times = []
        for k in range(30):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            N.call("hs_advect", args, stream_ptr())
            b.record()
            torch.cuda.synchronize()
            if k >= 5:
                times.append(a.elapsed_time(b) * 1e3)
        times.sort()
        print(f"two_pass={os.environ.get('HS_TWO_PASS', '1')} chunks={os.environ.get('HS_ADVECT_CHUNKS', '1')} splat={splat} live={int(out_count.sum())} "
              f"median_us={times[len(times) // 2]:.1f} min_us={times[0]:.1f}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
