"""Per-kernel device times of a warmed scene, each stage replayed alone
(not product code): builds the scene, warms it, then re-launches the frame's
kernels one stage at a time K times with CUDA events (no L2 flush: the
steady-state inputs stay resident, the in-frame situation of compose/smooth),
printing median us per stage.  Library under test: HS_LIB (default product).

    python tools/bench_kernels.py [--config C3] [--reps 200] [--stages compose,smooth,fft,advect]
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--stages", default="compose,smooth,fft,advect")
    ap.add_argument("--flush", action="store_true", help="flush L2 before every launch")
    args = ap.parse_args()
    import torch
    from bench import scene_config
    from paper_2511_02852_b200 import Simulation
    from paper_2511_02852_b200 import _native as N
    from paper_2511_02852_b200._layout import stream_ptr
    from paper_2511_02852_b200.fft_background import fft_args
    cfg, keys, _, _ = scene_config(args.config, 0, 1)
    sim = Simulation(cfg, device="cuda:0", rng_seed_keys=keys)
    sim.run_frames(2000, dt=0.1)
    sim.run_frames(5)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
    captured = {}

    # record the frame's launches by wrapping N.call
    real_call = N.call

    def spy(name, a, stream):
        captured.setdefault(name, []).append(a)
        return real_call(name, a, stream)
    N.call = spy
    sim.config = sim.config.__class__(**{**sim.config.__dict__, "graph": False})
    sim.step(stats=False)
    torch.cuda.synchronize()
    N.call = real_call
    groups = {"compose": ["hs_compose"], "smooth": ["hs_smooth"], "fft": ["hs_fft_evolve"],
              "advect": ["hs_advect_resident"], "inject": ["hs_inject"]}
    out = {}
    for st in args.stages.split(","):
        names = groups[st]
        calls = [(n, a) for n in names for a in captured.get(n, [])]
        if not calls:
            continue
        # advect is in place: each replay moves the particles on (a few percent
        # cull per 50 replays), so it gets fewer replays
        reps = min(args.reps, 50) if st == "advect" else args.reps
        ts = []
        for _ in range(reps):
            if args.flush:
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for n, a in calls:
                real_call(n, a, stream_ptr())
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        out[st] = (float(np.median(ts)), float(np.percentile(ts, 10)))
    for k, (m, p10) in out.items():
        print(f"{k:8s} median {m:7.2f} us  p10 {p10:7.2f} us")
    return 0


if __name__ == "__main__":
    sys.exit(main())
