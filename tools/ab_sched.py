"""A/B of frame-schedule knobs on one warmed scene (not product code):
FFT fork point (after inject / frame start) x stream priorities.  Each variant
recaptures the frame graphs and times K flushed graph steps with CUDA events.

    python tools/ab_sched.py [--config C3] [--steps 300]
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
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--rounds", type=int, default=2)
    args = ap.parse_args()
    import torch
    from bench import scene_config
    from paper_2511_02852_b200 import Simulation
    cfg, keys, _, _ = scene_config(args.config, 0, 1)
    sim = Simulation(cfg, device="cuda:0", rng_seed_keys=keys)
    sim.run_frames(2000, dt=0.1)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
    variants = {"after_inject": (False, False), "start": (True, False), "after_inject+prio": (False, True),
                "start+prio": (True, True)}
    res = {k: [] for k in variants}
    for _ in range(args.rounds):
        for name, (start, prio) in variants.items():
            sim.fft_fork_at_start, sim.sched_priorities = start, prio
            sim._graphs = {}
            sim._sides = {}
            sim.prepare_graphs()
            for _ in range(10):
                sim.step(stats=False)
            torch.cuda.synchronize()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
            for a, b in ev:
                flush.zero_()
                a.record()
                sim.step(stats=False)
                b.record()
            torch.cuda.synchronize()
            t = np.array([a.elapsed_time(b) for a, b in ev]) * 1e3
            res[name].append((float(np.median(t)), float(np.mean(t)), float(np.percentile(t, 90))))
    sim.check()
    for name, r in res.items():
        print(f"{name:20s} " + "  ".join(f"p50 {a:6.1f} mean {b:6.1f} p90 {c:6.1f}" for a, b, c in r))
    return 0


if __name__ == "__main__":
    sys.exit(main())
