"""Profiling driver: warm a preset scene to steady state, then run a few
eager frames (for `ncu -k <kernel> -s <skip>`).  Not part of the product.

    python tools/prof_frame.py --config C3 --frames 5
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--frames", type=int, default=5)
    ap.add_argument("--warm-frames", type=int, default=2000)
    ap.add_argument("--patches", type=int, default=None, help="first N patches of a multi-patch scene")
    args = ap.parse_args()
    import torch
    from paper_2511_02852_b200 import Simulation
    from bench import scene_config
    cfg, keys, _, _ = scene_config(args.config, 0, 1, args.patches)
    sim = Simulation(cfg, device="cuda:0", rng_seed_keys=keys)
    sim.run_frames(args.warm_frames, dt=0.1)
    sim.run_frames(3)
    torch.cuda.synchronize()
    sim.config = sim.config.__class__(**{**sim.config.__dict__, "graph": False})
    torch.cuda.cudart().cudaProfilerStart()      # ncu --profile-from-start off
    for _ in range(args.frames):
        sim.step(stats=False)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    sim.check()
    print("live", sim.live_particles(), "launches/frame", sim.kernel_launches_per_frame())
    return 0


if __name__ == "__main__":
    sys.exit(main())
