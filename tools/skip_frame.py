"""Frame-time attribution (not product code): with a -DHS_EXP_SKIP build
(HS_LIB), re-capture the C3 frame graphs with one or more stages' launches
skipped (HS_EXP_SKIP=<stages>) after a normal warm-up, and time frames as
bench.py does (L2 flush between frames, CUDA events).  The drop in frame time
when a stage is skipped is how much of the frame it holds.

    HS_LIB=/tmp/skip/libhybridsea_b200.so python tools/skip_frame.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    import torch
    from bench import WARM_DT, WARM_SECONDS, scene_config
    from paper_2511_02852_b200 import Simulation
    cfg, keys, _, _ = scene_config(sys.argv[1] if len(sys.argv) > 1 else "C3", 0, 1)
    sim = Simulation(cfg, device="cuda:0", rng_seed_keys=keys)
    sim.run_frames(int(round(WARM_SECONDS / WARM_DT)), dt=WARM_DT)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
    sets = os.environ.get("SKIP_SETS", "|fft|inject|advect|smooth|compose|inject,advect|fft,inject|"
                          "smooth,compose|fft,smooth,compose|").split("|")
    if os.environ.get("FORK_AT_START"):
        sim.fft_fork_at_start = True
    # AB_ATTR="name=v1|name=v2": time frames with a Simulation attribute set to each value
    # (graphs re-captured per value), instead of the skip sets
    ab = os.environ.get("AB_ATTR")
    if ab:
        for spec in ab.split("|") * 2:
            for kv in spec.split(","):              # "a=1,b=2": several attributes at once
                k, v = kv.split("=")
                setattr(sim, k, eval(v))
            sim._graphs = {}
            sim.prepare_graphs()
            for _ in range(5):
                sim.step(stats=False)
            ts = []
            for _ in range(300):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                sim.step(stats=False)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            print(f"{spec:30s} frame median {np.median(ts):7.2f} us  mean {np.mean(ts):7.2f}  p10 "
                  f"{np.percentile(ts, 10):7.2f}", flush=True)
        return 0
    for tag in sets:
        os.environ["HS_EXP_SKIP"] = tag
        sim._graphs = {}
        sim.prepare_graphs()
        for _ in range(5):
            sim.step(stats=False)
        ts = []
        for _ in range(300):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sim.step(stats=False)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        print(f"skip {tag or '(none)':22s} frame median {np.median(ts):7.2f} us  mean {np.mean(ts):7.2f}  p10 "
              f"{np.percentile(ts, 10):7.2f}", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
