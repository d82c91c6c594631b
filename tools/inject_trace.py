"""Phase timeline of hs_inject's CTA 0 (trace build: -DHS_INJECT_TRACE) in a
steady-state C3 frame (graph replay).  HS_LIB must point at the trace build.
Not product code."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from bench import WARM_DT, WARM_SECONDS, scene_config
    from paper_2511_02852_b200 import Simulation
    from paper_2511_02852_b200 import _native as N
    cfg, keys, _, _ = scene_config(sys.argv[1] if len(sys.argv) > 1 else "C3", 0, 1)
    sim = Simulation(cfg, device="cuda:0", rng_seed_keys=keys)
    sim.run_frames(int(round(WARM_SECONDS / WARM_DT)), dt=WARM_DT)
    sim.prepare_graphs()
    names = ["ledger+scan", "amplitudes", "sums+scan", "positions", "append flush"]
    rows = []
    for _ in range(40):
        sim.step(stats=False)
        torch.cuda.synchronize()
        buf = np.zeros(16, np.uint64)
        N.lib().hs_debug_itrace(C.c_void_p(buf.ctypes.data))
        t = buf[:6].astype(np.float64)
        rows.append(np.diff(t) / 1000.0)
    r = np.array(rows)
    for k, nm in enumerate(names):
        print(f"{nm:14s} p50 {np.median(r[:, k]):6.2f} us  max {r[:, k].max():6.2f}")
    print(f"total          p50 {np.median(r.sum(1)):6.2f} us")


if __name__ == "__main__":
    main()
