"""C3 steady-state live particles per bucket with the bucket's layer factor
(not product code): where the splat's reductions land."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from bench import WARM_DT, WARM_SECONDS, scene_config
from paper_2511_02852_b200 import Simulation
cfg, keys, _, _ = scene_config(sys.argv[1] if len(sys.argv) > 1 else "C3", 0, 1)
sim = Simulation(cfg, device="cuda:0", rng_seed_keys=keys)
sim.run_frames(int(round(WARM_SECONDS / WARM_DT)), dt=WARM_DT)
torch.cuda.synchronize()
c = sim.counts_host()[0]
for b, L in enumerate(sim.synth.pack.layers[:sim.nb]):
    print(b, "f", L.f, "H", L.H, "layer", L.ncx, "x", L.ncy, "live", int(c[b]), "per texel %.3f" % (c[b] / (L.ncx * L.ncy)))
print("total", int(c.sum()))
