import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2511_02852_b200 import Simulation, scenes
cuda = torch.device("cuda:0")
outs = []
for _ in range(3):
    cfg = scenes.c5(2, frames=40, fft_n=512, deterministic=True)
    sim = Simulation(cfg, device=cuda)
    rows = [sim.step() for _ in range(cfg.frames)]
    outs.append([(r.despawned_energy.copy(), r.patch_variance, r.fft_band_variance, r.particle_counts.copy(), r.injected_energy.copy()) for r in rows])
for k in range(40):
    a, b, c = outs[0][k], outs[1][k], outs[2][k]
    d = [not np.array_equal(a[i], b[i]) or not np.array_equal(a[i], c[i]) for i in range(5)]
    if any(d):
        print(k, d, a[1], b[1], c[1], a[2], b[2], c[2], np.abs(a[0]-b[0]).max(), np.abs(a[4]-b[4]).max())
