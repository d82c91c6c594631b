"""Dump the steady-state C3 resident pool (positions, buckets, slot order)
for offline splat-locality analysis: gpurun_out/pool_c3.npz."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2511_02852_b200 import Simulation, scenes  # noqa: E402

cfg = scenes.c3()
sim = Simulation(cfg, device=torch.device("cuda:0"))
sim.prepare_graphs()
for _ in range(2000):
    sim.step(0.1, stats=False)
for _ in range(40):
    sim.step(cfg.dt, stats=False)
torch.cuda.synchronize()
buf = sim._buf
x, y = sim.pools[buf][0].cpu().numpy(), sim.pools[buf][1].cpu().numpy()
np.savez_compressed("gpurun_out/pool_c3.npz", x=x, y=y, seg_base=sim.seg_base.cpu().numpy(),
                    seg_len=sim.seg_len[sim._lp].cpu().numpy(), live=sim.live.cpu().numpy())
print("saved", x.shape, sim.live.cpu().numpy())
