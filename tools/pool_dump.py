"""Dump the steady-state C3 resident pool (positions, buckets, slot order)
for offline splat-locality analysis: gpurun_out/pool_c3.npz."""
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2511_02852_b200 import Simulation, scenes  # noqa: E402

from bench import scene_config  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
npatch = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg, keys, _, _ = scene_config(name, 0, 1, npatch)
sim = Simulation(cfg, device=torch.device("cuda:0"), rng_seed_keys=keys)
sim.prepare_graphs()
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2000):
    sim.step(0.1, stats=False)
for _ in range(40):
    sim.step(cfg.dt, stats=False)
torch.cuda.synchronize()
buf = sim._buf
x, y = sim.pools[buf][0].cpu().numpy(), sim.pools[buf][1].cpu().numpy()
np.savez_compressed(f"gpurun_out/pool_{name}.npz", x=x, y=y, seg_base=sim.seg_base.cpu().numpy(),
                    seg_len=sim.seg_len[sim._lp].cpu().numpy(), live=sim.live.cpu().numpy(),
                    regions=np.array([[r.min_corner[0], r.min_corner[1]] for r in sim.current_regions()]),
                    factors=np.array(sim.plans[0].factors), texel=np.array([cfg.patches[0].size[0] / (cfg.patches[0].res - 1)]))
print("saved", x.shape, sim.live.cpu().numpy())
