"""Per-bucket live population and layer grid of the warmed C3 scene."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_02852_b200 import Simulation, scenes
sim = Simulation(scenes.c3(), device="cuda:0")
sim.run_frames(2000, dt=0.1)
torch.cuda.synchronize()
cnt = sim.counts[sim._parity].cpu().numpy().reshape(-1)
for b, L in enumerate(sim.synth.pack.layers):
    print(f"b={b:2d} f={L.f:3d} H={L.H:3d} wx={L.wx:5d} wy={L.wy:5d} cells={L.wx*L.wy:8d} live={int(cnt[b]):7d} per_cell={cnt[b]/(L.wx*L.wy):8.2f}")
print("total", int(cnt.sum()))
