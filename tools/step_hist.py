"""Per-step device times of the bench loop (C3), grouped by position in the
resident-pool compaction cycle: where does the mean - p50 gap come from?"""
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
    sim.step(stats=False)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
fs = torch.empty((), dtype=torch.int64, device="cuda:0")
K = 640
st = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
en = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
phase = []
torch.cuda.synchronize()
for k in range(K):
    flush.zero_()
    torch.sum(flush.view(torch.int64), dim=0, out=fs)
    phase.append(sim._since)
    st[k].record()
    sim.step(stats=False)
    en[k].record()
torch.cuda.synchronize()
t = np.array([a.elapsed_time(b) * 1e3 for a, b in zip(st, en)])
ph = np.array(phase)
print("mean %.1f p50 %.1f p90 %.1f max %.1f" % (t.mean(), np.median(t), np.percentile(t, 90), t.max()))
for p in range(0, 32):
    sel = t[ph == p]
    if sel.size:
        print(p, "n", sel.size, "mean %.1f min %.1f max %.1f" % (sel.mean(), sel.min(), sel.max()))
