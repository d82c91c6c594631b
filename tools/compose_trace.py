"""Per-phase timeline of hs_compose CTAs (trace build: -DHS_COMPOSE_TRACE),
steady-state C3 frame, graph replay.  HS_LIB must point at the trace build."""
import ctypes as C
import sys
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2511_02852_b200 import Simulation, scenes  # noqa: E402
from paper_2511_02852_b200 import _native as N  # noqa: E402

cfg = scenes.c3()
sim = Simulation(cfg, device=torch.device("cuda:0"))
sim.prepare_graphs()
for _ in range(2000):
    sim.step(0.1, stats=False)
for _ in range(5):
    sim.step(cfg.dt, stats=False)
torch.cuda.synchronize()
buf = np.zeros(4096 * 8, np.uint64)
N.lib().hs_debug_trace(C.c_void_p(buf.ctypes.data))
n = sim.synth.compose_tiles
t8 = buf.reshape(4096, 8)[:n, :8].astype(np.float64)
t = t8[:, :7]
t0 = t[:, 0].min()
t = (t - t0) / 1000.0
t7 = (t8[:, 7] - t0) / 1000.0          # after the texel loops, before the composite nodes
names = ["start", "plans", "stage+f1", "tc", "coarse", "bgprep", "epilogue"]
print("tiles", n, "kernel span us", t[:, 6].max())
print("start times: min %.2f p50 %.2f max %.2f" % (t[:, 0].min(), np.median(t[:, 0]), t[:, 0].max()))
for k in range(1, 7):
    d = t[:, k] - t[:, k - 1]
    print(f"{names[k]:9s} p10 {np.percentile(d,10):6.2f} p50 {np.median(d):6.2f} p90 {np.percentile(d,90):6.2f} max {d.max():6.2f}")
for lbl, d in (("texels", t7 - t[:, 5]), ("composite", t[:, 6] - t7)):
    print(f"  {lbl:9s} p10 {np.percentile(d,10):6.2f} p50 {np.median(d):6.2f} p90 {np.percentile(d,90):6.2f} max {d.max():6.2f}")
print("end times: p10 %.2f p50 %.2f max %.2f" % (np.percentile(t[:, 6], 10), np.median(t[:, 6]), t[:, 6].max()))
info = sim.synth.compose_info.cpu().numpy().reshape(-1, 3)[:n]
res = cfg.patches[0].res
band = 40   # margin / texel
edge = (info[:, 1] < band) | (info[:, 2] < band) | (info[:, 1] + 30 > res - band) | (info[:, 2] + 30 > res - band)
print("band tiles", edge.sum(), "end p50 %.2f max %.2f" % (np.median(t[edge, 6]), t[edge, 6].max()),
      "texels p50 %.2f composite p50 %.2f" % (np.median((t7 - t[:, 5])[edge]), np.median((t[:, 6] - t7)[edge])))
print("interior tiles", (~edge).sum(), "end p50 %.2f max %.2f" % (np.median(t[~edge, 6]), t[~edge, 6].max()))
slow = np.argsort(-t[:, 6])[:12]
for k in slow:
    print(k, info[k], " ".join("%.2f" % v for v in t[k, :7]))
# per-SM? blockIdx order
print("end vs block index (deciles):", [round(float(np.median(t[i * n // 10:(i + 1) * n // 10, 6])), 2) for i in range(10)])
