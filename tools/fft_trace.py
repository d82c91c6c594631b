"""Per-phase timeline of the FFT rows kernel CTAs (trace build:
-DHS_FFT_TRACE), steady-state C3 frame.  HS_LIB must point at the trace build."""
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
for _ in range(300):
    sim.step(0.1, stats=False)
for _ in range(5):
    sim.step(cfg.dt, stats=False)
torch.cuda.synchronize()
buf = np.zeros(2048 * 8, np.uint64)
N.lib().hs_debug_ftrace(C.c_void_p(buf.ctypes.data))
n = cfg.fft_n // 2 + 1
t = buf.reshape(2048, 8)[:n, :5].astype(np.float64)
t = (t - t[:, 0].min()) / 1000.0
print("ctas", n, "span %.2f" % t[:, 4].max())
print("start p10 %.2f p50 %.2f p90 %.2f max %.2f" % tuple(np.percentile(t[:, 0], [10, 50, 90, 100])))
for k, nm in ((1, "load"), (2, "spectrum"), (3, "fft"), (4, "store")):
    d = t[:, k] - t[:, k - 1]
    print(f"{nm:9s} p10 {np.percentile(d,10):6.2f} p50 {np.median(d):6.2f} p90 {np.percentile(d,90):6.2f} max {d.max():6.2f}")
