"""Setup latency of the background init: device hs_init_h0 vs the host fp64
numpy formation (the reference's init_fft arithmetic), per grid size.
`kernels_ms` is the device time of the hs_init_h0 launches alone (CUDA
events on the launching stream); `device_ms` adds the host mirror download."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2511_02852_b200 import DirectionalSpectrum, derive_params, init_fft  # noqa: E402
from paper_2511_02852_b200 import _native as N  # noqa: E402
from paper_2511_02852_b200 import fft_background as F  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    sp = DirectionalSpectrum(derive_params(10.0, 1e5, 9.81), 0.0)
    out = []
    call = N.call
    for n, L in ((512, 2000.0), (1024, 4000.0), (2048, 8000.0), (4096, 8000.0)):
        init_fft(sp, n, L, 1, device=dev)          # warm (tables, allocator)
        torch.cuda.synchronize()
        ev = []

        def timed_call(name, args, stream, _ev=ev):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            call(name, args, stream)
            b.record()
            _ev.append((a, b))
        F.N.call = timed_call
        t = time.perf_counter()
        init_fft(sp, n, L, 5, device=dev)
        torch.cuda.synchronize()
        t_dev = time.perf_counter() - t
        F.N.call = call
        k_ms = sum(a.elapsed_time(b) for a, b in ev)
        t = time.perf_counter()
        init_fft(sp, n, L, 5, device=dev, on_device=False)
        torch.cuda.synchronize()
        t_host = time.perf_counter() - t
        out.append({"n": n, "kernels_ms": round(k_ms, 3), "device_ms": round(t_dev * 1e3, 2),
                    "host_ms": round(t_host * 1e3, 1)})
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
