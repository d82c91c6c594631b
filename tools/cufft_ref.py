"""Reference point (not product code): cuFFT (torch.fft) time of the
transforms this path's FFT stage does -- 1024^2 complex64 inverse 2-D FFT,
and 1.5 of them -- to size how far the hand-written transform is from the
library's."""
import torch
x = torch.randn(1024, 1024, dtype=torch.complex64, device="cuda")
y = torch.randn(513, 1024, dtype=torch.complex64, device="cuda")
for name, f in [("c2c 1024^2 ifft2", lambda: torch.fft.ifft2(x)),
                ("c2r 1024^2 irfft2 (half spectrum)", lambda: torch.fft.irfft2(y.T.contiguous(), s=(1024, 1024))),
                ("c2c ifft2 + c2r irfft2", lambda: (torch.fft.ifft2(x), torch.fft.irfft2(y.T.contiguous(), s=(1024, 1024))))]:
    for _ in range(10):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(50):
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"{name:40s} median {ts[len(ts)//2]:7.2f} us  min {ts[0]:7.2f} us")
