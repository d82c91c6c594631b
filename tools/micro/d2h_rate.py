"""Pinned D2H / H2D copy rate of a frame-sized buffer on this box (not product code)."""
import torch
dev = "cuda:0"
for mb in (1, 4, 16):
    n = mb << 18
    src = torch.randn(n, device=dev)
    dst = torch.empty(n, pin_memory=True)
    for _ in range(5):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(50):
        dst.copy_(src, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    us = s.elapsed_time(e) * 1e3 / 50
    print(f"D2H {mb} MiB: {us:.1f} us  {4 * n / us / 1e3:.1f} GB/s")
    s.record()
    for _ in range(50):
        src.copy_(dst, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    us = s.elapsed_time(e) * 1e3 / 50
    print(f"H2D {mb} MiB: {us:.1f} us  {4 * n / us / 1e3:.1f} GB/s")
