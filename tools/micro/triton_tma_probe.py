"""Probe (not product code): does a TMA load work on this box?  Triton's
tensor-descriptor load compiles to cp.async.bulk.tensor; dumps its PTX."""
import torch, triton, triton.language as tl
from triton.tools.tensor_descriptor import TensorDescriptor

@triton.jit
def k(desc, out):
    x = desc.load([0, 0])
    offs = tl.arange(0, 16)[:, None] * 16 + tl.arange(0, 16)[None, :]
    tl.store(out + offs, x)

a = torch.arange(40 * 40, dtype=torch.float32, device="cuda").reshape(40, 40)
out = torch.zeros(256, device="cuda")
d = TensorDescriptor.from_tensor(a, [16, 16])
triton.set_allocator(lambda size, align, stream: torch.empty(size, dtype=torch.int8, device="cuda"))
h = k[(1,)](d, out)
torch.cuda.synchronize()
print("ok", out[:5].tolist(), out[17].item())
ptx = h.asm["ptx"]
for line in ptx.splitlines():
    if "tensor" in line or "mbarrier" in line or "fence" in line:
        print(line.strip())
open("gpurun_out/triton_tma.ptx", "w").write(ptx)
open("gpurun_out/triton_tma.cubin", "wb").write(h.asm["cubin"])
