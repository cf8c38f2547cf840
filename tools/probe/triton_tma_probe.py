# Cross-check that tensor TMA works on this box at all (probe only; not product code).
import torch, triton, triton.language as tl

@triton.jit
def k(desc, out_ptr):
    x = desc.load([0, 0])
    offs = tl.arange(0, 64)
    tl.store(out_ptr + offs, tl.reshape(x, [64]))

def alloc(size, align, stream):
    return torch.empty(size, dtype=torch.int8, device="cuda")

triton.set_allocator(alloc)
a = torch.arange(64 * 16, dtype=torch.float32, device="cuda").reshape(16, 64)
from triton.tools.tensor_descriptor import TensorDescriptor
d = TensorDescriptor.from_tensor(a, [1, 64])
o = torch.empty(64, device="cuda")
k[(1,)](d, o)
torch.cuda.synchronize()
print("triton TMA:", "ok" if torch.equal(o, a[0]) else "MISMATCH")
