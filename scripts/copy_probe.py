"""Copy-rate probes for the c6 buffer shape (timing context for the stencil)."""
import torch
R, LD = 16386, 16416
a = torch.rand(R * LD, device="cuda"); b = torch.empty_like(a)
def t(fn, n=100):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
nb = 2 * R * LD * 4
ms = t(lambda: b.copy_(a)); print(f"copy a->b           {ms:.4f} ms {nb / ms / 1e6:.0f} GB/s")
st = [0]
def pp():
    if st[0]: a.copy_(b)
    else: b.copy_(a)
    st[0] ^= 1
ms = t(pp); print(f"copy ping-pong      {ms:.4f} ms {nb / ms / 1e6:.0f} GB/s")
a2, b2 = a.view(R, LD), b.view(R, LD)
ms = t(lambda: b2[1:-1, 1:16385].copy_(a2[1:-1, 1:16385])); print(f"copy 2-D interior   {ms:.4f} ms {2 * 16384 * 16384 * 4 / ms / 1e6:.0f} GB/s")
ms = t(lambda: torch.add(a, 1.0, out=b)); print(f"add a+1 -> b        {ms:.4f} ms {nb / ms / 1e6:.0f} GB/s")
