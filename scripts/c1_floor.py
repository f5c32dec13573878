"""Floor of bench.py's c1 timing bracket: a 256 MB L2 flush, then an event pair
around (a) a 1-element torch kernel, (b) a 4 MiB int32 torch sum — context for
the teams_threads kernel's ~12.5 us."""
import torch
flush = torch.empty(2 * 126 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
tiny = torch.zeros(1, device="cuda")
x = torch.randint(0, 1 << 30, (1 << 20,), dtype=torch.int32, device="cuda")
def t(fn, n=300):
    for _ in range(5): flush.fill_(1.0); fn()
    evs = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(n)]
    torch.cuda.synchronize()
    for a, b in evs:
        flush.fill_(1.0); a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs) / n * 1000
print(f"1-element add after flush: {t(lambda: tiny.add_(1)):.2f} us")
print(f"torch.sum int32 2^20 after flush: {t(lambda: x.sum(dtype=torch.int64)):.2f} us")
