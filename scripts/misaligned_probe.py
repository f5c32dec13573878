"""Flat fp32 total of 2^28 elements: 16-byte aligned vs 4/8/12 bytes off
(device time per call, back-to-back, inputs > L2 so every call streams HBM).
    python scripts/misaligned_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_01906_b200 import hpar as H, nests  # noqa: E402

n = 1 << 28
raw = torch.rand(n + 8, device="cuda")
for off in (0, 1, 2, 3):
    x = raw[off:off + n]
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    nest = H.Nest(nests.c5_nest(2), device=0, cluster_dim=2, warps_per_cta=4, clusters=148)
    d = H.make_desc(x, out, n0=n)
    for _ in range(3):
        nest.parallel_for_reduce(d)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        nest.parallel_for_reduce(d)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"offset {4 * off:2d} B  {nest.last_kernel():10s} {ms:.4f} ms  {n * 4 / ms / 1e6:.0f} GB/s  "
          f"total {out.item():.6f}")
