"""Which kernel serves the edge shapes of C2/C3, and at what rate: dense
rows whose length or leading dimension is not a multiple of 4 (rows not
16-byte aligned), and input pointers off a 16-byte boundary; CSR values
off a 16-byte boundary.  Device time per call (back-to-back; inputs > L2).
    python scripts/edge_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import gen  # noqa: E402
from paper_2309_01906_b200 import hpar as H, nests  # noqa: E402


def timeit(nest, d, reps=5):
    for _ in range(2):
        nest.parallel_for_reduce(d)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        nest.parallel_for_reduce(d)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


rows = 65536
for cols, ld, off in ((4096, 4096, 0), (4096, 4096, 1), (4095, 4095, 0), (4095, 4096, 0), (4100, 4100, 0),
                      (4092, 4092, 0)):
    raw = torch.rand(rows * ld + 8, device="cuda")
    x = raw[off:off + rows * ld]
    out = torch.empty(rows, dtype=torch.float32, device="cuda")
    nest = H.Nest(nests.c2_nest(), device=0, cluster_dim=2, warps_per_cta=4, clusters=444)
    d = H.make_desc(x, out, n0=rows, n1=cols, ld=ld, nloops=2, keyed=True)
    ms = timeit(nest, d)
    ref = x.view(rows, ld)[:, :cols].double().sum(1)
    err = ((out.double() - ref).abs() / ref.abs().clamp_min(1e-30)).max().item()
    print(f"C2 {rows}x{cols} ld {ld} ptr+{4 * off}B  {nest.last_kernel():18s} {ms:.4f} ms  "
          f"{rows * cols * 4 / ms / 1e6:.0f} GB/s  max rel err {err:.1e}")
    del raw, x
R, NNZ = 1 << 24, 1 << 28
off_h = gen.csr_offsets(R, NNZ)
offs = torch.from_numpy(off_h).cuda()
raw = torch.rand(NNZ + 8, device="cuda")
for o in (0, 1):
    v = raw[o:o + NNZ]
    out = torch.empty(R, dtype=torch.float32, device="cuda")
    nest = H.Nest(nests.c3_fast_nest(), device=0)
    d = H.make_desc(v, out, n0=R, n1=NNZ, nloops=2, keyed=True, offsets=offs)
    try:
        ms = timeit(nest, d, reps=3)
    except H.HparError as e:
        print(f"C3 2^24 rows 2^28 nnz ptr+{4 * o}B  rejected: {e}")
        continue
    print(f"C3 2^24 rows 2^28 nnz ptr+{4 * o}B  {nest.last_kernel():18s} {ms:.4f} ms  "
          f"{(NNZ * 4 + (R + 1) * 8 + R * 4) / ms / 1e6:.0f} GB/s")
