"""Debug helper: run the C3 segmented kernel at growing sizes, report the first failure."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from inputs import gen
from paper_2309_01906_b200 import hpar as H, nests
from oracle import oracle as O

sizes = [(int(a), int(b)) for a, b in (s.split(":") for s in sys.argv[1:])] or [(1 << 16, 1 << 20), (1 << 20, 1 << 24), (1 << 22, 1 << 26)]
for rows, nnz in sizes:
    off = gen.csr_offsets(rows, nnz)
    v = gen.gen_f32(gen.SEED_C3, 0, nnz)
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8)
    x = torch.from_numpy(v).cuda()
    offd = torch.from_numpy(off).cuda()
    out = torch.full((rows,), -1.0, dtype=torch.float32, device="cuda")
    import os
    if os.environ.get("PRESYNC"):
        torch.cuda.synchronize()
    for it in range(int(os.environ.get("CALLS", "3"))):
        nest.parallel_for_reduce(H.make_desc(x, out, n0=rows, n1=nnz, nloops=2, keyed=True, offsets=offd))
        torch.cuda.synchronize()
        print("call", it, "ok", flush=True)
    if os.environ.get("HPAR_SEG_DEBUG"):
        continue
    got = out.cpu().numpy().astype(np.float64)
    want = O.segsum_f32(v, off)
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
    bad = np.nonzero(rel > 1e-5)[0]
    print(rows, nnz, "max long row", int(np.diff(off).max()), "bad", bad.size, bad[:5], flush=True)
