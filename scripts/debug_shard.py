import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from inputs import gen
from oracle import oracle as O
from paper_2309_01906_b200 import hpar as H, nests
off = gen.csr_offsets(20000, 300000)
v = gen.gen_f32(gen.SEED_C3, 0, int(off[-1]))
want = O.segsum_f32(v, off)
for G in (3,):
    for g in range(G):
        b, c = H.hpar_shard_range_csr(off, G, g)
        nest = H.Nest(nests.c3_fast_nest(), device=0, rank=g, nranks=G, cluster_dim=2, warps_per_cta=8, clusters=5)
        lo = (off[b:b + c + 1] - off[b]).astype(np.int64)
        vals = v[off[b]:off[b + c]]
        xd = torch.from_numpy(vals).cuda()
        out = torch.full((c,), -1.0, dtype=torch.float64, device="cuda")
        d = H.make_desc(xd, out, n0=20000, n1=int(vals.size), nloops=2, keyed=True, offsets=torch.from_numpy(lo).cuda(), out_dtype=H.F64, local_n0=c)
        nest.parallel_for_reduce(d)
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        w = want[b:b + c]
        bad = np.nonzero(np.abs(got - w) > 1e-5 * np.maximum(np.abs(w), 1e-30))[0]
        print(G, g, b, c, "nnz", vals.size, "bad", bad.size, bad[:10], [(int(lo[i+1]-lo[i]), got[i], w[i]) for i in bad[:5]], flush=True)
