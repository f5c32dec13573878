import os, sys, torch
sys.path.insert(0, "/root/repo")
from inputs import gen
from paper_2309_01906_b200 import hpar as H, nests
R, NNZ = 1 << 24, 1 << 28
offs = torch.from_numpy(gen.csr_offsets(R, NNZ)).cuda()
v = torch.rand(NNZ, device="cuda", dtype=torch.float64 if os.environ.get("SR_F64") else torch.float32)
out = torch.zeros(R, dtype=v.dtype, device="cuda")
nest = H.Nest(nests.c3_fast_nest(), device=0)
d = H.make_desc(v, out, n0=R, n1=NNZ, nloops=2, keyed=True, offsets=offs, op=H.OP_SUM if os.environ.get("SR_F64") else H.OP_MIN)
for _ in range(3): nest.parallel_for_reduce(d)
torch.cuda.synchronize()
print(nest.last_kernel())
