import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from inputs import gen
from paper_2309_01906_b200 import hpar as H, nests
from tests.test_gpu_parity import run_nest
off = gen.csr_offsets(3000, 40000)
v = gen.gen_f32(gen.SEED_C3, 0, 40000)
for rc in (16, 64):
    levels = nests.c3_nest(with_gpu=True, rows_chunk=rc, width=8)
    res = run_nest(H, torch, levels, v, n0=3000, offsets=off, keyed=True, C=4, K=2, W=4)
    print(rc, res["kernel"], np.bincount(res["count"])[:4], res["owner"][:20])
levels = nests.c3_nest(with_gpu=False, rows_chunk=16, width=8)
res = run_nest(H, torch, levels, v, n0=3000, offsets=off, keyed=True, C=4, K=2, W=4)
print("nogpu", res["kernel"], np.bincount(res["count"])[:4])
