import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2309_01906_b200 import hpar as H, nests
from inputs import gen
import ctypes, os
L = ctypes.CDLL("/root/repo/inputs/libhpar_inputs.so")
L.hpar_inputs_fill_f32.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
L2B = 126 * 2**20
for mb in (1074, 134):
    n = mb * 2**20 // 4
    k = max(1, -(-3 * L2B // (n * 4)) + 1)
    xs = [torch.empty(n, device="cuda") for _ in range(k)]
    for x in xs: L.hpar_inputs_fill_f32(5, 0, n, x.data_ptr(), None)
    outs = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(k)]
    for C in (0, 148, 296):
        nest = H.Nest(nests.c5_nest(2), device=0, cluster_dim=2, warps_per_cta=8, clusters=C)
        ds = [H.make_desc(xs[i], outs[i], n0=n) for i in range(k)]
        for i in range(5): nest.parallel_for_reduce(ds[i % k])
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        ev = [(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True)) for _ in range(60)]
        with torch.cuda.graph(g, capture_error_mode="relaxed"):
            for i in range(60):
                ev[i][0].record(); nest.parallel_for_reduce(ds[i % k], torch.cuda.current_stream().cuda_stream); ev[i][1].record()
        g.replay(); torch.cuda.synchronize()
        t = sorted(a.elapsed_time(b) for a, b in ev)[30]
        print(f"flat_tma {mb} MB C={nest.info().C}: {t*1e3:.1f} us = {mb*2**20/(t*1e-3)/1e9:.0f} GB/s", flush=True)
    # torch copy
    ys = [torch.empty_like(x) for x in xs]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(60)]
    for i in range(60):
        ev[i][0].record(); ys[i % k].copy_(xs[i % k]); ev[i][1].record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)[30]
    print(f"torch copy {mb} MB: {t*1e3:.1f} us = {2*mb*2**20/(t*1e-3)/1e9:.0f} GB/s (read+write)", flush=True)
    del xs, ys, outs
    torch.cuda.empty_cache()
