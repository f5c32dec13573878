"""Which kernel serves the calls outside the benchmarked shapes, and at
what rate: 8-byte element types, MIN/MAX, CSR through the generic nest.
Device time per call (back-to-back; inputs > L2).
    python scripts/generic_probe.py"""
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


def line(name, nest, d, nbytes):
    try:
        ms = timeit(nest, d)
    except H.HparError as e:
        print(f"{name:40s} rejected: {e}")
        return
    print(f"{name:40s} {nest.last_kernel():18s} {ms:.4f} ms  {nbytes / ms / 1e6:.0f} GB/s")


n = 1 << 28
for dt, name in ((torch.float32, "f32"), (torch.int32, "i32"), (torch.float64, "f64"), (torch.int64, "i64")):
    x = (torch.rand(n, device="cuda") * 100).to(dt)
    for op, on in ((H.OP_SUM, "sum"), (H.OP_MIN, "min"), (H.OP_MAX, "max")):
        odt = torch.float64 if dt.is_floating_point else torch.int64
        out = torch.zeros(1, dtype=odt, device="cuda")
        nest = H.Nest(nests.c5_nest(2), device=0, cluster_dim=2, warps_per_cta=4, clusters=148)
        line(f"flat {name} {on} 2^28", nest, H.make_desc(x, out, n0=n, op=op), n * x.element_size())
    del x
rows, cols = 65536, 4096
x = torch.rand(rows * cols, device="cuda")
for op, on in ((H.OP_SUM, "sum"), (H.OP_MIN, "min"), (H.OP_MAX, "max")):
    out = torch.zeros(rows, dtype=torch.float32, device="cuda")
    nest = H.Nest(nests.c2_nest(), device=0, cluster_dim=2, warps_per_cta=4, clusters=444)
    line(f"rows f32 {on} 65536x4096", nest, H.make_desc(x, out, n0=rows, n1=cols, ld=cols, nloops=2, keyed=True, op=op),
         rows * cols * 4)
del x
R, NNZ = 1 << 24, 1 << 28
offs = torch.from_numpy(gen.csr_offsets(R, NNZ)).cuda()
v = torch.rand(NNZ, device="cuda")
out = torch.zeros(R, dtype=torch.float32, device="cuda")
nest = H.Nest(nests.c3_nest(), device=0, cluster_dim=2, warps_per_cta=8)
line("CSR f32 sum, generic c3_nest", nest, H.make_desc(v, out, n0=R, n1=NNZ, nloops=2, keyed=True, offsets=offs),
     NNZ * 4 + (R + 1) * 8 + R * 4)
for op, on in ((H.OP_MIN, "min"), (H.OP_MAX, "max")):
    nest = H.Nest(nests.c3_fast_nest(), device=0)
    line(f"CSR f32 {on}, c3_fast_nest", nest, H.make_desc(v, out, n0=R, n1=NNZ, nloops=2, keyed=True, offsets=offs,
                                                          op=op), NNZ * 4 + (R + 1) * 8 + R * 4)
for dt, odt, on in ((torch.float64, torch.float64, "f64 sum"), (torch.int32, torch.int64, "i32 sum"),
                    (torch.int64, torch.int64, "i64 sum")):
    vv = (v * 1000).to(dt)
    o2 = torch.zeros(R, dtype=odt, device="cuda")
    nest = H.Nest(nests.c3_fast_nest(), device=0)
    line(f"CSR {on}, c3_fast_nest", nest, H.make_desc(vv, o2, n0=R, n1=NNZ, nloops=2, keyed=True, offsets=offs),
         NNZ * vv.element_size() + (R + 1) * 8 + R * 8)
    del vv
# the ordered AFFINE op (NEXT f2) on a flat nest of int64
x = torch.randint(-(1 << 62), 1 << 62, (n,), dtype=torch.int64, device="cuda")
out = torch.zeros(2, dtype=torch.int64, device="cuda")
nest = H.Nest(nests.c5_nest(2), device=0, cluster_dim=2, warps_per_cta=4, clusters=148)
line("flat i64 affine 2^28", nest, H.make_desc(x, out, n0=n, op=H.OP_AFFINE), n * 8)
lv = nests.c5_nest(2)
lv[-1].chunk = 2  # lane static(2): not the fused flat shape -> the generic interpreter
nest = H.Nest(lv, device=0, cluster_dim=2, warps_per_cta=4, clusters=148)
line("flat i64 affine 2^28, lane static(2)", nest, H.make_desc(x, out, n0=n, op=H.OP_AFFINE), n * 8)
# lane static(1) / static(2) flat nests (warp static(32 V)) on the fused flat kernel
xf = torch.rand(n, device="cuda")
for V in (1, 2):
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    nest = H.Nest(nests.flat_nest(2, 4096, V), device=0, cluster_dim=2, warps_per_cta=4, clusters=148)
    line(f"flat f32 sum 2^28, lane static({V})", nest, H.make_desc(xf, out, n0=n), n * 4)
# row sums with lane static(1) / static(2) over the columns (warp static(32 V))
x = torch.rand(rows * cols, device="cuda")
for V in (1, 2):
    lv = nests.c2_nest()
    lv[-1].chunk, lv[-2].chunk = V, 32 * V
    out = torch.zeros(rows, dtype=torch.float32, device="cuda")
    nest = H.Nest(lv, device=0, cluster_dim=2, warps_per_cta=4, clusters=444)
    line(f"rows f32 sum 65536x4096, lane static({V})", nest,
         H.make_desc(x, out, n0=rows, n1=cols, ld=cols, nloops=2, keyed=True), rows * cols * 4)
