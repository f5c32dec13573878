#!/usr/bin/env python3
"""One small launch of every libhpar kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck; scripts/sanitize.sh).

Each case checks its result against the oracle so that a run under the
sanitizer is also a parity run; the process exits non-zero on a mismatch.
Sizes are small (the sanitizer slows kernels by 10-1000x) but span several
tiles and a ragged tail.  `--only NAME` runs one case; `--probe-no-barrier`
adds the negative-control probes (the barrier removed) for racecheck.
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--probe-no-barrier", action="store_true")
    args = ap.parse_args()
    import torch

    from inputs import gen
    from oracle import oracle as O
    from paper_2309_01906_b200 import hpar as H
    from paper_2309_01906_b200 import nests
    torch.cuda.set_device(0)
    cases = {}

    def case(fn):
        cases[fn.__name__] = fn
        return fn

    def rel_ok(got, want, tol=1e-5):
        got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
        return bool(np.all(np.abs(got - want) <= tol * np.abs(want)))

    @case
    def flat():
        n = 4096 * 2 * 5 + 4 * 77 + 3
        x = gen.gen_f32(gen.SEED_C5, 0, n)
        nest = H.Nest(nests.c5_nest(2), device=0, cluster_dim=2, warps_per_cta=8, clusters=3)
        out = torch.zeros(1, dtype=torch.float64, device="cuda")
        fp = torch.zeros(3, dtype=torch.int64, device="cuda")
        nest.parallel_for_reduce(H.make_desc(torch.from_numpy(x).cuda(), out, n0=n))
        nest.parallel_for_reduce(H.make_desc(torch.from_numpy(x).cuda(), out, n0=n, verify=H.VERIFY_FINGERPRINT,
                                             fingerprint=fp))
        torch.cuda.synchronize()
        assert nest.last_kernel() == "flat_tma"
        return rel_ok(out.item(), O.sum_f32(x))

    @case
    def teams():
        x = gen.gen_i32(gen.SEED_C1, 0, 64 * 1024)
        nest = H.Nest(nests.c1_nest(outer=64), device=0, cluster_dim=2, warps_per_cta=8)
        out = torch.zeros(1, dtype=torch.int64, device="cuda")
        nest.parallel_for_reduce(H.make_desc(torch.from_numpy(x).cuda(), out, n0=64, n1=1024, ld=1024, nloops=2))
        torch.cuda.synchronize()
        assert nest.last_kernel() == "teams_threads", nest.last_kernel()
        return int(out.item()) == O.sum_i32(x)

    @case
    def rowwise():
        rows, cols = 19, 4096
        a = gen.gen_f32(gen.SEED_C2, 0, rows * cols)
        nest = H.Nest(nests.c2_nest(), device=0, cluster_dim=2, warps_per_cta=4, clusters=5)
        out = torch.zeros(rows, dtype=torch.float32, device="cuda")
        nest.parallel_for_reduce(H.make_desc(torch.from_numpy(a).cuda(), out, n0=rows, n1=cols, ld=cols, nloops=2,
                                             keyed=True))
        torch.cuda.synchronize()
        assert nest.last_kernel() == "rowwise_tma_dsmem"
        return rel_ok(out.cpu().numpy(), O.rowsum_f32(a, rows, cols))

    @case
    def hist():
        ok = True
        for W, mis in ((8, 0), (4, 0), (4, 5)):
            n = 16384 * 2 * 3 + 1000 + 7
            x = gen.gen_u8(gen.SEED_C4, 0, n)
            nest = H.Nest(nests.c4_nest(2), device=0, cluster_dim=2, warps_per_cta=W, clusters=2)
            raw = torch.zeros(n + 32, dtype=torch.uint8, device="cuda")
            xd = raw[mis:mis + n]
            xd.copy_(torch.from_numpy(x).cuda())
            out = torch.zeros(256, dtype=torch.int64, device="cuda")
            nest.parallel_for_reduce(H.make_desc(xd, out, n0=n, op=H.OP_HIST256))
            torch.cuda.synchronize()
            ok &= np.array_equal(out.cpu().numpy().astype(np.uint64), O.hist256(x))
        return ok

    @case
    def segmented():
        rng = np.random.default_rng(5)
        rows = 700
        lens = np.where(rng.random(rows) < 0.01, rng.integers(4097, 20000, rows), rng.geometric(0.1, rows))
        lens[::50] = 0
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        v = gen.gen_f32(gen.SEED_C3, 0, int(off[-1]))
        nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8, clusters=2)
        out = torch.zeros(rows, dtype=torch.float32, device="cuda")
        for _ in range(2):
            nest.parallel_for_reduce(H.make_desc(torch.from_numpy(v).cuda(), out, n0=rows, n1=v.size, nloops=2,
                                                 keyed=True, offsets=torch.from_numpy(off).cuda()))
        torch.cuda.synchronize()
        assert nest.last_kernel() == "segmented_csr"
        return rel_ok(out.cpu().numpy(), O.segsum_f32(v, off))

    @case
    def generic():
        ok = True
        # dynamic teams, keyed CSR with lane groups (the generic C3 nest)
        off = gen.csr_offsets(300, 4000)
        v = gen.gen_f32(gen.SEED_C3, 0, 4000)
        nest = H.Nest(nests.c3_nest(rows_chunk=16, width=8), device=0, cluster_dim=2, warps_per_cta=4, clusters=2)
        out = torch.zeros(300, dtype=torch.float64, device="cuda")
        nest.parallel_for_reduce(H.make_desc(torch.from_numpy(v).cuda(), out, n0=300, nloops=2, keyed=True,
                                             offsets=torch.from_numpy(off).cuda(), out_dtype=H.F64))
        torch.cuda.synchronize()
        assert nest.last_kernel() == "generic"
        ok &= rel_ok(out.cpu().numpy(), O.segsum_f32(v, off))
        # ordered affine op, block schedules: the direct recurrence
        x = gen.gen_i32(77, 0, 5003).astype(np.int64)
        nest = H.Nest([H.Level(1, 3, H.STATIC), H.Level(4, 5, H.STATIC)], device=0, cluster_dim=2, warps_per_cta=2,
                      clusters=2)
        out = torch.zeros(2, dtype=torch.int64, device="cuda")
        nest.parallel_for_reduce(H.make_desc(torch.from_numpy(x).cuda(), out, n0=x.size, op=H.OP_AFFINE))
        torch.cuda.synchronize()
        A, B = (int(t) for t in out.cpu().numpy().view(np.uint64))
        ok &= (A * 3 + B) % (1 << 64) == O.affine_run(x, 3)
        return ok

    @case
    def probe():
        ok = True
        C, K, W = 3, 2, 4
        nest = H.Nest([H.Level(H.HPAR_GPU, H.HPAR_LANE)], device=0, cluster_dim=K, warps_per_cta=W, clusters=C)
        for lvl, ntask in ((H.HPAR_LANE, C * K * W * 32), (H.HPAR_WARP, C * K * W), (H.HPAR_CTA, C * K)):
            folds = torch.zeros(ntask, dtype=torch.int64, device="cuda")
            nest.barrier_probe(lvl, folds.data_ptr(), rounds=4)
            if args.probe_no_barrier:
                nest.barrier_probe(lvl, folds.data_ptr(), rounds=4, no_barrier=True, delay_ns=1000)
        torch.cuda.synchronize()
        return ok

    @case
    def stencil():
        from oracle import ghostmap as G
        R, C = 200, 333
        A = gen.gen_f32(gen.SEED_C5, 0, R * C).reshape(R, C)
        ld = (C + 3) // 4 * 4
        a = torch.zeros((R, ld), dtype=torch.float32, device="cuda")
        a[:, :C] = torch.from_numpy(A).cuda()
        b = a.clone()
        nest = H.Nest(nests.stencil_nest(), device=0)
        whole = H.Rect((0, 0), (R, C))
        H.hpar_stencil5(nest, H.stencil_desc(a, b, ld, whole, whole, (R, C)))
        torch.cuda.synchronize()
        return np.array_equal(b[:, :C].cpu().numpy(), G.stencil5(A, 1))

    names = [args.only] if args.only else list(cases)
    bad = []
    for nm in names:
        ok = cases[nm]()
        print(f"sanitize case {nm}: {'ok' if ok else 'MISMATCH'}", flush=True)
        if not ok:
            bad.append(nm)
    torch.cuda.synchronize()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
