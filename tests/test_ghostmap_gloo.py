"""Device-level ghost refresh across ranks on CPU (gloo, world_size 4 = the
§4 example's 4 devices): each rank holds only its to-section,
steps it with the oracle's local step, and refreshes its ghosts by the C
ABI's exchange plan (hpar_map_exchange_plan) with point-to-point send/recv —
the host logic of hpar_map_exchange, whose NCCL transfer runs only on GPUs.
After T steps the gathered from-sections equal the sequential stencil."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N, T = 24, 4


def _worker(rank, world, store, q):
    # file rendezvous: no TCP port to race for (127.0.0.1 TCP works too)
    dist.init_process_group("gloo", init_method=f"file://{store}", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import ghostmap as G
        from paper_2309_01906_b200 import build as pbuild
        pbuild.build()
        from paper_2309_01906_b200 import hpar as H
        sp = G.paper_example_spec(N)
        m = H.map_spec(sp.extent, sp.siblings, sp.grid_cols, [(d.mul, d.add, d.len) for d in sp.to],
                       [(d.mul, d.add, d.len) for d in sp.frm])
        H.hpar_map_validate(m)
        to, fr = H.hpar_map_sections(m, rank)
        A = np.random.default_rng(9).standard_normal((N, N)).astype(np.float32)  # every rank: same parent
        local = A[to.off[0]:to.off[0] + to.len[0], to.off[1]:to.off[1] + to.len[1]].copy()
        plan = H.hpar_map_exchange_plan(m, rank)
        for _ in range(T):
            local = G.local_step(local, sp, rank)
            reqs, inbox = [], []
            for (peer, kind, (r0, c0, nr, nc)) in plan:
                a0, b0 = r0 - to.off[0], c0 - to.off[1]
                if kind == "send":
                    reqs.append(dist.isend(torch.from_numpy(local[a0:a0 + nr, b0:b0 + nc].copy()), peer))
                else:
                    t = torch.empty((nr, nc), dtype=torch.float32)
                    reqs.append(dist.irecv(t, peer))
                    inbox.append((t, a0, b0, nr, nc))
            for r in reqs:
                r.wait()
            for (t, a0, b0, nr, nc) in inbox:
                local[a0:a0 + nr, b0:b0 + nc] = t.numpy()
        a0, b0 = fr.off[0] - to.off[0], fr.off[1] - to.off[1]
        q.put((rank, (fr.tup(), local[a0:a0 + fr.len[0], b0:b0 + fr.len[1]].copy())))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_four_rank_ghost_exchange():
    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    import tempfile
    store = os.path.join(tempfile.mkdtemp(prefix="hpar_gloo_"), "rendezvous")  # a FileStore path
    procs = [ctx.Process(target=_worker, args=(r, world, store, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    from oracle import ghostmap as G
    A = np.random.default_rng(9).standard_normal((N, N)).astype(np.float32)
    want = G.stencil5(A, T)
    got = np.full_like(want, np.nan)
    for r in range(world):
        (r0, c0, nr, nc), tile = res[r]
        got[r0:r0 + nr, c0:c0 + nc] = tile
    assert np.array_equal(got, want)
