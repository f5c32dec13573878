"""Multi-rank host logic on CPU (gloo, world_size 2): the GPU level's shard
ranges (§8(a) A2), the node-level combine semantics (A9: per-rank results
folded across ranks equal the whole-node result) and bench.py's
max-over-ranks timing rule.  The NCCL node level itself runs only on GPUs."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, store, q):
    # file rendezvous: no TCP port to race for (127.0.0.1 TCP works too)
    dist.init_process_group("gloo", init_method=f"file://{store}", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from inputs import gen
        from oracle import oracle as O
        from paper_2309_01906_b200 import build as pbuild
        pbuild.build()
        from paper_2309_01906_b200 import hpar as H
        from paper_2309_01906_b200 import nests
        d = H.b200_desc()
        out = {}
        # (1) shards of the flat nest (config 5 shape) and the collapsed nest
        for name, levels in (("flat", nests.c5_nest()), ("collapsed", [H.Level(1, 5)])):
            nest = H.Nest(levels, device=-1, desc=d, nranks=world, rank=rank, clusters=3, warps_per_cta=2)
            n0 = 1_000_003
            b, c = nest.shard_range(n0, rank)
            t = torch.tensor([b, c], dtype=torch.int64)
            allt = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(allt, t)
            out[name] = [tuple(x.tolist()) for x in allt]
        # (2) node combine: each rank reduces its shard (oracle), allreduce == whole
        nest = H.Nest(nests.c5_nest(), device=-1, desc=d, nranks=world, rank=rank, clusters=3, warps_per_cta=2)
        n0 = 300_007
        b, c = nest.shard_range(n0, rank)
        xi = gen.gen_i32(gen.SEED_C1, b, c)  # global indices: rank-count invariant
        part = torch.tensor([O.sum_i32(xi)], dtype=torch.int64)
        dist.all_reduce(part)
        out["int_total"] = int(part.item())
        k = gen.gen_f32_k(gen.SEED_C5, b, c)
        pk = torch.tensor([O.sum_u64(k)], dtype=torch.int64)
        dist.all_reduce(pk)
        out["f32_numerators"] = int(pk.item())
        # (3) max-over-ranks timing (bench.py rule)
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out["max_ms"] = float(t.item())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo():
    world = 2
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
    from inputs import gen
    from oracle import oracle as O
    for name in ("flat", "collapsed"):
        shards = res[0][name]
        assert shards == res[1][name]
        assert shards[0][0] == 0 and shards[0][0] + shards[0][1] == shards[1][0]
        assert shards[1][0] + shards[1][1] == 1_000_003
        assert abs(shards[0][1] - shards[1][1]) <= 3 * 2 * 2 * 32  # static block over GPU tasks
    whole_i = O.sum_i32(gen.gen_i32(gen.SEED_C1, 0, 300_007))
    whole_k = O.sum_u64(gen.gen_f32_k(gen.SEED_C5, 0, 300_007))
    for r in range(world):
        assert res[r]["int_total"] == whole_i
        assert res[r]["f32_numerators"] == whole_k
        assert res[r]["max_ms"] == 2.0
    assert np.isfinite(whole_k)
