"""The node level across real GPUs (§8(a) A9, A10; §8(e); NEXT f1, f3):
one process per GPU, torch's ProcessGroupNCCL communicator borrowed by the
nests.  Runs only where >= 2 GPUs are visible (the round-end box has one; the
CPU side of the same host logic is covered by the gloo tests), and then:

* ncclAllReduce node level: C1 (teams, int64), C4 (hist, u64 x 256), C5
  (flat, f64) totals on every rank vs the oracle over the whole input;
* the ordered AFFINE op: allgather + rank-order fold vs the oracle's direct
  recurrence (block schedules);
* the in-kernel node level (HPAR_NEST_NODE_FUSED, NCCL LSA stores + barrier)
  for flat and hist vs the same oracle values, over repeated calls;
* hpar_barrier(GPU): a cross-rank rendezvous that completes on every rank;
* hpar_map_exchange: two sibling stencil tiles refreshed over NCCL vs the
  sequential stencil (oracle/ghostmap.py);
* `bench.py --gpus G` spawns G ranks and reports n_gpus = G.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus() -> int:
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


needs_2 = pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs (one process per GPU)")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


N_FLAT = (1 << 22) + 12345
N_C1 = 1024


def _worker(rank, world, port, q):
    try:
        sys.path.insert(0, ROOT)
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                                device_id=dev)
        t = torch.ones(1, device=dev)
        dist.all_reduce(t)
        from inputs import gen
        from paper_2309_01906_b200 import hpar as H
        from paper_2309_01906_b200 import nests
        comm = H.torch_nccl_comm()
        res = {"gpu_num": int(H.hpar_hierarchy_query(rank, comm)[H.HPAR_GPU].num)}

        def total(levels, x_full_fn, op, n0, *, flags=0, reps=2, inner=0, **kw):
            nest = H.Nest(levels, device=rank, nccl_comm=comm, flags=flags, **kw)
            b, c = nest.shard_range(n0, rank)
            per = inner if inner else 1
            x = torch.from_numpy(x_full_fn(b * per, c * per)).to(dev)
            if op == H.OP_HIST256:
                out = torch.zeros(256, dtype=torch.int64, device=dev)
            elif op == H.OP_AFFINE:
                out = torch.zeros(2, dtype=torch.int64, device=dev)
            else:
                out = torch.zeros(1, dtype=torch.float64 if x.dtype == torch.float32 else torch.int64, device=dev)
            got = []
            for _ in range(reps):
                out.zero_()
                d = H.make_desc(x, out, op=op, n0=n0, n1=inner, ld=inner, nloops=2 if inner else 1)
                nest.parallel_for_reduce(d)
                torch.cuda.synchronize()
                got.append(out.cpu().numpy().copy())
            kern = nest.last_kernel()
            nest.close()
            return kern, got

        res["c5"] = total(nests.c5_nest(2), lambda b, c: gen.gen_f32(gen.SEED_C5, b, c), H.OP_SUM, N_FLAT,
                          cluster_dim=2, warps_per_cta=8)
        res["c4"] = total(nests.c4_nest(2), lambda b, c: gen.gen_u8(gen.SEED_C4, b, c), H.OP_HIST256, N_FLAT,
                          cluster_dim=2, warps_per_cta=8, clusters=7)
        res["c1"] = total(nests.c1_nest(outer=N_C1), lambda b, c: gen.gen_i32(gen.SEED_C1, b, c), H.OP_SUM, N_C1,
                          inner=1024, cluster_dim=2, warps_per_cta=8)
        res["affine"] = total([H.Level(1, 3, H.STATIC), H.Level(4, 5, H.STATIC)],
                              lambda b, c: gen.gen_i32(gen.SEED_C1, b, c).astype(np.int64), H.OP_AFFINE, 70_001,
                              cluster_dim=2, warps_per_cta=2, clusters=2)
        for name, lv, fn, op in (("c5_fused", nests.c5_nest(2), lambda b, c: gen.gen_f32(gen.SEED_C5, b, c), H.OP_SUM),
                                 ("c4_fused", nests.c4_nest(2), lambda b, c: gen.gen_u8(gen.SEED_C4, b, c),
                                  H.OP_HIST256)):
            res[name] = total(lv, fn, op, N_FLAT, flags=H.HPAR_NEST_NODE_FUSED, reps=3, cluster_dim=2,
                              warps_per_cta=8, clusters=7 if op == H.OP_HIST256 else 0)
        # GPU-level barrier: a rendezvous that completes on every rank
        nest = H.Nest(nests.c5_nest(2), device=rank, nccl_comm=comm)
        nest.barrier(H.HPAR_GPU, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        res["barrier"] = True
        nest.close()
        # ghost exchange (f3): a 2 x 1 sibling grid of tile x tile from-sections
        from oracle import ghostmap as G
        tile, T = 96, 3
        extent = (world * tile + 2, tile + 2)
        m = H.map_spec(extent, world, 1, [(tile, 0, tile + 2), (tile, 0, tile + 2)], [(tile, 1, tile), (tile, 1, tile)])
        H.hpar_map_validate(m)
        to, fr = H.hpar_map_sections(m, rank)
        A = gen.gen_f32(gen.SEED_C5, 0, extent[0] * extent[1]).reshape(extent)
        snest = H.Nest(nests.stencil_nest(), device=rank, nccl_comm=comm)
        ld = (to.len[1] + 31) // 32 * 32
        a = torch.zeros((to.len[0], ld), dtype=torch.float32, device=dev)
        a[:, :to.len[1]] = torch.from_numpy(A[to.off[0]:to.off[0] + to.len[0], to.off[1]:to.off[1] + to.len[1]].copy()).to(dev)
        b_ = a.clone()
        s = torch.cuda.current_stream().cuda_stream
        for _ in range(T):
            H.hpar_stencil5(snest, H.stencil_desc(a, b_, ld, to, fr, extent), s)
            H.hpar_map_exchange(snest, m, b_, ld, s)
            a, b_ = b_, a
        torch.cuda.synchronize()
        r0, c0 = fr.off[0] - to.off[0], fr.off[1] - to.off[1]
        res["stencil"] = (fr.tup(), a[r0:r0 + fr.len[0], c0:c0 + fr.len[1]].cpu().numpy(), G.stencil5(A, T),
                          (fr.off[0], fr.off[1], fr.len[0], fr.len[1]))
        snest.close()
        q.put((rank, "ok", res))
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, "err", traceback.format_exc()))


@needs_2
@pytest.mark.timeout(900)
def test_node_level_across_gpus(oracle):
    import torch.multiprocessing as mp
    from inputs import gen
    world = min(_ngpus(), 8)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, status, res = q.get(timeout=800)
        assert status == "ok", res
        out[r] = res
    for p in procs:
        p.join(60)
    exact5 = oracle.sum_u64(gen.gen_f32_k(gen.SEED_C5, 0, N_FLAT)) * 2.0 ** -24
    bins4 = oracle.hist256(gen.gen_u8(gen.SEED_C4, 0, N_FLAT))
    sum1 = oracle.sum_i32(gen.gen_i32(gen.SEED_C1, 0, N_C1 * 1024))
    xa = gen.gen_i32(gen.SEED_C1, 0, 70_001).astype(np.int64)
    for r, res in out.items():
        assert res["gpu_num"] == world
        for name in ("c5", "c5_fused"):
            kern, got = res[name]
            assert kern == "flat_tma"
            for g in got:
                assert abs(g[0] - exact5) <= 1e-5 * exact5, (r, name)
        for name in ("c4", "c4_fused"):
            kern, got = res[name]
            assert kern.startswith("hist256_lanepriv")
            for g in got:
                assert np.array_equal(g.astype(np.uint64), bins4), (r, name)
        kern, got = res["c1"]
        assert kern == "teams_threads"
        assert all(int(g[0]) == sum1 for g in got)
        kern, got = res["affine"]
        for g in got:
            A, B = (int(v) for v in g.view(np.uint64))
            assert (A * 7 + B) % (1 << 64) == oracle.affine_run(xa, 7)
        assert res["barrier"]
        _, tile_got, whole, (r0, c0, nr, nc) = res["stencil"]
        assert np.array_equal(tile_got, whole[r0:r0 + nr, c0:c0 + nc]), r


@needs_2
@pytest.mark.timeout(900)
def test_bench_spawns_ranks_on_gpus():
    """`bench.py --gpus 2` (no launcher) spawns two ranks over NCCL and times
    the strong-scaled C2 matrix on both: n_gpus 2 in the JSON line."""
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "c2", "--steps", "20", "--warmup", "3",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=800, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["elements_total"] == 65536 * 4096
