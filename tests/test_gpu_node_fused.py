"""NEXT f1 on the GPU: the node level inside the kernel (HPAR_NEST_NODE_FUSED,
node_fused.cuh) through a real NCCL communicator — symmetric window, device
communicator, LSA stores and barrier.  One GPU here, so the communicator has
one rank: the slot write / barrier / rank-order fold all run, with G = 1.
Results must equal the oracle and the host-NCCL path, for every kernel that
has a node level (flat, hist, teams, generic incl. the ordered AFFINE op),
over repeated calls (slot halves alternate).  HPAR_NEST_NODE_ALWAYS runs the
host-enqueued node level (ncclAllReduce; the ordered op's ncclAllGather +
rank-fold kernel) and the GPU barrier's NCCL rendezvous through the same
one-rank communicator: the collective path executes, as an identity."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(port, q):
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
        t = torch.ones(1, device="cuda")
        dist.all_reduce(t)
        from inputs import gen
        from paper_2309_01906_b200 import build
        build.build()
        from paper_2309_01906_b200 import hpar as H
        from paper_2309_01906_b200 import nests
        comm = H.torch_nccl_comm()
        res = {}
        # A0: the GPU level's num through ncclCommCount of the borrowed communicator
        t = H.hpar_hierarchy_query(0, comm)
        q_gpu_num = (int(t[H.HPAR_GPU].num), dist.get_world_size())

        def run(levels, x, op, n0, reps=3, **kw):
            outs = []
            for flags in (H.HPAR_NEST_NODE_FUSED, 0, H.HPAR_NEST_NODE_ALWAYS):
                nest = H.Nest(levels, device=0, nccl_comm=comm, flags=flags, **kw)
                xd = torch.from_numpy(x).cuda()
                if op == H.OP_HIST256:
                    out = torch.zeros(256, dtype=torch.int64, device="cuda")
                elif op == H.OP_AFFINE:
                    out = torch.zeros(2, dtype=torch.int64, device="cuda")
                else:
                    out = torch.zeros(1, dtype=torch.float64 if x.dtype.kind == "f" else torch.int64, device="cuda")
                got = []
                for _ in range(reps):
                    out.zero_()
                    nest.parallel_for_reduce(H.make_desc(xd, out, n0=n0, op=op))
                    torch.cuda.synchronize()
                    got.append(out.cpu().numpy().copy())
                outs.append((nest.last_kernel(), got))
                nest.close()
            return outs

        n = (1 << 22) + 5
        res["flat"] = run(nests.c5_nest(2), gen.gen_f32(gen.SEED_C5, 0, n), H.OP_SUM, n, cluster_dim=2,
                          warps_per_cta=8)
        res["hist"] = run(nests.c4_nest(2), gen.gen_u8(gen.SEED_C4, 0, n), H.OP_HIST256, n, cluster_dim=2,
                          warps_per_cta=4)
        res["generic_min"] = run([H.Level(1, 2, H.STATIC), H.Level(3, 5, H.STATIC_CHUNK, chunk=3)],
                                 gen.gen_i32(gen.SEED_C1, 0, 100_003), H.OP_MIN, 100_003, clusters=3)
        res["generic_affine"] = run([H.Level(1, 3, H.STATIC), H.Level(4, 5, H.STATIC)],
                                    gen.gen_i32(gen.SEED_C1, 0, 70_001).astype(np.int64), H.OP_AFFINE, 70_001,
                                    clusters=2)
        # the GPU-level barrier's NCCL rendezvous through the same communicator
        bnest = H.Nest([H.Level(1, 5)], device=0, nccl_comm=comm, flags=H.HPAR_NEST_NODE_ALWAYS)
        bnest.barrier(H.HPAR_GPU, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        bnest.close()
        q.put(("ok", (res, q_gpu_num)))
        dist.destroy_process_group()
    except Exception as e:  # report, do not hang the parent
        import traceback
        q.put(("err", traceback.format_exc()))


@pytest.mark.timeout(600)
def test_node_level_in_kernel():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(_free_port(), q))
    p.start()
    status, res = q.get(timeout=540)
    p.join(60)
    assert status == "ok", res
    res, (gpu_num, world) = res
    assert gpu_num == world == 1, "hierarchy query GPU num = ncclCommCount of the communicator"
    from inputs import gen
    from oracle import oracle as O
    n = (1 << 22) + 5
    want = {
        "flat": None,
        "hist": O.hist256(gen.gen_u8(gen.SEED_C4, 0, n)),
        "generic_min": O.min_i32(gen.gen_i32(gen.SEED_C1, 0, 100_003)),
    }
    for name, ((k_fused, fused), (k_host, host), (k_coll, coll)) in res.items():
        assert k_fused == k_host == k_coll, name
        for a, b, c in zip(fused, host, coll):
            assert np.array_equal(a, b), (name, a, b)   # same kernel, same tree: bit-identical
            assert np.array_equal(c, b), (name, c, b)   # + the node collective (1 rank: identity)
        if want.get(name) is not None:
            assert np.array_equal(fused[0].astype(np.int64).ravel()[: np.size(want[name])], np.asarray(want[name]).ravel())
    # the ordered op against the oracle (not only fused vs host): block
    # schedules at every level, so the composed map is the oracle's direct
    # recurrence y <- (2x+1) y + x^2 over the 70,001 elements in order
    xa = gen.gen_i32(gen.SEED_C1, 0, 70_001).astype(np.int64)
    for got in res["generic_affine"][0][1]:
        A, B = (int(v) for v in np.asarray(got).view(np.uint64).ravel()[:2])
        for y0 in (0, 5, 123456789):
            assert (A * y0 + B) % (1 << 64) == O.affine_run(xa, y0)
    whole = O.sum_u64(gen.gen_f32_k(gen.SEED_C5, 0, n))
    assert abs(res["flat"][0][1][0][0] - whole * 2.0 ** -24) <= 1e-9 * whole * 2.0 ** -24
