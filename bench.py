#!/usr/bin/env python3
"""bench.py — throughput of the hpar hot path on B200 (BASELINE.json metric:
"elements/s and HBM GB/s (% of peak) for nested reductions at 1/2/4/8 B200").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5|c2|c4|c1|c3|c6] [--impl hpar|reference]

A step is one hpar_parallel_for_reduce over one batch of the config's
synthetic workload (seeded generator, inputs/gen.py recipe), inputs resident
in HBM.  Default workload: config 5 (BASELINE.json configs[4], the largest
single-GPU configuration): the 5-level flat nest GPU -> cluster -> CTA ->
warp -> lane summing 2^34 fp32 (64 GiB), strong-scaled over the GPUs with
one NCCL allreduce at the node level.  Config 2 (configs[1], the 4-level
row-wise nest over ONE 65536 x 4096 fp32 matrix) is strong-scaled too: its
rows are sharded over the GPUs.  `--gpus N` without a
launcher spawns N ranks itself (torch.distributed.run, one process per GPU,
127.0.0.1 rendezvous); under torchrun WORLD_SIZE must equal N.  Rank 0 prints
ONE JSON line.  `--impl reference` times the CPU oracle (the reference arm
for this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "elements/s and HBM GB/s (% of peak) for nested reductions at 1/2/4/8 B200"
NOMINAL_HBM_GBS = 8000.0
RED_SHARED_PEAK_UPS = 8.785e12  # red.shared.add.u32, lane-private (profiles/r01_red_shared_peak.txt)
L2_BYTES = 126 * 2 ** 20


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        j = json.load(open(p))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


# ---------------------------------------------------------------- clocks --
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.marks = [None, None]

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def mark(self, i):
        self.marks[i] = time.time()

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()
        rows = []
        t0, t1 = self.marks
        for ts, line in self.samples:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            rows.append((ts, parts))
        inside = [r for r in rows if t0 and t1 and t0 - 0.05 <= r[0] <= t1 + 0.05] or rows
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(p[0]) for _, p in inside if p[0].replace(".", "").isdigit()]
        smax = [float(p[1]) for _, p in inside if p[1].replace(".", "").isdigit()]
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        reasons = sorted({names[k] for _, p in inside for k in range(4) if p[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(inside)}


# --------------------------------------------------------------- configs --
def config_spec(name: str, nranks: int):
    from inputs import gen
    if name == "c2":  # one 65536 x 4096 matrix, rows sharded over the GPUs
        rows, cols = 65536, 4096
        return dict(workload="c2_rowwise_4level_65536x4096_f32", kind="rowwise", cols=cols,
                    n0=rows, scaling="strong", seed=gen.SEED_C2, dtype="f32", elems_total=rows * cols)
    if name == "c5":
        n = 1 << 34
        return dict(workload="c5_flat_5level_2^34_f32", kind="flat", n0=n, scaling="strong", seed=gen.SEED_C5,
                    dtype="f32", elems_total=n)
    if name == "c4":
        n = 1 << 32
        return dict(workload="c4_hist256_2^32_u8", kind="hist", n0=n, scaling="strong", seed=gen.SEED_C4,
                    dtype="u8", elems_total=n)
    if name == "c1":
        return dict(workload="c1_2level_1024x1024_i32", kind="c1", n0=1024, cols=1024, scaling="weak",
                    seed=gen.SEED_C1, dtype="i32", elems_per_rank=1 << 20, bytes_per_rank=(1 << 22) + 8)
    if name == "c3":  # one 2^24-row matrix; rows sharded at nnz-balanced boundaries (§8(e))
        return dict(workload="c3_csr_segmented_2^24rows_2^28nnz_f32", kind="csr", rows=1 << 24, nnz=1 << 28,
                    n0=1 << 24, scaling="strong", seed=gen.SEED_C3, dtype="f32", elems_total=1 << 28)
    if name == "c6":  # NEXT f3: §4 ghost maps + 5-point stencil, one Jacobi sweep per step
        tile = 16384
        return dict(workload="c6_stencil5_16384x16384_per_gpu_f32", kind="stencil", tile=tile, n0=tile * tile,
                    scaling="weak", seed=gen.SEED_C5, dtype="f32", elems_per_rank=tile * tile,
                    bytes_per_rank=tile * tile * 8)
    raise SystemExit(f"unknown config {name}")


# ------------------------------------------------------------- hpar arm ---
def run_hpar(args):
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2309_01906_b200 import build as pbuild
    if int(os.environ.get("RANK", "0")) == 0:
        pbuild.build()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        dist.barrier()
        pbuild.build()  # no-op after rank 0 built
    from paper_2309_01906_b200 import hpar as H
    from paper_2309_01906_b200 import nests

    comm = None
    if world > 1:
        t = torch.ones(1, device=dev)
        dist.all_reduce(t)
        comm = H.torch_nccl_comm()
    spec = config_spec(args.config, world)
    # --shard G (diagnostic, one GPU): time rank 0's shard of a G-GPU run of a
    # keyed config (rows are independent: a rank's kernel is exactly this)
    sim_world, sim_rank = world, rank
    shard_kw = {}
    flat_shard = 1  # c4 / c5: a rank's shard is n0 / G elements of the same kernel
    if args.shard > 1:
        if world > 1 or args.config not in ("c2", "c3", "c4", "c5"):
            raise SystemExit("--shard G: one process, configs c2, c3, c4, c5")
        if args.config in ("c2", "c3"):
            sim_world, sim_rank = args.shard, 0
            shard_kw = dict(nranks=sim_world, rank=sim_rank)
        else:  # the GPU level is host-applied: rank 0's launch is the nest over its n0 / G elements
            flat_shard = args.shard
    L = ctypes.CDLL(os.path.join(ROOT, "inputs", "libhpar_inputs.so"))
    for f in ("hpar_inputs_fill_f32", "hpar_inputs_fill_u8", "hpar_inputs_fill_i32"):
        getattr(L, f).argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    # tuned geometry per config (sweeps in profiles/)
    tuned = {"c2": (4, 444), "c4": (8, 74), "c5": (4, 148), "c1": (8, 148)}.get(args.config, (8, 0))
    K = int(os.environ.get("HPAR_K", "2"))  # CTAs per cluster (knob; 2 = tuned)
    W = args.warps or tuned[0]
    if args.clusters < 0:
        args.clusters = tuned[1]
    kind = spec["kind"]
    extra_inputs = []
    step = e2e_step = None
    if kind == "stencil":
        # sibling grid: gx = 2 columns once there are 2+ GPUs; each GPU's from-
        # tile is tile x tile with a 1-cell ghost ring (P:376-377 form)
        tile = spec["tile"]
        gx = 1 if world == 1 else 2
        gy = world // gx
        extent = (gy * tile + 2, gx * tile + 2)
        mspec = H.map_spec(extent, world, gx, [(tile, 0, tile + 2), (tile, 0, tile + 2)],
                           [(tile, 1, tile), (tile, 1, tile)])
        H.hpar_map_validate(mspec)
        to, fr = H.hpar_map_sections(mspec, rank)
        nest = H.Nest(nests.stencil_nest(), device=local, nccl_comm=comm)
        lda = int(os.environ.get("HPAR_C6_LDA", "32"))  # row pitch: whole 128-byte lines (knob; 4 = 16 B, 2.5% slower)
        ld = (tile + 2 + lda - 1) // lda * lda
        x = torch.empty((tile + 2, ld), dtype=torch.float32, device=dev)
        L.hpar_inputs_fill_f32(spec["seed"], rank * x.numel(), x.numel(), x.data_ptr(), sptr)
        out = x.clone()
        descs = [H.stencil_desc(x, out, ld, to, fr, extent), H.stencil_desc(out, x, ld, to, fr, extent)]
        bufs = [x, out]
        phase = [0]

        def step():
            cs = torch.cuda.current_stream().cuda_stream
            H.hpar_stencil5(nest, descs[phase[0]], cs)
            H.hpar_map_exchange(nest, mspec, bufs[1 - phase[0]], ld, cs)
            phase[0] ^= 1

        def e2e_step():  # host input -> x, one sweep into out (+ ghost refresh), out -> host
            H.hpar_stencil5(nest, descs[0], sptr)
            H.hpar_map_exchange(nest, mspec, out, ld, sptr)

        elems_rank = tile * tile
        alg_bytes = tile * tile * 8
        host_in_bytes, host_out_bytes = x.numel() * 4, out.numel() * 4
    elif kind == "rowwise":
        nest = H.Nest(nests.c2_nest(), device=local, nccl_comm=comm, cluster_dim=K, warps_per_cta=W,
                      clusters=args.clusters, **shard_kw)
        b, cnt = nest.shard_range(spec["n0"], sim_rank)
        cols = spec["cols"]
        x = torch.empty(cnt * cols, dtype=torch.float32, device=dev)
        L.hpar_inputs_fill_f32(spec["seed"], b * cols, cnt * cols, x.data_ptr(), sptr)
        out = torch.empty(cnt, dtype=torch.float32, device=dev)
        mk = lambda xx, oo, ex: H.make_desc(xx, oo, n0=spec["n0"], n1=cols, ld=cols, nloops=2, keyed=True)
        desc = mk(x, out, [])
        elems_rank = cnt * cols
        alg_bytes = cnt * cols * 4 + cnt * 4
        host_in_bytes, host_out_bytes = cnt * cols * 4, cnt * 4
    elif kind in ("flat", "hist"):
        nflags = H.HPAR_NEST_NODE_FUSED if (args.node == "fused" and comm is not None) else 0
        if kind == "flat":
            nest = H.Nest(nests.c5_nest(K), device=local, nccl_comm=comm, cluster_dim=K, warps_per_cta=W,
                          clusters=args.clusters, flags=nflags)
        else:
            nest = H.Nest(nests.c4_nest(K, tile=int(os.environ.get("HPAR_C4_TILE", nests.TILE_U8))),
                          device=local, nccl_comm=comm, cluster_dim=K, warps_per_cta=W,
                          clusters=args.clusters, flags=nflags)
        b, cnt = nest.shard_range(spec["n0"] // flat_shard, rank)
        if kind == "flat":
            x = torch.empty(cnt, dtype=torch.float32, device=dev)
            L.hpar_inputs_fill_f32(spec["seed"], b, cnt, x.data_ptr(), sptr)
            out = torch.empty(1, dtype=torch.float64, device=dev)
            alg_bytes = cnt * 4 + 8
            host_in_bytes = cnt * 4
        else:
            x = torch.empty(cnt, dtype=torch.uint8, device=dev)
            L.hpar_inputs_fill_u8(spec["seed"], b, cnt, x.data_ptr(), sptr)
            out = torch.empty(256, dtype=torch.int64, device=dev)
            alg_bytes = cnt + 2048
            host_in_bytes = cnt
        mk = lambda xx, oo, ex: H.make_desc(xx, oo, n0=spec["n0"] // flat_shard,
                                            op=H.OP_HIST256 if kind == "hist" else H.OP_SUM)
        desc = mk(x, out, [])
        elems_rank = cnt
        host_out_bytes = out.numel() * out.element_size()
    elif kind == "c1":
        # teams: 0 = C clusters x K CTAs (bench default C = 148: 296 teams of
        # 3-4 rows, 10.8 us; 1024 teams of one row each: 14.9 us); HPAR_C1_TEAMS
        # = 1024 is the one-row-per-team form
        teams = int(os.environ.get("HPAR_C1_TEAMS", "0"))
        nest = H.Nest(nests.c1_nest(outer=teams), device=local, nccl_comm=comm, cluster_dim=K, warps_per_cta=W,
                      clusters=args.clusters if teams == 0 else 0,
                      flags=H.HPAR_NEST_NODE_FUSED if (args.node == "fused" and comm is not None) else 0)
        b, cnt = nest.shard_range(spec["n0"] * world, rank)
        x = torch.empty(cnt * 1024, dtype=torch.int32, device=dev)
        L.hpar_inputs_fill_i32(spec["seed"], b * 1024, cnt * 1024, x.data_ptr(), sptr)
        out = torch.empty(1, dtype=torch.int64, device=dev)
        mk = lambda xx, oo, ex: H.make_desc(xx, oo, n0=spec["n0"] * world, n1=1024, ld=1024, nloops=2)
        desc = mk(x, out, [])
        elems_rank = cnt * 1024
        alg_bytes = cnt * 1024 * 4 + 8
        host_in_bytes, host_out_bytes = cnt * 4096, 8
    else:  # c3: CSR segmented rows
        from inputs import gen
        rows, nnz = spec["rows"], spec["nnz"]
        off_host = gen.csr_offsets(rows, nnz)
        nest = H.Nest(nests.c3_fast_nest(lane_chunk=int(os.environ.get("HPAR_C3_LPL", "16"))), device=local, nccl_comm=comm, cluster_dim=K, warps_per_cta=W,
                      clusters=args.clusters, **shard_kw)
        b, cnt = H.hpar_shard_range_csr(off_host, sim_world, sim_rank)  # nnz-balanced row shard
        lo = off_host[b:b + cnt + 1] - off_host[b]
        nnz_l = int(lo[-1])
        off = torch.from_numpy(lo).to(dev)
        x = torch.empty(max(nnz_l, 4), dtype=torch.float32, device=dev)
        L.hpar_inputs_fill_f32(spec["seed"], int(off_host[b]), nnz_l, x.data_ptr(), sptr)  # global indices
        out = torch.empty(max(cnt, 1), dtype=torch.float32, device=dev)
        mx = int((lo[1:] - lo[:-1]).max()) if cnt else 0
        mk = lambda xx, oo, ex: H.make_desc(xx, oo, n0=rows, n1=nnz_l, nloops=2, keyed=True, offsets=ex[0],
                                            local_n0=cnt, max_inner=mx)
        desc = mk(x, out, [off])
        elems_rank = nnz_l
        alg_bytes = nnz_l * 4 + (cnt + 1) * 8 + cnt * 4
        host_in_bytes, host_out_bytes = nnz_l * 4 + (cnt + 1) * 8, cnt * 4
        extra_inputs = [off]
    torch.cuda.synchronize()

    # L2: a working set under 3 x L2 (c1; c2 / c3 shards at 4+ GPUs) is timed
    # over rotating input copies (>= 3 x L2 together), so no step finds its
    # inputs in L2 and no flush leaves dirty lines to write back during the
    # kernel; larger inputs need neither
    rot_descs = [desc] if step is None else []
    rot_keep = []  # the copies' tensors: a desc holds raw pointers only
    if step is None and alg_bytes < 3 * L2_BYTES:
        ncopy = min(128, -(-3 * L2_BYTES // max(alg_bytes, 1)) + 1)
        for _ in range(ncopy - 1):
            xc, oc, ec = x.clone(), out.clone(), [t.clone() for t in extra_inputs]
            rot_keep.append((xc, oc, ec))
            rot_descs.append(mk(xc, oc, ec))
        assert len({d.in_ for d in rot_descs}) == len(rot_descs), "rotating copies must be distinct buffers"
    rot = [0]
    if step is None:
        def step():
            nest.parallel_for_reduce(rot_descs[rot[0]], torch.cuda.current_stream().cuda_stream)
            rot[0] = (rot[0] + 1) % len(rot_descs)
    if e2e_step is None:
        def e2e_step():
            nest.parallel_for_reduce(desc, sptr)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # external=True: inside a graph capture the records become event-record
    # nodes that timestamp when the graph runs (not capture-time dependencies)
    ev = [(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
          for _ in range(args.steps)]
    t_all0 = torch.cuda.Event(enable_timing=True, external=True)
    t_all1 = torch.cuda.Event(enable_timing=True, external=True)

    def timed_steps():
        t_all0.record()
        for i in range(args.steps):
            ev[i][0].record()
            step()
            ev[i][1].record()
        t_all1.record()

    graph = None
    # multi-rank runs stay eager (the node level's NCCL call inside a capture is
    # not exercised on this round's one-GPU boxes; --graph forces it)
    if not args.no_graph and (world == 1 or args.graph):
        # the K timed steps as ONE CUDA graph, event records included: the
        # device runs them back to back, so a step's events bracket its
        # kernel(s), not the host's launch latency (launch-bound configs)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, capture_error_mode="relaxed"):
            timed_steps()
        torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.15)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark(0)
    if graph is None:
        timed_steps()
    else:
        graph.replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks.mark(1)
    time.sleep(0.1)
    clk = clocks.stop()
    kern_ms = [a.elapsed_time(b_) for a, b_ in ev]
    step_ms_local = sum(kern_ms) / len(kern_ms)
    # max over ranks
    t = torch.tensor([step_ms_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms = float(t.item())
    # whole-job HBM rate: every rank's algorithmic bytes / the slowest rank's time
    tb = torch.tensor([float(alg_bytes)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tb)
    bytes_all = float(tb.item())
    elems_total = elems_rank * world if spec["scaling"] == "weak" else spec["n0"] * (1024 if kind == "c1" else 1)
    if spec["scaling"] == "strong":
        elems_total = spec.get("elems_total", spec["n0"])
    if args.shard > 1:
        elems_total = elems_rank  # the one shard timed here
    value = elems_total / (step_ms * 1e-3)
    peak, peak_src = measured_peak()
    achieved = alg_bytes / (step_ms_local * 1e-3) / 1e9

    # ---------------- e2e: host buffers through the C ABI ----------------
    e2e = None
    if not args.no_e2e:
        e2e_steps = max(1, min(args.steps, args.e2e_steps))
        dev_inputs = [x] + extra_inputs
        host_inputs = []
        for t_ in dev_inputs:
            h_ = torch.empty(tuple(t_.shape), dtype=t_.dtype, pin_memory=True)
            h_.copy_(t_)
            host_inputs.append(h_)
        host_out = torch.empty(tuple(out.shape), dtype=out.dtype, pin_memory=True)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            for d_, h_ in zip(dev_inputs, host_inputs):
                d_.copy_(h_, non_blocking=True)
            e2e_step()
            host_out.copy_(out, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = torch.tensor([e0.elapsed_time(e1) / e2e_steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": elems_total / (float(e2e_ms.item()) * 1e-3), "unit": "elements/s",
               "h2d_bytes_per_step": int(host_in_bytes), "d2h_bytes_per_step": int(host_out_bytes),
               "steps": e2e_steps, "ms_per_step": float(e2e_ms.item())}

    kernel = nest.last_kernel()
    traffic = None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic = tj.get(f"{args.config}:{kernel}")
    except Exception:
        pass
    line = {
        "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": spec["scaling"],
        "vs_baseline": None, "dtype": spec["dtype"], "data": "synthetic (seeded splitmix64, inputs/gen.py recipe)",
        "config": {"workload": spec["workload"] + (f" (rank 0 shard of {args.shard} GPUs, diagnostic)" if args.shard > 1 else ""),
                   "kernel": kernel, "n0_global": spec["n0"],
                   "elements_total": elems_total, "parallelism": f"gpu{world}",
                   "l2": (f"{len(rot_descs)} rotating input copies ({len(rot_descs) * alg_bytes / 2**20:.0f} MiB >= 3 x L2)"
                          if len(rot_descs) > 1 else "inputs > 3 x L2, no flush"),
                   "geometry": {"C": nest.info().C, "K": K, "W": W},
                   "node_level": ("in-kernel (NCCL LSA)" if args.node == "fused" else "ncclAllReduce")
                   if world > 1 and kind in ("flat", "hist", "c1") else None},
        "hbm_gbs": achieved,  # this rank's kernel, algorithmic bytes / device time
        "pct_of_8tbs": achieved / NOMINAL_HBM_GBS,
        "hbm_gbs_all_gpus": bytes_all / (step_ms * 1e-3) / 1e9,
        "pct_of_aggregate_peak": bytes_all / (step_ms * 1e-3) / 1e9 / (measured_peak()[0] * world),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src, "kernel": kernel,
                     "algorithmic_bytes_per_launch": int(alg_bytes)},
        "clocks": clk, "e2e": e2e, "gpu_launches": args.steps,
        "timing": ("eager launches" if graph is None else f"one CUDA graph of the {args.steps} steps (event records inside)")
                  + ", CUDA events per step, max over ranks",
    }
    if kind == "hist":  # the second ceiling: shared-memory RED throughput (profiles/r01_red_shared_peak.txt)
        ups = elems_rank / (step_ms_local * 1e-3)
        line["roofline_smem_red"] = {"bound": "smem_red", "achieved": ups, "peak": RED_SHARED_PEAK_UPS,
                                     "unit": "updates/s", "frac": ups / RED_SHARED_PEAK_UPS,
                                     "peak_source": "measured, scripts/red_shared_peak.cu"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, budget_s=args.cpu_budget)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------ CPU oracle legs ---
def host_cpu() -> dict:
    """The box's CPU model and logical core count (reported next
    to the oracle's one-core timing)."""
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "host_cores": os.cpu_count()}


def cpu_baseline(config: str, budget_s: float = 10.0, samples: int = 1):
    """Time the oracle (plain sequential C, one core) on a bounded sample of
    the workload; returns elements/s, what was sampled and the host CPU."""
    r = _cpu_baseline(config, budget_s)
    if r is not None:
        r.update(host_cpu())
    return r


def _cpu_baseline(config: str, budget_s: float = 10.0):
    import numpy as np

    from inputs import gen
    from oracle import oracle as O
    O.build()
    cores = 1
    if config == "c2":
        cols = 4096
        rows = 8192
        a = gen.gen_f32(gen.SEED_C2, 0, rows * cols)
        O.rowsum_f32(a[: 64 * cols], 64, cols)  # warm
        t0 = time.perf_counter()
        reps = 0
        while True:
            O.rowsum_f32(a, rows, cols)
            reps += 1
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
        return {"value": reps * rows * cols / dt, "unit": "elements/s", "cores": cores, "kind": "oracle",
                "sample": f"or_rowsum_f32 over {rows} rows x {cols} of the c2 matrix, {reps} passes, {dt:.1f} s"}
    if config in ("c5", "c1"):
        n = 1 << 26
        x = gen.gen_f32(gen.SEED_C5, 0, n) if config == "c5" else gen.gen_i32(gen.SEED_C1, 0, n)
        f = O.sum_f32 if config == "c5" else O.sum_i32
        t0 = time.perf_counter()
        reps = 0
        while True:
            f(x)
            reps += 1
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
        return {"value": reps * n / dt, "unit": "elements/s", "cores": cores, "kind": "oracle",
                "sample": f"{f.__name__} over the first 2^26 elements, {reps} passes, {dt:.1f} s"}
    if config in ("c3", "c6"):
        f, n, what = oracle_step_fn(config, 1 << 24)
        t0 = time.perf_counter()
        reps = 0
        while True:
            f()
            reps += 1
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
        return {"value": reps * n / dt, "unit": "elements/s", "cores": cores, "kind": "oracle",
                "sample": f"{what}, {reps} passes, {dt:.1f} s"}
    if config == "c4":
        n = 1 << 26
        x = gen.gen_u8(gen.SEED_C4, 0, n)
        t0 = time.perf_counter()
        reps = 0
        while True:
            O.hist256(x)
            reps += 1
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
        return {"value": reps * n / dt, "unit": "elements/s", "cores": cores, "kind": "oracle",
                "sample": f"or_hist256 over the first 2^26 bytes, {reps} passes, {dt:.1f} s"}
    return None


def oracle_step_fn(config: str, n_elems: int):
    """(callable, elements per call, description): the oracle's plain
    definition over a bounded sample of the config's workload."""
    from inputs import gen
    from oracle import oracle as O
    O.build()
    if config == "c2":
        cols = 4096
        rows = max(1, min(65536, n_elems // cols))
        a = gen.gen_f32(gen.SEED_C2, 0, rows * cols)
        return (lambda: O.rowsum_f32(a, rows, cols)), rows * cols, f"or_rowsum_f32 over rows [0,{rows}) x 4096"
    if config == "c3":
        off = gen.csr_offsets(1 << 24, 1 << 28)
        rows = int(np.searchsorted(off, min(n_elems, 1 << 28))) if n_elems else 1
        rows = max(1, min(1 << 24, rows))
        nnz = int(off[rows])
        v = gen.gen_f32(gen.SEED_C3, 0, nnz)
        o = off[: rows + 1].copy()
        return (lambda: O.segsum_f32(v, o)), nnz, f"or_segsum_f32 over rows [0,{rows}) ({nnz} nonzeros)"
    if config == "c6":
        from oracle import ghostmap as G
        side = int(max(64, min(16386, int(np.sqrt(max(n_elems, 1))))))
        a = gen.gen_f32(gen.SEED_C5, 0, side * side).reshape(side, side)
        return (lambda: G.stencil5_step(a)), side * side, f"ghostmap.stencil5_step (numpy fp32) on {side} x {side}"
    # the sample is bounded: c1's whole workload is 2^20 elements; c4/c5 at
    # most 2^28 elements (1 GiB of fp32) per step
    n = max(1024, min(n_elems, (1 << 20) if config == "c1" else (1 << 28)))
    if config == "c4":
        x = gen.gen_u8(gen.SEED_C4, 0, n)
        return (lambda: O.hist256(x)), n, f"or_hist256 over bytes [0,{n})"
    if config == "c1":
        x = gen.gen_i32(gen.SEED_C1, 0, n)
        return (lambda: O.sum_i32(x)), n, f"or_sum_i32 over elements [0,{n})"
    x = gen.gen_f32(gen.SEED_C5, 0, n)
    return (lambda: O.sum_f32(x)), n, f"or_sum_f32 over elements [0,{n})"


def run_reference(args):
    """The reference arm of this tier: the CPU oracle as it stands, one core,
    W untimed + K timed steps, each step a bounded sample of the workload
    (sized so the whole run takes about a minute)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    spec = config_spec(args.config, 1)
    f, n, _ = oracle_step_fn(args.config, 1 << 20)
    t0 = time.perf_counter()
    f()
    per_elem = (time.perf_counter() - t0) / n
    target = min(10.0, 60.0 / max(1, args.steps + args.warmup))
    f, n, what = oracle_step_fn(args.config, int(target / max(per_elem, 1e-12)))
    for _ in range(args.warmup):
        f()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        f()
    dt = time.perf_counter() - t0
    value = n * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": spec["scaling"], "vs_baseline": None, "dtype": spec["dtype"],
        "data": "synthetic (seeded splitmix64, inputs/gen.py recipe)",
        "config": {"workload": spec["workload"],
                   "kernel": "oracle (CPU, numpy fp32)" if args.config == "c6" else "oracle (CPU, sequential C)"},
        "cpu_baseline": {"value": value, "unit": "elements/s", "cores": 1, "kind": "oracle",
                         "sample": f"{what} per step, {args.steps} timed steps, {dt:.1f} s", **host_cpu()},
        "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch_ranks(n: int, argv: list[str]) -> int:
    """Run this script as n ranks (one process per GPU) under
    torch.distributed.run on this node, 127.0.0.1 rendezvous; returns the
    launcher's exit code.  The native library is built once, before the
    ranks start."""
    if "--check-launch" not in argv:
        from paper_2309_01906_b200 import build as pbuild
        pbuild.build()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


def check_launch(args):
    """--check-launch: the launcher's plumbing without a GPU — every rank
    joins a gloo process group, the ranks' ids are summed, rank 0 prints the
    world size it saw (tests/test_bench_contract.py)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([rank], dtype=torch.int64)
    if world > 1:
        dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"check_launch": True, "n_gpus": world, "rank_sum": int(t.item())}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5", "c6"])
    ap.add_argument("--check-launch", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--shard", type=int, default=1,
                    help="diagnostic: time rank 0's shard of a G-GPU run on this one GPU (c2, c3, c4, c5)")
    ap.add_argument("--impl", default="hpar", choices=["hpar", "reference"])
    ap.add_argument("--node", default="nccl", choices=["nccl", "fused"],
                    help="node level of total reductions at N>1: host ncclAllReduce, or in-kernel (NEXT f1)")
    ap.add_argument("--clusters", type=int, default=-1, help="C (0 = resident clusters, -1 = tuned default)")
    ap.add_argument("--warps", type=int, default=0, help="W warps per CTA (0 = tuned default)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of one CUDA graph of K steps")
    ap.add_argument("--graph", action="store_true", help="capture the K steps in a CUDA graph also when N > 1")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if "WORLD_SIZE" in os.environ:
        if int(os.environ["WORLD_SIZE"]) != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started WORLD_SIZE="
                             f"{os.environ['WORLD_SIZE']} ranks")
    elif args.gpus > 1:
        sys.exit(launch_ranks(args.gpus, sys.argv[1:]))
    if args.check_launch:
        check_launch(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_hpar(args)


if __name__ == "__main__":
    main()
