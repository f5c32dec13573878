"""CPU-only tests of libhpar.so's host side: the library loads and exports
every symbol include/*.h declares; the level table (Table 2 for B200);
nest validation and its diagnostics (describe-only nests, no GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def H():
    from paper_2309_01906_b200 import build
    build.build()
    from paper_2309_01906_b200 import hpar
    return hpar


def declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return set(re.findall(r"\b(hpar_[a-z_0-9]+)\s*\(", txt))


def test_exports_every_declared_symbol(H):
    lib = ctypes.CDLL(H.LIB_PATH)
    names = declared("hpar.h")
    assert {"hpar_hierarchy_query", "hpar_nest_create", "hpar_parallel_for_reduce", "hpar_barrier"} <= names
    for n in names:
        assert hasattr(lib, n), n
    inp = ctypes.CDLL(os.path.join(ROOT, "inputs", "libhpar_inputs.so"))
    for n in declared("hpar_inputs.h"):
        assert hasattr(inp, n), n


def test_level_table_b200(H):
    t = H.hpar_hierarchy_describe(H.b200_desc(), nranks=8, cluster_dim=2, warps_per_cta=8)
    names = [r.name.decode() for r in t]
    assert names == ["node", "gpu", "cluster", "cta", "warp", "lane"]
    f = {r.name.decode(): r.flags() for r in t}
    assert t[1].num == 8 and t[3].num == 2 and t[4].num == 8 and t[5].num == 32
    assert "barrier" not in f["cluster"]          # P:178 read as "does not support"
    assert "atomic" not in f["gpu"]               # P:72 no cross-GPU atomics
    assert "shuffle" in f["lane"] and "lockstep" not in f["lane"]   # P:616-619 ITS
    assert "dynamic" in f["cluster"] and "dynamic" not in f["lane"]
    assert "oversubscribable" in f["cluster"]
    assert t[3].localmem_bytes == 2 * t[4].localmem_bytes   # DSMEM = K x smem
    g = [r.grainedness for r in t]
    assert g == sorted(g, reverse=True)           # P:140 grainedness shrinks inward


def test_collapse_is_intersection_and_product(H):
    """S:83-91 / acceptance #6 over all contiguous runs of the B200 levels."""
    d = H.b200_desc()
    t = H.hpar_hierarchy_describe(d, nranks=4, cluster_dim=2, warps_per_cta=8, clusters=10)
    for first in range(1, 6):
        for last in range(first, 6):
            levels = []
            if first > 1:
                levels.append(H.Level(1, first - 1))
            levels.append(H.Level(first, last))
            if last < 5:
                levels.append(H.Level(last + 1, 5))
            nest = H.Nest(levels, device=-1, desc=d, cluster_dim=2, warps_per_cta=8, clusters=10,
                          nranks=4, rank=1)
            info = nest.info()
            a = 1 if first > 1 else 0
            flags = 0xFFFFFFFF
            num = 1
            for hw in range(first, last + 1):
                flags &= t[hw].props
                num *= t[hw].num
            assert info.props[a] == flags and info.tasks[a] == num


def test_partition_algebra(H):
    """width divides num, outer num/width, inner width; width = num
    is the identity; width 5 is an error."""
    d = H.b200_desc()
    for w in (1, 2, 4, 8, 16, 32):
        nest = H.Nest([H.Level(1, 4), H.Level(5, 5, width=w), H.Level(5, 5)], device=-1, desc=d,
                      clusters=3, warps_per_cta=2)
        info = nest.info()
        assert info.tasks[1] == 32 // w and info.tasks[2] == w and info.lane_width == (w if w else 0)
        assert info.props[1] == info.props[2]   # the inner slice keeps the lane's flags
    for bad in (5, 3, 64):
        with pytest.raises(H.HparError) as e:
            H.Nest([H.Level(1, 4), H.Level(5, 5, width=bad), H.Level(5, 5)], device=-1, desc=d)
        assert e.value.code == H.HPAR_E_PARTITION


def test_capability_and_structure_errors(H):
    d = H.b200_desc()
    cases = [
        ([H.Level(1, 4), H.Level(5, 5, H.DYNAMIC, chunk=4)], H.HPAR_E_CAPABILITY),   # lanes: no dynamic
        ([H.Level(1, 1, H.DYNAMIC, chunk=4), H.Level(2, 5)], H.HPAR_E_CAPABILITY),   # GPUs: no dynamic
        ([H.Level(1, 2), H.Level(4, 5)], H.HPAR_E_INVALID),                          # not contiguous
        ([H.Level(1, 3)], H.HPAR_E_INVALID),                                         # must end at lane
        ([H.Level(1, 5, H.STATIC_CHUNK, chunk=0)], H.HPAR_E_INVALID),                # chunk >= 1
        ([H.Level(1, 3, width=2), H.Level(3, 5)], H.HPAR_E_UNSUPPORTED),             # only lanes split
        ([H.Level(1, 1), H.Level(2, 3, fanout=7), H.Level(4, 5)], H.HPAR_E_INVALID),  # 7 teams, K=2
    ]
    for levels, code in cases:
        with pytest.raises(H.HparError) as e:
            H.Nest(levels, device=-1, desc=d)
        assert e.value.code == code, (levels, e.value)
    # more ranks than GPU-level: the nest must bind the GPU level
    with pytest.raises(H.HparError) as e:
        H.Nest([H.Level(2, 5)], device=-1, desc=d, nranks=2)
    assert e.value.code == H.HPAR_E_INVALID
    # fanout on teams fixes the cluster count (config 1: 1024 teams)
    nest = H.Nest([H.Level(1, 1), H.Level(2, 3, fanout=1024), H.Level(4, 5, H.STATIC_CHUNK, loop=1, chunk=4)],
                  device=-1, desc=d)
    assert nest.info().C == 512


def test_schedule_none_overflow_diagnosed(H):
    """P:251 / S:342: schedule(none) with more iterations than tasks is an
    error before any launch (validated on a describe-only nest)."""
    import torch
    d = H.b200_desc()
    nest = H.Nest([H.Level(1, 4, H.STATIC), H.Level(5, 5, H.NONE)], device=-1, desc=d, clusters=2,
                  warps_per_cta=2)
    x = torch.zeros(10, dtype=torch.int32)
    out = torch.zeros(1, dtype=torch.int64)
    # 2 clusters x 2 CTAs x 2 warps = 8 warps; each warp's list has ceil(n/8) iterations
    desc = H.make_desc(x, out, n0=8 * 32)
    with pytest.raises(H.HparError) as e:   # fits: 32 per warp -> validated, then "cannot execute"
        nest.parallel_for_reduce(desc)
    assert e.value.code == H.HPAR_E_INVALID and "cannot execute" in str(e.value)
    desc = H.make_desc(x, out, n0=8 * 32 + 1)
    with pytest.raises(H.HparError) as e:
        nest.parallel_for_reduce(desc)
    assert e.value.code == H.HPAR_E_SCHEDULE


def test_barrier_capability(H):
    d = H.b200_desc()
    nest = H.Nest([H.Level(1, 5)], device=-1, desc=d)
    with pytest.raises(H.HparError) as e:
        nest.barrier(H.HPAR_CLUSTER)
    assert e.value.code == H.HPAR_E_CAPABILITY


def test_shard_ranges(H):
    """§8(a) A2: static block of the outer loop over the GPUs, also when the
    GPU level is collapsed with the levels below it."""
    d = H.b200_desc()
    for levels in ([H.Level(1, 1), H.Level(2, 5)], [H.Level(1, 5)]):
        for G in (1, 2, 3, 8):
            nest = H.Nest(levels, device=-1, desc=d, nranks=G, rank=0, clusters=3, warps_per_cta=2)
            for n0 in (0, 1, 7, 1000, 12345):
                prev = 0
                for g in range(G):
                    b, c = nest.shard_range(n0, g)
                    assert b == prev and c >= 0
                    prev = b + c
                assert prev == n0


def test_shard_range_csr_is_nnz_balanced(H):
    """§8(e) C3: contiguous, covering row shards whose nonzero counts differ
    from nnz/G by less than one row (brute force over the definition)."""
    import numpy as np
    from inputs import gen
    rng = np.random.default_rng(3)
    cases = [gen.csr_offsets(5000, 70000), np.zeros(11, np.int64), np.array([0, 10**6], np.int64)]
    lens = rng.integers(0, 50, 777)
    cases.append(np.concatenate([[0], np.cumsum(lens)]).astype(np.int64))
    for off in cases:
        rows, nnz = off.size - 1, int(off[-1])
        for G in (1, 2, 3, 4, 8):
            shards = [H.hpar_shard_range_csr(off, G, g) for g in range(G)]
            assert shards[0][0] == 0 and sum(c for _, c in shards) == rows
            for (b0, c0), (b1, _) in zip(shards, shards[1:]):
                assert b0 + c0 == b1
            for g, (b, c) in enumerate(shards):
                # the definition: b_g = first row whose start offset >= ceil(g nnz / G)
                target = -(-g * nnz // G)
                hit = np.nonzero(off[:rows] >= target)[0]
                want = 0 if g == 0 else (int(hit[0]) if hit.size else rows)
                assert b == want
                if rows and nnz:
                    maxlen = int(np.diff(off).max())
                    assert abs(int(off[b + c] - off[b]) - nnz / G) <= maxlen + 1


def test_caller_sharded_csr_local_n0(H):
    """local_n0 (§8(e) C3): rows of a caller-sharded CSR shard; an empty
    shard (HPAR_LOCAL_N0_EMPTY, what make_desc passes for 0) validates and
    returns without a launch — never the GPU level's static block of n0 rows
    with a 1-entry offsets array; other negatives are rejected;
    a non-CSR call with local_n0 is rejected."""
    import torch
    from paper_2309_01906_b200 import nests
    d = H.b200_desc()
    nest = H.Nest(nests.c3_fast_nest(), device=-1, desc=d, nranks=4, rank=3, cluster_dim=2, warps_per_cta=8,
                  clusters=4)
    x = torch.zeros(4, dtype=torch.float32)
    out = torch.zeros(1, dtype=torch.float32)
    off = torch.zeros(1, dtype=torch.int64)
    desc = H.make_desc(x, out, n0=1000, n1=0, nloops=2, keyed=True, offsets=off, local_n0=0)
    assert desc.local_n0 == H.LOCAL_N0_EMPTY
    nest.parallel_for_reduce(desc)  # OK: nothing to do on this rank
    assert nest.last_kernel().startswith("none")
    desc.local_n0 = -5
    with pytest.raises(H.HparError) as e:
        nest.parallel_for_reduce(desc)
    assert e.value.code == H.HPAR_E_INVALID
    flat = H.make_desc(x, torch.zeros(1, dtype=torch.float64), n0=4, local_n0=2)
    with pytest.raises(H.HparError) as e:
        H.Nest(nests.c5_nest(), device=-1, desc=d).parallel_for_reduce(flat)
    assert e.value.code == H.HPAR_E_INVALID


def test_barrier_levels_host(H):
    """A10 at host level (reading #26): node / CTA / warp / lane barriers are
    the kernel boundary, the cluster level has none, the probe is for
    in-kernel levels only; a describe-only nest cannot execute the GPU-level
    rendezvous or the probe."""
    d = H.b200_desc()
    nest = H.Nest([H.Level(1, 5)], device=-1, desc=d)
    for lvl in (H.HPAR_CLUSTER,):
        with pytest.raises(H.HparError) as e:
            nest.barrier(lvl)
        assert e.value.code == H.HPAR_E_CAPABILITY
    with pytest.raises(H.HparError) as e:
        nest.barrier_probe(H.HPAR_CLUSTER, 0)
    assert e.value.code == H.HPAR_E_CAPABILITY
    with pytest.raises(H.HparError) as e:
        nest.barrier_probe(H.HPAR_GPU, 0)
    assert e.value.code == H.HPAR_E_INVALID
    with pytest.raises(H.HparError) as e:
        nest.barrier(H.HPAR_LANE)
    assert e.value.code == H.HPAR_E_INVALID and "describe-only" in str(e.value)


def test_nest_validation_fuzz(H):
    """Random level lists (slices of the hierarchy, schedules, chunks,
    partitions, fanouts, loops, geometries) through hpar_nest_create on
    describe-only nests: every call either succeeds with a consistent info
    (per-level tasks = the product of the collapsed hardware counts, a lane
    partition dividing 32) or fails with one of the model's error codes —
    never another exception or a crash."""
    import random
    d = H.b200_desc()
    rng = random.Random(4242)
    codes = {H.HPAR_E_INVALID, H.HPAR_E_CAPABILITY, H.HPAR_E_SCHEDULE, H.HPAR_E_PARTITION, H.HPAR_E_UNSUPPORTED}
    ok = 0
    for _ in range(600):
        cuts = sorted(rng.sample(range(2, 6), rng.randint(0, 4)))
        first = rng.choice([1, 1, 1, 2, 3])
        bounds = [first] + [c for c in cuts if c > first] + [6]
        levels = []
        for i in range(len(bounds) - 1):
            sch = rng.choice([H.STATIC, H.STATIC_CHUNK, H.DYNAMIC, H.NONE])
            chunk = rng.choice([0, 1, 3, 64]) if sch in (H.STATIC_CHUNK, H.DYNAMIC) else 0
            lv = H.Level(bounds[i], bounds[i + 1] - 1, sch, loop=rng.choice([0, 0, 1]), chunk=chunk)
            if rng.random() < 0.1:
                lv.width = rng.choice([2, 3, 4, 8])
            if rng.random() < 0.1:
                lv.fanout = rng.choice([1, 7, 64, 1024])
            levels.append(lv)
        K, W = rng.choice([1, 2, 4, 8, 16]), rng.choice([1, 4, 8, 32, 33])
        try:
            nest = H.Nest(levels, device=-1, desc=d, cluster_dim=K, warps_per_cta=W, clusters=rng.choice([0, 1, 148]),
                          nranks=rng.choice([1, 2, 8]), rank=0)
        except H.HparError as e:
            assert e.code in codes, (levels, e)
            continue
        info = nest.info()
        assert info.nlevels == len(levels)
        assert info.lane_width == 0 or 32 % max(info.lane_width, 1) == 0
        ok += 1
    assert ok > 20  # (most random lists violate some rule; those must fail cleanly)
