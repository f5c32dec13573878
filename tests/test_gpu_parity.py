"""GPU parity: libhpar.so (through the C ABI) against the oracle, element by
element, on seeded inputs.  Bit-exact for integers, coverage maps and bins;
1e-5 relative for fp32 (north_star).  Runs on the B200 box (-m gpu)."""
import os
import random

import numpy as np
import pytest

from inputs import gen
from tests.nestutil import assert_rel, fanouts, oracle_levels

# HPAR_FUZZ_N=<n>: run every randomized fuzz test with n seeds (a long sweep)
FUZZ_N = int(os.environ.get("HPAR_FUZZ_N", "0"))

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2309_01906_b200 import build
    build.build()
    from paper_2309_01906_b200 import hpar
    return hpar


@pytest.fixture(scope="module")
def torch_mod():
    import torch
    return torch


@pytest.fixture(scope="module")
def inputs_lib():
    import ctypes
    import os
    from paper_2309_01906_b200 import build
    build.build()
    L = ctypes.CDLL(os.path.join(os.path.dirname(gen.__file__), "libhpar_inputs.so"))
    for name in ("hpar_inputs_fill_i32", "hpar_inputs_fill_f32", "hpar_inputs_fill_u8"):
        f = getattr(L, name)
        f.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        f.restype = ctypes.c_int
    return L


def dev_fill(L, torch, kind, seed, begin, n):
    dt = {"i32": torch.int32, "f32": torch.float32, "u8": torch.uint8}[kind]
    t = torch.empty(n, dtype=dt, device="cuda")
    rc = getattr(L, f"hpar_inputs_fill_{kind}")(seed, begin, n, t.data_ptr(), None)
    assert rc == 0
    return t


def test_device_generator_matches_numpy(inputs_lib, torch_mod):
    torch = torch_mod
    for kind, f in (("i32", gen.gen_i32), ("f32", gen.gen_f32), ("u8", gen.gen_u8)):
        for seed, begin in ((1, 0), (5, (1 << 34) - 5000)):
            t = dev_fill(inputs_lib, torch, kind, seed, begin, 5000)
            assert np.array_equal(t.cpu().numpy(), f(seed, begin, 5000))


# ---------------------------------------------------------------------------
def run_nest(H, torch, levels, x, *, n0, n1=0, offsets=None, keyed=False, op=0, C=4, K=2, W=4,
             partials=True, coverage=True, max_inner=0, out_f64=True, misalign=0, ld=0, nest=None,
             fingerprint=False):
    if nest is None:  # (a caller may pass one Nest to reuse across calls)
        nest = H.Nest(levels, device=0, cluster_dim=K, warps_per_cta=W, clusters=C)
    nloops = 2 if (n1 or offsets is not None) else 1
    if offsets is not None:
        n_iter = int(offsets[-1])
    else:
        n_iter = n0 * (n1 if nloops == 2 else 1)
    xd = torch.from_numpy(x).cuda()
    if ld and ld != n1:  # rows at stride ld; the padding columns hold poison (NaN / a huge int) that a read would show
        assert nloops == 2 and ld > n1
        xp = np.full((n0, ld), np.nan if x.dtype.kind == "f" else np.iinfo(x.dtype).max // 3, dtype=x.dtype)
        xp[:, :n1] = x.reshape(n0, n1)
        x_dev_src = xp.reshape(-1)
    else:
        x_dev_src = x
    xd = torch.from_numpy(x_dev_src).cuda()
    if misalign:  # the input starts `misalign` bytes past a 16-byte boundary
        assert misalign % x.itemsize == 0
        e0 = misalign // x.itemsize
        raw = torch.zeros(x_dev_src.size + 32, dtype=xd.dtype, device="cuda")
        xd = raw[e0:e0 + x_dev_src.size]
        xd.copy_(torch.from_numpy(x_dev_src).cuda())
        assert xd.data_ptr() % 16 == misalign
    fp = x.dtype.kind == "f"
    if op == H.OP_AFFINE:
        out = torch.zeros((n0, 2) if keyed else (2,), dtype=torch.int64, device="cuda")
    elif keyed:
        out = torch.zeros(n0, dtype=torch.float64 if fp else torch.int64, device="cuda")
    elif op == H.OP_HIST256:
        out = torch.zeros(256, dtype=torch.int64, device="cuda")
    else:
        out = torch.zeros(1, dtype=torch.float64 if fp else torch.int64, device="cuda")
    owner = torch.full((max(n_iter, 1),), -1, dtype=torch.int64, device="cuda") if coverage else None
    count = torch.zeros(max(n_iter, 1), dtype=torch.int32, device="cuda") if coverage else None
    Ts = fanouts(levels, 1, C, K, W)
    parts = []
    if partials:
        first_inner = 0
        if keyed:
            while first_inner < len(levels) and levels[first_inner].loop == 0:
                first_inner += 1
        tot = 1
        for a, T in enumerate(Ts):
            if keyed:
                if a < first_inner:
                    parts.append(None)
                    continue
                per = int(np.prod(Ts[first_inner:a + 1]))
                size = n0 * per
            else:
                tot *= T
                size = tot
            shape = (size, 256) if op == H.OP_HIST256 else ((size, 2) if op == H.OP_AFFINE else (size,))
            parts.append(torch.full(shape, -7, dtype=torch.float64 if (fp and op != H.OP_HIST256) else torch.int64,
                                    device="cuda"))
    offs = torch.from_numpy(offsets).cuda() if offsets is not None else None
    verify = (H.VERIFY_COVERAGE if coverage else 0) | (H.VERIFY_PARTIALS if partials else 0)
    fpt = torch.zeros(3, dtype=torch.int64, device="cuda") if fingerprint else None
    if fingerprint:
        verify |= H.VERIFY_FINGERPRINT
    d = H.make_desc(xd, out, op=op, n0=n0, n1=n1, ld=ld or n1, nloops=nloops, keyed=keyed, offsets=offs,
                    max_inner=max_inner, verify=verify, partials=parts, owner=owner, count=count, fingerprint=fpt,
                    out_dtype=(H.U64 if op == H.OP_AFFINE else (H.F64 if fp else H.I64)) if keyed else -1)
    nest.parallel_for_reduce(d)
    torch.cuda.synchronize()
    res = out.cpu().numpy()
    return dict(nest=nest, out=res, owner=owner.cpu().numpy()[:n_iter] if coverage else None,
                count=count.cpu().numpy()[:n_iter] if coverage else None,
                parts=[p.cpu().numpy() if p is not None else None for p in parts], kernel=nest.last_kernel(),
                fp=fpt.cpu().numpy().view(np.uint64) if fingerprint else None)


def compare(oracle, H, levels, res, x, *, n0, n1=0, offsets=None, keyed=False, op=0, C, K, W,
            dynamic=False, partials=True, unmaterialised=()):
    """unmaterialised: the nest levels whose partials the kernel documents it
    does not produce (they must stay at the -7 fill); every other requested
    level must equal the oracle's."""
    ol = oracle_levels(oracle, levels, 1, C, K, W)
    o = oracle.nest_run(ol, n0=n0, n1=n1, offsets=offsets, x=x, op=op, keyed=keyed,
                        nloops=2 if (n1 or offsets is not None) else 1)
    fp = x.dtype.kind == "f"
    # result
    if op in (H.OP_HIST256, H.OP_AFFINE):
        assert np.array_equal(res["out"].view(np.uint64), o.result)
    elif fp:
        assert_rel(res["out"] if keyed else res["out"][0], o.result)
    else:
        assert np.array_equal(res["out"] if keyed else res["out"][0], o.result)
    # coverage
    if res["count"] is not None:
        assert (res["count"] == 1).all(), "every iteration executes exactly once"
        if not dynamic:
            assert np.array_equal(res["owner"], o.owner), "owner map differs from the oracle"
    # partials (static nests; dynamic assignment differs from the round-robin model)
    if partials and not dynamic:
        for a, p in enumerate(res["parts"]):
            if p is None or o.partials[a] is None:
                continue
            if a in unmaterialised:
                assert np.all(p == -7), f"level {a}: documented as not materialised, but written"
                continue
            if op in (H.OP_HIST256, H.OP_AFFINE):
                assert np.array_equal(p.view(np.uint64), o.partials[a]), f"level {a} partials"
            elif fp:
                assert_rel(p, o.partials[a])
            else:
                assert np.array_equal(p, o.partials[a]), f"level {a} partials"
    return o


# ---------------------------------------------------------------------------
def test_c1_generic_bit_exact(H, torch_mod, oracle):
    """Config 1 at full size (2^20 int32, outer 1024 x inner 1024): int64 sum,
    coverage owner map and per-level partials bit-exact."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    x = gen.gen_i32(gen.SEED_C1, 0, 1 << 20)
    # bench.py's launch: 148 clusters x 2 CTAs = 296 teams of 3-4 rows; and
    # the one-row-per-team form (1024 teams)
    for levels, C in ((nests.c1_nest(with_gpu=True, outer=0), 148), (nests.c1_nest(with_gpu=True), 512)):
        K, W = 2, 8
        res = run_nest(H, torch, levels, x, n0=1024, n1=1024, C=C, K=K, W=W)
        assert res["out"][0] == oracle.sum_i32(x)
        assert res["kernel"] == "teams_threads"
        compare(oracle, H, levels, res, x, n0=1024, n1=1024, C=C, K=K, W=W)


SCHEDS = [(0, 0), (1, 1), (1, 3), (1, 8), (3, 0)]


def random_flat_nest(H, rng, n):
    """random nest over gpu..lane with collapses and an optional lane partition"""
    hw = [H.HPAR_GPU, H.HPAR_CLUSTER, H.HPAR_CTA, H.HPAR_WARP, H.HPAR_LANE]
    cuts = sorted(rng.sample(range(1, 5), rng.randint(1, 4)))
    bounds = [0] + cuts + [5]
    levels = []
    for i in range(len(bounds) - 1):
        s, c = rng.choice(SCHEDS)
        levels.append(H.Level(hw[bounds[i]], hw[bounds[i + 1] - 1], s, loop=0, chunk=c))
    if rng.random() < 0.4:
        w = rng.choice([2, 4, 8, 16])
        levels[-1].width = w
        levels.append(H.Level(H.HPAR_LANE, H.HPAR_LANE, rng.choice([0, 1]), loop=0, chunk=rng.choice([1, 2])))
    return levels


def test_generic_random_flat_nests(H, torch_mod, oracle):
    """≥40 random flat nests (collapses, partitions, every static schedule,
    ragged sizes): results, owner maps and partials vs the oracle."""
    torch = torch_mod
    rng = random.Random(2309)
    done = 0
    while done < (FUZZ_N or 40):
        levels = random_flat_nest(H, rng, 0)
        C, K, W = rng.choice([1, 3, 5]), rng.choice([1, 2, 4]), rng.choice([1, 2, 4])
        n = rng.randint(0, 7000)
        Ts = fanouts(levels, 1, C, K, W)
        # skip nests whose schedule(none) would overflow (tested separately)
        try:
            oracle.nest_run(oracle_levels(oracle, levels, 1, C, K, W), n0=n)
        except oracle.OracleError:
            with pytest.raises(H.HparError) as e:
                run_nest(H, torch, levels, gen.gen_i32(7, 0, max(n, 1))[:n], n0=n, C=C, K=K, W=W)
            assert e.value.code == H.HPAR_E_SCHEDULE
            continue
        x = gen.gen_i32(done + 100, 0, n) if done % 2 == 0 else gen.gen_f32(done + 100, 0, n)
        res = run_nest(H, torch, levels, x, n0=n, C=C, K=K, W=W)
        compare(oracle, H, levels, res, x, n0=n, C=C, K=K, W=W)
        done += 1
        assert Ts


def test_generic_random_two_loop_nests(H, torch_mod, oracle):
    """Random two-loop dense nests on the generic interpreter (the runs of
    consecutive positions it maps once, chain_map_run): a random cut of the
    hierarchy between the rows' levels (loop 0) and the columns' levels
    (loop 1), random collapses and static / static(c) schedules, keyed or
    total, ragged shapes; results, owner maps and partials vs the oracle."""
    torch = torch_mod
    rng = random.Random(2310)
    hw = [H.HPAR_GPU, H.HPAR_CLUSTER, H.HPAR_CTA, H.HPAR_WARP, H.HPAR_LANE]
    done = tries = 0
    while done < (FUZZ_N or 30) and tries < 20 * (FUZZ_N or 30):
        tries += 1
        cuts = sorted(rng.sample(range(1, 5), rng.randint(1, 4)))
        bounds = [0] + cuts + [5]
        nl = len(bounds) - 1
        split = rng.randint(1, nl - 1) if nl > 1 else 1  # levels [0, split) on loop 0, the rest on loop 1
        levels = []
        for i in range(nl):
            sch, c = rng.choice([(0, 0), (1, 1), (1, 3), (1, 8)])
            levels.append(H.Level(hw[bounds[i]], hw[bounds[i + 1] - 1], sch, loop=0 if i < split else 1, chunk=c))
        keyed = rng.random() < 0.5
        C, K, W = rng.choice([1, 3, 5]), rng.choice([1, 2, 4]), rng.choice([1, 2, 4])
        n0, n1 = rng.randint(1, 60), rng.randint(1, 400)
        x = gen.gen_i32(done + 900, 0, n0 * n1) if done % 2 == 0 else gen.gen_f32(done + 900, 0, n0 * n1)
        try:
            res = run_nest(H, torch, levels, x, n0=n0, n1=n1, keyed=keyed, C=C, K=K, W=W)
        except H.HparError as e:  # nests the model rejects (e.g. a keyed combine needing a missing barrier)
            assert e.code in (H.HPAR_E_CAPABILITY, H.HPAR_E_INVALID, H.HPAR_E_UNSUPPORTED), e
            continue
        compare(oracle, H, levels, res, x, n0=n0, n1=n1, keyed=keyed, C=C, K=K, W=W)
        done += 1
    assert done >= (FUZZ_N or 30) // 2


@pytest.mark.parametrize("seed", range(FUZZ_N or 12))
def test_generic_csr_fuzz(H, torch_mod, oracle, seed):
    """Random CSR nests of the generic form (config-3 shape: rows
    dynamic(c) over teams, lanes(w) partitions over the rows, nonzeros
    static(1) over a row's lane group) on the generic interpreter: random
    rows_chunk, width, geometry, op and dtype; every row vs the oracle, every
    nonzero visited once (dynamic schedules: counts, not owner maps)."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    rng = np.random.default_rng(8000 + seed)
    rows = int(rng.integers(1, 1500))
    lens = np.where(rng.random(rows) < 0.2, 0, rng.geometric(0.1, rows))
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    nnz = int(off[-1])
    combos = [("f32", H.OP_SUM), ("f32", H.OP_MAX), ("i32", H.OP_SUM), ("i64", H.OP_MIN), ("f64", H.OP_SUM)]
    dt, op = combos[int(rng.integers(len(combos)))]
    if dt == "f32":
        v = gen.gen_f32(gen.SEED_C3 + seed, 0, nnz)
    elif dt == "i32":
        v = gen.gen_i32(gen.SEED_C1 + seed, 0, nnz)
    elif dt == "i64":
        v = rng.integers(-(1 << 62), 1 << 62, nnz, dtype=np.int64)
    else:
        v = rng.standard_normal(nnz)
    levels = nests.c3_nest(with_gpu=True, rows_chunk=int(rng.choice([1, 3, 16, 64])),
                           width=int(rng.choice([1, 2, 4, 8, 16, 32])))
    C, K, W = int(rng.integers(1, 8)), int(rng.choice([1, 2, 4])), int(rng.choice([1, 2, 4, 8]))
    res = run_nest(H, torch, levels, v, n0=rows, offsets=off, keyed=True, op=op, C=C, K=K, W=W, partials=False)
    assert res["kernel"] == "generic"
    compare(oracle, H, levels, res, v, n0=rows, offsets=off, keyed=True, op=op, C=C, K=K, W=W, dynamic=True,
            partials=False)


@pytest.mark.parametrize("family", ["flat", "hist", "rowwise", "teams", "segrows"])
def test_nest_reuse_fuzz(H, torch_mod, oracle, family):
    """One Nest per kernel family called (FUZZ_N or 30) times with random
    sizes, ops, dtypes and pointer offsets in a row: the self-resetting
    tickets, partial buffers and workspaces must leave every call exact
    against the oracle (a stale ticket or partial shows as a wrong result)."""
    from paper_2309_01906_b200 import nests
    from tests.nestutil import oracle_levels
    torch = torch_mod
    rng = np.random.default_rng({"flat": 1, "hist": 2, "rowwise": 3, "teams": 4, "segrows": 5}[family] + 9000)
    C, K, W = 5, 2, 4
    levels = {"flat": nests.c5_nest(K), "hist": nests.c4_nest(K), "rowwise": nests.c2_nest(),
              "teams": nests.c1_nest(outer=0), "segrows": nests.c3_fast_nest()}[family]
    if family == "segrows":
        W = 8
    nest = H.Nest(levels, device=0, cluster_dim=K, warps_per_cta=W, clusters=C)  # one Nest for every call
    for _ in range(FUZZ_N or 30):
        if family == "flat":
            n = int(rng.integers(0, 200000))
            dt, op = [("f32", H.OP_SUM), ("i32", H.OP_MAX), ("f64", H.OP_SUM), ("i64", H.OP_AFFINE)][int(rng.integers(4))]
            x = (gen.gen_f32(int(rng.integers(100)), 0, n) if dt == "f32" else gen.gen_i32(int(rng.integers(100)), 0, n)
                 if dt == "i32" else rng.standard_normal(n) if dt == "f64" else rng.integers(-(1 << 62), 1 << 62, n))
            mis = int(rng.integers(0, 16 // x.itemsize)) * x.itemsize if n else 0
            res = run_nest(H, torch, levels, x, n0=n, op=op, C=C, K=K, W=W, misalign=mis, coverage=False, partials=False, nest=nest)
            compare(oracle, H, levels, res, x, n0=n, op=op, C=C, K=K, W=W, partials=False)
        elif family == "hist":
            n = int(rng.integers(0, 300000))
            x = gen.gen_u8_zipf(int(rng.integers(100)), 0, n)
            mis = int(rng.integers(0, 16)) if n else 0
            res = run_nest(H, torch, levels, x, n0=n, op=H.OP_HIST256, C=C, K=K, W=W, misalign=mis, coverage=False,
                           partials=False, nest=nest)
            assert np.array_equal(res["out"].astype(np.uint64), oracle.hist256(x))
        elif family in ("rowwise", "teams"):
            n0, n1 = int(rng.integers(1, 80)), int(rng.integers(1, 3000))
            dt, op = [("f32", H.OP_SUM), ("i32", H.OP_MIN), ("f64", H.OP_MAX), ("i64", H.OP_AFFINE)][int(rng.integers(4))]
            x = (gen.gen_f32(int(rng.integers(100)), 0, n0 * n1) if dt == "f32" else
                 gen.gen_i32(int(rng.integers(100)), 0, n0 * n1) if dt == "i32" else
                 rng.standard_normal(n0 * n1) if dt == "f64" else rng.integers(-(1 << 62), 1 << 62, n0 * n1))
            keyed = family == "rowwise"
            res = run_nest(H, torch, levels, x, n0=n0, n1=n1, keyed=keyed, op=op, C=C, K=K, W=W, coverage=False,
                           partials=False, nest=nest)
            compare(oracle, H, levels, res, x, n0=n0, n1=n1, keyed=keyed, op=op, C=C, K=K, W=W, partials=False)
        else:
            rows = int(rng.integers(1, 2000))
            lens = np.where(rng.random(rows) < 0.01, rng.integers(4097, 20000, rows), rng.geometric(0.1, rows))
            off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
            v = rng.standard_normal(int(off[-1])) + 3.0  # no near-cancelling rows (the tolerance is relative)
            res = run_nest(H, torch, levels, v, n0=rows, offsets=off, keyed=True, C=C, K=2, W=W, coverage=False,
                           partials=False, nest=nest)
            ol = oracle_levels(oracle, nests.c3_nest(with_gpu=False, rows_chunk=16, width=8), 1, 2, 2, 4)
            assert_rel(res["out"], oracle.nest_run(ol, n0=rows, offsets=off, x=v, keyed=True, coverage=False,
                                                   partials=False).result)
        assert res["kernel"] != "generic", res["kernel"]


def test_csr_n1_zero_reads_nnz(H, torch_mod, oracle):
    """hpar.h lets a CSR call pass n1 = 0 (the value count is then read from
    offsets[n0_local] on the device): both fused CSR kernels, with long rows
    (> 4096, the chunk / segment lists sized from that count), vs the oracle;
    and inside graph capture such a call is refused (HPAR_E_INVALID)."""
    from paper_2309_01906_b200 import nests
    from tests.nestutil import oracle_levels
    torch = torch_mod
    rng = np.random.default_rng(77)
    rows = 3000
    lens = np.where(rng.random(rows) < 0.01, rng.integers(4097, 30000, rows), rng.geometric(0.1, rows))
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    offd = torch.from_numpy(off).cuda()
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8, clusters=5)
    v32 = gen.gen_f32(gen.SEED_C3, 0, int(off[-1]))
    out = torch.full((rows,), -1.0, dtype=torch.float64, device="cuda")
    nest.parallel_for_reduce(H.make_desc(torch.from_numpy(v32).cuda(), out, n0=rows, n1=0, nloops=2, keyed=True,
                                         offsets=offd, out_dtype=H.F64))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "segmented_csr"
    assert_rel(out.cpu().numpy(), oracle.segsum_f32(v32, off))
    v = rng.standard_normal(int(off[-1])) + 3.0
    out.fill_(-1.0)
    nest.parallel_for_reduce(H.make_desc(torch.from_numpy(v).cuda(), out, n0=rows, n1=0, nloops=2, keyed=True,
                                         offsets=offd, out_dtype=H.F64))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "segrows_csr"
    ol = oracle_levels(oracle, nests.c3_nest(with_gpu=False, rows_chunk=16, width=8), 1, 2, 2, 4)
    assert_rel(out.cpu().numpy(), oracle.nest_run(ol, n0=rows, offsets=off, x=v, keyed=True, coverage=False,
                                                  partials=False).result)
    xd = torch.from_numpy(v32).cuda()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with pytest.raises(H.HparError) as e:
        with torch.cuda.graph(g, stream=s):
            nest.parallel_for_reduce(H.make_desc(xd, out, n0=rows, n1=0, nloops=2, keyed=True, offsets=offd,
                                                 out_dtype=H.F64), s.cuda_stream)
    assert e.value.code == H.HPAR_E_INVALID


def test_desc_validation_fuzz(H, torch_mod):
    """Random malformed calls through hpar_parallel_for_reduce on real nests:
    bad ops / dtypes / out dtypes, negative extents, NULL pointers, loop and
    keyed mismatches, verify without its buffers.  Each must fail with one of
    the model's error codes before any launch — never a crash — and the nest
    must stay usable (a valid call afterwards is exact)."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    rng = np.random.default_rng(99)
    nest = H.Nest(nests.c5_nest(2), device=0, cluster_dim=2, warps_per_cta=4, clusters=3)
    x = torch.ones(1000, dtype=torch.float32, device="cuda")
    out = torch.zeros(4, dtype=torch.float64, device="cuda")
    codes = {H.HPAR_E_INVALID, H.HPAR_E_UNSUPPORTED, H.HPAR_E_CAPABILITY}
    for _ in range(200):
        d = H.make_desc(x, out, n0=1000)
        k = int(rng.integers(9))
        if k == 0:
            d.op = int(rng.choice([-1, 5, 99]))
        elif k == 1:
            d.in_dtype = int(rng.choice([-1, 9]))
        elif k == 2:
            d.op = H.OP_HIST256  # u8 only
        elif k == 3:
            d.n0 = -int(rng.integers(1, 100))
        elif k == 4:
            d.out = None
        elif k == 5:
            d.nloops = int(rng.choice([0, 3]))
        elif k == 6:
            d.in_ = None
        elif k == 7:
            d.verify = H.VERIFY_COVERAGE  # no owner / count buffers
        else:
            d.op = H.OP_AFFINE  # int64 only
        with pytest.raises(H.HparError) as e:
            nest.parallel_for_reduce(d)
        assert e.value.code in codes, (k, e.value)
    torch.cuda.synchronize()
    out.zero_()
    nest.parallel_for_reduce(H.make_desc(x, out, n0=1000))
    torch.cuda.synchronize()
    assert out[0].item() == 1000.0


def test_generic_min_max(H, torch_mod, oracle):
    torch = torch_mod
    levels = [H.Level(H.HPAR_CLUSTER, H.HPAR_CTA, 1, chunk=5), H.Level(H.HPAR_WARP, H.HPAR_LANE, 0)]
    for x in (gen.gen_f32(3, 0, 9999), gen.gen_i32(3, 0, 9999)):
        for op in (H.OP_MIN, H.OP_MAX):
            res = run_nest(H, torch, levels, x, n0=x.size, op=op, C=3, K=2, W=2)
            compare(oracle, H, levels, res, x, n0=x.size, op=op, C=3, K=2, W=2)


def test_generic_two_loop_total_and_keyed(H, torch_mod, oracle):
    """Multi-loop nests (P:215-225 bind_ancestor): dense and CSR, total and
    keyed, including a lane partition for the keyed CSR rows."""
    torch = torch_mod
    rng = random.Random(5)
    # dense keyed: rows over cluster(s) or CTAs, cols over the rest
    for rows_to in (H.HPAR_CLUSTER, H.HPAR_CTA, H.HPAR_WARP):
        levels = [H.Level(H.HPAR_GPU, H.HPAR_GPU, 0, loop=0),
                  H.Level(H.HPAR_CLUSTER, rows_to, rng.choice([0, 1]), loop=0, chunk=2)]
        if rows_to < H.HPAR_LANE:
            levels.append(H.Level(rows_to + 1, H.HPAR_LANE, rng.choice([0, 1]), loop=1, chunk=rng.choice([1, 4])))
        n0, n1 = 37, 301
        x = gen.gen_f32(11, 0, n0 * n1)
        res = run_nest(H, torch, levels, x, n0=n0, n1=n1, keyed=True, C=3, K=2, W=4)
        compare(oracle, H, levels, res, x, n0=n0, n1=n1, keyed=True, C=3, K=2, W=4)
        xi = gen.gen_i32(12, 0, n0 * n1)
        res = run_nest(H, torch, levels, xi, n0=n0, n1=n1, keyed=False, C=3, K=2, W=4)
        compare(oracle, H, levels, res, xi, n0=n0, n1=n1, keyed=False, C=3, K=2, W=4)
    # CSR keyed with lanes(8) groups owning rows
    off = gen.csr_offsets(500, 9000)
    v = gen.gen_f32(gen.SEED_C3, 0, 9000)
    levels = [H.Level(H.HPAR_GPU, H.HPAR_GPU, 0, loop=0), H.Level(H.HPAR_CLUSTER, H.HPAR_CTA, 0, loop=0),
              H.Level(H.HPAR_WARP, H.HPAR_LANE, 1, loop=0, chunk=1, width=8),
              H.Level(H.HPAR_LANE, H.HPAR_LANE, 1, loop=1, chunk=1)]
    res = run_nest(H, torch, levels, v, n0=500, offsets=off, keyed=True, C=2, K=2, W=2)
    compare(oracle, H, levels, res, v, n0=500, offsets=off, keyed=True, C=2, K=2, W=2)


def test_generic_dynamic_levels(H, torch_mod, oracle):
    """dynamic(c) at the cluster, CTA and warp levels: every iteration once,
    each task's iterations a union of whole chunks of its parent list, results
    equal (reading #9)."""
    torch = torch_mod
    for dyn_first, dyn_last in ((H.HPAR_CLUSTER, H.HPAR_CLUSTER), (H.HPAR_CLUSTER, H.HPAR_CTA),
                                (H.HPAR_WARP, H.HPAR_WARP)):
        levels = []
        hw = H.HPAR_CLUSTER
        if dyn_first > hw:
            levels.append(H.Level(hw, dyn_first - 1, 0))
        levels.append(H.Level(dyn_first, dyn_last, H.DYNAMIC, chunk=37))
        if dyn_last < H.HPAR_LANE:
            levels.append(H.Level(dyn_last + 1, H.HPAR_LANE, 1, chunk=1))
        x = gen.gen_i32(21, 0, 50000)
        res = run_nest(H, torch, levels, x, n0=x.size, C=5, K=2, W=4)
        compare(oracle, H, levels, res, x, n0=x.size, C=5, K=2, W=4, dynamic=True)
        if (dyn_first, dyn_last) == (H.HPAR_CLUSTER, H.HPAR_CLUSTER):
            # chunk alignment: every chunk of 37 consecutive iterations belongs to one cluster
            cl = res["owner"] // (2 * 4 * 32)
            pad = (-x.size) % 37
            chunks = np.concatenate([cl, np.full(pad, -1)]).reshape(-1, 37)
            for row in chunks:
                vals = row[row >= 0]
                assert (vals == vals[0]).all()
    # keyed CSR with dynamic rows over teams (config-3 generic nest)
    from paper_2309_01906_b200 import nests
    off = gen.csr_offsets(3000, 40000)
    v = gen.gen_f32(gen.SEED_C3, 0, 40000)
    levels = nests.c3_nest(with_gpu=True, rows_chunk=16, width=8)
    res = run_nest(H, torch, levels, v, n0=3000, offsets=off, keyed=True, C=4, K=2, W=4)
    compare(oracle, H, levels, res, v, n0=3000, offsets=off, keyed=True, C=4, K=2, W=4, dynamic=True)


# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n", [0, 1, 5, 4096 * 2 * 7 + 3, 1 << 20, (1 << 22) + 4 * 12345 + 2])
def test_flat_fused_kernel(H, torch_mod, oracle, n):
    """The fused TMA flat kernel (config-5 nest) at reduced sizes with ragged
    tails: sum bit-comparable within 1e-5, owner map and partials vs oracle."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    levels = nests.c5_nest(K=2)
    C, K, W = 7, 2, 8
    x = gen.gen_f32(gen.SEED_C5, 0, n)
    res = run_nest(H, torch, levels, x, n0=n, C=C, K=K, W=W, coverage=n <= (1 << 20))
    assert res["kernel"] == "flat_tma"
    compare(oracle, H, levels, res, x, n0=n, C=C, K=K, W=W, partials=n <= (1 << 20))
    xi = gen.gen_i32(gen.SEED_C1, 0, n)
    res = run_nest(H, torch, levels, xi, n0=n, C=C, K=K, W=W, coverage=False, partials=False)
    assert res["out"][0] == oracle.sum_i32(xi)


@pytest.mark.parametrize("mis", [4, 8, 12])
def test_flat_misaligned_input(H, torch_mod, oracle, mis):
    """An fp32/int32 input 4, 8 or 12 bytes off a 16-byte boundary stays on
    the fused flat kernel (SURVEY §8(b) alignment; P:252's peel done by the
    copy): tiles copy their enclosing granules and each lane takes its four
    elements from two aligned vectors.  Total, owner map (the nominal static
    closed form) and every level's partials vs the oracle; the int32 total
    exact; the fp32 total bitwise equal to the aligned call's (same owner
    map, same arithmetic order)."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    levels = nests.c5_nest(K=2)
    C, K, W = 5, 2, 8
    for n in (1, 3, 7, 4096 * 2 * 5, 4096 * 2 * 7 + 4 * 99 + 3, 300001):
        x = gen.gen_f32(gen.SEED_C5, 0, n)
        res = run_nest(H, torch, levels, x, n0=n, C=C, K=K, W=W, misalign=mis)
        assert res["kernel"] == "flat_tma"
        compare(oracle, H, levels, res, x, n0=n, C=C, K=K, W=W)
        ref = run_nest(H, torch, levels, x, n0=n, C=C, K=K, W=W, coverage=False, partials=False)
        assert res["out"].tobytes() == ref["out"].tobytes()
        xi = gen.gen_i32(gen.SEED_C1, 0, n)
        res = run_nest(H, torch, levels, xi, n0=n, C=C, K=K, W=W, coverage=False, partials=False, misalign=mis)
        assert res["kernel"] == "flat_tma"
        assert res["out"][0] == oracle.sum_i32(xi)


@pytest.mark.parametrize("n0,n1,ld,mis", [(50, 4095, 4095, 0), (37, 4100, 4100, 0), (29, 4092, 4092, 8),
                                          (40, 4096, 4096, 4), (33, 4095, 4096, 0), (21, 1001, 1003, 12),
                                          (9, 3, 5, 4), (6, 1, 1, 0), (300, 777, 777, 0)])
def test_rowwise_ragged_rows(H, torch_mod, oracle, n0, n1, ld, mis):
    """Rows the aligned copy cannot take whole — n1 not a multiple of 4K,
    ld not a multiple of 4 (NaN padding columns), the base pointer off a
    16-byte boundary — stay on the fused row-wise kernel: each CTA copies the
    granules enclosing its static column block of the row and its lanes
    shift by the row's offset.  Rows, owner map and every level's partials
    vs the oracle."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    levels = nests.c2_nest()
    for K, W, C in ((2, 4, 7), (4, 8, 3)):
        x = gen.gen_f32(gen.SEED_C2, 0, n0 * n1)
        res = run_nest(H, torch, levels, x, n0=n0, n1=n1, keyed=True, C=C, K=K, W=W, ld=ld, misalign=mis)
        assert res["kernel"] == "rowwise_tma_dsmem"
        compare(oracle, H, levels, res, x, n0=n0, n1=n1, keyed=True, C=C, K=K, W=W)


@pytest.mark.parametrize("mis", [0, 8])
@pytest.mark.parametrize("dt", ["f64", "i64"])
def test_flat_8byte_elements(H, torch_mod, oracle, dt, mis):
    """fp64 and int64 inputs (SURVEY §8(b) dtypes) on the fused flat kernel:
    a lane's four elements are 32 bytes (two aligned vectors, three when the
    input sits 8 bytes off a granule).  SUM / MIN / MAX results, owner map
    and every level's partials vs the oracle; int64 sums of values near 2^62
    wrap mod 2^64 exactly as the oracle's."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    levels = nests.c5_nest(K=2)
    C, K, W = 5, 2, 8
    rng = np.random.default_rng(64)
    for n in (0, 1, 3, 4096 * 2 * 5, 4096 * 2 * 7 + 4 * 99 + 3, 300001):
        if dt == "f64":
            x = rng.standard_normal(n) * 1e3
        else:
            x = rng.integers(-(1 << 62), 1 << 62, n, dtype=np.int64)
        for op in (H.OP_SUM, H.OP_MIN, H.OP_MAX):
            res = run_nest(H, torch, levels, x, n0=n, op=op, C=C, K=K, W=W, misalign=mis if n else 0)
            assert res["kernel"] == "flat_tma"
            compare(oracle, H, levels, res, x, n0=n, op=op, C=C, K=K, W=W)


@pytest.mark.parametrize("mis", [0, 8])
def test_flat_affine_op(H, torch_mod, oracle, mis):
    """The ordered AFFINE operator (NEXT f2) on the fused flat kernel: the
    lane folds its elements in ascending position order and every level
    folds its children in ascending task order, which is the nest's fold
    (the oracle's nest walk); result, owner map and every level's partials
    bit-exact, aligned and 8 bytes off a granule."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    levels = nests.c5_nest(K=2)
    C, K, W = 5, 2, 8
    rng = np.random.default_rng(65)
    for n in (1, 4096 * 2 * 5 + 1, 4096 * 2 * 7 + 4 * 99 + 3, 200001):
        x = rng.integers(-(1 << 62), 1 << 62, n, dtype=np.int64)
        res = run_nest(H, torch, levels, x, n0=n, op=H.OP_AFFINE, C=C, K=K, W=W, misalign=mis)
        assert res["kernel"] == "flat_tma"
        compare(oracle, H, levels, res, x, n0=n, op=H.OP_AFFINE, C=C, K=K, W=W)


@pytest.mark.parametrize("dt", ["f32", "f64", "i32", "i64"])
def test_rowwise_dtypes_and_ops(H, torch_mod, oracle, dt):
    """SUM / MIN / MAX over fp32, fp64, int32 and int64 rows (SURVEY §8(b)
    ops and dtypes) on the fused row-wise kernel, aligned and ragged: rows
    (fp: within the §8(c) tolerance, MIN/MAX and integers exact), owner map
    and every level's partials vs the oracle.  fp32 sums keep the fp32 lane /
    warp tree; the others carry 64-bit partials through 8-byte DSMEM slots."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    levels = nests.c2_nest()
    rng = np.random.default_rng(77)
    for n0, n1, ld, mis, K, W, C in ((50, 4096, 4096, 0, 2, 4, 7), (21, 1001, 1003, 8, 4, 8, 3),
                                     (13, 1000, 1000, 0, 2, 8, 5), (7, 5, 6, 0, 2, 4, 3)):
        if dt == "f32":  # the workload's nonnegative values: reading #6 bounds the fp32 tree relative to sum |x|
            x = gen.gen_f32(gen.SEED_C2, 0, n0 * n1)
        elif dt == "f64":
            x = rng.standard_normal(n0 * n1)
        elif dt == "i32":
            x = rng.integers(-(1 << 31), (1 << 31) - 1, n0 * n1, dtype=np.int64).astype(np.int32)
        else:
            x = rng.integers(-(1 << 62), 1 << 62, n0 * n1, dtype=np.int64)
        if mis % x.itemsize:
            mis = 0
        for op in (H.OP_SUM, H.OP_MIN, H.OP_MAX):
            res = run_nest(H, torch, levels, x, n0=n0, n1=n1, keyed=True, op=op, C=C, K=K, W=W, ld=ld,
                           misalign=mis)
            assert res["kernel"] == "rowwise_tma_dsmem", (dt, op, n1)
            compare(oracle, H, levels, res, x, n0=n0, n1=n1, keyed=True, op=op, C=C, K=K, W=W)


def test_rowwise_affine_op(H, torch_mod, oracle):
    """The ordered AFFINE op per row (keyed, int64) on the fused row-wise
    kernel: lane 0 of every butterfly combines (own, higher lanes), the
    combiner folds warp partials and CTA partials in ascending order, 16-byte
    partials travel as two 8-byte st.async transactions.  Rows, owner map and
    every level's partials bit-exact vs the oracle's nest fold, aligned and
    ragged."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    levels = nests.c2_nest()
    rng = np.random.default_rng(99)
    for n0, n1, ld, mis, K, W, C in ((40, 4096, 4096, 0, 2, 4, 7), (21, 1001, 1003, 8, 4, 8, 3), (7, 5, 6, 0, 2, 4, 3)):
        x = rng.integers(-(1 << 62), 1 << 62, n0 * n1, dtype=np.int64)
        res = run_nest(H, torch, levels, x, n0=n0, n1=n1, keyed=True, op=H.OP_AFFINE, C=C, K=K, W=W, ld=ld,
                       misalign=mis)
        assert res["kernel"] == "rowwise_tma_dsmem"
        compare(oracle, H, levels, res, x, n0=n0, n1=n1, keyed=True, op=H.OP_AFFINE, C=C, K=K, W=W)


@pytest.mark.parametrize("V", [1, 2])
def test_flat_lane_chunks(H, torch_mod, oracle, V):
    """The flat nest with lane static(1) / static(2) (warp static(32 V)) on
    the fused flat kernel: fp32 sums (pairwise inside a lane chunk), int32,
    fp64 MIN and the int64 AFFINE op; results, owner maps and partials vs
    the oracle, aligned and off a granule."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    C, K, W = 5, 2, 8
    rng = np.random.default_rng(70 + V)
    levels = nests.flat_nest(K=K, tile=4096, vec=V)
    for n in (0, 5, 4096 * 2 * 5 + 77, 200003):
        for dt, op in (("f32", H.OP_SUM), ("i32", H.OP_SUM), ("f64", H.OP_MIN), ("i64", H.OP_AFFINE)):
            if dt == "f32":
                x = gen.gen_f32(gen.SEED_C5, 0, n)
            elif dt == "i32":
                x = gen.gen_i32(gen.SEED_C1, 0, n)
            elif dt == "f64":
                x = rng.standard_normal(n)
            else:
                x = rng.integers(-(1 << 62), 1 << 62, n, dtype=np.int64)
            for mis in ((0, x.itemsize) if n else (0,)):
                res = run_nest(H, torch, levels, x, n0=n, op=op, C=C, K=K, W=W, misalign=mis)
                assert res["kernel"] == "flat_tma"
                compare(oracle, H, levels, res, x, n0=n, op=op, C=C, K=K, W=W)


def test_rowwise_fused_kernel_small(H, torch_mod, oracle):
    """The fused row-wise kernel (config-2 nest) on 50 x 4096 and ragged
    columns: rows, owner map, per-row lane/warp/CTA partials vs oracle."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    levels = nests.c2_nest()
    for n0, n1, C in ((50, 4096, 7), (13, 1000, 3), (5, 8, 9)):
        x = gen.gen_f32(gen.SEED_C2, 0, n0 * n1)
        res = run_nest(H, torch, levels, x, n0=n0, n1=n1, keyed=True, C=C, K=2, W=8)
        assert res["kernel"] == "rowwise_tma_dsmem"
        compare(oracle, H, levels, res, x, n0=n0, n1=n1, keyed=True, C=C, K=2, W=8)


@pytest.mark.parametrize("n", [0, 17, 16384 * 2 * 5 + 7, 1 << 20])
def test_hist_fused_kernel(H, torch_mod, oracle, n):
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    levels = nests.c4_nest(K=2)
    C, K, W = 5, 2, 4
    for x in (gen.gen_u8(gen.SEED_C4, 0, n), gen.gen_u8_zipf(gen.SEED_C4, 0, n), np.zeros(n, np.uint8)):
        res = run_nest(H, torch, levels, x, n0=n, op=H.OP_HIST256, C=C, K=K, W=W, coverage=n <= 200000,
                       partials=n <= 200000)
        assert res["kernel"].startswith("hist256_lanepriv")
        assert np.array_equal(res["out"].astype(np.uint64), oracle.hist256(x))
        if n <= 200000:
            compare(oracle, H, levels, res, x, n0=n, op=H.OP_HIST256, C=C, K=K, W=W)


@pytest.mark.parametrize("mis", [1, 7, 15])
def test_hist_misaligned_input(H, torch_mod, oracle, mis):
    """An input pointer off a 16-byte boundary is not rejected (SURVEY §8(b)
    alignment): tiles copy their enclosing 16-byte granules and the lanes
    read bytes at the offset; result, coverage (owner = the nominal static
    closed form) and every level's partials vs the oracle."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    levels = nests.c4_nest(K=2)
    C, K, W = 3, 2, 4
    for n in (1, 17, 16384 * 2 * 5 + 7, 200000):
        for x in (gen.gen_u8(gen.SEED_C4, 0, n), gen.gen_u8_zipf(gen.SEED_C4, 0, n)):
            res = run_nest(H, torch, levels, x, n0=n, op=H.OP_HIST256, C=C, K=K, W=W, misalign=mis)
            assert res["kernel"].startswith("hist256_lanepriv")
            assert np.array_equal(res["out"].astype(np.uint64), oracle.hist256(x))
            compare(oracle, H, levels, res, x, n0=n, op=H.OP_HIST256, C=C, K=K, W=W)


@pytest.mark.parametrize("W,tile", [(8, 16384), (16, 8192), (12, 12288)])
def test_hist_shared_regions(H, torch_mod, oracle, W, tile):
    """W > 6 consumer warps: warp pairs share one lane-table region (the
    atomics keep it exact; the warp level is folded into the shared counters
    in timed runs).  Totals, coverage (every byte once, owner = static closed
    form) and the partials of EVERY level vs the oracle — the lane and warp
    bins of verify runs come from direct per-byte atomics — on uniform,
    skewed and all-zero bytes (reading #23)."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    levels = nests.c4_nest(K=2, tile=tile)
    C, K = 3, 2
    for n in (0, 5, tile * 2 * 7 + 9, 1 << 20):
        for x in (gen.gen_u8(gen.SEED_C4, 0, n), gen.gen_u8_zipf(gen.SEED_C4, 0, n), np.zeros(n, np.uint8)):
            small = n <= 300000
            res = run_nest(H, torch, levels, x, n0=n, op=H.OP_HIST256, C=C, K=K, W=W, coverage=small,
                           partials=small)
            assert res["kernel"].startswith("hist256_lanepriv")
            assert np.array_equal(res["out"].astype(np.uint64), oracle.hist256(x))
            if small:  # every level incl. lane / warp bins (built directly in verify runs), owner map
                compare(oracle, H, levels, res, x, n0=n, op=H.OP_HIST256, C=C, K=K, W=W)
    # outer-level partials (cluster, CTA) with shared regions
    n = tile * 2 * 5 + 3
    x = gen.gen_u8(gen.SEED_C4, 1, n)
    nest = H.Nest(levels, device=0, cluster_dim=K, warps_per_cta=W, clusters=C)
    xd = torch.from_numpy(x).cuda()
    out = torch.zeros(256, dtype=torch.int64, device="cuda")
    cl = torch.zeros((C, 256), dtype=torch.int64, device="cuda")
    cta = torch.zeros((C * K, 256), dtype=torch.int64, device="cuda")
    parts = [None, cl, cta, None, None]
    nest.parallel_for_reduce(H.make_desc(xd, out, n0=n, op=H.OP_HIST256, verify=H.VERIFY_PARTIALS, partials=parts))
    torch.cuda.synchronize()
    cta_h = cta.cpu().numpy().astype(np.uint64)
    for b in range(C * K):
        h = np.zeros(256, dtype=np.uint64)
        for s in range(b * tile, n, C * K * tile):
            h += oracle.hist256(x[s:s + tile])
        assert np.array_equal(cta_h[b], h), f"CTA {b}"
    assert np.array_equal(cl.cpu().numpy().astype(np.uint64).sum(axis=0), oracle.hist256(x))


def _csr_cases():
    off_z = gen.csr_offsets(3000, 40000)
    yield "zipf", off_z
    yield "all_empty", np.zeros(501, dtype=np.int64)
    yield "one_huge_row", np.array([0, (1 << 20) + 3], dtype=np.int64)
    lens = np.array([0, 1, 0, 0, 1024, 1025, 0, 3, 2048 + 5, 0, 0, 127, 128, 129, 0, 4096, 4097, 0, 8192, 8193, 1, 0],
                    dtype=np.int64)
    lens = np.tile(lens, 20)
    off = np.zeros(lens.size + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    yield "edges", off
    yield "short_only", np.arange(0, 2 * 70001, 2, dtype=np.int64)
    # nnz % 4 != 0 with short rows at the very end: the unaligned array tail
    # (< 4 values past the last whole 16 bytes) at odd and even row ends
    tail = np.concatenate([[0], np.cumsum(np.tile([3, 1, 16, 2, 5, 1, 1], 1001))]).astype(np.int64)
    yield "unaligned_tail", tail


@pytest.mark.parametrize("case", ["zipf", "all_empty", "one_huge_row", "edges", "short_only", "unaligned_tail"])
def test_segmented_csr_kernel(H, torch_mod, oracle, case):
    """Config-3 fused kernel: every row sum within 1e-5 of the oracle's fp64
    segment sums (0 exactly for empty rows), every nonzero visited once, each
    block of 128 rows' short rows handled by one warp (dynamic chunk alignment)."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    off = dict(_csr_cases())[case]
    rows, nnz = off.size - 1, int(off[-1])
    v = gen.gen_f32(gen.SEED_C3, 0, nnz)
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8, clusters=5)
    xd = torch.from_numpy(v).cuda() if nnz else torch.zeros(4, dtype=torch.float32, device="cuda")
    offd = torch.from_numpy(off).cuda()
    out = torch.full((max(rows, 1),), -1.0, dtype=torch.float64, device="cuda")
    owner = torch.full((max(nnz, 1),), -1, dtype=torch.int64, device="cuda")
    count = torch.zeros(max(nnz, 1), dtype=torch.int32, device="cuda")
    for verify in (0, H.VERIFY_COVERAGE):
        out.fill_(-1.0)
        d = H.make_desc(xd, out, n0=rows, n1=nnz, nloops=2, keyed=True, offsets=offd, out_dtype=H.F64,
                        verify=verify, owner=owner if verify else None, count=count if verify else None)
        nest.parallel_for_reduce(d)
        torch.cuda.synchronize()
        assert nest.last_kernel() == "segmented_csr"
        assert_rel(out.cpu().numpy()[:rows], oracle.segsum_f32(v, off))
    if nnz:
        assert (count.cpu().numpy()[:nnz] == 1).all()
        own = owner.cpu().numpy()[:nnz] // 32  # warp of the owner
        lens = np.diff(off)
        rb = nests.c3_fast_nest()[1].chunk
        for b0 in range(0, rows, rb):
            rs = [r for r in range(b0, min(b0 + rb, rows)) if 0 < lens[r] <= 4096]
            if rs:
                ws_ = np.concatenate([own[off[r]:off[r + 1]] for r in rs])
                assert (ws_ == ws_[0]).all(), "a block's short rows span several warps"


@pytest.mark.parametrize("mis", [4, 8, 12])
@pytest.mark.parametrize("case", ["zipf", "one_huge_row", "edges", "unaligned_tail"])
def test_segmented_misaligned_values(H, torch_mod, oracle, case, mis):
    """CSR values 4, 8 or 12 bytes off a 16-byte boundary (a slice of a
    larger tensor) stay on the fused kernel: it sees the array from the
    granule boundary before them with every offset moved by the same shift.
    Row sums vs the oracle, every nonzero visited exactly once (coverage
    indexed by the caller's positions), over both output dtypes."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    off = dict(_csr_cases())[case]
    rows, nnz = off.size - 1, int(off[-1])
    v = gen.gen_f32(gen.SEED_C3, 0, nnz)
    raw = torch.full((nnz + 16,), float("nan"), dtype=torch.float32, device="cuda")
    e0 = mis // 4
    xd = raw[e0:e0 + nnz]
    xd.copy_(torch.from_numpy(v).cuda())
    assert xd.data_ptr() % 16 == mis
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8, clusters=5)
    offd = torch.from_numpy(off).cuda()
    owner = torch.full((nnz,), -1, dtype=torch.int64, device="cuda")
    count = torch.zeros(nnz, dtype=torch.int32, device="cuda")
    for dt, odt in ((torch.float64, H.F64), (torch.float32, H.F32)):
        out = torch.full((rows,), -1.0, dtype=dt, device="cuda")
        count.zero_()
        d = H.make_desc(xd, out, n0=rows, n1=nnz, nloops=2, keyed=True, offsets=offd, out_dtype=odt,
                        verify=H.VERIFY_COVERAGE, owner=owner, count=count)
        nest.parallel_for_reduce(d)
        torch.cuda.synchronize()
        assert nest.last_kernel() == "segmented_csr"
        assert_rel(out.cpu().numpy().astype(np.float64), oracle.segsum_f32(v, off))
        assert (count.cpu().numpy() == 1).all()
        d = H.make_desc(xd, out, n0=rows, n1=nnz, nloops=2, keyed=True, offsets=offd, out_dtype=odt)
        out.fill_(-1.0)
        nest.parallel_for_reduce(d)
        torch.cuda.synchronize()
        assert_rel(out.cpu().numpy().astype(np.float64), oracle.segsum_f32(v, off))


@pytest.mark.parametrize("dt,op", [("f32", "min"), ("f32", "max"), ("f64", "sum"), ("f64", "min"), ("i32", "sum"),
                                   ("i64", "sum"), ("i64", "max"), ("i64", "affine")])
@pytest.mark.parametrize("case", ["zipf", "all_empty", "one_huge_row", "edges", "short_only", "unaligned_tail"])
def test_segrows_ops_and_dtypes(H, torch_mod, oracle, case, dt, op):
    """The collapsed CSR nest (c3_fast_nest) for the ops and dtypes the fp32
    sum kernel does not take (kernel_segrows.cu): every row vs the oracle's
    nest walk (MIN/MAX and integers exact, fp64 within the tolerance; empty
    rows the identity), every nonzero visited once, each block's short rows
    on one warp; the long rows (> 4096) through the chunk list."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    off = dict(_csr_cases())[case]
    rows, nnz = off.size - 1, int(off[-1])
    rng = np.random.default_rng(12)
    if dt == "f32":
        v = gen.gen_f32(gen.SEED_C3, 0, nnz) - np.float32(0.5)
    elif dt == "f64":
        v = rng.standard_normal(nnz) + 3.0
    elif dt == "i32":
        v = rng.integers(-(1 << 31), (1 << 31) - 1, nnz, dtype=np.int64).astype(np.int32)
    else:
        v = rng.integers(-(1 << 62), 1 << 62, nnz, dtype=np.int64)
    hop = {"sum": H.OP_SUM, "min": H.OP_MIN, "max": H.OP_MAX, "affine": H.OP_AFFINE}[op]
    fp = dt in ("f32", "f64")
    for lpl in (16, 8):
        nest = H.Nest(nests.c3_fast_nest(lane_chunk=lpl), device=0, cluster_dim=2, warps_per_cta=8, clusters=5)
        xd = torch.from_numpy(v).cuda() if nnz else torch.zeros(4, dtype=torch.from_numpy(v).dtype, device="cuda")
        offd = torch.from_numpy(off).cuda()
        shape = (max(rows, 1), 2) if op == "affine" else (max(rows, 1),)
        out = torch.full(shape, -1, dtype=torch.float64 if fp else torch.int64, device="cuda")
        owner = torch.full((max(nnz, 1),), -1, dtype=torch.int64, device="cuda")
        count = torch.zeros(max(nnz, 1), dtype=torch.int32, device="cuda")
        for verify in (0, H.VERIFY_COVERAGE):
            out.fill_(-1)
            d = H.make_desc(xd, out, n0=rows, n1=nnz, nloops=2, keyed=True, offsets=offd, op=hop,
                            out_dtype=H.F64 if fp else (H.U64 if op == "affine" else H.I64), verify=verify,
                            owner=owner if verify else None, count=count if verify else None)
            nest.parallel_for_reduce(d)
            torch.cuda.synchronize()
            assert nest.last_kernel() == "segrows_csr"
            ref_levels = nests.c3_nest(with_gpu=False, rows_chunk=16, width=8)
            o = None if op == "affine" else oracle.nest_run(oracle_levels(oracle, ref_levels, 1, 2, 2, 4), n0=rows, offsets=off, x=v, op=hop,
                                keyed=True, coverage=False, partials=False)
            got = out.cpu().numpy()[:rows]
            if op == "affine":
                # DESIGN reading #28: per row, the sequential composition (the
                # direct recurrence); (A, B) pinned by y0 = 0 -> B, y0 = 1 -> A + B
                g = got.view(np.uint64)
                for r in range(rows):
                    xr = v[off[r]:off[r + 1]]
                    B = oracle.affine_run(xr, 0)
                    assert int(g[r, 1]) == B and (int(g[r, 0]) + B) % (1 << 64) == oracle.affine_run(xr, 1), (case, r)
            elif fp and op == "sum":
                assert_rel(got, o.result)
            else:
                assert np.array_equal(got, o.result), (case, dt, op)
        if nnz:
            assert (count.cpu().numpy()[:nnz] == 1).all()
            own = owner.cpu().numpy()[:nnz] // 32
            lens = np.diff(off)
            for b0 in range(0, rows, 256):
                rs = [r for r in range(b0, min(b0 + 256, rows)) if 0 < lens[r] <= 4096]
                if rs:
                    ws_ = np.concatenate([own[off[r]:off[r + 1]] for r in rs])
                    assert (ws_ == ws_[0]).all(), "a block's short rows span several warps"


def test_segrows_zero_rows(H, torch_mod):
    """A CSR call with no rows on the CSR rows kernel: nothing written, both
    launches exit at once (the block ticket and the empty chunk list)."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8, clusters=3)
    x = torch.zeros(4, dtype=torch.float64, device="cuda")
    out = torch.full((1,), -3.0, dtype=torch.float64, device="cuda")
    off = torch.zeros(1, dtype=torch.int64, device="cuda")
    nest.parallel_for_reduce(H.make_desc(x, out, n0=0, n1=0, nloops=2, keyed=True, offsets=off, out_dtype=H.F64))
    torch.cuda.synchronize()
    assert out.item() == -3.0


def _probe_expect(oracle, level, C, K, W, rounds):
    """The oracle's fold for every task of the probe (hpar_barrier_probe):
    sum over rounds of the sum over the task's sibling group of
    fp_mix((round << 40) ^ sibling id), mod 2^64.  Groups: the 32 lanes of a
    warp, the W warps of a CTA, the K CTAs of a cluster."""
    M = (1 << 64) - 1
    group = {"lane": 32, "warp": W, "cta": K}[level]
    ntask = {"lane": C * K * W * 32, "warp": C * K * W, "cta": C * K}[level]
    out = np.zeros(ntask, dtype=np.uint64)
    for g0 in range(0, ntask, group):
        f = 0
        for r in range(rounds):
            f += sum(oracle.fp_mix((r << 40) ^ (g0 + j)) for j in range(group))
        out[g0:g0 + group] = f & M
    return out


def test_barrier_probes(H, torch_mod, oracle):
    """§8(a) A10 / §8(c) #5: with the lane / warp / CTA barriers of the hot
    path (__syncwarp, bar.sync, barrier.cluster) every task's folds over its
    siblings' slots equal the oracle's group folds; host-level hpar_barrier
    on those levels is the kernel boundary (OK, nothing enqueued); the
    cluster level has no barrier."""
    torch = torch_mod
    C, K, W, R = 37, 2, 8, 8
    nest = H.Nest([H.Level(H.HPAR_GPU, H.HPAR_LANE)], device=0, cluster_dim=K, warps_per_cta=W, clusters=C)
    for name, lvl in (("lane", H.HPAR_LANE), ("warp", H.HPAR_WARP), ("cta", H.HPAR_CTA)):
        want = _probe_expect(oracle, name, C, K, W, R)
        folds = torch.zeros(want.size, dtype=torch.int64, device="cuda")
        nest.barrier_probe(lvl, folds.data_ptr(), rounds=R)
        torch.cuda.synchronize()
        assert np.array_equal(folds.cpu().numpy().view(np.uint64), want), f"{name}: folds differ from the oracle's"
    for lvl in (H.HPAR_LANE, H.HPAR_WARP, H.HPAR_CTA, H.HPAR_NODE, H.HPAR_GPU):
        nest.barrier(lvl)
    torch.cuda.synchronize()
    for call in (lambda: nest.barrier(H.HPAR_CLUSTER),
                 lambda: nest.barrier_probe(H.HPAR_CLUSTER, folds.data_ptr())):
        with pytest.raises(H.HparError) as e:
            call()
        assert e.value.code == H.HPAR_E_CAPABILITY


@pytest.mark.parametrize("level", ["warp", "cta"])
def test_barrier_probe_negative_control(H, torch_mod, oracle, level):
    """The probe pins something: with the level barrier removed and sibling k
    writing (k+1) x 2 us late, readers fold stale slots and the folds differ
    from the oracle's.  (The lane level's control is left to racecheck:
    lanes reconverge after the divergent delay, profiles/r02_sanitizer.md.)"""
    torch = torch_mod
    C, K, W, R = 37, 2, 8, 4
    nest = H.Nest([H.Level(H.HPAR_GPU, H.HPAR_LANE)], device=0, cluster_dim=K, warps_per_cta=W, clusters=C)
    lvl = {"warp": H.HPAR_WARP, "cta": H.HPAR_CTA}[level]
    want = _probe_expect(oracle, level, C, K, W, R)
    folds = torch.zeros(want.size, dtype=torch.int64, device="cuda")
    nest.barrier_probe(lvl, folds.data_ptr(), rounds=R, no_barrier=True, delay_ns=2000)
    torch.cuda.synchronize()
    bad = int((folds.cpu().numpy().view(np.uint64) != want).sum())
    assert bad > 0, "a probe without its barrier still folded every slot correctly"


def test_hierarchy_query_matches_device(H, torch_mod):
    torch = torch_mod
    t = H.hpar_hierarchy_query(0)
    p = torch.cuda.get_device_properties(0)
    assert [r.name.decode() for r in t] == H.LEVEL_NAMES
    assert t[H.HPAR_GPU].num == 1 and t[H.HPAR_LANE].num == 32
    assert t[H.HPAR_GPU].groupmem_bytes == p.total_memory
    assert t[H.HPAR_CLUSTER].num >= p.multi_processor_count // 2
    assert "barrier" not in t[H.HPAR_CLUSTER].flags() and "shuffle" in t[H.HPAR_LANE].flags()


def test_ordered_affine_op(H, torch_mod, oracle):
    """NEXT f2: a non-commutative user-defined operator
    (affine-map composition mod 2^64) through the generic kernel.  Every GPU
    tree is order-preserving, so results and per-level partials equal the
    oracle's ascending-task-order fold BIT FOR BIT for any static nest; with
    block schedules that is the sequential recurrence itself."""
    torch = torch_mod
    rng = random.Random(86)
    done = 0
    while done < (FUZZ_N or 25):
        levels = random_flat_nest(H, rng, 0)
        for l in levels:
            if l.schedule == H.NONE:
                l.schedule = H.STATIC
        C, K, W = rng.choice([1, 3, 5]), rng.choice([1, 2, 4]), rng.choice([1, 2, 4])
        n = rng.randint(0, 6000)
        x = gen.gen_i32(done + 300, 0, n).astype(np.int64)
        res = run_nest(H, torch, levels, x, n0=n, op=H.OP_AFFINE, C=C, K=K, W=W)
        assert res["kernel"] == "generic"
        compare(oracle, H, levels, res, x, n0=n, op=H.OP_AFFINE, C=C, K=K, W=W)
        done += 1
    # block schedules everywhere: the fold is the sequential recurrence
    levels = [H.Level(H.HPAR_GPU), H.Level(H.HPAR_CLUSTER), H.Level(H.HPAR_CTA), H.Level(H.HPAR_WARP),
              H.Level(H.HPAR_LANE)]
    x = gen.gen_i32(4242, 0, 100003).astype(np.int64)
    res = run_nest(H, torch, levels, x, n0=x.size, op=H.OP_AFFINE, C=7, K=2, W=4, coverage=False, partials=False)
    A, B = (int(v) for v in res["out"].view(np.uint64))
    assert (A * 5 + B) % (1 << 64) == oracle.affine_run(x, 5)
    # keyed rows (2 loops): per-row composed maps
    levels = [H.Level(H.HPAR_GPU, H.HPAR_GPU, 0, loop=0), H.Level(H.HPAR_CLUSTER, H.HPAR_CTA, 0, loop=0),
              H.Level(H.HPAR_WARP, H.HPAR_LANE, 1, loop=1, chunk=2)]
    x = gen.gen_i32(77, 0, 29 * 333).astype(np.int64)
    res = run_nest(H, torch, levels, x, n0=29, n1=333, keyed=True, op=H.OP_AFFINE, C=3, K=2, W=2)
    compare(oracle, H, levels, res, x, n0=29, n1=333, keyed=True, op=H.OP_AFFINE, C=3, K=2, W=2)


def test_teams_affine_op(H, torch_mod, oracle):
    """The ordered AFFINE op on the teams x threads kernel (config-1 nest,
    int64): each thread folds its (row, chunk) iterations in nest order and
    every level in ascending task order — results, owner map and partials
    bit-exact vs the oracle's nest fold, for chunk 4 and a ragged chunk."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    rng = np.random.default_rng(3)
    for n0, n1, chunk, C in ((64, 1024, 4, 8), (37, 1000, 3, 5), (5, 7, 4, 3)):
        levels = nests.c1_nest(outer=0)
        levels[-1].chunk = chunk
        x = rng.integers(-(1 << 62), 1 << 62, n0 * n1, dtype=np.int64)
        res = run_nest(H, torch, levels, x, n0=n0, n1=n1, op=H.OP_AFFINE, C=C, K=2, W=4)
        assert res["kernel"] == "teams_threads"
        compare(oracle, H, levels, res, x, n0=n0, n1=n1, op=H.OP_AFFINE, C=C, K=2, W=4)


@pytest.mark.parametrize("seed", range(FUZZ_N or 16))
def test_teams_fuzz(H, torch_mod, oracle, seed):
    """Random two-level teams x threads nests (config-1 shape: teams =
    cluster..CTA static over rows, threads = warp..lane static(c) over
    columns) on the fused teams kernel: rows, columns, ld, chunk c, K, W, C,
    op and dtype (AFFINE over int64) at random; total, owner map and every
    level's partials vs the oracle."""
    torch = torch_mod
    rng = np.random.default_rng(6000 + seed)
    n0 = int(rng.integers(1, 300))
    n1 = int(rng.choice([int(rng.integers(1, 64)), int(rng.integers(64, 3000))]))
    ld = n1 + int(rng.choice([0, 0, int(rng.integers(1, 9))]))
    K, W = int(rng.choice([1, 2, 4, 8])), int(rng.choice([1, 2, 4, 8, 16]))
    C = int(rng.integers(1, 12))
    chunk = int(rng.choice([1, 2, 3, 4, 8, 16]))
    combos = [("i32", H.OP_SUM), ("i32", H.OP_MAX), ("f32", H.OP_SUM), ("f64", H.OP_MIN), ("i64", H.OP_SUM),
              ("i64", H.OP_AFFINE)]
    dt, op = combos[int(rng.integers(len(combos)))]
    if dt == "i32":
        x = gen.gen_i32(gen.SEED_C1 + seed, 0, n0 * n1)
    elif dt == "f32":
        x = gen.gen_f32(gen.SEED_C1 + seed, 0, n0 * n1)
    elif dt == "f64":
        x = rng.standard_normal(n0 * n1)
    else:
        x = rng.integers(-(1 << 62), 1 << 62, n0 * n1, dtype=np.int64)
    levels = [H.Level(H.HPAR_GPU, H.HPAR_GPU, H.STATIC, loop=0),
              H.Level(H.HPAR_CLUSTER, H.HPAR_CTA, H.STATIC, loop=0),
              H.Level(H.HPAR_WARP, H.HPAR_LANE, H.STATIC_CHUNK, loop=1, chunk=chunk)]
    res = run_nest(H, torch, levels, x, n0=n0, n1=n1, op=op, C=C, K=K, W=W, ld=ld)
    assert res["kernel"] == "teams_threads", (n0, n1, chunk, K, W, dt)
    compare(oracle, H, levels, res, x, n0=n0, n1=n1, op=op, C=C, K=K, W=W)


def test_generic_keyed_dynamic_repeated_calls(H, torch_mod, oracle):
    """Regression: in keyed mode every CTA of a cluster must be done before the
    cluster's leader arrives at the grid ticket (whose last arriver resets the
    dynamic tickets).  Same nest, several calls, K = 2 and 4."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    off = gen.csr_offsets(3000, 40000)
    v = gen.gen_f32(gen.SEED_C3, 0, 40000)
    want = oracle.segsum_f32(v, off)
    for K in (2, 4):
        nest = H.Nest(nests.c3_nest(with_gpu=True, rows_chunk=64, width=8), device=0, cluster_dim=K,
                      warps_per_cta=4, clusters=3)
        xd = torch.from_numpy(v).cuda()
        offd = torch.from_numpy(off).cuda()
        for _ in range(4):
            out = torch.zeros(3000, dtype=torch.float64, device="cuda")
            owner = torch.zeros(40000, dtype=torch.int64, device="cuda")
            count = torch.zeros(40000, dtype=torch.int32, device="cuda")
            nest.parallel_for_reduce(H.make_desc(xd, out, n0=3000, nloops=2, keyed=True, offsets=offd,
                                                 out_dtype=H.F64, verify=H.VERIFY_COVERAGE, owner=owner,
                                                 count=count))
            torch.cuda.synchronize()
            assert (count.cpu().numpy() == 1).all()
            assert_rel(out.cpu().numpy(), want)


@pytest.mark.parametrize("G", [2, 3, 8])
def test_segmented_nnz_balanced_ranks(H, torch_mod, oracle, G):
    """§8(e) C3: the GPU level shards rows at nnz-balanced boundaries
    (hpar_shard_range_csr); each rank's call sees only its rows (local_n0)
    and values; the concatenated keyed results equal the oracle.  The ranks
    run one after another on this GPU (keyed results: no node collective)."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    off = gen.csr_offsets(20000, 300000)
    v = gen.gen_f32(gen.SEED_C3, 0, int(off[-1]))
    got = np.full(20000, np.nan)
    for g in range(G):
        b, c = H.hpar_shard_range_csr(off, G, g)
        nest = H.Nest(nests.c3_fast_nest(), device=0, rank=g, nranks=G, cluster_dim=2, warps_per_cta=8, clusters=5)
        lo = (off[b:b + c + 1] - off[b]).astype(np.int64)
        vals = v[off[b]:off[b + c]]
        xd = torch.from_numpy(vals).cuda() if vals.size else torch.zeros(4, dtype=torch.float32, device="cuda")
        out = torch.full((max(c, 1),), -1.0, dtype=torch.float64, device="cuda")
        d = H.make_desc(xd, out, n0=20000, n1=int(vals.size), nloops=2, keyed=True,
                        offsets=torch.from_numpy(lo).cuda(), out_dtype=H.F64, local_n0=c)
        nest.parallel_for_reduce(d)
        torch.cuda.synchronize()
        assert nest.last_kernel() == "segmented_csr"
        got[b:b + c] = out.cpu().numpy()[:c]
    assert_rel(got, oracle.segsum_f32(v, off))


@pytest.mark.parametrize("seed", range(FUZZ_N or 10))
def test_segmented_fuzz(H, torch_mod, oracle, seed):
    """Random CSR shapes through the fused kernel: empty / short / medium /
    split (> 4096) rows in random order, nnz with any residue mod 4, and
    value sets that keep every window on the exact prefix path (the input
    recipe), push windows onto the in-order fp64 path (magnitudes over 60
    decades), or mix both.  Results within 1e-5 of the oracle; every
    nonzero visited once."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    rng = np.random.default_rng(1000 + seed)
    rows = int(rng.integers(1, 2500))
    kind = rng.choice(4, size=rows, p=[0.3, 0.5, 0.17, 0.03])
    lens = np.where(kind == 0, 0, np.where(kind == 1, rng.geometric(0.2, rows),
                    np.where(kind == 2, rng.integers(30, 2500, rows), rng.integers(4097, 40000, rows))))
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    nnz = int(off[-1])
    v = gen.gen_f32(gen.SEED_C3 + seed, 0, nnz)
    if seed % 3 == 1:
        v = (10.0 ** rng.uniform(-30, 30, nnz)).astype(np.float32)
    elif seed % 3 == 2:
        spikes = rng.random(nnz) < 0.001
        v = np.where(spikes, (10.0 ** rng.uniform(-20, 20, nnz)).astype(np.float32), v).astype(np.float32)
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8, clusters=int(rng.integers(1, 9)))
    if seed % 4 == 3:  # a CSR slice: rows start at b0 > 0, the b0 values before them are NaN (never read into a row)
        b0 = int(rng.integers(1, 41))
        off = off + b0
        v = np.concatenate([np.full(b0, np.nan, dtype=np.float32), v])
        nnz = int(off[-1])
    xd = torch.from_numpy(v).cuda() if nnz else torch.zeros(4, dtype=torch.float32, device="cuda")
    offd = torch.from_numpy(off).cuda()
    out = torch.full((rows,), -1.0, dtype=torch.float64, device="cuda")
    owner = torch.full((max(nnz, 1),), -1, dtype=torch.int64, device="cuda")
    count = torch.zeros(max(nnz, 1), dtype=torch.int32, device="cuda")
    want = oracle.segsum_f32(v, off)
    for verify in (0, H.VERIFY_COVERAGE):
        out.fill_(-1.0)
        d = H.make_desc(xd, out, n0=rows, n1=nnz, nloops=2, keyed=True, offsets=offd, out_dtype=H.F64,
                        verify=verify, owner=owner if verify else None, count=count if verify else None)
        nest.parallel_for_reduce(d)
        torch.cuda.synchronize()
        assert nest.last_kernel() == "segmented_csr"
        assert_rel(out.cpu().numpy(), want)
    if nnz:
        cnt = count.cpu().numpy()[:nnz]
        assert (cnt[int(off[0]):] == 1).all() and (cnt[:int(off[0])] == 0).all()


@pytest.mark.parametrize("seed", range(FUZZ_N or 12))
def test_segrows_fuzz(H, torch_mod, oracle, seed):
    """Random CSR shapes on the CSR rows kernel: empty / short / medium /
    long (> 4096) rows in random order, a random op and dtype (MIN / MAX over
    fp32; SUM / MIN / MAX over fp64, int32, int64; AFFINE over int64), a
    random lane chunk, grid and value-pointer offset.  Every row vs the
    oracle (the nest walk of the generic CSR nest; AFFINE per row against the
    direct recurrence), every nonzero visited once."""
    from paper_2309_01906_b200 import nests
    from tests.nestutil import oracle_levels
    torch = torch_mod
    rng = np.random.default_rng(2000 + seed)
    rows = int(rng.integers(1, 2500))
    kind = rng.choice(4, size=rows, p=[0.3, 0.5, 0.17, 0.03])
    lens = np.where(kind == 0, 0, np.where(kind == 1, rng.geometric(0.2, rows),
                    np.where(kind == 2, rng.integers(30, 2500, rows), rng.integers(4097, 40000, rows))))
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    nnz = int(off[-1])
    combos = [("f32", H.OP_MIN), ("f32", H.OP_MAX), ("f64", H.OP_SUM), ("f64", H.OP_MIN), ("f64", H.OP_MAX),
              ("i32", H.OP_SUM), ("i32", H.OP_MIN), ("i64", H.OP_SUM), ("i64", H.OP_MAX), ("i64", H.OP_AFFINE)]
    dt, op = combos[int(rng.integers(len(combos)))]
    if dt == "f32":
        v = (rng.standard_normal(nnz) * 10 ** rng.uniform(-3, 3)).astype(np.float32)
    elif dt == "f64":
        v = rng.standard_normal(nnz) + float(rng.uniform(-2, 2))
    elif dt == "i32":
        v = rng.integers(-(1 << 31), (1 << 31) - 1, nnz, dtype=np.int64).astype(np.int32)
    else:
        v = rng.integers(-(1 << 62), 1 << 62, nnz, dtype=np.int64)
    if seed % 4 == 3:  # a CSR slice: rows start at b0 > 0 after b0 poison values no row covers
        b0 = int(rng.integers(1, 41))
        off = off + b0
        poison = np.full(b0, np.nan if v.dtype.kind == "f" else np.iinfo(v.dtype).max // 3, dtype=v.dtype)
        v = np.concatenate([poison, v])
        nnz = int(off[-1])
    lpl = int(rng.choice([8, 16]))
    nest = H.Nest(nests.c3_fast_nest(lane_chunk=lpl), device=0, cluster_dim=2, warps_per_cta=8,
                  clusters=int(rng.integers(1, 9)))
    shift = int(rng.integers(0, 16 // v.itemsize))  # elements off a 16-byte granule
    raw = torch.zeros(nnz + 16, dtype=torch.from_numpy(v[:0]).dtype, device="cuda")
    xd = raw[shift:shift + nnz]
    if nnz:
        xd.copy_(torch.from_numpy(v).cuda())
    offd = torch.from_numpy(off).cuda()
    fp = dt in ("f32", "f64")
    shape = (rows, 2) if op == H.OP_AFFINE else (rows,)
    out = torch.full(shape, -1, dtype=torch.float64 if fp else torch.int64, device="cuda")
    owner = torch.full((max(nnz, 1),), -1, dtype=torch.int64, device="cuda")
    count = torch.zeros(max(nnz, 1), dtype=torch.int32, device="cuda")
    odt = H.F64 if fp else (H.U64 if op == H.OP_AFFINE else H.I64)
    d = H.make_desc(xd, out, n0=rows, n1=nnz, nloops=2, keyed=True, offsets=offd, op=op, out_dtype=odt,
                    verify=H.VERIFY_COVERAGE, owner=owner, count=count)
    nest.parallel_for_reduce(d)
    torch.cuda.synchronize()
    assert nest.last_kernel() == "segrows_csr"
    got = out.cpu().numpy()
    if op == H.OP_AFFINE:
        g = got.view(np.uint64)
        for r in range(rows):
            xr = v[off[r]:off[r + 1]]
            B = oracle.affine_run(xr, 0)
            assert int(g[r, 1]) == B and (int(g[r, 0]) + B) % (1 << 64) == oracle.affine_run(xr, 1), r
    else:
        ol = oracle_levels(oracle, nests.c3_nest(with_gpu=False, rows_chunk=16, width=8), 1, 2, 2, 4)
        want = oracle.nest_run(ol, n0=rows, offsets=off, x=v, op=op, keyed=True, coverage=False,
                               partials=False).result
        if fp and op == H.OP_SUM:
            assert_rel(got, want)
        else:
            assert np.array_equal(got, want)
    if nnz:
        cnt = count.cpu().numpy()[:nnz]
        assert (cnt[int(off[0]):] == 1).all() and (cnt[:int(off[0])] == 0).all()


@pytest.mark.parametrize("seed", range(FUZZ_N or 24))
def test_flat_fuzz(H, torch_mod, oracle, seed):
    """Random flat shapes on the fused flat kernel: length (empty, ragged,
    several tiles), tile, lane chunk (static(1) / static(2) / static(4)), the
    nest's spelling (separate or collapsed cluster..CTA and warp..lane
    levels), K, W, C, op, dtype (fp32 / int32 / fp64 / int64, AFFINE over
    int64) and pointer offset at random; total, owner map and every level's
    partials vs the oracle."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    rng = np.random.default_rng(4000 + seed)
    K, W = int(rng.choice([1, 2, 4, 8])), int(rng.choice([1, 2, 4, 8, 16]))
    combos = [("f32", H.OP_SUM), ("f32", H.OP_MAX), ("i32", H.OP_SUM), ("i32", H.OP_MIN), ("f64", H.OP_SUM),
              ("f64", H.OP_MIN), ("i64", H.OP_SUM), ("i64", H.OP_AFFINE)]
    dt, op = combos[int(rng.integers(len(combos)))]
    esz = 8 if dt in ("f64", "i64") else 4
    V = int(rng.choice([1, 2, 4]))  # lane static(V), warp static(32 V)
    tile = 32 * V * W * int(rng.choice([1, 2, 4, 8]))
    tile = min(tile, 32768 // esz) // (32 * V * W) * (32 * V * W) or 32 * V * W
    C = int(rng.integers(1, 10))
    n = int(rng.choice([0, int(rng.integers(1, 3000)), int(rng.integers(3000, 400000))]))
    if dt == "f32":
        x = gen.gen_f32(gen.SEED_C5 + seed, 0, n)
    elif dt == "i32":
        x = gen.gen_i32(gen.SEED_C1 + seed, 0, n)
    elif dt == "f64":
        x = rng.standard_normal(n) + 1.0
    else:
        x = rng.integers(-(1 << 62), 1 << 62, n, dtype=np.int64)
    mis = int(rng.integers(0, 16 // esz)) * esz if n else 0
    # any of the four equivalent spellings: cluster + CTA or cluster..CTA,
    # warp + lane or warp..lane (the same owner map, so the same kernel)
    spell = int(rng.integers(4))
    levels = [H.Level(H.HPAR_GPU, H.HPAR_GPU, H.STATIC)]
    if spell & 1:
        levels.append(H.Level(H.HPAR_CLUSTER, H.HPAR_CTA, H.STATIC_CHUNK, chunk=tile))
    else:
        levels += [H.Level(H.HPAR_CLUSTER, H.HPAR_CLUSTER, H.STATIC_CHUNK, chunk=K * tile),
                   H.Level(H.HPAR_CTA, H.HPAR_CTA, H.STATIC_CHUNK, chunk=tile)]
    if spell & 2:
        levels.append(H.Level(H.HPAR_WARP, H.HPAR_LANE, H.STATIC_CHUNK, chunk=V))
    else:
        levels += [H.Level(H.HPAR_WARP, H.HPAR_WARP, H.STATIC_CHUNK, chunk=32 * V),
                   H.Level(H.HPAR_LANE, H.HPAR_LANE, H.STATIC_CHUNK, chunk=V)]
    fpr = bool(rng.random() < 0.5)  # also the coverage fingerprints (F_once, F_owner, count) vs the oracle's
    res = run_nest(H, torch, levels, x, n0=n, op=op, C=C, K=K, W=W, misalign=mis, fingerprint=fpr)
    assert res["kernel"] == "flat_tma", (n, tile, K, W, V, dt, spell)
    compare(oracle, H, levels, res, x, n0=n, op=op, C=C, K=K, W=W)
    if fpr:
        once, own = oracle.fp_flat_range(oracle_levels(oracle, levels, 1, C, K, W), n, 0, n)
        assert (int(res["fp"][0]), int(res["fp"][1]), int(res["fp"][2])) == (once, own, n)


@pytest.mark.parametrize("seed", range(FUZZ_N or 20))
def test_hist_fuzz(H, torch_mod, oracle, seed):
    """Random shapes on the histogram kernel: length, tile, K, W (private or
    shared lane-table regions), C, pointer offset, the nest's spelling
    (separate or collapsed levels), uniform / skewed / constant bytes; bins,
    owner map and every level's partials vs the oracle."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    rng = np.random.default_rng(5000 + seed)
    K, W = int(rng.choice([1, 2, 4, 8])), int(rng.choice([1, 2, 4, 6, 8, 12, 16]))
    tile = 512 * W * int(rng.choice([1, 2, 4]))
    tile = min(tile, 32768) // (512 * W) * (512 * W) or 512 * W
    C = int(rng.integers(1, 8))
    n = int(rng.choice([0, int(rng.integers(1, 5000)), int(rng.integers(5000, 300000))]))
    kind = int(rng.integers(3))
    x = (gen.gen_u8(gen.SEED_C4 + seed, 0, n) if kind == 0 else gen.gen_u8_zipf(gen.SEED_C4 + seed, 0, n)
         if kind == 1 else np.full(n, int(rng.integers(256)), dtype=np.uint8))
    mis = int(rng.integers(0, 16)) if n else 0
    spell = int(rng.integers(4))  # separate or collapsed cluster..CTA / warp..lane levels
    levels = [H.Level(H.HPAR_GPU, H.HPAR_GPU, H.STATIC)]
    if spell & 1:
        levels.append(H.Level(H.HPAR_CLUSTER, H.HPAR_CTA, H.STATIC_CHUNK, chunk=tile))
    else:
        levels += [H.Level(H.HPAR_CLUSTER, H.HPAR_CLUSTER, H.STATIC_CHUNK, chunk=K * tile),
                   H.Level(H.HPAR_CTA, H.HPAR_CTA, H.STATIC_CHUNK, chunk=tile)]
    if spell & 2:
        levels.append(H.Level(H.HPAR_WARP, H.HPAR_LANE, H.STATIC_CHUNK, chunk=16))
    else:
        levels += [H.Level(H.HPAR_WARP, H.HPAR_WARP, H.STATIC_CHUNK, chunk=512),
                   H.Level(H.HPAR_LANE, H.HPAR_LANE, H.STATIC_CHUNK, chunk=16)]
    fpr = bool(rng.random() < 0.5)  # also the coverage fingerprints vs the oracle's
    res = run_nest(H, torch, levels, x, n0=n, op=H.OP_HIST256, C=C, K=K, W=W, misalign=mis, fingerprint=fpr)
    assert res["kernel"].startswith("hist256_lanepriv"), (n, tile, K, W, spell)
    if fpr:
        once, own = oracle.fp_flat_range(oracle_levels(oracle, levels, 1, C, K, W), n, 0, n)
        assert (int(res["fp"][0]), int(res["fp"][1]), int(res["fp"][2])) == (once, own, n)
    assert np.array_equal(res["out"].astype(np.uint64), oracle.hist256(x))
    compare(oracle, H, levels, res, x, n0=n, op=H.OP_HIST256, C=C, K=K, W=W)


@pytest.mark.parametrize("seed", range(FUZZ_N or 24))
def test_rowwise_fuzz(H, torch_mod, oracle, seed):
    """Random dense-row shapes on the fused row-wise kernel: rows, columns,
    leading dimension, pointer offset, lane chunk (1, 2, 4), K, W, C, op and
    dtype at random (ragged or aligned); rows, owner map and every level's
    partials vs the oracle."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    rng = np.random.default_rng(3000 + seed)
    n0 = int(rng.integers(1, 120))
    n1 = int(rng.choice([int(rng.integers(1, 40)), int(rng.integers(40, 5000))]))
    ld = n1 + int(rng.choice([0, 0, int(rng.integers(1, 9))]))
    K, W = int(rng.choice([1, 2, 4, 8])), int(rng.choice([1, 2, 4, 8]))
    if K * W > 32:
        W = 32 // K
    C = int(rng.integers(1, 12))
    combos = [("f32", H.OP_SUM), ("f32", H.OP_MIN), ("f64", H.OP_SUM), ("f64", H.OP_MAX), ("i32", H.OP_SUM),
              ("i64", H.OP_MIN), ("i64", H.OP_AFFINE)]
    dt, op = combos[int(rng.integers(len(combos)))]
    if dt == "f32":
        x = gen.gen_f32(gen.SEED_C2 + seed, 0, n0 * n1)
    elif dt == "f64":
        x = rng.standard_normal(n0 * n1)
    elif dt == "i32":
        x = rng.integers(-(1 << 31), (1 << 31) - 1, n0 * n1, dtype=np.int64).astype(np.int32)
    else:
        x = rng.integers(-(1 << 62), 1 << 62, n0 * n1, dtype=np.int64)
    mis = int(rng.integers(0, 16 // x.itemsize)) * x.itemsize
    levels = nests.c2_nest()
    V = int(rng.choice([1, 2, 4]))  # lane static(V), warp static(32 V) over the columns
    levels[-1].chunk, levels[-2].chunk = V, 32 * V
    if rng.random() < 0.5:  # the collapsed spelling: one warp..lane level static(V)
        levels = levels[:-2] + [H.Level(H.HPAR_WARP, H.HPAR_LANE, H.STATIC_CHUNK, loop=1, chunk=V)]
    res = run_nest(H, torch, levels, x, n0=n0, n1=n1, keyed=True, op=op, C=C, K=K, W=W, ld=ld, misalign=mis)
    assert res["kernel"] == "rowwise_tma_dsmem", (n0, n1, ld, K, W, V, dt, op)
    compare(oracle, H, levels, res, x, n0=n0, n1=n1, keyed=True, op=op, C=C, K=K, W=W)


@pytest.mark.parametrize("values", ["zeros_normal", "zeros_tiny", "subnormal_only", "zero_rows"])
def test_segmented_explicit_zeros(H, torch_mod, oracle, values):
    """Explicit zeros and subnormals in the CSR values (DESIGN reading on the
    C3 exactness guard): a window's min |v| is taken over all its values, so a
    zero counts as binade 0 — windows holding zeros among normal values take
    the in-order fp64 path, windows of zeros and values below 2^-106 (binades
    <= 20) stay on the exact prefix path.  Both must match the oracle's fp64
    segment sums within 1e-5, rows of zeros exactly 0."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    rng = np.random.default_rng(77)
    rows = 3000
    lens = np.where(rng.random(rows) < 0.02, rng.integers(4097, 20000, rows), rng.geometric(0.08, rows))
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    nnz = int(off[-1])
    v = gen.gen_f32(gen.SEED_C3, 0, nnz)
    zero = rng.random(nnz) < 0.3
    if values == "zeros_normal":
        v = np.where(zero, 0.0, v).astype(np.float32)
    elif values == "zeros_tiny":
        tiny = np.ldexp(rng.random(nnz) + 0.5, rng.integers(-150, -107, nnz)).astype(np.float32)
        v = np.where(zero, 0.0, tiny).astype(np.float32)
    elif values == "subnormal_only":
        v = (rng.integers(1, 1 << 23, nnz).astype(np.uint32)).view(np.float32).copy()
    else:  # every third row all zeros, the rest recipe values
        rz = np.repeat(np.arange(rows) % 3 == 0, lens)
        v = np.where(rz, 0.0, v).astype(np.float32)
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8, clusters=4)
    xd = torch.from_numpy(v).cuda()
    offd = torch.from_numpy(off).cuda()
    out = torch.full((rows,), -1.0, dtype=torch.float64, device="cuda")
    d = H.make_desc(xd, out, n0=rows, n1=nnz, nloops=2, keyed=True, offsets=offd, out_dtype=H.F64)
    nest.parallel_for_reduce(d)
    torch.cuda.synchronize()
    assert nest.last_kernel() == "segmented_csr"
    assert_rel(out.cpu().numpy(), oracle.segsum_f32(v, off))


def test_segmented_nest_reuse_shrinking_nnz(H, torch_mod, oracle):
    """One Nest called with a large CSR (long rows > 4096 nonzeros), then with
    smaller ones that still hold long rows, then the large one again: the
    segment workspace keeps the layout of its capacity, so tickets and the
    empty queue slots stay where the kernel looks."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    rng = np.random.default_rng(4242)
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8, clusters=6)

    def case(rows, p_long):
        lens = np.where(rng.random(rows) < p_long, rng.integers(4097, 60000, rows), rng.geometric(0.1, rows))
        off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        return off, gen.gen_f32(gen.SEED_C3, 0, int(off[-1]))

    cases = [case(4000, 0.02), case(600, 0.05), case(50, 0.2), case(4000, 0.02)]
    for off, v in cases + cases[::-1]:
        rows = off.size - 1
        out = torch.full((rows,), -1.0, dtype=torch.float64, device="cuda")
        d = H.make_desc(torch.from_numpy(v).cuda(), out, n0=rows, n1=v.size, nloops=2, keyed=True,
                        offsets=torch.from_numpy(off).cuda(), out_dtype=H.F64)
        nest.parallel_for_reduce(d)
        torch.cuda.synchronize()
        assert nest.last_kernel() == "segmented_csr"
        assert_rel(out.cpu().numpy(), oracle.segsum_f32(v, off))


def test_segrows_nest_reuse_shrinking_nnz(H, torch_mod, oracle):
    """The CSR rows kernel's workspace keeps the layout of its capacity too:
    one Nest, fp64 sums over a large CSR with long rows, smaller ones, and
    the large one again, interleaved with an int64 MAX call (another
    instantiation on the same workspace); every call vs the oracle."""
    from paper_2309_01906_b200 import nests
    from tests.nestutil import oracle_levels
    torch = torch_mod
    rng = np.random.default_rng(4243)
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8, clusters=6)
    ol = oracle_levels(oracle, nests.c3_nest(with_gpu=False, rows_chunk=16, width=8), 1, 2, 2, 4)

    def case(rows, p_long):
        lens = np.where(rng.random(rows) < p_long, rng.integers(4097, 60000, rows), rng.geometric(0.1, rows))
        return np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)

    offs = [case(4000, 0.02), case(600, 0.05), case(50, 0.2), case(4000, 0.02)]
    for k, off in enumerate(offs + offs[::-1]):
        rows, nnz = off.size - 1, int(off[-1])
        if k % 2 == 0:
            v, op, odt, tdt = rng.standard_normal(nnz), H.OP_SUM, H.F64, torch.float64
        else:
            v, op, odt, tdt = rng.integers(-(1 << 40), 1 << 40, nnz, dtype=np.int64), H.OP_MAX, H.I64, torch.int64
        out = torch.full((rows,), -1, dtype=tdt, device="cuda")
        d = H.make_desc(torch.from_numpy(v).cuda(), out, n0=rows, n1=nnz, nloops=2, keyed=True, op=op,
                        offsets=torch.from_numpy(off).cuda(), out_dtype=odt)
        nest.parallel_for_reduce(d)
        torch.cuda.synchronize()
        assert nest.last_kernel() == "segrows_csr"
        want = oracle.nest_run(ol, n0=rows, offsets=off, x=v, op=op, keyed=True, coverage=False,
                               partials=False).result
        if op == H.OP_SUM:
            assert_rel(out.cpu().numpy(), want)
        else:
            assert np.array_equal(out.cpu().numpy(), want)


def test_segmented_empty_caller_shard(H, torch_mod):
    """A caller-sharded CSR rank with no rows (local_n0 = 0 ->
    HPAR_LOCAL_N0_EMPTY) returns without a launch and writes nothing (ADVICE
    r01: it used to fall back to the static block of n0 rows)."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    nest = H.Nest(nests.c3_fast_nest(), device=0, rank=1, nranks=2, cluster_dim=2, warps_per_cta=8, clusters=2)
    off = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = torch.full((1,), -3.0, dtype=torch.float32, device="cuda")
    x = torch.zeros(4, dtype=torch.float32, device="cuda")
    nest.parallel_for_reduce(H.make_desc(x, out, n0=100, n1=0, nloops=2, keyed=True, offsets=off, local_n0=0))
    torch.cuda.synchronize()
    assert float(out.item()) == -3.0
    assert nest.last_kernel().startswith("none")


def test_hierarchy_query_cluster_num_is_occupancy(H, torch_mod):
    """P:139 num(c): the cluster level's num equals cudaOccupancyMaxActiveClusters
    for the flat kernel's launch shape (288 threads, a 64 KiB ring, clusters of
    2), cross-checked through the driver API on a stand-in kernel of the same
    footprint compiled here with NVRTC (cuda-python; nothing from libhpar)."""
    from cuda.bindings import driver as cu
    from cuda.bindings import nvrtc
    torch = torch_mod
    torch.cuda.init()
    t = H.hpar_hierarchy_query(0)
    src = b'extern "C" __global__ void standin(float* o) { extern __shared__ float s[]; ' \
          b'if (o) o[threadIdx.x] = s[threadIdx.x]; }'
    err, prog = nvrtc.nvrtcCreateProgram(src, b"standin.cu", 0, [], [])
    assert err == nvrtc.nvrtcResult.NVRTC_SUCCESS
    err, = nvrtc.nvrtcCompileProgram(prog, 1, [b"--gpu-architecture=sm_100a"])
    assert err == nvrtc.nvrtcResult.NVRTC_SUCCESS
    err, size = nvrtc.nvrtcGetCUBINSize(prog)
    cubin = b" " * size
    err, = nvrtc.nvrtcGetCUBIN(prog, cubin)
    assert err == nvrtc.nvrtcResult.NVRTC_SUCCESS
    err, = cu.cuInit(0)
    err, ctx = cu.cuDevicePrimaryCtxRetain(0)
    err, = cu.cuCtxSetCurrent(ctx)
    err, mod = cu.cuModuleLoadData(cubin)
    assert err == cu.CUresult.CUDA_SUCCESS, err
    err, fn = cu.cuModuleGetFunction(mod, b"standin")
    smem = 4 * 4096 * 4 + 256  # the ring + the kernel's static barriers / climb slots (< 1 KiB)
    err, = cu.cuFuncSetAttribute(fn, cu.CUfunction_attribute.CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem)
    cfg = cu.CUlaunchConfig()
    cfg.gridDimX, cfg.gridDimY, cfg.gridDimZ = 2, 1, 1
    cfg.blockDimX, cfg.blockDimY, cfg.blockDimZ = 9 * 32, 1, 1
    cfg.sharedMemBytes = smem
    attr = cu.CUlaunchAttribute()
    attr.id = cu.CUlaunchAttributeID.CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION
    attr.value.clusterDim.x, attr.value.clusterDim.y, attr.value.clusterDim.z = 2, 1, 1
    cfg.attrs = [attr]
    cfg.numAttrs = 1
    err, nclus = cu.cuOccupancyMaxActiveClusters(fn, cfg)
    assert err == cu.CUresult.CUDA_SUCCESS, err
    assert t[H.HPAR_CLUSTER].num == nclus
    assert t[H.HPAR_CTA].num == 2 and t[H.HPAR_WARP].num == 8
    # the default geometry of a nest is the same single wave
    from paper_2309_01906_b200 import nests
    assert H.Nest(nests.c5_nest(2), device=0, cluster_dim=2, warps_per_cta=8).info().C == nclus


def test_segmented_huge_values(H, torch_mod, oracle):
    """Values near FLT_MAX / 2^9: a window's fp32 segmented sums could
    overflow where fp64 does not, so windows holding a finite |v| >= 2^119
    take the in-order fp64 row loop (reading #24).  Rows of such values (sums
    above FLT_MAX, f64 output) beside rows of tiny and ordinary values,
    against the oracle's fp64 sums."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    rng = np.random.default_rng(119)
    rows = 2000
    lens = np.where(rng.random(rows) < 0.01, rng.integers(4097, 9000, rows), rng.integers(1, 700, rows))
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    nnz = int(off[-1])
    v = gen.gen_f32(gen.SEED_C3, 0, nnz)
    kind = rng.integers(0, 3, rows)
    scale = np.repeat(np.where(kind == 0, 1e37, np.where(kind == 1, 1e-30, 1.0)), lens)
    v = (v.astype(np.float64) * scale).astype(np.float32)
    assert np.isfinite(v).all()
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8, clusters=4)
    out = torch.full((rows,), -1.0, dtype=torch.float64, device="cuda")
    nest.parallel_for_reduce(H.make_desc(torch.from_numpy(v).cuda(), out, n0=rows, n1=nnz, nloops=2, keyed=True,
                                         offsets=torch.from_numpy(off).cuda(), out_dtype=H.F64))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "segmented_csr"
    want = oracle.segsum_f32(v, off)
    assert (want[kind == 0] > 3.5e38).any(), "the test needs row sums beyond FLT_MAX"
    assert_rel(out.cpu().numpy(), want)


def test_misaligned_fp32_inputs_not_rejected(H, torch_mod, oracle):
    """SURVEY §8(b) alignment: an fp32 input 4 bytes off a 16-byte boundary is
    never rejected — the flat and row-wise kernels copy enclosing granules
    (test_flat_misaligned_input, test_rowwise_ragged_rows); the CSR rows of
    the generic nest go to the interpreter (P:252 masked lanes) — flat
    total, dense rows and CSR rows, against the oracle."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    n = 4096 * 2 * 3 + 11
    x = gen.gen_f32(gen.SEED_C5, 0, n)
    raw = torch.zeros(n + 8, dtype=torch.float32, device="cuda")
    xd = raw[1:1 + n]
    xd.copy_(torch.from_numpy(x).cuda())
    assert xd.data_ptr() % 16 == 4
    tot = torch.zeros(1, dtype=torch.float64, device="cuda")
    nest = H.Nest(nests.c5_nest(2), device=0, cluster_dim=2, warps_per_cta=4, clusters=3)
    nest.parallel_for_reduce(H.make_desc(xd, tot, n0=n))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "flat_tma"
    assert_rel(tot.cpu().numpy(), [oracle.sum_f32(x)])
    rows, cols = 7, 4096
    a = gen.gen_f32(gen.SEED_C2, 0, rows * cols)
    raw = torch.zeros(rows * cols + 8, dtype=torch.float32, device="cuda")
    ad = raw[1:1 + rows * cols]
    ad.copy_(torch.from_numpy(a).cuda())
    out = torch.zeros(rows, dtype=torch.float64, device="cuda")
    nest = H.Nest(nests.c2_nest(), device=0, cluster_dim=2, warps_per_cta=4, clusters=3)
    nest.parallel_for_reduce(H.make_desc(ad, out, n0=rows, n1=cols, ld=cols, nloops=2, keyed=True, out_dtype=H.F64))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "rowwise_tma_dsmem"
    assert_rel(out.cpu().numpy(), oracle.rowsum_f32(a, rows, cols))
    off = gen.csr_offsets(300, 5000)
    v = gen.gen_f32(gen.SEED_C3, 0, 5000)
    raw = torch.zeros(5008, dtype=torch.float32, device="cuda")
    vd = raw[1:5001]
    vd.copy_(torch.from_numpy(v).cuda())
    out = torch.zeros(300, dtype=torch.float64, device="cuda")
    nest = H.Nest(nests.c3_nest(rows_chunk=16, width=8), device=0, cluster_dim=2, warps_per_cta=4, clusters=2)
    nest.parallel_for_reduce(H.make_desc(vd, out, n0=300, nloops=2, keyed=True, offsets=torch.from_numpy(off).cuda(),
                                         out_dtype=H.F64))
    torch.cuda.synchronize()
    assert_rel(out.cpu().numpy(), oracle.segsum_f32(v, off))


def test_rowwise_padded_rows(H, torch_mod, oracle):
    """Dense rows with a row stride larger than the row (ld > n1, 16-byte
    multiples): the fused row-wise kernel reads only the n1 columns of each
    row (the padding holds NaN, which would poison any row that read it);
    row sums against the oracle's."""
    from paper_2309_01906_b200 import nests
    torch = torch_mod
    levels = nests.c2_nest()
    for n0, n1, ld, C in ((37, 4096, 4096 + 64, 5), (11, 2048, 3000 + 4, 3)):
        a = gen.gen_f32(gen.SEED_C2, 0, n0 * ld).reshape(n0, ld)
        a[:, n1:] = np.float32(np.nan)  # the padding must never be read
        x = torch.from_numpy(a.ravel().copy()).cuda()
        out = torch.zeros(n0, dtype=torch.float64, device="cuda")
        nest = H.Nest(levels, device=0, cluster_dim=2, warps_per_cta=4, clusters=C)
        nest.parallel_for_reduce(H.make_desc(x, out, n0=n0, n1=n1, ld=ld, nloops=2, keyed=True, out_dtype=H.F64))
        torch.cuda.synchronize()
        assert nest.last_kernel() == "rowwise_tma_dsmem"
        assert_rel(out.cpu().numpy(), oracle.rowsum_f32(np.ascontiguousarray(a[:, :n1]), n0, n1))
