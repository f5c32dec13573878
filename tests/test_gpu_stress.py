"""Repetition stress for the synchronisation-heavy kernels (a stand-in for
the racecheck run the pool does not allow, profiles/r02_sanitizer.md): each
fused kernel runs many back-to-back calls on mid-size inputs; every call's
result must be BITWISE identical to the first (all combine trees are
ordered and the dynamic schedules' results do not depend on the claim
order) and equal to the oracle.  A race in a ticket, a queue publication, an
mbarrier phase or a self-reset would show up as a differing call."""
import numpy as np
import pytest

from inputs import gen
from tests.nestutil import assert_rel

pytestmark = pytest.mark.gpu
REPS = 60


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2309_01906_b200 import build
    build.build()
    from paper_2309_01906_b200 import hpar as H
    from paper_2309_01906_b200 import nests
    return torch, H, nests


def _repeat(torch, nest, desc, out):
    outs = []
    for _ in range(REPS):
        out.fill_(-5)
        nest.parallel_for_reduce(desc)
        outs.append(out.clone())
    torch.cuda.synchronize()
    first = outs[0].cpu().numpy()
    for k, o in enumerate(outs[1:], 1):
        assert np.array_equal(o.cpu().numpy().view(np.uint8), first.view(np.uint8)), f"call {k} differs"
    return first


def test_stress_segmented(env, oracle):
    torch, H, nests = env
    rng = np.random.default_rng(9)
    rows = 30000
    lens = np.where(rng.random(rows) < 0.003, rng.integers(4097, 60000, rows), rng.geometric(0.07, rows))
    lens[::11] = 0
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    v = gen.gen_f32(gen.SEED_C3, 0, int(off[-1]))
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8)
    x, o = torch.from_numpy(v).cuda(), torch.from_numpy(off).cuda()
    out = torch.empty(rows, dtype=torch.float64, device="cuda")
    d = H.make_desc(x, out, n0=rows, n1=v.size, nloops=2, keyed=True, offsets=o, out_dtype=H.F64)
    assert_rel(_repeat(torch, nest, d, out), oracle.segsum_f32(v, off))
    assert nest.last_kernel() == "segmented_csr"


def test_stress_segrows(env, oracle):
    """The CSR rows kernel for other ops / dtypes: fp64 sums with long rows
    (chunk list, last-chunk ordered fold, self-resetting tickets) bitwise
    identical over repeated calls and equal to the oracle."""
    torch, H, nests = env
    from tests.nestutil import oracle_levels
    rng = np.random.default_rng(19)
    rows = 20000
    lens = np.where(rng.random(rows) < 0.004, rng.integers(4097, 80000, rows), rng.geometric(0.07, rows))
    lens[::13] = 0
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    v = rng.standard_normal(int(off[-1])) + 1.0
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8)
    x, o = torch.from_numpy(v).cuda(), torch.from_numpy(off).cuda()
    out = torch.empty(rows, dtype=torch.float64, device="cuda")
    d = H.make_desc(x, out, n0=rows, n1=v.size, nloops=2, keyed=True, offsets=o, out_dtype=H.F64)
    got = _repeat(torch, nest, d, out)
    assert nest.last_kernel() == "segrows_csr"
    ol = oracle_levels(oracle, nests.c3_nest(with_gpu=False, rows_chunk=16, width=8), 1, 2, 2, 4)
    assert_rel(got, oracle.nest_run(ol, n0=rows, offsets=off, x=v, keyed=True, coverage=False,
                                    partials=False).result)


def test_stress_rowwise(env, oracle):
    torch, H, nests = env
    rows, cols = 3000, 4096
    a = gen.gen_f32(gen.SEED_C2, 0, rows * cols)
    nest = H.Nest(nests.c2_nest(), device=0, cluster_dim=2, warps_per_cta=4, clusters=444)
    x = torch.from_numpy(a).cuda()
    out = torch.empty(rows, dtype=torch.float32, device="cuda")
    d = H.make_desc(x, out, n0=rows, n1=cols, ld=cols, nloops=2, keyed=True)
    assert_rel(_repeat(torch, nest, d, out), oracle.rowsum_f32(a, rows, cols))
    assert nest.last_kernel() == "rowwise_tma_dsmem"


def test_stress_hist_and_flat(env, oracle):
    torch, H, nests = env
    n = (1 << 24) + 333
    b = gen.gen_u8_zipf(gen.SEED_C4, 0, n)
    nest = H.Nest(nests.c4_nest(2), device=0, cluster_dim=2, warps_per_cta=8, clusters=74)
    xb = torch.from_numpy(b).cuda()
    out = torch.empty(256, dtype=torch.int64, device="cuda")
    got = _repeat(torch, nest, H.make_desc(xb, out, n0=n, op=H.OP_HIST256), out)
    assert np.array_equal(got.astype(np.uint64), oracle.hist256(b))
    f = gen.gen_f32(gen.SEED_C5, 0, n)
    nest = H.Nest(nests.c5_nest(2), device=0, cluster_dim=2, warps_per_cta=4, clusters=148)
    xf = torch.from_numpy(f).cuda()
    tot = torch.empty(1, dtype=torch.float64, device="cuda")
    got = _repeat(torch, nest, H.make_desc(xf, tot, n0=n), tot)
    assert_rel(got, [oracle.sum_f32(f)])


def test_stress_teams_and_generic(env, oracle):
    torch, H, nests = env
    xi = gen.gen_i32(gen.SEED_C1, 0, 1 << 20)
    nest = H.Nest(nests.c1_nest(outer=0), device=0, cluster_dim=2, warps_per_cta=8, clusters=148)
    x = torch.from_numpy(xi).cuda()
    out = torch.empty(1, dtype=torch.int64, device="cuda")
    got = _repeat(torch, nest, H.make_desc(x, out, n0=1024, n1=1024, ld=1024, nloops=2), out)
    assert int(got[0]) == oracle.sum_i32(xi)
    assert nest.last_kernel() == "teams_threads"
    # generic interpreter with a dynamic level (tickets self-reset every call)
    levels = [H.Level(H.HPAR_CLUSTER, H.HPAR_CTA, H.DYNAMIC, chunk=37), H.Level(H.HPAR_WARP, H.HPAR_LANE, 1, chunk=1)]
    nest = H.Nest(levels, device=0, cluster_dim=2, warps_per_cta=4, clusters=5)
    xs = gen.gen_i32(21, 0, 50000)
    x = torch.from_numpy(xs).cuda()
    got = _repeat(torch, nest, H.make_desc(x, out, n0=xs.size), out)
    assert int(got[0]) == oracle.sum_i32(xs)
