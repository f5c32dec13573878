"""Out-of-bounds evidence without compute-sanitizer (closed on this pool:
profiles/r02_sanitizer.md).  Every kernel family runs on inputs and outputs
embedded in larger device buffers whose margins hold canaries:

* inputs are followed AND preceded by poison (NaN for fp32, 0xFF bytes for
  the histogram, huge ints for int32): a read past either end that reaches
  the result turns it into NaN / changes bin 255 / the int sum, which the
  oracle comparison catches;
* outputs, per-level partials, coverage owner / count and fingerprints sit
  between canary words that must be unchanged after the call (a write past
  either end is caught directly).

Sizes span several tiles with ragged tails; results are compared with the
oracle as in the parity tests."""
import numpy as np
import pytest

from inputs import gen
from tests.nestutil import assert_rel

pytestmark = pytest.mark.gpu
PAD = 4096  # elements of margin on each side


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


def poisoned_input(torch, x: np.ndarray, shift: int = 0):
    """x on the device with PAD (+ shift) poison elements before it and PAD
    after it (shift > 0: x starts off a 16-byte boundary)"""
    if x.dtype == np.float32:
        poison = np.float32(np.nan)
    elif x.dtype == np.uint8:
        poison = np.uint8(0xFF)
    elif x.dtype == np.int64:
        poison = np.int64(0x5A5A5A5A5A5A5A5A)
    else:
        poison = np.int32(0x7FFFFF00)
    buf = np.full(x.size + 2 * PAD + shift, poison, dtype=x.dtype)
    buf[PAD + shift:PAD + shift + x.size] = x
    d = torch.from_numpy(buf).cuda()
    return d, d[PAD + shift:PAD + shift + x.size]


class Canaried:
    """a device tensor of `shape`/dtype between two canary margins"""

    def __init__(self, torch, shape, dtype, fill=0):
        n = int(np.prod(shape)) if shape else 1
        self.n = n
        self.buf = torch.full((n + 2 * PAD,), 0, dtype=dtype, device="cuda")
        self.buf.view(torch.int8 if self.buf.element_size() == 1 else torch.int32)[:].fill_(-0x5B if self.buf.element_size() == 1 else 0x5B5B5B5B)
        self.ref = self.buf.clone()
        self.t = self.buf[PAD:PAD + n].view(*shape) if shape else self.buf[PAD:PAD + 1]
        self.t.fill_(fill)

    def check(self, torch):
        head = torch.equal(self.buf[:PAD], self.ref[:PAD])
        tail = torch.equal(self.buf[PAD + self.n:], self.ref[PAD + self.n:])
        assert head and tail, f"canary overwritten (head ok: {head}, tail ok: {tail})"


def test_flat_and_teams_bounds(env, oracle):
    torch, H, nests = env
    n = 4096 * 2 * 7 + 4 * 99 + 3
    x = gen.gen_f32(gen.SEED_C5, 0, n)
    _, xd = poisoned_input(torch, x)
    nest = H.Nest(nests.c5_nest(2), device=0, cluster_dim=2, warps_per_cta=8, clusters=5)
    out = Canaried(torch, (1,), torch.float64)
    clus = Canaried(torch, (5,), torch.float64)
    owner = Canaried(torch, (n,), torch.int64, fill=-1)
    count = Canaried(torch, (n,), torch.int32)
    fp = Canaried(torch, (3,), torch.int64)
    parts = [None, clus.t, None, None, None]
    nest.parallel_for_reduce(H.make_desc(xd, out.t, n0=n, verify=H.VERIFY_PARTIALS | H.VERIFY_COVERAGE |
                                         H.VERIFY_FINGERPRINT, partials=parts, owner=owner.t, count=count.t,
                                         fingerprint=fp.t))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "flat_tma"
    for c in (out, clus, owner, count, fp):
        c.check(torch)
    assert_rel(out.t.cpu().numpy(), [oracle.sum_f32(x)])
    assert (count.t.cpu().numpy() == 1).all()
    # teams (C1 shape, 64 rows)
    xi = gen.gen_i32(gen.SEED_C1, 0, 64 * 1024)
    _, xid = poisoned_input(torch, xi)
    nest = H.Nest(nests.c1_nest(outer=64), device=0, cluster_dim=2, warps_per_cta=8)
    out = Canaried(torch, (1,), torch.int64)
    nest.parallel_for_reduce(H.make_desc(xid, out.t, n0=64, n1=1024, ld=1024, nloops=2))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "teams_threads"
    out.check(torch)
    assert int(out.t.item()) == oracle.sum_i32(xi)


def test_rowwise_bounds(env, oracle):
    torch, H, nests = env
    for rows, cols in ((37, 4096), (5, 1000), (11, 1003), (3, 5)):  # the last two: ragged (granule) copies
        a = gen.gen_f32(gen.SEED_C2, 0, rows * cols)
        _, ad = poisoned_input(torch, a)
        nest = H.Nest(nests.c2_nest(), device=0, cluster_dim=2, warps_per_cta=4, clusters=7)
        out = Canaried(torch, (rows,), torch.float32)
        nest.parallel_for_reduce(H.make_desc(ad, out.t, n0=rows, n1=cols, ld=cols, nloops=2, keyed=True))
        torch.cuda.synchronize()
        assert nest.last_kernel() == "rowwise_tma_dsmem"
        out.check(torch)
        assert_rel(out.t.cpu().numpy(), oracle.rowsum_f32(a, rows, cols))


@pytest.mark.parametrize("W", [4, 8])
def test_hist_bounds(env, oracle, W):
    torch, H, nests = env
    n = 16384 * 2 * 5 + 777
    x = gen.gen_u8(gen.SEED_C4, 0, n)
    _, xd = poisoned_input(torch, x)
    nest = H.Nest(nests.c4_nest(2), device=0, cluster_dim=2, warps_per_cta=W, clusters=3)
    out = Canaried(torch, (256,), torch.int64)
    clus = Canaried(torch, (3, 256), torch.int64)
    fp = Canaried(torch, (3,), torch.int64)
    parts = [None, clus.t, None, None, None]
    nest.parallel_for_reduce(H.make_desc(xd, out.t, n0=n, op=H.OP_HIST256, verify=H.VERIFY_PARTIALS |
                                         H.VERIFY_FINGERPRINT, partials=parts, fingerprint=fp.t))
    torch.cuda.synchronize()
    for c in (out, clus, fp):
        c.check(torch)
    assert np.array_equal(out.t.cpu().numpy().astype(np.uint64), oracle.hist256(x))


def test_segmented_bounds(env, oracle):
    torch, H, nests = env
    rng = np.random.default_rng(31)
    rows = 900
    lens = np.where(rng.random(rows) < 0.01, rng.integers(4097, 30000, rows), rng.geometric(0.1, rows))
    lens[::37] = 0
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    nnz = int(off[-1])
    v = gen.gen_f32(gen.SEED_C3, 0, nnz)
    offd = torch.from_numpy(off).cuda()  # offsets are not poisoned: a wild offset could hang the box
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8, clusters=3)
    for dt, shift in ((torch.float32, 0), (torch.float64, 0), (torch.float32, 1), (torch.float64, 3)):
        _, vd = poisoned_input(torch, v, shift)  # shift: values 4 / 12 bytes off a granule
        out = Canaried(torch, (rows,), dt)
        owner = Canaried(torch, (nnz,), torch.int64, fill=-1)
        count = Canaried(torch, (nnz,), torch.int32)
        nest.parallel_for_reduce(H.make_desc(vd, out.t, n0=rows, n1=nnz, nloops=2, keyed=True, offsets=offd,
                                             verify=H.VERIFY_COVERAGE, owner=owner.t, count=count.t))
        torch.cuda.synchronize()
        assert nest.last_kernel() == "segmented_csr"
        for c in (out, owner, count):
            c.check(torch)
        assert_rel(out.t.cpu().numpy(), oracle.segsum_f32(v, off))
        assert (count.t.cpu().numpy() == 1).all()


def test_segrows_bounds(env, oracle):
    """The CSR rows kernel for other ops / dtypes (kernel_segrows.cu): fp64
    values between poison (NaN) margins, also 8 bytes off a granule, rows
    and coverage between canaries; long rows through the chunk list."""
    torch, H, nests = env
    rng = np.random.default_rng(41)
    rows = 700
    lens = np.where(rng.random(rows) < 0.01, rng.integers(4097, 40000, rows), rng.geometric(0.1, rows))
    lens[::29] = 0
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    nnz = int(off[-1])
    v = rng.standard_normal(nnz) + 2.0
    offd = torch.from_numpy(off).cuda()
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8, clusters=3)
    for shift, op in ((0, H.OP_SUM), (1, H.OP_MIN), (1, H.OP_SUM)):
        _, vd = poisoned_input(torch, v, shift)
        out = Canaried(torch, (rows,), torch.float64)
        owner = Canaried(torch, (nnz,), torch.int64, fill=-1)
        count = Canaried(torch, (nnz,), torch.int32)
        nest.parallel_for_reduce(H.make_desc(vd, out.t, n0=rows, n1=nnz, nloops=2, keyed=True, offsets=offd, op=op,
                                             out_dtype=H.F64, verify=H.VERIFY_COVERAGE, owner=owner.t,
                                             count=count.t))
        torch.cuda.synchronize()
        assert nest.last_kernel() == "segrows_csr"
        for c in (out, owner, count):
            c.check(torch)
        got = out.t.cpu().numpy()
        if op == H.OP_SUM:
            assert_rel(got, oracle.nest_run(_c3_oracle_levels(oracle, nests), n0=rows, offsets=off, x=v, op=op,
                                            keyed=True, coverage=False, partials=False).result)
        else:
            assert np.array_equal(got, oracle.nest_run(_c3_oracle_levels(oracle, nests), n0=rows, offsets=off, x=v,
                                                       op=op, keyed=True, coverage=False, partials=False).result)
        assert (count.t.cpu().numpy() == 1).all()


def _c3_oracle_levels(oracle, nests):
    from tests.nestutil import oracle_levels
    return oracle_levels(oracle, nests.c3_nest(with_gpu=False, rows_chunk=16, width=8), 1, 2, 2, 4)


def test_generic_bounds(env, oracle):
    torch, H, nests = env
    off = gen.csr_offsets(300, 4000)
    v = gen.gen_f32(gen.SEED_C3, 0, 4000)
    _, vd = poisoned_input(torch, v)
    offd = torch.from_numpy(off).cuda()
    nest = H.Nest(nests.c3_nest(rows_chunk=16, width=8), device=0, cluster_dim=2, warps_per_cta=4, clusters=2)
    out = Canaried(torch, (300,), torch.float64)
    nest.parallel_for_reduce(H.make_desc(vd, out.t, n0=300, nloops=2, keyed=True, offsets=offd, out_dtype=H.F64))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "generic"
    out.check(torch)
    assert_rel(out.t.cpu().numpy(), oracle.segsum_f32(v, off))
