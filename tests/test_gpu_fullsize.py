"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (same nests, geometry and kernels):

  C2  65536 x 4096 fp32: every row vs the oracle's fp64 row sums
  C3  2^24 rows / 2^28 nonzeros: every row vs the oracle's segment sums
  C4  2^32 bytes: all bins vs the oracle's histogram of the whole input;
      coverage fingerprints (F_once, F_owner, count) vs the oracle's; cluster
      partials sum to the bins, sampled ones vs the oracle
  C5  2^34 fp32 (64 GiB): the total vs the oracle's exact sum; coverage
      fingerprints vs the oracle's; sampled cluster partials vs the oracle
  c6  16384^2 + ghost ring at the 128-byte pitch: two sweeps bit-exact vs
      the oracle's numpy steps over the whole array
Edge cases at their stated sizes: C4 with 2^32 equal bytes (bin 0 = 2^32,
beyond any u32 counter), C3 with one row of 2^26 nonzeros between empty rows,
C3 past 2^31 nonzeros per rank (sampled rows around position 2^31), C2 with
ragged rows (4095 columns) and C3 with fp64 values (the CSR rows kernel);
C3's coverage at full size (every one of 2^28 nonzeros visited once); the
8-byte flat path past 4 GiB of input (fp64 and int64, exact totals) and the
row-wise fp64 path past 4 GiB (rows equal to the oracle's exact sums); the CSR
rows kernel past 2^31 nonzeros (int32 sums, sampled rows).
The oracle runs range by range in a process pool (tests/fullsize_oracle.py:
every quantity is exact and additive over disjoint ranges).
Inputs come from the device generator, which is cross-checked bit for bit
against inputs/gen.py in test_gpu_parity.py."""
import ctypes
import os

import numpy as np
import pytest

from inputs import gen
from tests.nestutil import assert_rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2309_01906_b200 import build
    build.build()
    from paper_2309_01906_b200 import hpar as H
    from paper_2309_01906_b200 import nests
    L = ctypes.CDLL(os.path.join(os.path.dirname(gen.__file__), "libhpar_inputs.so"))
    for f in ("hpar_inputs_fill_f32", "hpar_inputs_fill_u8", "hpar_inputs_fill_i32"):
        getattr(L, f).argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    return torch, H, nests, L


def bench_geometry(config):
    """the tuned geometry bench.py uses (K, W, C)"""
    return {"c2": (2, 4, 444), "c4": (2, 8, 74), "c5": (2, 4, 148)}.get(config, (2, 8, 0))


def test_c2_full(env, oracle):
    torch, H, nests, L = env
    K, W, C = bench_geometry("c2")
    rows, cols = 65536, 4096
    nest = H.Nest(nests.c2_nest(), device=0, cluster_dim=K, warps_per_cta=W, clusters=C)
    x = torch.empty(rows * cols, dtype=torch.float32, device="cuda")
    L.hpar_inputs_fill_f32(gen.SEED_C2, 0, rows * cols, x.data_ptr(), None)
    out = torch.empty(rows, dtype=torch.float32, device="cuda")
    nest.parallel_for_reduce(H.make_desc(x, out, n0=rows, n1=cols, ld=cols, nloops=2, keyed=True))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "rowwise_tma_dsmem"
    a = gen.gen_f32(gen.SEED_C2, 0, rows * cols)
    assert_rel(out.cpu().numpy(), oracle.rowsum_f32(a, rows, cols))


def test_c3_full(env, oracle):
    torch, H, nests, L = env
    rows, nnz = 1 << 24, 1 << 28
    off = gen.csr_offsets(rows, nnz)
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8)
    x = torch.empty(nnz, dtype=torch.float32, device="cuda")
    L.hpar_inputs_fill_f32(gen.SEED_C3, 0, nnz, x.data_ptr(), None)
    offd = torch.from_numpy(off).cuda()
    out = torch.empty(rows, dtype=torch.float32, device="cuda")
    want = oracle.segsum_f32(gen.gen_f32(gen.SEED_C3, 0, nnz), off)
    for _ in range(2):  # second call exercises the self-reset of tickets and queues
        out.fill_(-1.0)
        nest.parallel_for_reduce(H.make_desc(x, out, n0=rows, n1=nnz, nloops=2, keyed=True, offsets=offd))
        torch.cuda.synchronize()
        assert nest.last_kernel() == "segmented_csr"
        assert_rel(out.cpu().numpy(), want)


def _cluster_tiles(c, C, K, tile, n):
    """global element ranges of cluster c under cluster static(K*tile)"""
    chunk = K * tile
    return [(b, min(b + chunk, n)) for b in range(c * chunk, n, C * chunk)]


def _flat_levels(C, K, W, tile, V):
    """the c4/c5 nest [GPU static, cluster static(K tile), CTA static(tile),
    warp static(32 V), lane static(V)] at G = 1, in the oracle's numbering"""
    return [(1, 0, 0), (C, 1, K * tile), (K, 1, tile), (W, 1, 32 * V), (32, 1, V)]


def test_c4_full(env, oracle):
    """C4 at 2^32 bytes in bench.py's timed launch (K, W, C) = (2, 8, 74):
    all 256 bins bit-exact against the oracle's histogram of the whole input;
    then a verify run of the same geometry: per-iteration coverage by
    fingerprints (F_once = every byte exactly once, F_owner = each byte's
    owner is the oracle's leaf for it, count = 2^32), cluster partials summing
    to the bins, sampled cluster partials against the oracle's bytes."""
    from tests import fullsize_oracle as F
    torch, H, nests, L = env
    K, W, C = bench_geometry("c4")
    n = 1 << 32
    tile = nests.TILE_U8
    nest = H.Nest(nests.c4_nest(K), device=0, cluster_dim=K, warps_per_cta=W, clusters=C)
    assert nest.info().C == C
    x = torch.empty(n, dtype=torch.uint8, device="cuda")
    L.hpar_inputs_fill_u8(gen.SEED_C4, 0, n, x.data_ptr(), None)
    out = torch.zeros(256, dtype=torch.int64, device="cuda")
    nest.parallel_for_reduce(H.make_desc(x, out, n0=n, op=H.OP_HIST256))
    torch.cuda.synchronize()
    assert nest.last_kernel().startswith("hist256_lanepriv")
    bins = out.cpu().numpy().astype(np.uint64)
    want = F.histogram(gen.SEED_C4, n)
    assert np.array_equal(bins, want)
    # verify run: fingerprints + cluster partials
    out.zero_()
    clus = torch.zeros((C, 256), dtype=torch.int64, device="cuda")
    fp = torch.zeros(3, dtype=torch.int64, device="cuda")
    parts = [None] * len(nest.levels)
    parts[1] = clus  # level 1 = the cluster level of c4_nest
    nest.parallel_for_reduce(H.make_desc(x, out, n0=n, op=H.OP_HIST256, verify=H.VERIFY_PARTIALS | H.VERIFY_FINGERPRINT,
                                         partials=parts, fingerprint=fp))
    torch.cuda.synchronize()
    assert nest.last_kernel().startswith("hist256_lanepriv")
    assert np.array_equal(out.cpu().numpy().astype(np.uint64), want)
    f = [int(v) for v in fp.cpu().numpy().view(np.uint64)]
    once, own = F.flat_fingerprints(_flat_levels(C, K, W, tile, 16), n)
    assert f[2] == n, "iterations executed"
    assert f[0] == once, "F_once: some byte missed or visited twice"
    assert f[1] == own, "F_owner: some byte executed by another leaf than the oracle's"
    cl = clus.cpu().numpy().astype(np.uint64)
    assert np.array_equal(cl.sum(axis=0), want)
    for c in (0, C // 2, C - 1):
        h = np.zeros(256, dtype=np.uint64)
        for b, e in _cluster_tiles(c, C, K, tile, n):
            h += oracle.hist256(gen.gen_u8(gen.SEED_C4, b, e - b))
        assert np.array_equal(cl[c], h), f"cluster {c}"


def test_c5_full(env, oracle):
    """C5 at 2^34 fp32 (64 GiB) in bench.py's timed launch: the total within
    1e-5 of the oracle's (the exact sum: every input is k 2^-24, so the
    oracle's Σk over the whole input, range by range, gives it exactly); a
    verify run of the same geometry: fingerprints (F_once, F_owner, count
    = 2^34) against the oracle's, sampled cluster partials against the
    oracle's sums of those clusters' elements, total = fold of the cluster
    partials."""
    from tests import fullsize_oracle as F
    torch, H, nests, L = env
    K, W, C = bench_geometry("c5")
    n = 1 << 34
    tile = nests.TILE_F32
    nest = H.Nest(nests.c5_nest(K), device=0, cluster_dim=K, warps_per_cta=W, clusters=C)
    C = nest.info().C  # bench's default: the resident clusters (a launch parameter, checked by F_owner)
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    L.hpar_inputs_fill_f32(gen.SEED_C5, 0, n, x.data_ptr(), None)
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    nest.parallel_for_reduce(H.make_desc(x, out, n0=n))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "flat_tma"
    tot = float(out.item())
    exact = F.exact_numerator_sum(gen.SEED_C5, n) * 2.0 ** -24
    assert_rel(np.array([tot]), np.array([exact]))
    # verify run
    out.zero_()
    clus = torch.zeros(C, dtype=torch.float64, device="cuda")
    fp = torch.zeros(3, dtype=torch.int64, device="cuda")
    parts = [None] * len(nest.levels)
    parts[1] = clus
    nest.parallel_for_reduce(H.make_desc(x, out, n0=n, verify=H.VERIFY_PARTIALS | H.VERIFY_FINGERPRINT,
                                         partials=parts, fingerprint=fp))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "flat_tma"
    f = [int(v) for v in fp.cpu().numpy().view(np.uint64)]
    once, own = F.flat_fingerprints(_flat_levels(C, K, W, tile, 4), n)
    assert f[2] == n, "iterations executed"
    assert f[0] == once, "F_once: some element missed or visited twice"
    assert f[1] == own, "F_owner: some element executed by another leaf than the oracle's"
    cl = clus.cpu().numpy()
    assert_rel(np.array([float(out.item())]), np.array([float(np.sum(cl))]), tol=1e-9)
    assert_rel(np.array([float(out.item())]), np.array([exact]))
    for c in (0, C - 1):
        s = 0
        for b, e in _cluster_tiles(c, C, K, tile, n):
            s += oracle.sum_u64(gen.gen_f32_k(gen.SEED_C5, b, e - b))
        assert_rel(np.array([cl[c]]), np.array([s * 2.0 ** -24]))
    del x
    torch.cuda.empty_cache()


def test_c6_full(env):
    """c6 (NEXT f3) at bench.py's size and layout: one sibling's 16384^2
    from-section with its 1-cell ghost ring, rows at the 128-byte pitch
    (ld = 16416), one Jacobi sweep through hpar_stencil5 — bit-exact against
    the oracle's numpy step over the whole (16384+2)^2 array, two steps
    (ping-pong, as timed) likewise."""
    from oracle import ghostmap as G
    torch, H, nests, L = env
    tile = 16384
    ld = (tile + 2 + 31) // 32 * 32
    extent = (tile + 2, tile + 2)
    mspec = H.map_spec(extent, 1, 1, [(tile, 0, tile + 2), (tile, 0, tile + 2)], [(tile, 1, tile), (tile, 1, tile)])
    H.hpar_map_validate(mspec)
    to, fr = H.hpar_map_sections(mspec, 0)
    nest = H.Nest(nests.stencil_nest(), device=0)
    x = torch.empty((tile + 2, ld), dtype=torch.float32, device="cuda")
    L.hpar_inputs_fill_f32(gen.SEED_C5, 0, x.numel(), x.data_ptr(), None)
    out = x.clone()
    A = x[:, :tile + 2].cpu().numpy()
    want = G.stencil5_step(A)
    H.hpar_stencil5(nest, H.stencil_desc(x, out, ld, to, fr, extent))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "stencil5_tma"
    assert np.array_equal(out[:, :tile + 2].cpu().numpy(), want)
    H.hpar_stencil5(nest, H.stencil_desc(out, x, ld, to, fr, extent))
    torch.cuda.synchronize()
    assert np.array_equal(x[:, :tile + 2].cpu().numpy(), G.stencil5_step(want))


def test_c4_full_all_zero(env):
    """C4's degenerate skew at full size (SURVEY §8(d) skew variants): 2^32
    equal bytes — every increment lands in bin 0, so bin 0 = 2^32 exactly,
    which no u32 counter could hold (reading #8: lane / warp / CTA counters
    stay below 2^32 per task, cluster and GPU bins are u64)."""
    torch, H, nests, L = env
    K, W, C = bench_geometry("c4")
    n = 1 << 32
    nest = H.Nest(nests.c4_nest(K), device=0, cluster_dim=K, warps_per_cta=W, clusters=C)
    x = torch.zeros(n, dtype=torch.uint8, device="cuda")
    out = torch.zeros(256, dtype=torch.int64, device="cuda")
    nest.parallel_for_reduce(H.make_desc(x, out, n0=n, op=H.OP_HIST256))
    torch.cuda.synchronize()
    bins = out.cpu().numpy().astype(np.uint64)
    assert int(bins[0]) == n and int(bins[1:].sum()) == 0


def test_c3_single_huge_row(env, oracle):
    """C3's edge case at its stated size: one row of 2^26
    nonzeros (split into 4096 long-row segments, folded in ascending order by
    the last one) between empty rows, against the oracle's exact sum (the
    values are k 2^-24, so the oracle's integer numerator sum is exact)."""
    torch, H, nests, L = env
    nnz = 1 << 26
    off = np.array([0, 0, nnz, nnz, nnz], dtype=np.int64)  # empty, the huge row, two empty
    x = torch.empty(nnz, dtype=torch.float32, device="cuda")
    L.hpar_inputs_fill_f32(gen.SEED_C3, 0, nnz, x.data_ptr(), None)
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8)
    out = torch.full((4,), -1.0, dtype=torch.float64, device="cuda")
    nest.parallel_for_reduce(H.make_desc(x, out, n0=4, n1=nnz, nloops=2, keyed=True,
                                         offsets=torch.from_numpy(off).cuda(), out_dtype=H.F64))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "segmented_csr"
    got = out.cpu().numpy()
    exact = oracle.sum_u64(gen.gen_f32_k(gen.SEED_C3, 0, nnz)) * 2.0 ** -24
    assert got[0] == 0 and got[2] == 0 and got[3] == 0
    assert_rel(got[1:2], np.array([exact]))


def test_c3_beyond_2e31_nonzeros(env, oracle):
    """C3 past 32-bit sizes (the 180 GB HBM budget allows ~4e10 fp32
    nonzeros per GPU): 2^23 zipf rows (the longest 1.8e7 nonzeros) over
    2^31 + 49383 nonzeros.  Positions inside a 256-row block stay 32-bit;
    the launch proves every block spans < 2^31 (the block-span check, no
    max_inner given).  Sampled rows — those around positions 2^31 and 2^32 /
    the array end, the longest, random ones — vs the oracle's segment sums;
    the sum of all rows vs the oracle's exact total."""
    torch, H, nests, L = env
    from tests import fullsize_oracle as F
    rows, nnz = 1 << 23, (1 << 31) + 4 * 12345 + 3
    off = gen.csr_offsets(rows, nnz)
    assert int(off[-1]) == nnz
    lens = np.diff(off)
    x = torch.empty(nnz, dtype=torch.float32, device="cuda")
    L.hpar_inputs_fill_f32(gen.SEED_C3, 0, nnz, x.data_ptr(), None)
    offd = torch.from_numpy(off).cuda()
    out = torch.full((rows,), -1.0, dtype=torch.float64, device="cuda")
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8)
    d = H.make_desc(x, out, n0=rows, n1=nnz, nloops=2, keyed=True, offsets=offd, out_dtype=H.F64)
    for _ in range(2):
        out.fill_(-1.0)
        nest.parallel_for_reduce(d)
        torch.cuda.synchronize()
        assert nest.last_kernel() == "segmented_csr"
    got = out.cpu().numpy()
    r31 = int(np.searchsorted(off, 1 << 31, side="right")) - 1  # the row holding position 2^31
    rng = np.random.default_rng(5)
    sample = set(range(max(0, r31 - 300), min(rows, r31 + 300))) | set(range(rows - 300, rows))
    sample |= set(np.argsort(lens)[-8:].tolist()) | set(rng.integers(0, rows, 500).tolist())
    for r in sorted(sample):
        b, n = int(off[r]), int(lens[r])
        want = oracle.segsum_f32(gen.gen_f32(gen.SEED_C3, b, n), np.array([0, n], dtype=np.int64))
        assert_rel(got[r:r + 1], want)
    exact = F.exact_numerator_sum(gen.SEED_C3, nnz) * 2.0 ** -24
    assert abs(got.sum() - exact) <= 1e-9 * exact


def test_c2_full_ragged_rows(env, oracle):
    """C2's matrix with ragged rows at full size: 65536 x 4095 at ld 4095
    (every row starts at a different offset inside a 16-byte granule) on the
    fused row-wise kernel in bench.py's geometry; every row vs the oracle."""
    torch, H, nests, L = env
    K, W, C = bench_geometry("c2")
    rows, cols = 65536, 4095
    nest = H.Nest(nests.c2_nest(), device=0, cluster_dim=K, warps_per_cta=W, clusters=C)
    x = torch.empty(rows * cols, dtype=torch.float32, device="cuda")
    L.hpar_inputs_fill_f32(gen.SEED_C2, 0, rows * cols, x.data_ptr(), None)
    out = torch.empty(rows, dtype=torch.float32, device="cuda")
    nest.parallel_for_reduce(H.make_desc(x, out, n0=rows, n1=cols, ld=cols, nloops=2, keyed=True))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "rowwise_tma_dsmem"
    assert_rel(out.cpu().numpy(), oracle.rowsum_f32(gen.gen_f32(gen.SEED_C2, 0, rows * cols), rows, cols))


def test_c3_full_fp64_values(env, oracle):
    """C3's matrix (2^24 rows, 2^28 nonzeros, the longest row 1.8e7) with
    fp64 values on the CSR rows kernel: the values are the fp32 inputs
    widened exactly, so every row vs the oracle's fp64 segment sums of the
    same numbers; a second call checks the self-resetting chunk tickets."""
    torch, H, nests, L = env
    rows, nnz = 1 << 24, 1 << 28
    off = gen.csr_offsets(rows, nnz)
    v32 = gen.gen_f32(gen.SEED_C3, 0, nnz)
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8)
    x = torch.from_numpy(v32).cuda().double()
    offd = torch.from_numpy(off).cuda()
    out = torch.empty(rows, dtype=torch.float64, device="cuda")
    want = oracle.segsum_f32(v32, off)
    for _ in range(2):
        out.fill_(-1.0)
        nest.parallel_for_reduce(H.make_desc(x, out, n0=rows, n1=nnz, nloops=2, keyed=True, offsets=offd,
                                             out_dtype=H.F64))
        torch.cuda.synchronize()
        assert nest.last_kernel() == "segrows_csr"
        assert_rel(out.cpu().numpy(), want)


def test_c3_full_coverage(env):
    """C3 at full size with the coverage outputs (§8(c) "no loss, no
    duplication" at 2^28 iterations): every nonzero visited exactly once,
    owners valid leaf ids, and each sampled block's short rows on one warp
    (the dynamic(256) row blocks are warp tasks; reading #14)."""
    torch, H, nests, L = env
    rows, nnz = 1 << 24, 1 << 28
    off = gen.csr_offsets(rows, nnz)
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8)
    x = torch.empty(nnz, dtype=torch.float32, device="cuda")
    L.hpar_inputs_fill_f32(gen.SEED_C3, 0, nnz, x.data_ptr(), None)
    offd = torch.from_numpy(off).cuda()
    out = torch.empty(rows, dtype=torch.float32, device="cuda")
    owner = torch.full((nnz,), -1, dtype=torch.int64, device="cuda")
    count = torch.zeros(nnz, dtype=torch.int32, device="cuda")
    nest.parallel_for_reduce(H.make_desc(x, out, n0=rows, n1=nnz, nloops=2, keyed=True, offsets=offd,
                                         verify=H.VERIFY_COVERAGE, owner=owner, count=count))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "segmented_csr"
    assert int((count != 1).sum().item()) == 0, "a nonzero visited zero or several times"
    threads = int(nest.info().threads_per_gpu)
    own = owner.cpu().numpy()
    assert own.min() >= 0 and own.max() < threads
    lens = np.diff(off)
    rng = np.random.default_rng(8)
    for b0 in rng.integers(0, rows // 256, 400) * 256:
        rs = [r for r in range(b0, b0 + 256) if 0 < lens[r] <= 4096]
        if rs:
            w = np.concatenate([own[off[r]:off[r + 1]] for r in rs]) // 32
            assert (w == w[0]).all(), f"block {b0}: short rows on several warps"


def test_flat_fp64_and_int64_past_4gib(env, oracle):
    """The 8-byte flat path past 32-bit BYTE offsets: 2^30 + 12345 fp64
    (8.6 GB) — C5's fp32 inputs widened exactly, so the oracle's exact
    Σk 2^-24 is the total — and the same count of int64 (their numerators
    k), whose sum is exact; bench.py's C5 geometry; also 8 bytes off a
    granule."""
    from tests import fullsize_oracle as F
    torch, H, nests, L = env
    K, W, C = bench_geometry("c5")
    n = (1 << 30) + 12345
    nest = H.Nest(nests.c5_nest(K), device=0, cluster_dim=K, warps_per_cta=W, clusters=C)
    x32 = torch.empty(n, dtype=torch.float32, device="cuda")
    L.hpar_inputs_fill_f32(gen.SEED_C5, 0, n, x32.data_ptr(), None)
    ksum = F.exact_numerator_sum(gen.SEED_C5, n)
    raw = torch.empty(n + 2, dtype=torch.float64, device="cuda")
    for off in (0, 1):
        x = raw[off:off + n]
        x.copy_(x32)
        out = torch.zeros(1, dtype=torch.float64, device="cuda")
        nest.parallel_for_reduce(H.make_desc(x, out, n0=n))
        torch.cuda.synchronize()
        assert nest.last_kernel() == "flat_tma"
        assert_rel(out.cpu().numpy(), np.array([ksum * 2.0 ** -24]), tol=1e-12)
    del raw
    xi = (x32.double() * float(1 << 24)).long()
    del x32
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    nest.parallel_for_reduce(H.make_desc(xi, out, n0=n))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "flat_tma"
    assert int(out.item()) == ksum


def test_rowwise_fp64_past_4gib(env, oracle):
    """The row-wise kernel's 64-bit partial path past 4 GiB of input:
    150000 x 4096 fp64 rows (4.9 GB) holding C2's fp32 values widened
    exactly; every row sum is exact in fp64 (36 significant bits), so the
    rows must EQUAL the oracle's fp64 row sums of the same numbers."""
    torch, H, nests, L = env
    K, W, C = bench_geometry("c2")
    rows, cols = 150000, 4096
    nest = H.Nest(nests.c2_nest(), device=0, cluster_dim=K, warps_per_cta=W, clusters=C)
    x32 = torch.empty(rows * cols, dtype=torch.float32, device="cuda")
    L.hpar_inputs_fill_f32(gen.SEED_C2, 0, rows * cols, x32.data_ptr(), None)
    x = x32.double()
    del x32
    out = torch.empty(rows, dtype=torch.float64, device="cuda")
    nest.parallel_for_reduce(H.make_desc(x, out, n0=rows, n1=cols, ld=cols, nloops=2, keyed=True, out_dtype=H.F64))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "rowwise_tma_dsmem"
    want = oracle.rowsum_f32(gen.gen_f32(gen.SEED_C2, 0, rows * cols), rows, cols)
    assert np.array_equal(out.cpu().numpy(), want)


def test_segrows_beyond_2e31_nonzeros(env, oracle):
    """The CSR rows kernel past 2^31 nonzeros (its positions are 64-bit
    outside a window): 2^23 zipf rows over 2^31 + 12345 int32 values, SUM
    into int64 rows (exact).  Sampled rows — around position 2^31, the
    longest, the last, random ones — vs the oracle's nest walk of each row."""
    from tests.nestutil import oracle_levels
    torch, H, nests, L = env
    rows, nnz = 1 << 23, (1 << 31) + 12345
    off = gen.csr_offsets(rows, nnz)
    lens = np.diff(off)
    x = torch.empty(nnz, dtype=torch.int32, device="cuda")
    L.hpar_inputs_fill_i32(gen.SEED_C1, 0, nnz, x.data_ptr(), None)
    out = torch.full((rows,), -1, dtype=torch.int64, device="cuda")
    nest = H.Nest(nests.c3_fast_nest(), device=0, cluster_dim=2, warps_per_cta=8)
    nest.parallel_for_reduce(H.make_desc(x, out, n0=rows, n1=nnz, nloops=2, keyed=True,
                                         offsets=torch.from_numpy(off).cuda(), out_dtype=H.I64))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "segrows_csr"
    got = out.cpu().numpy()
    ol = oracle_levels(oracle, nests.c3_nest(with_gpu=False, rows_chunk=16, width=8), 1, 1, 1, 1)
    r31 = int(np.searchsorted(off, 1 << 31, side="right")) - 1
    rng = np.random.default_rng(6)
    sample = set(range(max(0, r31 - 200), min(rows, r31 + 200))) | set(range(rows - 200, rows))
    sample |= set(np.argsort(lens)[-4:].tolist()) | set(rng.integers(0, rows, 300).tolist())
    for r in sorted(sample):
        b, n = int(off[r]), int(lens[r])
        v = gen.gen_i32(gen.SEED_C1, b, n)
        want = oracle.nest_run(ol, n0=1, offsets=np.array([0, n], dtype=np.int64), x=v, keyed=True,
                               coverage=False, partials=False).result
        assert int(got[r]) == int(want[0]), r
