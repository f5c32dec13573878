"""NEXT f3 on the GPU: the 5-point stencil kernel (kernel_stencil.cu) and
the §4 device-level ghost maps, bit-exact against oracle/ghostmap.py."""
import os

import numpy as np
import pytest

from inputs import gen
from oracle import ghostmap as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    from paper_2309_01906_b200 import build
    build.build()
    from paper_2309_01906_b200 import hpar as H
    from paper_2309_01906_b200 import nests
    nest = H.Nest(nests.stencil_nest(), device=0)
    return torch, H, nest


def field(R, C, seed=gen.SEED_C5):
    return gen.gen_f32(seed, 0, R * C).reshape(R, C)


def run_whole(torch, H, nest, A, T):
    R, C = A.shape
    ld = (C + 3) // 4 * 4
    a = torch.zeros((R, ld), dtype=torch.float32, device="cuda")
    b = torch.zeros_like(a)
    a[:, :C] = torch.from_numpy(A).cuda()
    b.copy_(a)
    whole = H.Rect((0, 0), (R, C))
    for _ in range(T):
        H.hpar_stencil5(nest, H.stencil_desc(a, b, ld, whole, whole, (R, C)))
        a, b = b, a
    torch.cuda.synchronize()
    assert nest.last_kernel() == "stencil5_tma"
    return a[:, :C].cpu().numpy()


@pytest.mark.parametrize("shape", [(1, 1), (1, 7), (3, 3), (2, 9), (5, 200), (33, 129), (64, 256), (1000, 777)])
def test_stencil_whole_array(env, shape):
    torch, H, nest = env
    A = field(*shape)
    for T in (1, 3):
        assert np.array_equal(run_whole(torch, H, nest, A, T), G.stencil5(A, T))


def test_stencil_large(env):
    torch, H, nest = env
    A = field(2048, 4100, seed=gen.SEED_C3)
    assert np.array_equal(run_whole(torch, H, nest, A, 2), G.stencil5(A, 2))


def test_stencil_subsection_writes_only_from(env):
    """Cells of `out` outside the from-section are not written (only
    from elements go back); misaligned from-offsets take the scalar stores."""
    torch, H, nest = env
    R, C = 70, 300
    A = field(R, C)
    ld = 300
    a = torch.from_numpy(A).cuda().contiguous()
    b = torch.full_like(a, -7.0)
    to = H.Rect((0, 0), (R, C))
    fr = H.Rect((5, 3), (41, 229))
    H.hpar_stencil5(nest, H.stencil_desc(a, b, ld, to, fr, (R, C)))
    torch.cuda.synchronize()
    got = b.cpu().numpy()
    want = np.full_like(A, -7.0)
    full = G.stencil5(A, 1)
    want[5:46, 3:232] = full[5:46, 3:232]
    assert np.array_equal(got, want)


def _mapped_on_one_gpu(torch, H, nest, sp, A, T):
    m = H.map_spec(sp.extent, sp.siblings, sp.grid_cols, [(d.mul, d.add, d.len) for d in sp.to],
                   [(d.mul, d.add, d.len) for d in sp.frm])
    H.hpar_map_validate(m)
    secs = [H.hpar_map_sections(m, d) for d in range(sp.siblings)]
    ld = (sp.to[1].len + 3) // 4 * 4
    ins, outs = [], []
    for d, (to, fr) in enumerate(secs):
        t = torch.zeros((to.len[0], ld), dtype=torch.float32, device="cuda")
        t[:, :to.len[1]] = torch.from_numpy(A[to.off[0]:to.off[0] + to.len[0], to.off[1]:to.off[1] + to.len[1]].copy()).cuda()
        ins.append(t)
        outs.append(t.clone())
    for _ in range(T):
        for d, (to, fr) in enumerate(secs):
            H.hpar_stencil5(nest, H.stencil_desc(ins[d], outs[d], ld, to, fr, sp.extent))
        H.hpar_map_exchange_local(m, outs, ld)  # ghost refresh between the siblings' buffers
        ins, outs = outs, ins
    torch.cuda.synchronize()
    got = A.copy()
    for d, (to, fr) in enumerate(secs):
        loc = ins[d].cpu().numpy()
        r0, c0 = fr.off[0] - to.off[0], fr.off[1] - to.off[1]
        got[fr.off[0]:fr.off[0] + fr.len[0], fr.off[1]:fr.off[1] + fr.len[1]] = loc[r0:r0 + fr.len[0], c0:c0 + fr.len[1]]
    return got


def test_paper_geometry_four_siblings(env):
    """§4 verbatim: A[1024][1024] on 4 siblings, to = 513 x 513 with the
    ghost surface, from = 512 x 512; T steps == the sequential stencil."""
    torch, H, nest = env
    sp = G.paper_example_spec(1024)
    A = field(1024, 1024, seed=gen.SEED_C2)
    T = 4
    assert np.array_equal(_mapped_on_one_gpu(torch, H, nest, sp, A, T), G.stencil5(A, T))


def test_three_by_two_siblings_with_ghost_ring(env):
    torch, H, nest = env
    ty, tx = 45, 130
    sp = G.MapSpec((3 * ty + 2, 2 * tx + 2), 6, 2, (G.MapDim(ty, 0, ty + 2), G.MapDim(tx, 0, tx + 2)),
                   (G.MapDim(ty, 1, ty), G.MapDim(tx, 1, tx)))
    A = field(*sp.extent, seed=gen.SEED_C4)
    assert np.array_equal(_mapped_on_one_gpu(torch, H, nest, sp, A, 3), G.stencil5(A, 3))


def test_stencil_division_special_values(env):
    """Every fp32 class through the kernel's division by 5 (±0, ±inf, NaN,
    subnormals, FLT_MAX, random bit patterns): cell x sits between -0 cells,
    so its sum is x itself and the output is x / 5, compared with numpy's
    IEEE division via the oracle (scripts/div5_exhaustive.cu covers all 2^32
    inputs of the same sequence)."""
    torch, H, nest = env
    rng = np.random.default_rng(17)
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, -1e-45, 1.1754942e-38, 3.4028235e38,
                        -3.4028235e38, 5.0, 1.0, 0.2, 1e-40, 7.0e37], dtype=np.float32)
    vals = np.concatenate([special, rng.integers(0, 2 ** 32, 1 << 18, dtype=np.uint64).astype(np.uint32).view(np.float32)])
    n = vals.size
    A = np.full((3, 2 * n + 1), -0.0, dtype=np.float32)
    A[1, 1::2] = vals
    got = run_whole(torch, H, nest, A, 1)
    want = G.stencil5(A, 1)
    assert np.array_equal(got.view(np.uint32)[1, 1::2][~np.isnan(vals)], want.view(np.uint32)[1, 1::2][~np.isnan(vals)])
    assert np.array_equal(np.isnan(got), np.isnan(want))


@pytest.mark.parametrize("seed", range(int(os.environ.get("HPAR_FUZZ_N", "0")) or 16))
def test_stencil_fuzz(env, seed):
    """Random single-sibling stencils: array shape, row pitch (a multiple of
    4 >= the width), a random from-section inside the array and one sweep;
    the from-section vs the oracle's numpy step, every other cell of `out`
    untouched."""
    torch, H, nest = env
    rng = np.random.default_rng(7000 + seed)
    R, C = int(rng.integers(1, 400)), int(rng.integers(1, 700))
    ld = (C + 3) // 4 * 4 + 4 * int(rng.integers(0, 4))
    A = field(R, C, seed=gen.SEED_C5 + seed)
    r0, c0 = int(rng.integers(0, R)), int(rng.integers(0, C))
    nr, nc = int(rng.integers(1, R - r0 + 1)), int(rng.integers(1, C - c0 + 1))
    a = torch.zeros((R, ld), dtype=torch.float32, device="cuda")
    a[:, :C] = torch.from_numpy(A).cuda()
    b = torch.full_like(a, -7.0)
    H.hpar_stencil5(nest, H.stencil_desc(a, b, ld, H.Rect((0, 0), (R, C)), H.Rect((r0, c0), (nr, nc)), (R, C)))
    torch.cuda.synchronize()
    assert nest.last_kernel() == "stencil5_tma"
    got = b.cpu().numpy()[:, :C]
    want = np.full_like(A, -7.0)
    want[r0:r0 + nr, c0:c0 + nc] = G.stencil5(A, 1)[r0:r0 + nr, c0:c0 + nc]
    assert np.array_equal(got, want), (R, C, ld, r0, c0, nr, nc)
    assert (b.cpu().numpy()[:, C:] == -7.0).all(), "padding columns written"


@pytest.mark.parametrize("seed", range(int(os.environ.get("HPAR_FUZZ_N", "0")) or 8))
def test_mapped_siblings_fuzz(env, seed):
    """Random sibling grids with a one-cell ghost ring (the §4 mapping
    generalised: gy x gx siblings, ty x tx from-tiles, to = from + ring): T
    sweeps, each followed by the ghost refresh between the siblings'
    buffers, equal the sequential stencil over the whole array bit for bit."""
    torch, H, nest = env
    rng = np.random.default_rng(7500 + seed)
    gy, gx = int(rng.integers(1, 4)), int(rng.integers(1, 4))
    ty, tx = int(rng.integers(1, 70)), int(rng.integers(1, 150))
    sp = G.MapSpec((gy * ty + 2, gx * tx + 2), gy * gx, gx, (G.MapDim(ty, 0, ty + 2), G.MapDim(tx, 0, tx + 2)),
                   (G.MapDim(ty, 1, ty), G.MapDim(tx, 1, tx)))
    A = field(*sp.extent, seed=gen.SEED_C4 + seed)
    T = int(rng.integers(1, 5))
    assert np.array_equal(_mapped_on_one_gpu(torch, H, nest, sp, A, T), G.stencil5(A, T)), (gy, gx, ty, tx, T)
