"""§4 ghost maps through the C ABI (hpar_map_sections / _validate /
_exchange_plan) against the oracle (oracle/ghostmap.py), and the stencil's
argument checks.  CPU only: these entry points are host code."""
import itertools
import random

import numpy as np
import pytest

from oracle import ghostmap as G


@pytest.fixture(scope="module")
def H():
    from paper_2309_01906_b200 import build
    build.build()
    from paper_2309_01906_b200 import hpar
    return hpar


def to_c(H, sp: G.MapSpec):
    return H.map_spec(sp.extent, sp.siblings, sp.grid_cols,
                      [(d.mul, d.add, d.len) for d in sp.to], [(d.mul, d.add, d.len) for d in sp.frm])


def random_spec(rng):
    """Equal tiles of a gy x gx sibling grid with ghost depth g (clipped specs are
    not expressible: keep every section inside the array)."""
    gy, gx = rng.randint(1, 3), rng.randint(1, 3)
    ty, tx = rng.randint(1, 6), rng.randint(1, 6)
    g = rng.randint(0, 1)
    R, C = gy * ty + 2 * g, gx * tx + 2 * g
    to = (G.MapDim(ty, 0, ty + 2 * g), G.MapDim(tx, 0, tx + 2 * g))
    fr = (G.MapDim(ty, g, ty), G.MapDim(tx, g, tx))
    return G.MapSpec((R, C), gy * gx, gx, to, fr)


def test_sections_match_oracle(H):
    rng = random.Random(5)
    specs = [G.paper_example_spec(1024), G.paper_example_spec(16)] + [random_spec(rng) for _ in range(40)]
    for sp in specs:
        m = to_c(H, sp)
        for d in range(sp.siblings):
            to, fr = H.hpar_map_sections(m, d)
            (to_off, to_len), (fr_off, fr_len) = G.sections(sp, d)
            assert to.tup() == (to_off[0], to_off[1], to_len[0], to_len[1])
            assert fr.tup() == (fr_off[0], fr_off[1], fr_len[0], fr_len[1])
        with pytest.raises(H.HparError):
            H.hpar_map_sections(m, sp.siblings)


def _first_overlap_brute(sp):
    best = None
    for a, b in itertools.combinations(range(sp.siblings), 2):
        (_, _), (fa, la) = G.sections(sp, a)
        (_, _), (fb, lb) = G.sections(sp, b)
        for i in range(max(fa[0], fb[0]), min(fa[0] + la[0], fb[0] + lb[0])):
            for j in range(max(fa[1], fb[1]), min(fa[1] + la[1], fb[1] + lb[1])):
                if best is None or (i, j, a, b) < best:
                    best = (i, j, a, b)
    return best


def test_validate_matches_oracle(H):
    rng = random.Random(11)
    cases = [G.paper_example_spec(16)]
    for _ in range(60):
        sp = random_spec(rng)
        # perturb: overlapping from-sections, from outside to, out of bounds
        k = rng.randint(0, 3)
        if k == 1:
            fr = (G.MapDim(sp.frm[0].mul, sp.frm[0].add, sp.frm[0].len + 1), sp.frm[1])
            sp = G.MapSpec(sp.extent, sp.siblings, sp.grid_cols, sp.to, fr)
        elif k == 2:
            fr = (sp.frm[0], G.MapDim(max(sp.frm[1].mul - 1, 0), sp.frm[1].add, sp.frm[1].len))
            sp = G.MapSpec(sp.extent, sp.siblings, sp.grid_cols, sp.to, fr)
        cases.append(sp)
    for sp in cases:
        m = to_c(H, sp)
        try:
            G.validate(sp)
            want_ok = True
        except G.MapError:
            want_ok = False
        if want_ok:
            H.hpar_map_validate(m)
        else:
            with pytest.raises(H.HparError) as e:
                H.hpar_map_validate(m)
            ov = _first_overlap_brute(sp)
            if ov is not None and e.value.where is not None:
                assert e.value.where == ov


def test_validate_reports_pair(H):
    sp = G.MapSpec((16, 16), 2, 2, (G.MapDim(0, 0, 16), G.MapDim(0, 0, 16)), (G.MapDim(0, 0, 8), G.MapDim(0, 0, 8)))
    with pytest.raises(H.HparError) as e:
        H.hpar_map_validate(to_c(H, sp))
    assert e.value.where == (0, 0, 0, 1)


def test_exchange_plan_matches_oracle(H):
    rng = random.Random(2)
    for sp in [G.paper_example_spec(1024), G.paper_example_spec(12)] + [random_spec(rng) for _ in range(30)]:
        m = to_c(H, sp)
        for d in range(sp.siblings):
            assert H.hpar_map_exchange_plan(m, d) == G.exchange_plan(sp, d)


class _Buf:
    def __init__(self, a):
        self.a = a

    def data_ptr(self):
        return self.a.ctypes.data


def test_stencil_argument_checks(H):
    from paper_2309_01906_b200 import nests
    nest = H.Nest(nests.stencil_nest(), device=-1, desc=H.b200_desc(), clusters=4)
    a = np.zeros(64 * 64 + 16, np.float32)
    b = np.zeros(64 * 64 + 16, np.float32)
    off = (-a.ctypes.data % 16) // 4
    ia, ib = _Buf(a[off:]), _Buf(b[off:])
    R = H.Rect
    whole = R((0, 0), (64, 64))
    bad = [
        (whole, R((0, 0), (65, 64)), 64),            # from not inside to
        (R((0, 0), (32, 64)), R((0, 0), (32, 64)), 64),  # row 32 needed as a ghost, not held
        (whole, whole, 62),                           # pitch not a multiple of 4
    ]
    for to, fr, ld in bad:
        with pytest.raises(H.HparError) as e:
            H.hpar_stencil5(nest, H.stencil_desc(ia, ib, ld, to, fr, (64, 64)))
        assert e.value.code == H.HPAR_E_INVALID
    with pytest.raises(H.HparError):
        H.hpar_stencil5(nest, H.stencil_desc(ia, ia, 64, whole, whole, (64, 64)))  # in == out
