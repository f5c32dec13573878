"""Pins of the ghost-map / stencil oracle (oracle/ghostmap.py) against what
the paper and the mathematics fix: the §4 sections printed in the paper
(tests/golden/ghost_maps.json), closed forms of the 5-point average,
brute-force loops, and the SPEC conservation property (mapped execution ==
unmapped sequential execution, exactly).  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import ghostmap as G

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ghost_maps.json")


def spec_from_json(g):
    to = tuple(G.MapDim(*t) for t in g["to"])
    fr = tuple(G.MapDim(*t) for t in g["from"])
    return G.MapSpec(tuple(g["extent"]), g["siblings"], g["grid_cols"], to, fr)


def test_paper_sections_golden():
    g = json.load(open(GOLD))
    spec = spec_from_json(g)
    assert spec == G.paper_example_spec(1024)
    for e in g["expected"]:
        (to_off, to_len), (fr_off, fr_len) = G.sections(spec, e["d"])
        assert [to_off[0], to_off[0] + to_len[0]] == e["to_rows"]
        assert [to_off[1], to_off[1] + to_len[1]] == e["to_cols"]
        assert [fr_off[0], fr_off[0] + fr_len[0]] == e["from_rows"]
        assert [fr_off[1], fr_off[1] + fr_len[1]] == e["from_cols"]
        assert to_len[0] * to_len[1] == g["buffer_elements"]
    (t0, _), _ = G.sections(spec, 0)
    (t2, l2), _ = G.sections(spec, 2)
    assert sorted(set(range(0, 513)) & set(range(t2[0], t2[0] + l2[0]))) == g["overlap_rows_0_2"]
    G.validate(spec)  # disjoint from-sections: passes


def test_validate_errors():
    # two siblings write back the same elements (report coordinates and pair)
    bad = G.MapSpec((16, 16), 2, 2, (G.MapDim(0, 0, 16), G.MapDim(0, 0, 16)), (G.MapDim(0, 0, 8), G.MapDim(0, 0, 8)))
    with pytest.raises(G.MapError) as e:
        G.validate(bad)
    assert e.value.where == (0, 0, 0, 1)
    # from not inside to
    with pytest.raises(G.MapError):
        G.validate(G.MapSpec((16, 16), 4, 2, (G.MapDim(8, 0, 8), G.MapDim(8, 0, 8)),
                             (G.MapDim(8, 0, 9), G.MapDim(8, 0, 8))))
    # out of bounds
    with pytest.raises(G.MapError):
        G.validate(G.MapSpec((16, 16), 4, 2, (G.MapDim(8, 0, 10), G.MapDim(7, 0, 9)),
                             (G.MapDim(8, 0, 8), G.MapDim(8, 0, 8))))


def test_stencil_closed_forms():
    R, C = 9, 13
    A = np.full((R, C), 3.25, dtype=np.float32)
    assert np.array_equal(G.stencil5(A, 4), A)                       # constants are fixed points
    i, j = np.meshgrid(np.arange(R), np.arange(C), indexing="ij")
    L = (i + 2 * j).astype(np.float32)                                # harmonic: the average keeps it
    assert np.array_equal(G.stencil5(L, 3), L)
    S = np.zeros((R, C), dtype=np.float32)
    S[4, 6] = 5.0                                                     # impulse: 1/5 to itself and 4 neighbours
    B = G.stencil5_step(S)
    want = np.zeros_like(S)
    for (a, b) in ((4, 6), (3, 6), (5, 6), (4, 5), (4, 7)):
        want[a, b] = 1.0
    assert np.array_equal(B, want)
    # boundary cells keep their value whatever the interior does
    X = np.random.default_rng(1).random((R, C), dtype=np.float32)
    Y = G.stencil5(X, 5)
    assert np.array_equal(Y[0], X[0]) and np.array_equal(Y[-1], X[-1])
    assert np.array_equal(Y[:, 0], X[:, 0]) and np.array_equal(Y[:, -1], X[:, -1])


@pytest.mark.parametrize("shape", [(1, 7), (2, 5), (3, 3), (4, 9), (7, 4), (11, 6)])
def test_stencil_vs_brute(shape):
    A = np.random.default_rng(shape[0] * 31 + shape[1]).standard_normal(shape).astype(np.float32)
    for T in (1, 2, 3):
        assert np.array_equal(G.stencil5(A, T), G.stencil5_brute(A, T))


def test_mapped_equals_sequential():
    """mapped execution == unmapped sequential stencil, exactly."""
    rng = np.random.default_rng(7)
    for sp in (G.paper_example_spec(16), G.paper_example_spec(10)):
        A = rng.standard_normal(sp.extent).astype(np.float32)
        for T in (1, 3):
            assert np.array_equal(G.mapped_stencil5(A, sp, T), G.stencil5(A, T))


def test_neighbor_of_neighbor_is_an_error():
    """only declared ghosts are present."""
    sp = G.MapSpec((8, 8), 4, 2, (G.MapDim(4, 0, 4), G.MapDim(4, 0, 4)), (G.MapDim(4, 0, 4), G.MapDim(4, 0, 4)))
    with pytest.raises(G.MapError):
        G.mapped_stencil5(np.ones((8, 8), np.float32), sp, 1)


def test_exchange_plan_reproduces_repacking():
    """After a local step + write-back, applying sibling d's receive list to
    its stale buffer gives exactly pack(parent) — the halo exchange is the
    re-pack from parent memory."""
    rng = np.random.default_rng(3)
    sp = G.paper_example_spec(12)
    A = rng.standard_normal(sp.extent).astype(np.float32)
    locs = [G.pack(A, sp, d) for d in range(sp.siblings)]
    locs = [G.local_step(locs[d], sp, d) for d in range(sp.siblings)]
    for d in range(sp.siblings):
        G.writeback(A, locs[d], sp, d)
    sends = {}
    for d in range(sp.siblings):
        for (peer, kind, (r0, c0, nr, nc)) in G.exchange_plan(sp, d):
            if kind == "send":
                (to_off, _), _ = G.sections(sp, d)
                sends[(d, peer)] = locs[d][r0 - to_off[0]:r0 - to_off[0] + nr, c0 - to_off[1]:c0 - to_off[1] + nc].copy()
    for d in range(sp.siblings):
        (to_off, _), _ = G.sections(sp, d)
        for (peer, kind, (r0, c0, nr, nc)) in G.exchange_plan(sp, d):
            if kind == "recv":
                locs[d][r0 - to_off[0]:r0 - to_off[0] + nr, c0 - to_off[1]:c0 - to_off[1] + nc] = sends[(peer, d)]
        assert np.array_equal(locs[d], G.pack(A, sp, d))
