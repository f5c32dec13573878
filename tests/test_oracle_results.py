"""Pins of the oracle's results and per-level partials against closed forms,
library routines on special cases, invariants and the paper's worked example.
CPU only."""
import json
import math
import os
import random

import numpy as np
import pytest

from inputs import gen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "workshare_examples.json")


def test_sibling_sum_worked_example(oracle):
    """8 lanes with partial sums 1..8; fold of all siblings = 36."""
    g = json.load(open(GOLDEN))["sibling_sum"]
    x = np.array(g["values"], dtype=np.int32)
    # schedule(none): lane t owns iteration t, 8 lanes
    r = oracle.nest_run([oracle.Level(T=8, sched=oracle.NONE)], n0=8, x=x)
    assert r.result == g["expect"]
    assert list(r.partials[0]) == g["values"]


def test_sum_i32_exact_vs_python(oracle):
    x = gen.gen_i32(gen.SEED_C1, 0, 1 << 20)
    assert oracle.sum_i32(x) == sum(int(v) for v in x)


def test_sum_f32_closed_form_bit_exact(oracle):
    """Inputs are k * 2^-24: the exact sum is (sum k) * 2^-24, representable in
    fp64 while the partial sums stay below 2^29."""
    for seed, n in [(gen.SEED_C5, 1 << 20), (gen.SEED_C2, 4096), (9, 12345)]:
        x = gen.gen_f32(seed, 0, n)
        k = gen.gen_f32_k(seed, 0, n)
        exact = oracle.sum_u64(k)
        assert exact == sum(int(v) for v in k)
        assert oracle.sum_f32(x) == exact * 2.0 ** -24
        assert oracle.sum_f32(x) == math.fsum(float(v) for v in x)


def test_min_max(oracle):
    x = gen.gen_f32(3, 0, 5000)
    assert oracle.min_f32(x) == float(x.min()) and oracle.max_f32(x) == float(x.max())
    xi = gen.gen_i32(3, 0, 5000)
    assert oracle.min_i32(xi) == int(xi.min()) and oracle.max_i32(xi) == int(xi.max())
    assert oracle.min_f32(np.zeros(0, np.float32)) == math.inf  # empty -> identity (§8(b))


def test_hist256_vs_bincount(oracle):
    for x in [gen.gen_u8(gen.SEED_C4, 0, 1 << 18), np.zeros(1000, np.uint8),
              gen.gen_u8_zipf(gen.SEED_C4, 0, 1 << 16)]:
        assert (oracle.hist256(x) == np.bincount(x, minlength=256).astype(np.uint64)).all()


def test_rowsum_and_segsum_closed_form(oracle):
    rows, cols = 37, 515
    a = gen.gen_f32(gen.SEED_C2, 0, rows * cols)
    k = gen.gen_f32_k(gen.SEED_C2, 0, rows * cols).reshape(rows, cols)
    out = oracle.rowsum_f32(a, rows, cols)
    for r in range(rows):
        assert out[r] == int(k[r].sum()) * 2.0 ** -24
    off = np.array([0, 0, 5, 5, 300, 1000, 1000], dtype=np.int64)  # empty segments too
    v = gen.gen_f32(gen.SEED_C3, 0, 1000)
    kv = gen.gen_f32_k(gen.SEED_C3, 0, 1000)
    seg = oracle.segsum_f32(v, off)
    for r in range(len(off) - 1):
        assert seg[r] == int(kv[off[r]:off[r + 1]].sum()) * 2.0 ** -24
    assert seg[0] == 0.0 and seg[2] == 0.0


NESTS = [
    # (levels as (T, sched, chunk, loop))
    [(2, 0, 0, 0), (3, 1, 4, 0), (4, 0, 0, 0), (32, 1, 4, 0)],
    [(1, 0, 0, 0), (5, 2, 7, 0), (2, 1, 16, 0), (8, 1, 128, 0), (32, 1, 4, 0)],
    [(3, 0, 0, 0), (2, 0, 0, 0), (8, 0, 0, 0), (32, 0, 0, 0)],
    [(7, 1, 1, 0), (32, 1, 1, 0)],
]


def test_result_invariant_under_nest_shape(oracle):
    """north_star: 'the reduction result is independent of how levels are nested
    or partitioned' (exact for integers)."""
    x = gen.gen_i32(gen.SEED_C1, 0, 30011)
    ref = oracle.sum_i32(x)
    for lv in NESTS:
        levels = [oracle.Level(T=T, sched=s, chunk=c, loop=l) for (T, s, c, l) in lv]
        r = oracle.nest_run(levels, n0=x.size, x=x)
        assert r.result == ref
        assert (r.count == 1).all()
    for op, f in [(oracle.MIN, oracle.min_i32), (oracle.MAX, oracle.max_i32)]:
        levels = [oracle.Level(T=T, sched=s, chunk=c, loop=l) for (T, s, c, l) in NESTS[0]]
        assert oracle.nest_run(levels, n0=x.size, x=x, op=op).result == f(x)


def test_partials_parent_is_fold_of_children(oracle):
    """Per-level partials: each parent = ordered fold of its children;
    the sum over any level equals the total."""
    x = gen.gen_i32(5, 0, 9999)
    for lv in NESTS:
        levels = [oracle.Level(T=T, sched=s, chunk=c, loop=l) for (T, s, c, l) in lv]
        r = oracle.nest_run(levels, n0=x.size, x=x)
        for a in range(len(lv)):
            p = r.partials[a]
            assert int(p.sum()) == r.result
            if a > 0:
                T = lv[a][0]
                assert (p.reshape(-1, T).sum(axis=1) == r.partials[a - 1]).all()
        # leaf partial = sum of the elements it owns
        leaf = r.partials[-1]
        want = np.zeros_like(leaf)
        np.add.at(want, r.owner, x.astype(np.int64))
        assert (leaf == want).all()


def test_hist_partials(oracle):
    x = gen.gen_u8(4, 0, 20000)
    levels = [oracle.Level(T=3, sched=1, chunk=512), oracle.Level(T=4, sched=1, chunk=64),
              oracle.Level(T=32, sched=1, chunk=16)]
    r = oracle.nest_run(levels, n0=x.size, x=x, op=oracle.HIST256)
    assert (r.result == np.bincount(x, minlength=256)).all()
    assert (r.partials[0].sum(axis=0) == r.result).all()
    assert (r.partials[2].reshape(-1, 32, 256).sum(axis=1) == r.partials[1]).all()


def test_keyed_rowwise_partials(oracle):
    """Config-2 shape in miniature: rows over clusters (loop 0), columns over
    CTA -> warp -> lane (loop 1); per-row results and per-row inner partials."""
    rows, cols = 13, 256
    a = gen.gen_f32(gen.SEED_C2, 0, rows * cols)
    levels = [oracle.Level(T=3, sched=0, loop=0), oracle.Level(T=2, sched=0, loop=1),
              oracle.Level(T=2, sched=1, chunk=16, loop=1), oracle.Level(T=4, sched=1, chunk=4, loop=1)]
    r = oracle.nest_run(levels, n0=rows, n1=cols, x=a, keyed=True)
    ref = oracle.rowsum_f32(a, rows, cols)
    assert np.array_equal(r.result, ref)  # exact: multiples of 2^-24
    assert (r.count == 1).all()
    lane = r.partials[3].reshape(rows, 2, 2, 4)
    assert np.array_equal(lane.sum(axis=3), r.partials[2].reshape(rows, 2, 2))
    assert np.array_equal(r.partials[1].reshape(rows, 2).sum(axis=1), ref)


def test_keyed_csr(oracle):
    off = gen.csr_offsets(300, 4000)
    v = gen.gen_f32(gen.SEED_C3, 0, 4000)
    levels = [oracle.Level(T=4, sched=2, chunk=8, loop=0), oracle.Level(T=8, sched=1, chunk=1, loop=1)]
    r = oracle.nest_run(levels, n0=300, offsets=off, x=v, keyed=True)
    assert np.array_equal(r.result, oracle.segsum_f32(v, off))
    assert (r.count == 1).all()


def test_fingerprints(oracle):
    """Coverage fingerprints: F_once over [b, b+n) is a plain sum of fp_mix; an
    owner map fingerprint changes if any single owner changes."""
    b, n = 1 << 33, 5000
    assert oracle.fp_once(b, n) == sum(oracle.fp_mix(b + e) for e in range(n)) % (1 << 64)
    owner = np.arange(n, dtype=np.int64) % 97
    f = oracle.fp_owner(owner, b)
    owner[1234] += 1
    assert oracle.fp_owner(owner, b) != f


def _compose(maps):
    a, b = 1, 0
    for ma, mb in maps:
        a, b = (int(ma) * a) % (1 << 64), (int(ma) * b + int(mb)) % (1 << 64)
    return a, b


def test_affine_ordered_fold(oracle):
    """NEXT f2: the ordered fold of a non-commutative
    operator.  With block (static, no chunk) schedules at every level each
    task owns a contiguous, in-order run, so the hierarchical fold in
    ascending task order equals running the recurrence y <- (2x+1) y + x
    directly; with round-robin schedules it is the S:377 task-order fold,
    which differs.  Every parent is the ordered composition of its children."""
    x = gen.gen_i32(17, 0, 5003).astype(np.int64)
    block = [[(2, 0, 0, 0), (3, 0, 0, 0), (4, 0, 0, 0), (32, 0, 0, 0)], [(5, 0, 0, 0), (7, 0, 0, 0)]]
    for lv in block:
        levels = [oracle.Level(T=T, sched=s, chunk=c, loop=l) for (T, s, c, l) in lv]
        r = oracle.nest_run(levels, n0=x.size, x=x, op=oracle.AFFINE)
        A, B = int(r.result[0]), int(r.result[1])
        for y0 in (0, 1, 987654321):
            assert (A * y0 + B) % (1 << 64) == oracle.affine_run(x, y0)
    for lv in NESTS:
        levels = [oracle.Level(T=T, sched=s, chunk=c, loop=l) for (T, s, c, l) in lv]
        r = oracle.nest_run(levels, n0=x.size, x=x, op=oracle.AFFINE)
        res = (int(r.result[0]), int(r.result[1]))
        assert _compose(r.partials[0]) == res
        for a in range(1, len(lv)):
            T = lv[a][0]
            kids = r.partials[a].reshape(-1, T, 2)
            for pidx in range(kids.shape[0]):
                assert _compose(kids[pidx]) == tuple(int(v) for v in r.partials[a - 1][pidx])
    assert oracle.affine_run(x[::-1].copy(), 3) != oracle.affine_run(x, 3)


def test_affine_run_pinned_to_python_recurrence(oracle):
    """or_affine_run against the recurrence written out in Python integers
    (S:377's ordered fold of the element maps y -> (2x+1) y + x^2, mod 2^64),
    including negative int64 inputs (two's complement) and the empty run."""
    M = 1 << 64
    rng = np.random.default_rng(7)
    for n in (0, 1, 2, 17, 300):
        x = rng.integers(-(1 << 62), 1 << 62, n, dtype=np.int64)
        for y0 in (0, 1, 3, M - 1):
            y = y0
            for v in x.tolist():
                u = v % M
                y = ((2 * u + 1) * y + u * u) % M
            assert oracle.affine_run(x, y0) == y
