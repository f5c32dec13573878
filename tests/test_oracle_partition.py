"""Pins of the oracle's partition (own() and the nest walk) against what the
paper/SPEC fix and against an independent brute force.  CPU only."""
import json
import os
import random

import numpy as np
import pytest

from oracle import brute

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "workshare_examples.json")
SCHED = {"static": 0, "static_chunk": 1, "dynamic": 2, "none": 3}


def test_own_worked_examples(oracle):
    g = json.load(open(GOLDEN))
    for ex in g["own"]:
        for t, expect in ex["expect"].items():
            got = oracle.own(SCHED[ex["sched"]], ex["chunk"], ex["n"], ex["T"], int(t))
            assert got == expect, ex["cite"]


def test_own_none_overflow_is_error(oracle):
    g = json.load(open(GOLDEN))
    for ex in g["own_errors"]:
        with pytest.raises(oracle.OracleError) as e:
            oracle.own(SCHED[ex["sched"]], ex["chunk"], ex["n"], ex["T"], 0)
        assert e.value.code == oracle.E_SCHEDULE, ex["cite"]


def test_own_partition_property_1000_random(oracle):
    """SPEC S:386 / acceptance #4: every schedule partitions [0,N)."""
    rng = random.Random(1234)
    for _ in range(1000):
        n = rng.randint(0, 200)
        T = rng.randint(1, 20)
        c = rng.randint(1, 17)
        for sched in (0, 1, 2, 3):
            if sched == 3 and n > T:
                with pytest.raises(oracle.OracleError):
                    oracle.own(sched, c, n, T, 0)
                continue
            got = []
            for t in range(T):
                lst = oracle.own(sched, c, n, T, t)
                assert lst == sorted(lst)
                assert lst == brute.own_brute(sched, c, list(range(n)), T, t)
                if sched == 3:  # schedule(none) identity: iteration == task id
                    assert lst == ([t] if t < n else [])
                got += lst
            assert sorted(got) == list(range(n))


def test_static_block_sizes_differ_by_at_most_one(oracle):
    for n in range(0, 60):
        for T in range(1, 9):
            sizes = [len(oracle.own(0, 0, n, T, t)) for t in range(T)]
            assert max(sizes) - min(sizes) <= 1
            assert sizes == sorted(sizes, reverse=True)  # earlier tasks larger


def _all_tiny_nests(rng, count):
    scheds = [(0, 0), (1, 1), (1, 2), (1, 3), (2, 2), (3, 0)]
    for _ in range(count):
        depth = rng.randint(1, 4)
        lv = []
        for _ in range(depth):
            T = rng.choice([1, 2, 3, 5])
            s, c = rng.choice(scheds)
            lv.append((T, s, c, 0))
        yield lv


def test_nest_partition_vs_brute_flat(oracle):
    """Brute force on tiny nests (depth <= 4, T in {1,2,3,5}, n in [0,40])."""
    rng = random.Random(7)
    checked = 0
    for lv in _all_tiny_nests(rng, 300):
        n = rng.randint(0, 40)
        levels = [oracle.Level(T=T, sched=s, chunk=c, loop=l) for (T, s, c, l) in lv]
        try:
            want = brute.partition_brute(lv, n)
        except brute.ScheduleError:
            with pytest.raises(oracle.OracleError):
                oracle.nest_run(levels, n0=n)
            continue
        r = oracle.nest_run(levels, n0=n)
        assert (r.count == 1).all()
        for it in range(n):
            assert want[it] == [int(r.owner[it])]
        checked += 1
    assert checked > 100


def test_nest_partition_vs_brute_two_loops(oracle):
    """Multi-loop nests (PAPER P:215-225 bind_ancestor): each level refines only
    the loop it is bound to; dense and CSR inner extents."""
    rng = random.Random(11)
    checked = 0
    for _ in range(200):
        depth = rng.randint(2, 4)
        lv = []
        for a in range(depth):
            T = rng.choice([1, 2, 3])
            s, c = rng.choice([(0, 0), (1, 1), (1, 2), (2, 3)])
            lv.append((T, s, c, rng.randint(0, 1)))
        n0 = rng.randint(0, 7)
        levels = [oracle.Level(T=T, sched=s, chunk=c, loop=l) for (T, s, c, l) in lv]
        if rng.random() < 0.5:
            n1 = rng.randint(1, 9)
            want = brute.partition_brute(lv, n0, n1=n1)
            r = oracle.nest_run(levels, n0=n0, n1=n1, nloops=2)
            total = n0 * n1
        else:
            lengths = [rng.randint(0, 9) for _ in range(n0)]
            off = np.zeros(n0 + 1, dtype=np.int64)
            off[1:] = np.cumsum(lengths)
            want = brute.partition_brute(lv, n0, offsets=off)
            r = oracle.nest_run(levels, n0=n0, offsets=off, nloops=2)
            total = int(off[-1])
        assert (r.count == 1).all()
        for it in range(total):
            assert want[it] == [int(r.owner[it])]
        checked += 1
    assert checked == 200


def test_device_tiles_paper_section4(oracle):
    """A[1024][1024] tiled over devices 0-3 as 512x512 owned
    tiles (d/2, d mod 2): a 2-loop nest, rows static over 2, cols static over 2."""
    g = json.load(open(GOLDEN))["device_tiles"]
    levels = [oracle.Level(T=2, sched=0, loop=0), oracle.Level(T=2, sched=0, loop=1)]
    n = g["n"]
    r = oracle.nest_run(levels, n0=n, n1=n, nloops=2)
    assert (r.count == 1).all()
    for key, d in g["expect_owner_of"].items():
        i, j = map(int, key.split(","))
        assert r.owner[i * n + j] == d, g["cite"]
    counts = np.bincount(r.owner, minlength=4)
    assert (counts == g["tile"] ** 2).all()
