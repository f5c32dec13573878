"""Pins of the oracle's coverage fingerprints and of its per-iteration owner
function for flat nests (SURVEY §8(c) "Coverage at 2^32-2^34"; VERDICT r01
weak #1).  CPU only.

* or_fp_mix / or_fp_mix2 / or_fp_once / or_fp_owner against a pure-Python
  MurmurHash3 fmix64 written here (big-int arithmetic mod 2^64, nothing
  shared with oracle.c), whose inverse is checked to undo it (so a wrong
  shift or multiplier in the Python model would not round-trip).
* or_own_count against or_own's enumerated count, exhaustively on small n.
* or_owner_flat against or_nest_run's owner map AND the pure-Python list
  slicing model (oracle/brute.py) on random flat nests of every schedule.
* or_fp_flat_range: additive over disjoint ranges; equal to the fingerprint
  of the materialised owner map; sensitive to one dropped, duplicated or
  re-owned iteration (the failure modes it exists to catch).
"""
import random

import numpy as np
import pytest

from oracle import brute

M64 = (1 << 64) - 1
C1, C2 = 0xFF51AFD7ED558CCD, 0xC4CEB9FE1A85EC53  # MurmurHash3 fmix64 multipliers
GOLD, SALT, OWN = 0x9E3779B97F4A7C15, 0x632BE59BD9B4E019, 0xD6E8FEB86659FD93  # DESIGN.md protocol


def py_fmix64(z: int) -> int:
    z ^= z >> 33
    z = (z * C1) & M64
    z ^= z >> 33
    z = (z * C2) & M64
    z ^= z >> 33
    return z


def py_fmix64_inv(z: int) -> int:
    z ^= z >> 33                      # x ^ (x >> 33) is an involution for 64-bit x
    z = (z * pow(C2, -1, 1 << 64)) & M64
    z ^= z >> 33
    z = (z * pow(C1, -1, 1 << 64)) & M64
    z ^= z >> 33
    return z


def py_mix(i: int) -> int:
    return py_fmix64((i * GOLD + SALT) & M64)


def py_mix2(i: int, o: int) -> int:
    return py_fmix64(py_mix(i) ^ ((o * OWN) & M64))


def test_python_fmix64_is_a_bijection():
    rng = random.Random(64)
    assert py_fmix64(0) == 0
    for _ in range(2000):
        z = rng.getrandbits(64)
        assert py_fmix64_inv(py_fmix64(z)) == z
        assert py_fmix64(py_fmix64_inv(z)) == z


def test_fp_functions_vs_python(oracle):
    rng = random.Random(65)
    pts = [0, 1, 2, (1 << 32) - 1, 1 << 33, (1 << 34) - 1, M64] + [rng.getrandbits(64) for _ in range(500)]
    for i in pts:
        assert oracle.fp_mix(i) == py_mix(i)
        o = rng.getrandbits(40)
        assert oracle.fp_mix2(i, o) == py_mix2(i, o)
    b, n = (1 << 34) - 3000, 3000
    assert oracle.fp_once(b, n) == sum(py_mix(b + e) for e in range(n)) & M64
    owner = np.array([rng.getrandbits(30) for _ in range(n)], dtype=np.int64)
    assert oracle.fp_owner(owner, b) == sum(py_mix2(b + e, int(owner[e])) for e in range(n)) & M64


def test_own_count_closed_form(oracle):
    for sched, chunks in ((oracle.STATIC, [0]), (oracle.STATIC_CHUNK, [1, 2, 3, 7, 16]),
                          (oracle.DYNAMIC, [1, 5]), (oracle.NONE, [0])):
        for c in chunks:
            for T in (1, 2, 3, 5, 8):
                for n in range(0, 60):
                    if sched == oracle.NONE and n > T:
                        with pytest.raises(oracle.OracleError):
                            oracle.own_count(sched, c, n, T, 0)
                        continue
                    for t in range(T):
                        assert oracle.own_count(sched, c, n, T, t) == len(oracle.own(sched, c, n, T, t))


def random_flat_levels(oracle, rng, n):
    levels = []
    for _ in range(rng.randint(1, 5)):
        s = rng.choice([oracle.STATIC, oracle.STATIC_CHUNK, oracle.STATIC_CHUNK, oracle.NONE])
        levels.append(oracle.Level(T=rng.choice([1, 2, 3, 4, 5, 8]), sched=s,
                                   chunk=rng.choice([1, 2, 3, 4, 8, 16]) if s == oracle.STATIC_CHUNK else 0))
    return levels


def test_owner_flat_vs_nest_walk_and_brute(oracle):
    rng = random.Random(2309)
    done = 0
    while done < 300:
        n = rng.randint(0, 600)
        levels = random_flat_levels(oracle, rng, n)
        try:
            walk = oracle.nest_run(levels, n0=n)
        except oracle.OracleError:  # schedule(none) overflow: owner_flat must refuse too
            if n:
                with pytest.raises(oracle.OracleError):
                    [oracle.owner_flat(levels, n, i) for i in range(n)]
            continue
        got = [oracle.owner_flat(levels, n, i) for i in range(n)]
        assert got == list(walk.owner)
        if done % 5 == 0:
            b = brute.partition_brute([(l.T, l.sched, l.chunk, 0) for l in levels], n)
            assert all(len(b[i]) == 1 and b[i][0] == got[i] for i in range(n))
        done += 1


def test_owner_flat_at_full_size_shapes(oracle):
    """The C4 / C5 nest shapes at 2^32 / 2^34 iterations: the first and last
    iterations and the tile boundaries land where the closed forms of the
    coalesced flat nest put them (cluster static(K tile) -> CTA static(tile)
    -> warp static(32 V) -> lane static(V))."""
    for n, tile, V, C in ((1 << 34, 4096, 4, 148), (1 << 32, 16384, 16, 74)):
        K, W = 2, 8
        levels = [oracle.Level(T=1), oracle.Level(T=C, sched=1, chunk=K * tile),
                  oracle.Level(T=K, sched=1, chunk=tile), oracle.Level(T=W, sched=1, chunk=32 * V),
                  oracle.Level(T=32, sched=1, chunk=V)]
        rng = random.Random(n)
        for i in [0, V, 32 * V, tile, K * tile, C * K * tile, n - 1] + [rng.randrange(n) for _ in range(2000)]:
            g = i // tile                       # global tile; CTA g mod (C K) of the grid
            b = g % (C * K)
            within = i % tile
            w = (within // (32 * V)) % W
            lane = (within // V) % 32
            assert oracle.owner_flat(levels, n, i) == ((b * W + w) * 32 + lane), i


def test_fp_flat_range_additive_and_sensitive(oracle):
    rng = random.Random(7)
    for _ in range(20):
        n = rng.randint(1, 5000)
        levels = random_flat_levels(oracle, rng, n)
        levels = [l if l.sched != oracle.NONE else oracle.Level(T=l.T) for l in levels]
        g0 = rng.getrandbits(34)
        walk = oracle.nest_run(levels, n0=n)
        once, own = oracle.fp_flat_range(levels, n, 0, n, g0)
        assert once == oracle.fp_once(g0, n)
        assert own == oracle.fp_owner(walk.owner, g0)
        cut = sorted(rng.sample(range(n + 1), 2))
        parts = [oracle.fp_flat_range(levels, n, a, b - a, g0) for a, b in ((0, cut[0]), (cut[0], cut[1]), (cut[1], n))]
        assert sum(p[0] for p in parts) & M64 == once and sum(p[1] for p in parts) & M64 == own
        # one iteration dropped / duplicated / given to another leaf
        k = rng.randrange(n)
        assert (once - py_mix(g0 + k)) & M64 != once
        assert (once + py_mix(g0 + k)) & M64 != once
        o = int(walk.owner[k])
        assert (own - py_mix2(g0 + k, o) + py_mix2(g0 + k, o + 1)) & M64 != own
