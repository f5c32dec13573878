"""Oracle work at BASELINE.json's full sizes, split into independent index
ranges so a process pool can run them (test infrastructure: only the -m gpu
full-size tests use it).  Every quantity here is EXACT and additive over
disjoint ranges — integer numerator sums of the fp32 inputs (x = k 2^-24),
histogram counts, and the mod-2^64 coverage fingerprints — so the range
results add up to the oracle's whole-input answer exactly.  Each worker calls
only oracle/ (one thread per worker) and the seeded generator in inputs/."""
from __future__ import annotations

import multiprocessing as mp
import os

CHUNK = 1 << 24


def _sum_k(args):
    seed, b, n = args
    from inputs import gen
    from oracle import oracle as O
    return O.sum_u64(gen.gen_f32_k(seed, b, n))


def _hist(args):
    seed, b, n = args
    from inputs import gen
    from oracle import oracle as O
    return O.hist256(gen.gen_u8(seed, b, n))


def _fp(args):
    levels, n, b, cnt, g0 = args
    from oracle import oracle as O
    lv = [O.Level(T=T, sched=s, chunk=c) for (T, s, c) in levels]
    return O.fp_flat_range(lv, n, b, cnt, g0)


def _ranges(n, chunk=CHUNK):
    return [(b, min(chunk, n - b)) for b in range(0, n, chunk)]


def _pool():
    return mp.get_context("spawn").Pool(max(1, os.cpu_count() or 1))


def exact_numerator_sum(seed: int, n: int) -> int:
    """sum_i k_i over the first n fp32 inputs of `seed` (x_i = k_i 2^-24)."""
    with _pool() as p:
        return sum(p.map(_sum_k, [(seed, b, c) for b, c in _ranges(n)]))


def histogram(seed: int, n: int):
    import numpy as np
    with _pool() as p:
        return np.sum(p.map(_hist, [(seed, b, c) for b, c in _ranges(n)]), axis=0, dtype=np.uint64)


def flat_fingerprints(levels, n: int, g0: int = 0) -> tuple[int, int]:
    """(F_once, F_owner) of a flat nest over n iterations; levels as
    (T, sched, chunk) in the oracle's numbering."""
    with _pool() as p:
        parts = p.map(_fp, [(levels, n, b, c, g0) for b, c in _ranges(n)])
    m = (1 << 64) - 1
    return sum(a for a, _ in parts) & m, sum(b for _, b in parts) & m
