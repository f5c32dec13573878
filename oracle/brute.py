"""Tiny pure-Python brute-force model of the nest partition (explicit list
slicing), used to cross-check the C oracle's partition on tiny nests.

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py).  Written independently of
oracle.c: it enumerates positions by scanning and uses Python slicing, never
the closed forms.  SPEC S:337 / PAPER P:244-253.
"""
from __future__ import annotations

import itertools

STATIC, STATIC_CHUNK, DYNAMIC, NONE = 0, 1, 2, 3


class ScheduleError(ValueError):
    pass


def own_brute(sched: int, chunk: int, parent: list, T: int, t: int) -> list:
    n = len(parent)
    if sched == STATIC:
        # split into T contiguous pieces, first (n mod T) pieces one longer
        sizes = [n // T + (1 if k < n % T else 0) for k in range(T)]
        start = sum(sizes[:t])
        return parent[start:start + sizes[t]]
    if sched in (STATIC_CHUNK, DYNAMIC):
        chunks = [parent[k:k + chunk] for k in range(0, n, chunk)]
        mine = chunks[t::T]
        return [p for c in mine for p in c]
    if sched == NONE:
        if n > T:
            raise ScheduleError("schedule(none) with more iterations than tasks")
        return parent[t:t + 1]
    raise ValueError(sched)


def partition_brute(levels, n0: int, n1: int = 0, offsets=None):
    """levels: list of (T, sched, chunk, loop).  Returns dict iteration -> [leaf ids]."""
    nloops = 2 if (n1 or offsets is not None) else 1
    seen = {}
    radices = [l[0] for l in levels]
    for ids in itertools.product(*[range(T) for T in radices]):
        leaf = 0
        for T, t in zip(radices, ids):
            leaf = leaf * T + t
        l0 = list(range(n0))
        for (T, sched, chunk, loop), t in zip(levels, ids):
            if loop == 0:
                l0 = own_brute(sched, chunk, l0, T, t)
        for i in l0:
            if nloops == 1:
                seen.setdefault(i, []).append(leaf)
                continue
            length = (offsets[i + 1] - offsets[i]) if offsets is not None else n1
            l1 = list(range(length))
            for (T, sched, chunk, loop), t in zip(levels, ids):
                if loop == 1:
                    l1 = own_brute(sched, chunk, l1, T, t)
            for j in l1:
                it = (offsets[i] + j) if offsets is not None else i * n1 + j
                seen.setdefault(it, []).append(leaf)
    return seen
