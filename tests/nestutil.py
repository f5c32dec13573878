"""Test helpers: translate an hpar nest description into the oracle's own nest
description.  The fan-outs T are computed HERE from the geometry the test
chose (G, C, K, W, lane width), never read back from the CUDA library."""
from __future__ import annotations

import numpy as np

HW_GPU, HW_CLUSTER, HW_CTA, HW_WARP, HW_LANE = 1, 2, 3, 4, 5


def fanouts(levels, G: int, C: int, K: int, W: int) -> list[int]:
    """T (tasks per parent) of every nest level for hardware radices G, C, K, W, 32."""
    width = 0
    for l in levels:
        if l.width:
            width = l.width
    out = []
    prev_width = 0
    for l in levels:
        last = l.first if l.last is None else l.last
        T = 1
        for hw in range(l.first, last + 1):
            if hw == HW_GPU:
                T *= G
            elif hw == HW_CLUSTER:
                T *= C
            elif hw == HW_CTA:
                T *= K
            elif hw == HW_WARP:
                T *= W
            elif hw == HW_LANE:
                if l.width:
                    T *= 32 // l.width
                elif prev_width:
                    T *= prev_width
                else:
                    T *= 32
        out.append(T)
        prev_width = l.width
    assert width == 0 or 32 % width == 0
    return out


def oracle_levels(O, levels, G: int, C: int, K: int, W: int):
    Ts = fanouts(levels, G, C, K, W)
    return [O.Level(T=T, sched=l.schedule, chunk=l.chunk, loop=l.loop) for l, T in zip(levels, Ts)]


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    denom = np.where(b == 0, 1.0, np.abs(b))
    with np.errstate(invalid="ignore"):
        err = np.where(b == 0, np.abs(a), np.abs(a - b) / denom)
    # equal values are exact, including the MIN/MAX identities +inf / -inf of
    # empty tasks (empty loops yield the identity)
    return np.where(a == b, 0.0, err)


def assert_rel(got, want, tol=1e-5):
    """§8(c) reading #5: |g - o| <= tol * |o|; o == 0 requires g == 0 exactly."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    zero = want == 0
    assert np.all(got[zero] == 0), "nonzero result where the oracle has 0 (empty segment)"
    err = rel_err(got, want)
    assert np.all(err <= tol), f"max rel err {err.max():.3e} > {tol}"
