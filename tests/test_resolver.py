"""NEXT f4: property-based level selection (§3.2-3.3; SPEC
resolver S:225-253, policy S:283) and the portable aliases.
CPU only: the resolver is pure host code over the B200 level table."""
import itertools
import random

import pytest


@pytest.fixture(scope="module")
def H():
    from paper_2309_01906_b200 import build
    build.build()
    from paper_2309_01906_b200 import hpar
    return hpar


@pytest.fixture(scope="module")
def table(H):
    return H.hpar_hierarchy_describe(H.b200_desc(), nranks=8, cluster_dim=2, warps_per_cta=8)


def flags(table, first, last):
    f = 0xFFFFFFFF
    for l in range(first, last + 1):
        f &= table[l].props
    return f


def test_aliases(H):
    assert H.hpar_level_alias("devices") == (1, 1)
    assert H.hpar_level_alias("teams") == (2, 3)     # P:157 teams = partitions..ctas
    assert H.hpar_level_alias("threads") == (4, 5)
    assert H.hpar_level_alias("simd") == (5, 5)
    with pytest.raises(H.HparError):
        H.hpar_level_alias("tbps")                   # P:157 names it but never defines it


def test_teams_threads_from_reserve(H, table):
    """`parallel sync() reserve(sync(barrier))` + `parallel
    sync(barrier)` — 'OpenMP's current teams and parallel constructs match
    this example': the outer construct gets gpu..cluster (no barrier across
    clusters), the inner one cta..lane."""
    lv = H.hpar_nest_resolve([{"reserve": {"barrier"}}, {"demand": {"barrier"}}], table)
    assert [(l.first, l.last) for l in lv] == [(1, 2), (3, 5)]


def test_shuffle_barrier_is_the_lane_level(H, table):
    """P:291 `parallel sync(shuffle,barrier)` lands on the lanes (SPEC S:241
    maps it to the warp in its group convention)."""
    lv = H.hpar_nest_resolve([{}, {"demand": {"shuffle", "barrier"}}], table)
    assert (lv[-1].first, lv[-1].last) == (5, 5)
    lv = H.hpar_nest_resolve([{"demand": {"shuffle", "barrier"}}], table)
    assert [(l.first, l.last) for l in lv] == [(5, 5)]


def test_sync_empty_takes_everything(H, table):
    """sync() 'would use all available parallelism'."""
    lv = H.hpar_nest_resolve([{}], table)
    assert [(l.first, l.last) for l in lv] == [(1, 5)]


def test_unsatisfiable_is_capability_error(H, table):
    with pytest.raises(H.HparError) as e:
        H.hpar_nest_resolve([{"demand": {"critical"}}], table)   # no B200 level offers critical
    assert e.value.code == H.HPAR_E_CAPABILITY
    with pytest.raises(H.HparError) as e:
        H.hpar_nest_resolve([{}, {"demand": {"dynamic", "shuffle"}}], table)
    assert e.value.code == H.HPAR_E_CAPABILITY


def test_resolver_invariants_random(H, table):
    """satisfaction (demand ⊆ collapsed flags), disjoint
    contiguous runs covering gpu..lane, maximal outer fan-out, monotonicity of
    reserve; cross-checked against an exhaustive search."""
    names = ["barrier", "atomic", "shuffle", "dynamic", "progress", "globalmem", "localmem", "cache"]
    rng = random.Random(4)
    for _ in range(300):
        n = rng.randint(1, 4)
        cons = []
        for _ in range(n):
            cons.append({"demand": set(rng.sample(names, rng.randint(0, 2))),
                         "reserve": set(rng.sample(names, rng.randint(0, 1))) if rng.random() < 0.3 else set()})
        # exhaustive: all cut positions, pick the lexicographically longest-first feasible one
        best = None
        for s0, cuts in ((s0, cuts) for s0 in range(1, 6) for cuts in itertools.combinations(range(s0 + 1, 6), n - 1)):
            if best is not None and s0 > best[2]:
                break  # the coarsest feasible start wins
            bounds = [s0] + list(cuts) + [6]
            runs = [(bounds[i], bounds[i + 1] - 1) for i in range(n)]
            ok = True
            for i, (f, l) in enumerate(runs):
                fl = flags(table, f, l)
                if any(not (fl & H.P[p]) for p in cons[i]["demand"]):
                    ok = False
                if cons[i]["reserve"]:
                    if l == 5:
                        ok = False
                    else:
                        rest = flags(table, l + 1, 5)
                        if any(not (rest & H.P[p]) for p in cons[i]["reserve"]):
                            ok = False
            if ok:
                # construct by construct: longest run first, or shortest with a reserve
                key = tuple((l if cons[i]["reserve"] else -l) for i, (_, l) in enumerate(runs))
                if best is None or key < best[0]:
                    best = (key, runs, s0)
        if best is None:
            with pytest.raises(H.HparError):
                H.hpar_nest_resolve(cons, table)
            continue
        lv = H.hpar_nest_resolve(cons, table)
        assert [(l.first, l.last) for l in lv] == best[1]
        for c, l in zip(cons, lv):
            fl = flags(table, l.first, l.last)
            assert all(fl & H.P[p] for p in c["demand"])
        # the resolved nest is accepted by nest creation
        H.Nest(lv, device=-1, desc=H.b200_desc(), nranks=8 if lv[0].first == H.HPAR_GPU else 1,
               clusters=4 if lv[0].first <= H.HPAR_CLUSTER else 0)
