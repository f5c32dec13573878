"""Hierarchical ghost maps and the 5-point stencil, written
from the paper, slow and plain.

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py): only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference``
legs may import this module.  It never imports the product package.

What it follows:

* PAPER §4: a parallel construct at the device level maps one
  array section per sibling ``d``::

      map(to(d):   A[(d/2)*511 : 513][(d%2)*511 : 513])
      map(from(d): A[(d/2)*512 : 512][(d%2)*512 : 512])

  Sections are ``offset : length`` (OpenMP array-section convention, SPEC
  S:416/S:452); the second subscript is truncated in the paper and is
  reconstructed symmetrically with the first.  The to-sections
  overlap ("so devices can access the immediate neighbors for reading,
  commonly referred to as a ghost surface"); the from-sections "must
  have unique sources".  Here a section is, per dimension,
  ``offset = mul * coord + add`` with ``coord = d // grid_cols`` for rows and
  ``d % grid_cols`` for columns, ``length = len``.
* SPEC hier_memory: evaluate_sections, validate (containment,
  bounds, unique from-sources), pack (global -> dense local buffer of the
  to-section), write back (from-section local -> global; to-only ghost
  writes discarded).
* The stencil ("5-point average, one halo exchange round"): every
  interior cell becomes ``((((c + n) + s) + w) + e) / 5`` in fp32 in exactly
  that order; cells on the array's boundary keep their value (Dirichlet).
  The parity check against the GPU is exact (same IEEE fp32 operations, no
  contraction possible: the division follows the complete sum).

The mapped execution of T steps re-packs every sibling's to-section from the
parent array after each step's write-back — the parent memory the paper
assumes "is always large enough to hold its child memories" — which
is what a halo exchange between siblings must reproduce.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class MapDim:
    mul: int   # offset = mul * coord + add
    add: int
    len: int


@dataclass(frozen=True)
class MapSpec:
    extent: tuple          # (rows, cols) of the parent array
    siblings: int          # S
    grid_cols: int         # sibling d -> (d // grid_cols, d % grid_cols)
    to: tuple              # (MapDim rows, MapDim cols)
    frm: tuple             # (MapDim rows, MapDim cols)


def paper_example_spec(n: int = 1024) -> MapSpec:
    """P:376-377 for A[n][n] on 4 devices (n = 1024 in the paper)."""
    h = n // 2
    return MapSpec((n, n), 4, 2, (MapDim(h - 1, 0, h + 1), MapDim(h - 1, 0, h + 1)),
                   (MapDim(h, 0, h), MapDim(h, 0, h)))


def sibling_coords(spec: MapSpec, d: int) -> tuple:
    return (d // spec.grid_cols, d % spec.grid_cols)


def sections(spec: MapSpec, d: int) -> tuple:
    """evaluate_sections: ((to_off, to_len), (from_off, from_len)),
    each a pair over (rows, cols)."""
    c = sibling_coords(spec, d)
    to_off = tuple(spec.to[k].mul * c[k] + spec.to[k].add for k in range(2))
    to_len = tuple(spec.to[k].len for k in range(2))
    fr_off = tuple(spec.frm[k].mul * c[k] + spec.frm[k].add for k in range(2))
    fr_len = tuple(spec.frm[k].len for k in range(2))
    return (to_off, to_len), (fr_off, fr_len)


class MapError(ValueError):
    def __init__(self, msg: str, where=None):
        super().__init__(msg)
        self.where = where


def validate(spec: MapSpec) -> None:
    """Bounds, positive lengths, from ⊆ to per sibling, and unique
    from-sources — by marking every element (brute force)."""
    R, C = spec.extent
    owner = np.full((R, C), -1, dtype=np.int64)
    for d in range(spec.siblings):
        (to_off, to_len), (fr_off, fr_len) = sections(spec, d)
        for k in range(2):
            if to_len[k] <= 0 or fr_len[k] <= 0:
                raise MapError(f"sibling {d}: non-positive section length")
            if to_off[k] < 0 or to_off[k] + to_len[k] > spec.extent[k]:
                raise MapError(f"sibling {d}: to-section outside the array")
            if fr_off[k] < 0 or fr_off[k] + fr_len[k] > spec.extent[k]:
                raise MapError(f"sibling {d}: from-section outside the array")
            if fr_off[k] < to_off[k] or fr_off[k] + fr_len[k] > to_off[k] + to_len[k]:
                raise MapError(f"sibling {d}: from-section not inside its to-section")
        for i in range(fr_off[0], fr_off[0] + fr_len[0]):
            for j in range(fr_off[1], fr_off[1] + fr_len[1]):
                if owner[i, j] >= 0:
                    raise MapError(f"element ({i}, {j}) written back by siblings {owner[i, j]} and {d}",
                                   (i, j, int(owner[i, j]), d))
                owner[i, j] = d


def pack(A: np.ndarray, spec: MapSpec, d: int) -> np.ndarray:
    (to_off, to_len), _ = sections(spec, d)
    return A[to_off[0]:to_off[0] + to_len[0], to_off[1]:to_off[1] + to_len[1]].copy()


def writeback(A: np.ndarray, local: np.ndarray, spec: MapSpec, d: int) -> None:
    (to_off, _), (fr_off, fr_len) = sections(spec, d)
    r0, c0 = fr_off[0] - to_off[0], fr_off[1] - to_off[1]
    A[fr_off[0]:fr_off[0] + fr_len[0], fr_off[1]:fr_off[1] + fr_len[1]] = \
        local[r0:r0 + fr_len[0], c0:c0 + fr_len[1]]


def stencil5_step(A: np.ndarray) -> np.ndarray:
    """One Jacobi step on the whole array (fp32, boundary kept)."""
    A = np.asarray(A, dtype=np.float32)
    B = A.copy()
    if A.shape[0] >= 3 and A.shape[1] >= 3:
        c = A[1:-1, 1:-1]
        s = (((c + A[:-2, 1:-1]) + A[2:, 1:-1]) + A[1:-1, :-2]) + A[1:-1, 2:]
        B[1:-1, 1:-1] = s / np.float32(5)
    return B


def stencil5(A: np.ndarray, steps: int) -> np.ndarray:
    for _ in range(steps):
        A = stencil5_step(A)
    return A


def stencil5_brute(A: np.ndarray, steps: int) -> np.ndarray:
    """Element-by-element loops (pure Python; tiny arrays only)."""
    A = np.asarray(A, dtype=np.float32).copy()
    R, C = A.shape
    for _ in range(steps):
        B = A.copy()
        for i in range(1, R - 1):
            for j in range(1, C - 1):
                t = np.float32(A[i, j]) + np.float32(A[i - 1, j])
                t = np.float32(t + A[i + 1, j])
                t = np.float32(t + A[i, j - 1])
                t = np.float32(t + A[i, j + 1])
                B[i, j] = np.float32(t / np.float32(5))
        A = B
    return A


def local_step(local: np.ndarray, spec: MapSpec, d: int) -> np.ndarray:
    """One step inside sibling d's packed buffer: every from-cell is updated
    from its to-section neighbours (global boundary cells copy); an access
    outside the to-section is the S:455 'neighbor of a neighbor' error."""
    (to_off, to_len), (fr_off, fr_len) = sections(spec, d)
    R, C = spec.extent
    out = local.copy()
    for i in range(fr_off[0], fr_off[0] + fr_len[0]):
        for j in range(fr_off[1], fr_off[1] + fr_len[1]):
            li, lj = i - to_off[0], j - to_off[1]
            if i == 0 or j == 0 or i == R - 1 or j == C - 1:
                continue
            for (a, b) in ((li - 1, lj), (li + 1, lj), (li, lj - 1), (li, lj + 1)):
                if not (0 <= a < to_len[0] and 0 <= b < to_len[1]):
                    raise MapError(f"sibling {d}: stencil reads global ({a + to_off[0]}, {b + to_off[1]}) "
                                   f"outside its to-section")
            t = np.float32(local[li, lj]) + np.float32(local[li - 1, lj])
            t = np.float32(t + local[li + 1, lj])
            t = np.float32(t + local[li, lj - 1])
            t = np.float32(t + local[li, lj + 1])
            out[li, lj] = np.float32(t / np.float32(5))
    return out


def mapped_stencil5(A: np.ndarray, spec: MapSpec, steps: int) -> np.ndarray:
    """§4 mapped execution: per step, pack every sibling's to-section from the
    parent, step locally, write the from-sections back (pure loops: small
    arrays only)."""
    validate(spec)
    A = np.asarray(A, dtype=np.float32).copy()
    for _ in range(steps):
        locals_ = [local_step(pack(A, spec, d), spec, d) for d in range(spec.siblings)]
        for d in range(spec.siblings):
            writeback(A, locals_[d], spec, d)
    return A


def exchange_plan(spec: MapSpec, d: int) -> list:
    """Halo exchange of sibling d (the device-level ghost refresh): for every
    other sibling e, the rectangle to(d) ∩ from(e) is received from e, and
    to(e) ∩ from(d) is sent to e.  Returns [(peer, 'recv'|'send', (r0, c0,
    rows, cols) in GLOBAL coordinates)], peers ascending, recv before send."""
    out = []
    (tod, tld), (fod, fld) = sections(spec, d)
    for e in range(spec.siblings):
        if e == d:
            continue
        (toe, tle), (foe, fle) = sections(spec, e)
        for kind, (ao, al), (bo, bl) in (("recv", (tod, tld), (foe, fle)), ("send", (toe, tle), (fod, fld))):
            r0, r1 = max(ao[0], bo[0]), min(ao[0] + al[0], bo[0] + bl[0])
            c0, c1 = max(ao[1], bo[1]), min(ao[1] + al[1], bo[1] + bl[1])
            if r1 > r0 and c1 > c0:
                out.append((e, kind, (r0, c0, r1 - r0, c1 - c0)))
    return out
