"""ctypes wrapper around oracle/liboracle.so (the sequential C oracle).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this module.  It never
imports the product package (paper_2309_01906_b200) and the product never
imports it.

Schedules / ops / dtypes use the oracle's own numbering (oracle/oracle.c).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC_PATH = os.path.join(HERE, "oracle.c")

STATIC, STATIC_CHUNK, DYNAMIC, NONE = 0, 1, 2, 3
SUM, MIN, MAX, HIST256, AFFINE = 0, 1, 2, 3, 4
I32, I64, F32, F64, U8 = 0, 1, 2, 3, 4
OK, E_SCHEDULE, E_INVALID, E_NOMEM = 0, -1, -2, -3


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"oracle error {code} in {what}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2, no fast-math, single thread)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC_PATH):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", SRC_PATH, "-o", LIB_PATH])
    return LIB_PATH


class _Level(ctypes.Structure):
    _fields_ = [("sched", ctypes.c_int32), ("loop", ctypes.c_int32),
                ("chunk", ctypes.c_int64), ("T", ctypes.c_int64)]


@dataclass
class Level:
    T: int
    sched: int = STATIC
    chunk: int = 0
    loop: int = 0


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        L.or_own.restype = ctypes.c_int64
        L.or_own.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                             ctypes.c_int64, ctypes.c_void_p]
        L.or_nest_run.restype = ctypes.c_int
        L.or_nest_run.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                  ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
                                  ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        for name, rt in [("or_sum_i32", ctypes.c_int64), ("or_min_i32", ctypes.c_int64),
                         ("or_max_i32", ctypes.c_int64), ("or_sum_f32", ctypes.c_double),
                         ("or_min_f32", ctypes.c_double), ("or_max_f32", ctypes.c_double),
                         ("or_sum_u64", ctypes.c_uint64)]:
            getattr(L, name).restype = rt
            getattr(L, name).argtypes = [ctypes.c_void_p, ctypes.c_int64]
        L.or_hist256.restype = None
        L.or_hist256.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.or_rowsum_f32.restype = None
        L.or_rowsum_f32.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_void_p]
        L.or_segsum_f32.restype = None
        L.or_segsum_f32.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.or_affine_run.restype = ctypes.c_uint64
        L.or_affine_run.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64]
        L.or_fp_mix.restype = ctypes.c_uint64
        L.or_fp_mix.argtypes = [ctypes.c_uint64]
        L.or_fp_mix2.restype = ctypes.c_uint64
        L.or_fp_mix2.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.or_fp_once.restype = ctypes.c_uint64
        L.or_fp_once.argtypes = [ctypes.c_uint64, ctypes.c_int64]
        L.or_own_count.restype = ctypes.c_int64
        L.or_own_count.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]
        L.or_owner_flat.restype = ctypes.c_int64
        L.or_owner_flat.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64]
        L.or_fp_flat_range.restype = ctypes.c_int
        L.or_fp_flat_range.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p]
        L.or_fp_owner.restype = ctypes.c_uint64
        L.or_fp_owner.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64]
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------
# own(): S:337
# --------------------------------------------------------------------------
def own(sched: int, chunk: int, n: int, T: int, t: int) -> list[int]:
    cnt = lib().or_own(sched, chunk, n, T, t, None)
    if cnt < 0:
        raise OracleError(int(cnt), "own")
    out = np.zeros(max(cnt, 1), dtype=np.int64)
    lib().or_own(sched, chunk, n, T, t, _ptr(out))
    return out[:cnt].tolist()


# --------------------------------------------------------------------------
# nest semantics
# --------------------------------------------------------------------------
_ACC_NP = {I32: np.int64, I64: np.int64, F32: np.float64, F64: np.float64, U8: np.int64}
_IN_CODE = {np.dtype(np.int32): I32, np.dtype(np.int64): I64, np.dtype(np.float32): F32,
            np.dtype(np.float64): F64, np.dtype(np.uint8): U8}


@dataclass
class NestResult:
    result: object            # scalar / bins[256] / per-row array
    owner: np.ndarray | None  # per iteration leaf id
    count: np.ndarray | None  # per iteration visits
    partials: list            # per nest level (None if not requested)


def nest_run(levels: list[Level], *, n0: int, n1: int = 0, offsets: np.ndarray | None = None,
             x: np.ndarray | None = None, ld: int = 0, op: int = SUM, keyed: bool = False,
             coverage: bool = True, partials: bool = True, nloops: int | None = None,
             dtype: int | None = None) -> NestResult:
    """Run the oracle nest walk.  See or_nest_run in oracle.c for semantics."""
    if nloops is None:
        nloops = 2 if (n1 or offsets is not None) else 1
    nlev = len(levels)
    arr = (_Level * nlev)(*[_Level(l.sched, l.loop, l.chunk, l.T) for l in levels])
    if offsets is not None:
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        n_iter = int(offsets[n0])
    else:
        n_iter = n0 * (n1 if nloops == 2 else 1)
    if x is not None:
        x = np.ascontiguousarray(x)
        dt = _IN_CODE[x.dtype]
    else:
        dt = F64 if dtype is None else dtype
    owner = np.full(n_iter, -1, dtype=np.int64) if coverage else None
    count = np.zeros(n_iter, dtype=np.uint32) if coverage else None
    # partial arrays
    part_arrays = [None] * nlev
    part_ptrs = (ctypes.c_void_p * nlev)()
    if partials and x is not None:
        first_inner = 0
        if keyed:
            while first_inner < nlev and levels[first_inner].loop == 0:
                first_inner += 1
        tasks = 1
        for a, l in enumerate(levels):
            if keyed:
                if a < first_inner:
                    continue
                tasks = 1
                for b in range(first_inner, a + 1):
                    tasks *= levels[b].T
                size = n0 * tasks
            else:
                tasks *= l.T
                size = tasks
            if op == HIST256:
                part_arrays[a] = np.zeros((size, 256), dtype=np.uint64)
            elif op == AFFINE:
                part_arrays[a] = np.zeros((size, 2), dtype=np.uint64)
            else:
                part_arrays[a] = np.zeros(size, dtype=_ACC_NP[dt])
            part_ptrs[a] = part_arrays[a].ctypes.data
    width = 256 if op == HIST256 else (2 if op == AFFINE else 0)
    if keyed:
        result = np.zeros((n0, width) if width else n0, dtype=np.uint64 if width else _ACC_NP[dt])
    else:
        result = np.zeros(width if width else 1, dtype=np.uint64 if width else _ACC_NP[dt])
    rc = lib().or_nest_run(ctypes.cast(arr, ctypes.c_void_p), nlev, nloops, n0, n1,
                           _ptr(offsets), dt, _ptr(x), ld if ld else n1, op, 1 if keyed else 0,
                           _ptr(result) if x is not None else None, _ptr(owner), _ptr(count),
                           ctypes.cast(part_ptrs, ctypes.c_void_p))
    if rc != 0:
        raise OracleError(rc, "nest_run")
    if not keyed and op not in (HIST256, AFFINE):
        result = result[0]
    return NestResult(result if x is not None else None, owner, count, part_arrays)


# --------------------------------------------------------------------------
# plain definitions
# --------------------------------------------------------------------------
def sum_i32(x: np.ndarray) -> int:
    x = np.ascontiguousarray(x, dtype=np.int32)
    return int(lib().or_sum_i32(_ptr(x), x.size))


def sum_f32(x: np.ndarray) -> float:
    x = np.ascontiguousarray(x, dtype=np.float32)
    return float(lib().or_sum_f32(_ptr(x), x.size))


def min_f32(x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    return float(lib().or_min_f32(_ptr(x), x.size))


def max_f32(x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    return float(lib().or_max_f32(_ptr(x), x.size))


def min_i32(x):
    x = np.ascontiguousarray(x, dtype=np.int32)
    return int(lib().or_min_i32(_ptr(x), x.size))


def max_i32(x):
    x = np.ascontiguousarray(x, dtype=np.int32)
    return int(lib().or_max_i32(_ptr(x), x.size))


def sum_u64(k: np.ndarray) -> int:
    k = np.ascontiguousarray(k, dtype=np.uint64)
    return int(lib().or_sum_u64(_ptr(k), k.size))


def hist256(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.uint8)
    bins = np.zeros(256, dtype=np.uint64)
    lib().or_hist256(_ptr(x), x.size, _ptr(bins))
    return bins


def rowsum_f32(a: np.ndarray, rows: int, cols: int, ld: int | None = None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    out = np.zeros(rows, dtype=np.float64)
    lib().or_rowsum_f32(_ptr(a), rows, cols, ld or cols, _ptr(out))
    return out


def segsum_f32(v: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    v = np.ascontiguousarray(v, dtype=np.float32)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    rows = offsets.size - 1
    out = np.zeros(rows, dtype=np.float64)
    lib().or_segsum_f32(_ptr(v), _ptr(offsets), rows, _ptr(out))
    return out


def fp_mix(i: int) -> int:
    return int(lib().or_fp_mix(i))


def fp_mix2(i: int, o: int) -> int:
    return int(lib().or_fp_mix2(i, o))


def fp_once(begin: int, n: int) -> int:
    return int(lib().or_fp_once(begin, n))


def fp_owner(owner: np.ndarray, begin: int) -> int:
    owner = np.ascontiguousarray(owner, dtype=np.int64)
    return int(lib().or_fp_owner(_ptr(owner), begin, owner.size))


def affine_run(x: np.ndarray, y0: int = 0) -> int:
    x = np.ascontiguousarray(x, dtype=np.int64)
    return int(lib().or_affine_run(_ptr(x), x.size, y0))


# --------------------------------------------------------------------------
# per-iteration owners of flat nests and range fingerprints (full sizes)
# --------------------------------------------------------------------------
def _levels_arr(levels):
    return (_Level * len(levels))(*[_Level(l.sched, l.loop, l.chunk, l.T) for l in levels])


def own_count(sched: int, chunk: int, n: int, T: int, t: int) -> int:
    c = int(lib().or_own_count(sched, chunk, n, T, t))
    if c < 0:
        raise OracleError(c, "own_count")
    return c


def owner_flat(levels: list[Level], n: int, i: int) -> int:
    arr = _levels_arr(levels)
    o = int(lib().or_owner_flat(ctypes.cast(arr, ctypes.c_void_p), len(levels), n, i))
    if o < 0:
        raise OracleError(o, "owner_flat")
    return o


def fp_flat_range(levels: list[Level], n: int, begin: int, count: int, g0: int = 0) -> tuple[int, int]:
    """(F_once, F_owner) of iterations [begin, begin + count) of a flat nest
    over n iterations (mod 2^64; disjoint ranges add)."""
    arr = _levels_arr(levels)
    out = np.zeros(2, dtype=np.uint64)
    rc = lib().or_fp_flat_range(ctypes.cast(arr, ctypes.c_void_p), len(levels), n, begin, count, g0, _ptr(out))
    if rc != 0:
        raise OracleError(rc, "fp_flat_range")
    return int(out[0]), int(out[1])
