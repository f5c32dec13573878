"""Thin ctypes binding of libhpar.so (include/hpar.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels of libhpar.so.  Functions keep the C names (hpar_nest_create, ...);
`Nest` is a small convenience wrapper that owns a nest handle.  PyTorch is
used for device memory, streams and the process group's NCCL communicator.

There is no fallback: if libhpar.so is missing or fails to load, importing
this module raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HPAR_LIB") or os.path.join(PKG, "libhpar.so")  # HPAR_LIB: an in-tree experiment build

# ---- enums (include/hpar.h) ---------------------------------------------
HPAR_OK, HPAR_E_INVALID, HPAR_E_CAPABILITY, HPAR_E_SCHEDULE, HPAR_E_PARTITION = 0, -1, -2, -3, -4
HPAR_E_UNSUPPORTED, HPAR_E_CUDA, HPAR_E_NCCL, HPAR_E_NOMEM = -5, -6, -7, -8
STATUS_NAMES = {0: "HPAR_OK", -1: "HPAR_E_INVALID", -2: "HPAR_E_CAPABILITY", -3: "HPAR_E_SCHEDULE",
                -4: "HPAR_E_PARTITION", -5: "HPAR_E_UNSUPPORTED", -6: "HPAR_E_CUDA", -7: "HPAR_E_NCCL",
                -8: "HPAR_E_NOMEM"}
HPAR_NODE, HPAR_GPU, HPAR_CLUSTER, HPAR_CTA, HPAR_WARP, HPAR_LANE, HPAR_NLEVELS = range(7)
LEVEL_NAMES = ["node", "gpu", "cluster", "cta", "warp", "lane"]
PROPS = ["barrier", "critical", "atomic", "shuffle", "oversubscribable", "dynamic", "lockstep",
         "progress", "globalmem", "localmem", "groupmem", "cache"]
P = {name: 1 << i for i, name in enumerate(PROPS)}
STATIC, STATIC_CHUNK, DYNAMIC, NONE = 0, 1, 2, 3
OP_SUM, OP_MIN, OP_MAX, OP_HIST256, OP_AFFINE = 0, 1, 2, 3, 4
I32, I64, F32, F64, U8, U64 = 0, 1, 2, 3, 4, 5
VERIFY_COVERAGE, VERIFY_PARTIALS, VERIFY_FINGERPRINT = 1, 2, 4
PROBE_NO_BARRIER = 1  # hpar_barrier_probe flag: the negative control
LOCAL_N0_EMPTY = -1  # hpar_reduce_desc.local_n0 of an empty caller-sharded shard
MAX_NEST = 8


class HparError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


# ---- structs ------------------------------------------------------------
class LevelInfo(ctypes.Structure):
    _fields_ = [("level", ctypes.c_int32), ("props", ctypes.c_uint32), ("name", ctypes.c_char * 16),
                ("num", ctypes.c_int64), ("max_num", ctypes.c_int64), ("localmem_bytes", ctypes.c_uint64),
                ("groupmem_bytes", ctypes.c_uint64), ("grainedness", ctypes.c_double)]

    def flags(self) -> set[str]:
        return {n for n, b in P.items() if self.props & b}


class DeviceDesc(ctypes.Structure):
    _fields_ = [("sm_count", ctypes.c_int32), ("max_threads_per_sm", ctypes.c_int32),
                ("max_blocks_per_sm", ctypes.c_int32), ("warp_size", ctypes.c_int32),
                ("smem_per_block_optin", ctypes.c_int64), ("smem_per_sm", ctypes.c_int64),
                ("l2_bytes", ctypes.c_int64), ("hbm_bytes", ctypes.c_int64), ("cc_major", ctypes.c_int32),
                ("cc_minor", ctypes.c_int32), ("cluster_launch", ctypes.c_int32),
                ("max_cluster_size", ctypes.c_int32)]


def b200_desc() -> DeviceDesc:
    """A synthetic B200 description (for host-only validation without a GPU)."""
    return DeviceDesc(sm_count=148, max_threads_per_sm=2048, max_blocks_per_sm=32, warp_size=32,
                      smem_per_block_optin=232448, smem_per_sm=233472, l2_bytes=126 * 2 ** 20,
                      hbm_bytes=183359 * 2 ** 20, cc_major=10, cc_minor=0, cluster_launch=1,
                      max_cluster_size=8)


class NestLevel(ctypes.Structure):
    _fields_ = [("first", ctypes.c_int32), ("last", ctypes.c_int32), ("schedule", ctypes.c_int32),
                ("loop", ctypes.c_int32), ("chunk", ctypes.c_int64), ("fanout", ctypes.c_int64),
                ("width", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class NestConfig(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("cluster_dim", ctypes.c_int32), ("warps_per_cta", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("clusters", ctypes.c_int64), ("nccl_comm", ctypes.c_void_p), ("desc", ctypes.POINTER(DeviceDesc))]


class SyncConstruct(ctypes.Structure):
    _fields_ = [("demand", ctypes.c_uint32), ("reserve", ctypes.c_uint32), ("schedule", ctypes.c_int32),
                ("loop", ctypes.c_int32), ("chunk", ctypes.c_int64)]


class NestInfo(ctypes.Structure):
    _fields_ = [("G", ctypes.c_int64), ("C", ctypes.c_int64), ("K", ctypes.c_int64), ("W", ctypes.c_int64),
                ("rank", ctypes.c_int32), ("nlevels", ctypes.c_int32), ("lane_width", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("tasks", ctypes.c_int64 * MAX_NEST),
                ("total", ctypes.c_int64 * MAX_NEST), ("props", ctypes.c_uint32 * MAX_NEST),
                ("threads_per_gpu", ctypes.c_int64)]


class ReduceDesc(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("in_dtype", ctypes.c_int32), ("nloops", ctypes.c_int32),
                ("keyed", ctypes.c_int32), ("in_", ctypes.c_void_p), ("n0", ctypes.c_int64),
                ("n1", ctypes.c_int64), ("ld", ctypes.c_int64), ("offsets", ctypes.c_void_p),
                ("max_inner", ctypes.c_int64), ("out", ctypes.c_void_p), ("out_dtype", ctypes.c_int32),
                ("verify", ctypes.c_int32), ("level_partials", ctypes.c_void_p * MAX_NEST),
                ("coverage_owner", ctypes.c_void_p), ("coverage_count", ctypes.c_void_p),
                ("fingerprint", ctypes.c_void_p), ("global_begin", ctypes.c_uint64), ("local_n0", ctypes.c_int64)]


class MapDim(ctypes.Structure):
    _fields_ = [("mul", ctypes.c_int64), ("add", ctypes.c_int64), ("len", ctypes.c_int64)]


class MapSpec(ctypes.Structure):
    _fields_ = [("extent", ctypes.c_int64 * 2), ("siblings", ctypes.c_int32), ("grid_cols", ctypes.c_int32),
                ("to", MapDim * 2), ("from_", MapDim * 2)]


class Rect(ctypes.Structure):
    _fields_ = [("off", ctypes.c_int64 * 2), ("len", ctypes.c_int64 * 2)]

    def tup(self) -> tuple:
        return (self.off[0], self.off[1], self.len[0], self.len[1])


class Halo(ctypes.Structure):
    _fields_ = [("peer", ctypes.c_int32), ("send", ctypes.c_int32), ("rect", Rect)]


class StencilDesc(ctypes.Structure):
    _fields_ = [("in_", ctypes.c_void_p), ("out", ctypes.c_void_p), ("ld", ctypes.c_int64), ("to", Rect),
                ("from_", Rect), ("extent", ctypes.c_int64 * 2)]


# ---- library --------------------------------------------------------------
_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run paper_2309_01906_b200/build.py (no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        sig = {
            "hpar_device_describe": [ctypes.c_int32, ctypes.POINTER(DeviceDesc)],
            "hpar_hierarchy_describe": [ctypes.POINTER(DeviceDesc), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_int64, ctypes.POINTER(LevelInfo), ctypes.POINTER(ctypes.c_int32)],
            "hpar_hierarchy_query": [ctypes.c_int32, ctypes.c_void_p, ctypes.POINTER(LevelInfo),
                                     ctypes.POINTER(ctypes.c_int32)],
            "hpar_nest_create": [ctypes.POINTER(NestLevel), ctypes.c_int32, ctypes.POINTER(NestConfig),
                                 ctypes.POINTER(ctypes.c_void_p)],
            "hpar_nest_destroy": [ctypes.c_void_p],
            "hpar_nest_info": [ctypes.c_void_p, ctypes.POINTER(NestInfo)],
            "hpar_shard_range": [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                                 ctypes.POINTER(ctypes.c_int64)],
            "hpar_parallel_for_reduce": [ctypes.c_void_p, ctypes.POINTER(ReduceDesc), ctypes.c_void_p],
            "hpar_barrier": [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p],
            "hpar_barrier_probe": [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint32,
                                   ctypes.c_void_p, ctypes.c_void_p],
            "hpar_nest_resolve": [ctypes.POINTER(SyncConstruct), ctypes.c_int32, ctypes.POINTER(LevelInfo),
                                  ctypes.POINTER(NestLevel)],
            "hpar_level_alias": [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)],
            "hpar_shard_range_csr": [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)],
            "hpar_map_sections": [ctypes.POINTER(MapSpec), ctypes.c_int32, ctypes.POINTER(Rect), ctypes.POINTER(Rect)],
            "hpar_map_validate": [ctypes.POINTER(MapSpec), ctypes.POINTER(ctypes.c_int64)],
            "hpar_map_exchange_plan": [ctypes.POINTER(MapSpec), ctypes.c_int32, ctypes.POINTER(Halo), ctypes.c_int32,
                                       ctypes.POINTER(ctypes.c_int32)],
            "hpar_stencil5": [ctypes.c_void_p, ctypes.POINTER(StencilDesc), ctypes.c_void_p],
            "hpar_map_exchange": [ctypes.c_void_p, ctypes.POINTER(MapSpec), ctypes.c_void_p, ctypes.c_int64,
                                  ctypes.c_void_p],
            "hpar_map_exchange_local": [ctypes.POINTER(MapSpec), ctypes.POINTER(ctypes.c_void_p), ctypes.c_int64,
                                        ctypes.c_void_p],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        for name, args in {"hpar_last_error": [], "hpar_last_kernel": [ctypes.c_void_p], "hpar_version": []}.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != HPAR_OK:
        raise HparError(rc, lib().hpar_last_error().decode())


# ---- the C calls under their own names ------------------------------------
def hpar_version() -> str:
    return lib().hpar_version().decode()


def hpar_device_describe(device: int) -> DeviceDesc:
    d = DeviceDesc()
    _check(lib().hpar_device_describe(device, ctypes.byref(d)))
    return d


def hpar_hierarchy_describe(desc: DeviceDesc, nranks: int = 1, cluster_dim: int = 0, warps_per_cta: int = 0,
                            clusters: int = 0) -> list[LevelInfo]:
    out = (LevelInfo * HPAR_NLEVELS)()
    n = ctypes.c_int32()
    _check(lib().hpar_hierarchy_describe(ctypes.byref(desc), nranks, cluster_dim, warps_per_cta, clusters, out,
                                         ctypes.byref(n)))
    return list(out[: n.value])


def hpar_hierarchy_query(device: int = 0, nccl_comm: int | None = None) -> list[LevelInfo]:
    out = (LevelInfo * HPAR_NLEVELS)()
    n = ctypes.c_int32()
    _check(lib().hpar_hierarchy_query(device, nccl_comm, out, ctypes.byref(n)))
    return list(out[: n.value])


def hpar_level_alias(name: str) -> tuple[int, int]:
    f, l = ctypes.c_int32(), ctypes.c_int32()
    _check(lib().hpar_level_alias(name.encode(), ctypes.byref(f), ctypes.byref(l)))
    return f.value, l.value


def hpar_nest_resolve(constructs: list[dict], table: list[LevelInfo]) -> list["Level"]:
    """constructs: dicts with demand / reserve (sets of Table-2 property names),
    schedule, loop, chunk.  Returns the resolved nest levels."""
    n = len(constructs)
    arr = (SyncConstruct * n)()
    for i, c in enumerate(constructs):
        arr[i].demand = sum(P[p] for p in c.get("demand", ()))
        arr[i].reserve = sum(P[p] for p in c.get("reserve", ()))
        arr[i].schedule = c.get("schedule", STATIC)
        arr[i].loop = c.get("loop", 0)
        arr[i].chunk = c.get("chunk", 0)
    tab = (LevelInfo * HPAR_NLEVELS)(*table)
    out = (NestLevel * n)()
    _check(lib().hpar_nest_resolve(arr, n, tab, out))
    return [Level(o.first, o.last, o.schedule, o.loop, o.chunk) for o in out]


@dataclass
class Level:
    """One nest level (include/hpar.h hpar_nest_level)."""
    first: int
    last: int | None = None
    schedule: int = STATIC
    loop: int = 0
    chunk: int = 0
    fanout: int = 0
    width: int = 0

    def c(self) -> NestLevel:
        return NestLevel(self.first, self.first if self.last is None else self.last, self.schedule, self.loop,
                         self.chunk, self.fanout, self.width, 0)


def torch_nccl_comm(group=None) -> int:
    """The ncclComm_t of torch's ProcessGroupNCCL (borrowed; torch owns it)."""
    import torch
    import torch.distributed as dist
    pg = group or dist.distributed_c10d._get_default_group()
    backend = pg._get_backend(torch.device("cuda"))
    return int(backend._comm_ptr())


class Nest:
    """Owns an hpar_nest_t.  levels: list[Level]."""

    def __init__(self, levels: list[Level], device: int = 0, nccl_comm: int | None = None, cluster_dim: int = 0,
                 warps_per_cta: int = 0, clusters: int = 0, rank: int = 0, nranks: int = 1,
                 desc: DeviceDesc | None = None, flags: int = 0):
        self.levels = list(levels)
        arr = (NestLevel * len(levels))(*[l.c() for l in levels])
        self._desc = desc
        cfg = NestConfig(device, rank, nranks, cluster_dim, warps_per_cta, flags, clusters, nccl_comm,
                         ctypes.pointer(desc) if desc is not None else None)
        h = ctypes.c_void_p()
        _check(lib().hpar_nest_create(arr, len(levels), ctypes.byref(cfg), ctypes.byref(h)))
        self.handle = h
        self.device = device

    def close(self):
        if getattr(self, "handle", None):
            lib().hpar_nest_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> NestInfo:
        i = NestInfo()
        _check(lib().hpar_nest_info(self.handle, ctypes.byref(i)))
        return i

    def shard_range(self, n0: int, rank: int) -> tuple[int, int]:
        b, c = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().hpar_shard_range(self.handle, n0, rank, ctypes.byref(b), ctypes.byref(c)))
        return b.value, c.value

    def last_kernel(self) -> str:
        return lib().hpar_last_kernel(self.handle).decode()

    def parallel_for_reduce(self, desc: ReduceDesc, stream: int = 0) -> None:
        _check(lib().hpar_parallel_for_reduce(self.handle, ctypes.byref(desc), stream))

    def barrier(self, level: int, stream: int = 0) -> None:
        _check(lib().hpar_barrier(self.handle, level, stream))

    def barrier_probe(self, level: int, folds_ptr: int, rounds: int = 8, no_barrier: bool = False,
                      delay_ns: int = 0, stream: int = 0) -> None:
        _check(lib().hpar_barrier_probe(self.handle, level, rounds, PROBE_NO_BARRIER if no_barrier else 0,
                                        delay_ns, folds_ptr, stream))


def hpar_parallel_for_reduce(nest: Nest, desc: ReduceDesc, stream: int = 0) -> None:
    nest.parallel_for_reduce(desc, stream)


def hpar_barrier(nest: Nest, level: int, stream: int = 0) -> None:
    nest.barrier(level, stream)


def hpar_barrier_probe(nest: Nest, level: int, folds_ptr: int, rounds: int = 8, no_barrier: bool = False,
                       delay_ns: int = 0, stream: int = 0) -> None:
    nest.barrier_probe(level, folds_ptr, rounds, no_barrier, delay_ns, stream)


# ---- torch convenience ------------------------------------------------------
_TORCH_DT = None


def dtype_code(t) -> int:
    import torch
    global _TORCH_DT
    if _TORCH_DT is None:
        _TORCH_DT = {torch.int32: I32, torch.int64: I64, torch.float32: F32, torch.float64: F64,
                     torch.uint8: U8}
    return _TORCH_DT[t.dtype]


def make_desc(x, out, *, op: int = OP_SUM, n0: int, n1: int = 0, ld: int = 0, nloops: int = 1,
              keyed: bool = False, offsets=None, max_inner: int = 0, out_dtype: int = -1, verify: int = 0,
              partials=None, owner=None, count=None, fingerprint=None, global_begin: int = 0,
              local_n0: int | None = None) -> ReduceDesc:
    """Build an hpar_reduce_desc from torch tensors (device pointers only)."""
    d = ReduceDesc()
    d.op = op
    d.in_dtype = dtype_code(x)
    d.nloops = nloops
    d.keyed = 1 if keyed else 0
    d.in_ = x.data_ptr() if x.numel() else None
    d.n0, d.n1, d.ld = n0, n1, ld or n1
    d.offsets = offsets.data_ptr() if offsets is not None else None
    d.max_inner = max_inner
    d.out = out.data_ptr()
    d.out_dtype = out_dtype if out_dtype >= 0 else dtype_code(out)
    d.verify = verify
    for i, p in enumerate(partials or []):
        d.level_partials[i] = p.data_ptr() if p is not None else None
    d.coverage_owner = owner.data_ptr() if owner is not None else None
    d.coverage_count = count.data_ptr() if count is not None else None
    d.fingerprint = fingerprint.data_ptr() if fingerprint is not None else None
    d.global_begin = global_begin
    # local_n0: None = not caller-sharded; a row count (0 = this rank's shard is empty)
    d.local_n0 = 0 if local_n0 is None else (local_n0 if local_n0 > 0 else LOCAL_N0_EMPTY)
    # the desc holds raw device pointers: keep the tensors alive with it, so a
    # temporary passed here cannot be freed (and its memory reused) before the
    # kernel that reads it has run
    d._keep = (x, out, offsets, list(partials or []), owner, count, fingerprint)
    return d


# ---- hierarchical memory: ghost maps + stencil (§4; NEXT f3) -----------------
def map_spec(extent, siblings: int, grid_cols: int, to, frm) -> MapSpec:
    """to / frm: ((mul, add, len) rows, (mul, add, len) cols) — P:376-377."""
    m = MapSpec()
    m.extent[0], m.extent[1] = extent
    m.siblings, m.grid_cols = siblings, grid_cols
    for k in range(2):
        m.to[k] = MapDim(*to[k])
        m.from_[k] = MapDim(*frm[k])
    return m


def hpar_map_sections(m: MapSpec, d: int) -> tuple[Rect, Rect]:
    to, fr = Rect(), Rect()
    _check(lib().hpar_map_sections(ctypes.byref(m), d, ctypes.byref(to), ctypes.byref(fr)))
    return to, fr


def hpar_map_validate(m: MapSpec):
    """None if valid; raises HparError (with .where = (row, col, a, b) on an overlap)."""
    w = (ctypes.c_int64 * 4)(-1, -1, -1, -1)
    rc = lib().hpar_map_validate(ctypes.byref(m), w)
    if rc != HPAR_OK:
        e = HparError(rc, lib().hpar_last_error().decode())
        e.where = tuple(w) if w[0] >= 0 else None
        raise e


def hpar_map_exchange_plan(m: MapSpec, d: int) -> list[tuple]:
    """[(peer, 'recv'|'send', (r0, c0, rows, cols))] in plan order."""
    n = ctypes.c_int32(0)
    _check(lib().hpar_map_exchange_plan(ctypes.byref(m), d, None, 0, ctypes.byref(n)))
    arr = (Halo * max(n.value, 1))()
    _check(lib().hpar_map_exchange_plan(ctypes.byref(m), d, arr, n.value, ctypes.byref(n)))
    return [(h.peer, "send" if h.send else "recv", h.rect.tup()) for h in arr[:n.value]]


def stencil_desc(inp, out, ld: int, to: Rect, frm: Rect, extent) -> StencilDesc:
    d = StencilDesc()
    d.in_, d.out, d.ld = inp.data_ptr(), out.data_ptr(), ld
    d.to, d.from_ = to, frm
    d.extent[0], d.extent[1] = extent
    d._keep = (inp, out)  # raw pointers: keep the tensors alive with the desc
    return d


def hpar_stencil5(nest: "Nest", desc: StencilDesc, stream: int = 0) -> None:
    _check(lib().hpar_stencil5(nest.handle, ctypes.byref(desc), ctypes.c_void_p(stream)))


def hpar_map_exchange(nest: "Nest", m: MapSpec, buf, ld: int, stream: int = 0) -> None:
    _check(lib().hpar_map_exchange(nest.handle, ctypes.byref(m), ctypes.c_void_p(buf.data_ptr()), ld,
                                   ctypes.c_void_p(stream)))


def hpar_map_exchange_local(m: MapSpec, bufs: list, ld: int, stream: int = 0) -> None:
    arr = (ctypes.c_void_p * len(bufs))(*[b.data_ptr() for b in bufs])
    _check(lib().hpar_map_exchange_local(ctypes.byref(m), arr, ld, ctypes.c_void_p(stream)))

HPAR_NEST_NODE_FUSED = 1  # hpar_nest_config.flags: the node level inside the kernel (NEXT f1)
HPAR_NEST_NODE_ALWAYS = 2  # hpar_nest_config.flags: the host node collective also with one rank (tests)


def hpar_shard_range_csr(offsets, nranks: int, rank: int) -> tuple[int, int]:
    """nnz-balanced row shard (§8(e) C3); offsets: host int64 numpy [rows + 1]."""
    import numpy as np
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    b, c = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().hpar_shard_range_csr(off.ctypes.data, off.size - 1, nranks, rank, ctypes.byref(b), ctypes.byref(c)))
    return b.value, c.value
