"""The nests of BASELINE.json's configs, as hpar nest descriptions.

Each function returns the list of nest levels (outermost first) that the
config's loop nest uses, in the paper's terms (P:104-118 level selection,
P:149-155 collapse, P:211-253 bind + schedule).  These are host-side data
only; the execution is libhpar.so's.
"""
from __future__ import annotations

from .hpar import (DYNAMIC, HPAR_CLUSTER, HPAR_CTA, HPAR_GPU, HPAR_LANE, HPAR_WARP, NONE, STATIC,
                   STATIC_CHUNK, Level)

TILE_F32 = 4096     # elements per CTA tile (16 KiB) for the flat fp32 stream
TILE_U8 = 16384     # bytes per CTA tile for the histogram stream


def c1_nest(with_gpu: bool = True, outer: int = 1024) -> list[Level]:
    """Config 1: `parallel level(teams)` over the 1024 outer iterations, with
    `for` static; nested `parallel level(threads)` over the 1024 inner ones,
    `for` static(4) (SURVEY §8(c) reading #15).  teams = cluster x CTA
    collapsed (P:157 alias), threads = warp x lane collapsed."""
    lv = []
    if with_gpu:
        lv.append(Level(HPAR_GPU, HPAR_GPU, STATIC, loop=0))
    lv.append(Level(HPAR_CLUSTER, HPAR_CTA, STATIC, loop=0, fanout=outer))
    lv.append(Level(HPAR_WARP, HPAR_LANE, STATIC_CHUNK, loop=1, chunk=4))
    return lv


def flat_nest(K: int = 2, tile: int = TILE_F32, vec: int = 4, with_gpu: bool = True) -> list[Level]:
    """Configs 5 (fp32, vec=4) and 4 (uint8, vec=16): the coalesced flat nest
    GPU static -> cluster static(K*tile) -> CTA static(tile) -> warp
    static(32*vec) -> lane static(vec)."""
    lv = []
    if with_gpu:
        lv.append(Level(HPAR_GPU, HPAR_GPU, STATIC))
    lv += [Level(HPAR_CLUSTER, HPAR_CLUSTER, STATIC_CHUNK, chunk=K * tile),
           Level(HPAR_CTA, HPAR_CTA, STATIC_CHUNK, chunk=tile),
           Level(HPAR_WARP, HPAR_WARP, STATIC_CHUNK, chunk=32 * vec),
           Level(HPAR_LANE, HPAR_LANE, STATIC_CHUNK, chunk=vec)]
    return lv


def c5_nest(K: int = 2, with_gpu: bool = True) -> list[Level]:
    return flat_nest(K, TILE_F32, 4, with_gpu)


def c4_nest(K: int = 2, with_gpu: bool = True, tile: int = TILE_U8) -> list[Level]:
    return flat_nest(K, tile, 16, with_gpu)


def c2_nest(with_gpu: bool = True) -> list[Level]:
    """Config 2: rows (loop 0) static over GPUs and clusters; columns (loop 1)
    static over the CTAs of a cluster, static(128) over warps, static(4) over
    lanes (SURVEY §8(c) reading #13).  One result per row."""
    lv = []
    if with_gpu:
        lv.append(Level(HPAR_GPU, HPAR_GPU, STATIC, loop=0))
    lv += [Level(HPAR_CLUSTER, HPAR_CLUSTER, STATIC, loop=0),
           Level(HPAR_CTA, HPAR_CTA, STATIC, loop=1),
           Level(HPAR_WARP, HPAR_WARP, STATIC_CHUNK, loop=1, chunk=128),
           Level(HPAR_LANE, HPAR_LANE, STATIC_CHUNK, loop=1, chunk=4)]
    return lv


def c3_nest(with_gpu: bool = True, rows_chunk: int = 64, width: int = 8) -> list[Level]:
    """Config 3 (generic form): rows (loop 0) dynamic(rows_chunk) over the
    teams (cluster x CTA), static over warps and over lane groups
    lanes(width); the nonzeros of a row (loop 1) static(1) over
    the `width` lanes of its group."""
    lv = []
    if with_gpu:
        lv.append(Level(HPAR_GPU, HPAR_GPU, STATIC, loop=0))
    lv += [Level(HPAR_CLUSTER, HPAR_CTA, DYNAMIC, loop=0, chunk=rows_chunk),
           Level(HPAR_WARP, HPAR_LANE, STATIC, loop=0, width=width),
           Level(HPAR_LANE, HPAR_LANE, STATIC_CHUNK, loop=1, chunk=1)]
    return lv


def c3_fast_nest(with_gpu: bool = True, rows_chunk: int = 256, lane_chunk: int = 16) -> list[Level]:
    """Config 3 (the fused CSR kernel's nest): rows (loop 0) dynamic(rows_chunk)
    over ALL warps of the GPU (cluster..warp collapsed: flags = intersection,
    dynamic and atomic hold); the block's nonzeros (loop 2 = the collapsed
    (row, nonzero) space) static(lane_chunk) over the lanes (8 or 16).  Rows longer than
    4096 nonzeros are re-bound by length class to dynamic(16384) segments over
    the warps (kernel_segmented.cu; reading #14)."""
    lv = []
    if with_gpu:
        lv.append(Level(HPAR_GPU, HPAR_GPU, STATIC, loop=0))
    lv += [Level(HPAR_CLUSTER, HPAR_WARP, DYNAMIC, loop=0, chunk=rows_chunk),
           Level(HPAR_LANE, HPAR_LANE, STATIC_CHUNK, loop=2, chunk=lane_chunk)]
    return lv


def stencil_nest(with_gpu: bool = True) -> list[Level]:
    """The §4 stencil workload (NEXT f3): the GPU level takes one sibling's
    map sections (hpar_map_*); below it the from-section's rows are static
    over the CTAs' tiles and warps (4 rows each), columns static(4) over the
    lanes (kernel_stencil.cu)."""
    lv = []
    if with_gpu:
        lv.append(Level(HPAR_GPU, HPAR_GPU, STATIC, loop=0))
    lv += [Level(HPAR_CLUSTER, HPAR_CTA, STATIC, loop=0),
           Level(HPAR_WARP, HPAR_WARP, STATIC, loop=0),
           Level(HPAR_LANE, HPAR_LANE, STATIC_CHUNK, loop=1, chunk=4)]
    return lv


__all__ = ["stencil_nest", "c3_fast_nest","c1_nest", "c2_nest", "c3_nest", "c4_nest", "c5_nest", "flat_nest", "TILE_F32", "TILE_U8",
           "NONE"]
