"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no partitioning, no reduction):
only the counter-based generator and the workload shapes, so that both sides of
every parity test see identical inputs.  The CUDA side has its own
implementation of the same generator (``inputs/gen_device.cu``); the two are
cross-checked on prefixes by ``tests/test_gpu_inputs.py``.

Recipe:

* z(seed, i) = splitmix64(seed * 2**40 + i), where
  splitmix64(x) = finalise(x + 0x9E3779B97F4A7C15) with the standard
  Stafford-13 finaliser.  Global indices are < 2**34, so streams of distinct
  seeds never overlap.
* int32  = low 32 bits of z (two's complement)
* fp32   = (z >> 40) * 2**-24  in [0, 1)  -- every value is an exact multiple
           of 2**-24, which gives the oracle an exact closed-form pin.
* uint8  = z >> 56
* CSR (config 3): Zipf(beta) row lengths, L_r = floor(w_r * nnz / sum w) with
  w_r = (r+1)**-beta, the remainder handed +1 to the top ranks so that the
  lengths sum to nnz exactly, then rows permuted by argsort of z(seed_perm, r).
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

# Seeds per BASELINE.json config.
SEED_C1, SEED_C2, SEED_C3, SEED_C4, SEED_C5 = 1, 2, 3, 4, 5
SEED_C3_PERM = 1003


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Stafford-13 splitmix64 of a uint64 array (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = (x.astype(np.uint64) + GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        return z ^ (z >> np.uint64(31))


def z_stream(seed: int, begin: int, n: int) -> np.ndarray:
    idx = np.arange(begin, begin + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return splitmix64(np.uint64(seed) * np.uint64(1 << 40) + idx)


def gen_i32(seed: int, begin: int, n: int) -> np.ndarray:
    return (z_stream(seed, begin, n) & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.int32)


def gen_f32(seed: int, begin: int, n: int) -> np.ndarray:
    k = (z_stream(seed, begin, n) >> np.uint64(40)).astype(np.float64)
    return (k * 2.0 ** -24).astype(np.float32)


def gen_f32_k(seed: int, begin: int, n: int) -> np.ndarray:
    """The integer numerators k with fp32 value = k * 2**-24 (exact)."""
    return (z_stream(seed, begin, n) >> np.uint64(40)).astype(np.uint64)


def gen_u8(seed: int, begin: int, n: int) -> np.ndarray:
    return (z_stream(seed, begin, n) >> np.uint64(56)).astype(np.uint8)


def gen_u8_zipf(seed: int, begin: int, n: int, s: float = 1.1) -> np.ndarray:
    """Skewed byte variant for config 4: inverse CDF of Zipf(s) over 256 symbols,
    driven by u = (z >> 11) * 2**-53."""
    p = (np.arange(1, 257, dtype=np.float64)) ** (-s)
    cdf = np.cumsum(p / p.sum())
    u = (z_stream(seed, begin, n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return np.minimum(np.searchsorted(cdf, u, side="right"), 255).astype(np.uint8)


def zipf_lengths(rows: int, nnz: int, beta: float = 0.8) -> np.ndarray:
    """Row lengths (before permutation), summing to nnz exactly."""
    w = (np.arange(1, rows + 1, dtype=np.float64)) ** (-beta)
    lengths = np.floor(w * (nnz / w.sum())).astype(np.int64)
    rem = nnz - int(lengths.sum())
    assert 0 <= rem <= rows
    lengths[:rem] += 1
    return lengths


def csr_offsets(rows: int, nnz: int, beta: float = 0.8, seed_perm: int = SEED_C3_PERM) -> np.ndarray:
    """int64 offsets[rows+1] of the config-3 CSR structure."""
    lengths = zipf_lengths(rows, nnz, beta)
    perm = np.argsort(z_stream(seed_perm, 0, rows), kind="stable")
    lengths = lengths[perm]
    off = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(lengths, out=off[1:])
    return off


# Workload shapes of BASELINE.json configs (full size) and the reduced sizes
# the oracle finishes in seconds (same level structure; DESIGN.md §Input recipe).
CONFIGS = {
    "c1": dict(outer=1024, inner=1024, dtype="i32", seed=SEED_C1),
    "c2": dict(rows=65536, cols=4096, dtype="f32", seed=SEED_C2),
    "c3": dict(rows=1 << 24, nnz=1 << 28, beta=0.8, dtype="f32", seed=SEED_C3),
    "c4": dict(n=1 << 32, dtype="u8", seed=SEED_C4),
    "c5": dict(n=1 << 34, dtype="f32", seed=SEED_C5),
}
