"""hpar — B200-native hierarchical nested-parallel reductions (arXiv 2309.01906).

The product is libhpar.so (C ABI in include/hpar.h); this package is its thin
ctypes binding (`hpar`) plus the nest descriptions of the benchmark configs
(`nests`).  Build with `python paper_2309_01906_b200/build.py`.
"""
from . import hpar, nests  # noqa: F401
from .hpar import Level, Nest, HparError  # noqa: F401
