"""B200-native PoocH: out-of-core CNN training-step executor (arXiv 1907.05013).

The product is ``libpooch.so`` (C ABI, ``include/pooch.h``): hand-written sm_100a
kernels and a C++ profiler / planner / three-stream executor. This package is
the thin ctypes binding over it.
"""
from ._lib import PoochError, lib  # noqa: F401
