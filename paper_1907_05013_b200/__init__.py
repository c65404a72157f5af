"""B200-native PoocH: out-of-core CNN training-step executor (arXiv 1907.05013).

The product is ``libpooch.so`` (C ABI, ``include/pooch.h``): hand-written sm_100a
kernels and a C++ profiler / planner / three-stream executor. This package is
the thin ctypes binding over it.

``lib`` and ``PoochError`` are resolved lazily so that ``paper_1907_05013_b200.build``
can be imported (and run) in a fresh checkout before ``libpooch.so`` exists; every other
module imports ``_lib`` directly and fails loudly when the library is missing.
"""


def __getattr__(name):
    if name in ("lib", "PoochError"):
        from . import _lib
        return getattr(_lib, name)
    raise AttributeError(name)
