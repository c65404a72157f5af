"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no layer math, no simulation,
no planning). It only draws random numbers with NumPy's PCG64 so that the CPU
oracle (``oracle/``) and the GPU path (``paper_1907_05013_b200``) see the same
fp32 values. Recipe:

* images   x ~ N(0, 1), fp32, NHWC ``[B, H, W, C]`` (seed 0 + rank)
* labels   t ~ U{0 .. classes-1}, int32 (seed 1 + rank)
* weights  He-normal fan-in, fp32, conv weights in OIHW order ``[O, C, R, S]``,
           FC weight ``[O, I]`` and bias zeros; BN gamma = 1, beta = 0 (seed 2)
* profiles random task graphs for simulator/planner tests (integer ns / bytes)
"""
from __future__ import annotations

import numpy as np

__all__ = ["images", "labels", "he_normal", "uniform_f32", "rng", "random_profile"]


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def images(batch: int, h: int, w: int, c: int, seed: int = 0) -> np.ndarray:
    """x ~ N(0,1) as fp32 NHWC."""
    return rng(seed).standard_normal((batch, h, w, c), dtype=np.float64).astype(np.float32)


def labels(batch: int, classes: int, seed: int = 1, shape=None) -> np.ndarray:
    shape = (batch,) if shape is None else shape
    return rng(seed).integers(0, classes, size=shape).astype(np.int32)


def he_normal(shape, fan_in: int, g: np.random.Generator) -> np.ndarray:
    """He-normal (fan-in) draw in fp32; ``g`` is advanced (call order matters)."""
    std = np.sqrt(2.0 / fan_in)
    return (g.standard_normal(shape, dtype=np.float64) * std).astype(np.float32)


def uniform_f32(shape, lo: float, hi: float, seed: int) -> np.ndarray:
    return rng(seed).uniform(lo, hi, size=shape).astype(np.float32)


def random_profile(n: int, seed: int, *, dag: bool = False, max_bytes: int = 64,
                   max_t: int = 20, max_x: int = 30):
    """Random task graph for simulator / planner tests (plain data only).

    Returns a dict with integer ``fwd``, ``bwd``, ``bytes``, ``d2h``, ``h2d``
    lists, ``inputs`` (each task consumes its predecessor; with ``dag`` a few
    skip edges are added) and ``needs`` (bwd(i) reads its inputs and its own
    output, the SPEC's convention).
    """
    g = rng(1000 + seed)
    fwd = [int(v) for v in g.integers(1, max_t + 1, n)]
    bwd = [int(v) for v in g.integers(1, max_t + 1, n)]
    nbytes = [int(v) for v in g.integers(1, max_bytes + 1, n)]
    d2h = [int(v) for v in g.integers(1, max_x + 1, n)]
    h2d = [int(v) for v in g.integers(1, max_x + 1, n)]
    inputs = [[] if i == 0 else [i - 1] for i in range(n)]
    if dag:
        for i in range(2, n):
            if g.random() < 0.3:
                j = int(g.integers(0, i - 1))
                inputs[i].append(j)
    needs = [sorted(set(inputs[i]) | {i}) for i in range(n)]
    return dict(fwd=fwd, bwd=bwd, bytes=nbytes, d2h=d2h, h2d=h2d, inputs=inputs, needs=needs)
