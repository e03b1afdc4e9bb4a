"""Host-side elementwise work and reductions on all cores, bit-identical to numpy.

The solve path's host pieces (forcing, Dirichlet values, error norms;
solver.py:184-186, :239-246) are elementwise or reductions over N doubles.
numpy runs them on one core; here they run in chunks on a shared thread pool
(numpy releases the GIL).  Elementwise results are the same bits by
construction.  The l2 norm's ``mean`` is numpy's pairwise sum
(numpy/_core/src/umath/loops_utils.h.src, pairwise_sum: blocks of 8
accumulators up to 128 elements, otherwise split at n2 = n/2 rounded down to a
multiple of 8); ``pairwise_sum`` below descends that same split tree and hands
the subtrees below a size to numpy in parallel, so the total has numpy's bits
(tests/test_host.py checks both against numpy).
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

PAR_MIN = 1 << 18  # elements; below this one numpy call is faster
_CHUNK = 1 << 17
_pool = None


def pool() -> ThreadPoolExecutor:
    global _pool
    if _pool is None:
        n = int(os.environ.get("RBFFD_HOST_THREADS", "0")) or min(32, os.cpu_count() or 1)
        _pool = ThreadPoolExecutor(max_workers=max(1, n))
    return _pool


def chunked(n: int, fn, chunk: int = _CHUNK):
    """fn(lo, hi) over [0, n) in chunks on the pool; returns the results in order."""
    return list(pool().map(lambda lo: fn(lo, min(lo + chunk, n)), range(0, n, chunk)))


def _split(n: int) -> int:
    n2 = n // 2
    return n2 - n2 % 8


def pairwise_sum(x: np.ndarray, leaf: int = 1 << 17) -> float:
    """np.add.reduce(x) for a contiguous float64 vector, in parallel, same bits."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = x.shape[0]
    if n < PAR_MIN:
        return float(np.add.reduce(x))
    leaves = []

    def walk(lo, m):
        if m <= leaf:
            leaves.append((lo, m))
            return ("leaf", len(leaves) - 1)
        m2 = _split(m)
        return ("node", walk(lo, m2), walk(lo + m2, m - m2))

    tree = walk(0, n)
    sums = list(pool().map(lambda t: np.add.reduce(x[t[0]:t[0] + t[1]]), leaves))

    def combine(t):
        if t[0] == "leaf":
            return sums[t[1]]
        return combine(t[1]) + combine(t[2])

    return float(combine(tree))


def error_norms(values: np.ndarray, exact: np.ndarray):
    """(max|v - e|, sqrt(mean((v - e)**2))) with numpy's bits (solver.py:239-246)."""
    v = np.asarray(values, dtype=np.float64)
    e = np.asarray(exact, dtype=np.float64)
    n = v.shape[0]
    if n < PAR_MIN:
        diff = v - e
        return float(np.max(np.abs(diff))), math.sqrt(float((diff ** 2).mean()))
    sq = np.empty(n)

    def part(lo, hi):
        d = v[lo:hi] - e[lo:hi]
        np.multiply(d, d, out=sq[lo:hi])
        return float(np.max(np.abs(d)))

    linf = max(chunked(n, part))
    mean = pairwise_sum(sq) / n
    return linf, math.sqrt(mean)


def scaled_gather(scale: float, src: np.ndarray, idx: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
    """scale * src[idx] (elementwise: numpy's bits) on the pool."""
    n = idx.shape[0]
    if n < PAR_MIN:
        if out is None:
            return scale * src[idx]
        np.multiply(scale, src[idx], out=out)
        return out
    if out is None:
        out = np.empty(n)

    def part(lo, hi):
        np.multiply(scale, src[idx[lo:hi]], out=out[lo:hi])

    chunked(n, part)
    return out
