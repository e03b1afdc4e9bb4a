"""CPU problem setup of the reference arm -- TEST INFRASTRUCTURE ONLY.

``bench.py --impl reference`` (and tests/) build the benchmark workloads here,
on the host, without loading anything from the product package: the node set
comes from oracle/libnodes_orc.so (the advancing-front generator compiled
into the oracle's own library), supports and weights are restated from the
reference in numpy / scipy:

  * ``spacing_for_node_count`` <- pkg/src/rbffd/geometry.py:97-101
  * ``reference_nodes``        <- geometry.py:105-198 (libnodes_orc.so; the
                                  node sets are pinned to the reference's own
                                  outputs, tests/golden/nodes.json)
  * ``build_stencils``         <- neighborhoods.py:51-94 (cKDTree query with
                                  the _TIE_PAD = 8 look-ahead, (distance,
                                  index) order, exact scan of ambiguous rows)
  * ``assemble_shapes``        <- weights.py:143-206, _weights_batch :218-259
                                  (PHS r^3 + monomials, np.linalg.cond guard
                                  with COND_LIMIT = 1e14, np.linalg.solve)

The product's own CPU setup (paper_2107_03632_b200.synth, the bench's GPU
arm) restates the same reference functions; tests/test_bench_setup.py checks
that both produce byte-identical arrays, which is what lets the two bench
arms time the loop on the same (positions, neighbors, weights).
"""

from __future__ import annotations

import ctypes
import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
NODES_LIB = HERE / "libnodes_orc.so"

COND_LIMIT = 1e14  # weights.py:29
_CHUNK_BUDGET = 4_000_000  # weights.py:32
_TIE_PAD = 8  # neighborhoods.py:22


@dataclass
class Nodes:
    positions: np.ndarray  # (N, 2)
    is_boundary: np.ndarray  # (N,) bool
    h: float

    @property
    def n_total(self) -> int:
        return int(self.positions.shape[0])

    @property
    def interior_indices(self) -> np.ndarray:
        return np.flatnonzero(~self.is_boundary)

    @property
    def boundary_indices(self) -> np.ndarray:
        return np.flatnonzero(self.is_boundary)


@dataclass
class Stencils:
    n: int
    neighbors: np.ndarray  # (N, n) int64


@dataclass
class Shapes:
    degree: int
    interior_nodes: np.ndarray  # (N_i,) int64
    weights: np.ndarray  # (N_i, n)
    stencils: Stencils

    @property
    def n_rows(self) -> int:
        return int(self.weights.shape[0])


def spacing_for_node_count(n: int) -> float:  # geometry.py:97-101
    if n < 30:
        raise ValueError(f"target node count {n} is too small (need >= 30)")
    return 1.0 / (math.sqrt(1.0 + n / math.pi) - 1.0)


def _seed_key(seed: int) -> np.ndarray:
    n = abs(int(seed))
    words = []
    while n:
        words.append(n & 0xFFFFFFFF)
        n >>= 32
    return np.asarray(words or [0], dtype=np.uint32)


_nodes_lib = None


def _lib():
    global _nodes_lib
    if _nodes_lib is None:
        if not NODES_LIB.exists():
            import subprocess

            subprocess.run(["make", "-C", str(HERE), "-s"], check=True)
        L = ctypes.CDLL(str(NODES_LIB))
        L.rbf_generate_unit_disk_nodes.argtypes = [ctypes.c_double, ctypes.c_void_p, ctypes.c_int32,
                                                   ctypes.POINTER(ctypes.c_void_p),
                                                   ctypes.POINTER(ctypes.c_int64),
                                                   ctypes.POINTER(ctypes.c_int64)]
        L.rbf_generate_unit_disk_nodes.restype = ctypes.c_int
        L.rbf_free_host.argtypes = [ctypes.c_void_p]
        L.orc_nodes_last_error.restype = ctypes.c_char_p
        _nodes_lib = L
    return _nodes_lib


def reference_nodes(h: float, seed: int) -> Nodes:
    """The reference's advancing-front node set for (h, seed), geometry.py:105-198."""
    L = _lib()
    key = _seed_key(seed)
    ptr, n_total, n_boundary = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int64()
    rc = L.rbf_generate_unit_disk_nodes(float(h), key.ctypes.data, int(key.size), ctypes.byref(ptr),
                                        ctypes.byref(n_total), ctypes.byref(n_boundary))
    if rc != 0:
        raise ValueError(L.orc_nodes_last_error().decode())
    try:
        N = n_total.value
        buf = (ctypes.c_double * (2 * N)).from_address(ptr.value)
        positions = np.frombuffer(buf, dtype=np.float64).reshape(N, 2).copy()
    finally:
        L.rbf_free_host(ptr)
    is_boundary = np.zeros(N, dtype=bool)
    is_boundary[: n_boundary.value] = True
    return Nodes(positions=positions, is_boundary=is_boundary, h=float(h))


def _exact_row(positions: np.ndarray, i: int, n: int) -> np.ndarray:  # neighborhoods.py:134-138
    diff = positions - positions[i]
    dist = np.sqrt(diff[:, 0] ** 2 + diff[:, 1] ** 2)
    order = np.lexsort((np.arange(len(positions)), dist))
    return order[:n]


def build_stencils(nodes: Nodes, n: int) -> Stencils:  # neighborhoods.py:51-94
    from scipy.spatial import cKDTree

    total = nodes.n_total
    if not 1 <= n <= total:
        raise ValueError(f"support size n={n} outside [1, N={total}]")
    positions = nodes.positions
    tree = cKDTree(positions)
    k_query = min(total, n + _TIE_PAD)
    dist, idx = tree.query(positions, k=k_query, workers=-1)
    if dist.ndim == 1:
        dist, idx = dist[:, None], idx[:, None]
    order = np.lexsort((idx, dist))
    dist = np.take_along_axis(dist, order, axis=1)
    idx = np.take_along_axis(idx, order, axis=1)
    if k_query < total:
        for i in np.flatnonzero(dist[:, n - 1] == dist[:, k_query - 1]):
            idx[i, :n] = _exact_row(positions, int(i), n)
    return Stencils(n=n, neighbors=np.ascontiguousarray(idx[:, :n], dtype=np.int64))


def _exponents(degree: int) -> np.ndarray:  # weights.py:46-57 (graded lex, x-exponent descending)
    return np.asarray([(a, t - a) for t in range(degree + 1) for a in range(t, -1, -1)], dtype=np.int64)


def _weights_batch(supports: np.ndarray, expo: np.ndarray):  # weights.py:218-259
    count, n, _ = supports.shape
    m_size = expo.shape[0]
    size = n + m_size
    local = supports - supports[:, :1, :]
    radius = np.sqrt((local**2).sum(-1)).max(axis=1)
    scaled = local / radius[:, None, None]
    diff = scaled[:, :, None, :] - scaled[:, None, :, :]
    dist = np.sqrt((diff**2).sum(-1))
    mat = np.zeros((count, size, size))
    mat[:, :n, :n] = dist**3
    mono = scaled[:, :, 0:1] ** expo[:, 0] * scaled[:, :, 1:2] ** expo[:, 1]
    mat[:, :n, n:] = mono
    mat[:, n:, :n] = mono.transpose(0, 2, 1)
    rhs = np.zeros((count, size))
    rhs[:, :n] = 9.0 * np.sqrt((scaled**2).sum(-1))
    lap0 = np.zeros(m_size)
    for k, (a, b) in enumerate(expo):
        if (a, b) in ((2, 0), (0, 2)):
            lap0[k] = 2.0
    rhs[:, n:] = lap0
    with np.errstate(divide="ignore", invalid="ignore"):
        cond = np.linalg.cond(mat)
    good = cond <= COND_LIMIT
    weights = np.full((count, n), np.nan)
    if good.all():
        sol = np.linalg.solve(mat, rhs[:, :, None])[:, :, 0]
        weights = sol[:, :n] / radius[:, None] ** 2
    elif good.any():
        sol = np.linalg.solve(mat[good], rhs[good][:, :, None])[:, :, 0]
        weights[good] = sol[:, :n] / radius[good][:, None] ** 2
    return weights, cond


def assemble_shapes(nodes: Nodes, stencils: Stencils, degree: int, workers: int | None = None,
                    cond_check: bool = True) -> Shapes:
    """weights.py:143-206.  `workers` threads over the reference's chunks
    (results are written by row index: independent of scheduling).
    cond_check=False skips the SVD condition estimate (the weights are the
    same bits: the estimate never feeds the solve) for large benchmark sets."""
    expo = _exponents(degree)
    n = stencils.n
    if n < expo.shape[0]:
        raise ValueError(f"support size {n} below the {expo.shape[0]} monomials of degree {degree}")
    interior = nodes.interior_indices.astype(np.int64)
    n_rows = interior.size
    weights = np.empty((n_rows, n))
    size = n + expo.shape[0]
    chunk = max(32, min(4096, _CHUNK_BUDGET // (size * size)))
    spans = [(lo, min(lo + chunk, n_rows)) for lo in range(0, n_rows, chunk)]

    def run(span):
        lo, hi = span
        sup = nodes.positions[stencils.neighbors[interior[lo:hi]]]
        if cond_check:
            w, cond = _weights_batch(sup, expo)
            bad = np.flatnonzero(~(cond <= COND_LIMIT))
            if bad.size:
                node = int(interior[lo + int(bad[0])])
                raise ValueError(f"degenerate stencil at node {node}: condition estimate "
                                 f"{cond[bad[0]]:.3e}")
        else:
            w = _solve_only(sup, expo)
        weights[lo:hi] = w

    workers = workers or min(32, os.cpu_count() or 1)
    if workers > 1 and len(spans) > 1:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            list(pool.map(run, spans))
    else:
        for s in spans:
            run(s)
    return Shapes(degree=degree, interior_nodes=interior, weights=weights, stencils=stencils)


def _solve_only(supports: np.ndarray, expo: np.ndarray) -> np.ndarray:
    """_weights_batch without the condition estimate (same solve, same bits)."""
    count, n, _ = supports.shape
    m_size = expo.shape[0]
    size = n + m_size
    local = supports - supports[:, :1, :]
    radius = np.sqrt((local**2).sum(-1)).max(axis=1)
    scaled = local / radius[:, None, None]
    diff = scaled[:, :, None, :] - scaled[:, None, :, :]
    dist = np.sqrt((diff**2).sum(-1))
    mat = np.zeros((count, size, size))
    mat[:, :n, :n] = dist**3
    mono = scaled[:, :, 0:1] ** expo[:, 0] * scaled[:, :, 1:2] ** expo[:, 1]
    mat[:, :n, n:] = mono
    mat[:, n:, :n] = mono.transpose(0, 2, 1)
    rhs = np.zeros((count, size))
    rhs[:, :n] = 9.0 * np.sqrt((scaled**2).sum(-1))
    lap0 = np.zeros(m_size)
    for k, (a, b) in enumerate(expo):
        if (a, b) in ((2, 0), (0, 2)):
            lap0[k] = 2.0
    rhs[:, n:] = lap0
    sol = np.linalg.solve(mat, rhs[:, :, None])[:, :, 0]
    return sol[:, :n] / radius[:, None] ** 2


def reference_problem(target: int, n: int, degree: int, seed: int = 1, cond_check: bool = False):
    """(nodes, stencils, shapes) of a benchmark workload: the reference
    pipeline (geometry -> neighborhoods -> weights) for (target, seed)."""
    nodes = reference_nodes(spacing_for_node_count(target), seed)
    stencils = build_stencils(nodes, n)
    shapes = assemble_shapes(nodes, stencils, degree, cond_check=cond_check)
    return nodes, stencils, shapes
