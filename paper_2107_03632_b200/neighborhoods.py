"""Exact kNN supports on the GPU.

Mirrors rbffd.neighborhoods.build_stencils (pkg/src/rbffd/neighborhoods.py:51-94)
over the C ABI ``rbf_knn``: row i holds node i's n nearest nodes sorted by
(distance, index) -- node i first -- the same contract as the reference's
cKDTree query + lexsort + exact-scan fallback, pinned by its brute-force
oracle (tests/oracles.py:16-24).
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from .errors import DeviceError, ParameterError
from .problem import StencilSet


def build_stencils(nodes, n: int, device: int = 0) -> StencilSet:
    """The n exact nearest neighbours of every node (neighborhoods.py:51-94)."""
    total = nodes.n_total
    if not 1 <= n <= total:
        raise ParameterError(f"support size n={n} outside [1, N={total}]")
    pos = np.ascontiguousarray(nodes.positions, dtype=np.float64)
    out = np.empty((total, n), dtype=np.int64)
    lib = _lib.load()
    rc = lib.rbf_knn(pos.ctypes.data, total, int(n), out.ctypes.data, int(device))
    if rc == _lib.RBF_ERR_PARAM:
        raise ParameterError(_lib.last_error(lib))
    if rc != _lib.RBF_OK:
        raise DeviceError(_lib.last_error(lib))
    return StencilSet(n=n, neighbors=out)


def build_stencils_subset(positions: np.ndarray, n: int, query: np.ndarray, device: int = 0) -> np.ndarray:
    """Supports of the nodes `query` only (a rank's own rows): (len(query), n)
    int64 global ids, the n nearest of all nodes, same order and ties as
    build_stencils (rbf_knn_subset)."""
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    q = np.ascontiguousarray(query, dtype=np.int64)
    total = pos.shape[0]
    if not 1 <= n <= total:
        raise ParameterError(f"support size n={n} outside [1, N={total}]")
    out = np.empty((q.size, n), dtype=np.int64)
    lib = _lib.load()
    rc = lib.rbf_knn_subset(pos.ctypes.data, total, int(n), q.ctypes.data, q.size, out.ctypes.data, int(device))
    if rc == _lib.RBF_ERR_PARAM:
        raise ParameterError(_lib.last_error(lib))
    if rc != _lib.RBF_OK:
        raise DeviceError(_lib.last_error(lib))
    return out


def recommended_support_size(degree: int, dim: int = 2, safety: int = 1) -> int:
    """binomial(degree + dim, degree) x safety (neighborhoods.py:38-48)."""
    if degree < 0 or dim < 1:
        raise ParameterError(f"invalid degree={degree} or dim={dim}")
    if safety not in (1, 2):
        raise ParameterError(f"safety factor must be 1 or 2, got {safety}")
    return safety * math.comb(degree + dim, degree)
