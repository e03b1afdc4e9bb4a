"""Input containers and manufactured solution of the solve path.

The hot path consumes exactly three objects from the reference's CPU setup:
``NodeSet`` (pkg/src/rbffd/geometry.py:34-71), ``StencilSet``
(pkg/src/rbffd/neighborhoods.py:25-35) and ``ShapeStore``
(pkg/src/rbffd/weights.py:71-86).  The solver here is duck-typed over them:
the reference's own instances work unchanged; the light-weight mirrors below
exist so the GPU box (which has no reference package) can hold committed
fixtures and synthetic domains.

``closed_form_solution`` / ``forcing`` are the same numpy expressions as
geometry.py:74-86, evaluated in the same order, so they produce the same bits
(the Dirichlet values and f_int the kernel consumes).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class NodeSet:
    """Mirror of rbffd.geometry.NodeSet (geometry.py:34-71)."""

    positions: np.ndarray  # (N, 2) float64
    is_boundary: np.ndarray  # (N,) bool
    h: float

    @property
    def n_total(self) -> int:
        return self.positions.shape[0]

    @property
    def n_boundary(self) -> int:
        return int(self.is_boundary.sum())

    @property
    def n_interior(self) -> int:
        return self.n_total - self.n_boundary

    @property
    def interior_indices(self) -> np.ndarray:
        return np.flatnonzero(~self.is_boundary)

    @property
    def boundary_indices(self) -> np.ndarray:
        return np.flatnonzero(self.is_boundary)


@dataclass(frozen=True)
class StencilSet:
    """Mirror of rbffd.neighborhoods.StencilSet (neighborhoods.py:25-35)."""

    n: int
    neighbors: np.ndarray  # (N, n) int64, neighbors[i][0] == i


@dataclass(frozen=True)
class ShapeStore:
    """Mirror of rbffd.weights.ShapeStore (weights.py:71-86).

    ``weights[k]`` applies to ``stencils.neighbors[interior_nodes[k]]``.
    """

    degree: int
    interior_nodes: np.ndarray  # (N_i,) int64
    weights: np.ndarray  # (N_i, n) float64
    stencils: StencilSet

    @property
    def n_rows(self) -> int:
        return self.weights.shape[0]


_PAR_MIN = 1 << 18  # points; below this one numpy call is faster
_PAR_CHUNK = 1 << 16


def _closed_form_serial(p):
    return np.sin(np.pi * p[..., 0]) * np.sin(np.pi * p[..., 1])


def closed_form_solution(points, out=None):
    """sin(pi x) sin(pi y) -- geometry.py:74-81.

    Large (N, 2) inputs are evaluated in 64 Ki-point chunks on a thread pool
    (numpy releases the GIL); the expression is elementwise, so every value
    has the same bits as one call (tests/test_host.py checks it).  `out`
    (optional, float64 [N]) receives the values."""
    p = np.asarray(points, dtype=float)
    if p.ndim != 2 or p.shape[0] < _PAR_MIN:
        if out is None:
            return _closed_form_serial(p)
        out[...] = _closed_form_serial(p)
        return out
    if out is None:
        out = np.empty(p.shape[0])
    from . import _par

    def run(lo):
        hi = min(lo + _PAR_CHUNK, p.shape[0])
        out[lo:hi] = _closed_form_serial(p[lo:hi])

    list(_par.pool().map(run, range(0, p.shape[0], _PAR_CHUNK)))  # the package's persistent pool
    return out


def forcing(points):
    """2 pi^2 sin(pi x) sin(pi y) -- geometry.py:84-86 (same evaluation order)."""
    return 2.0 * np.pi**2 * closed_form_solution(points)


def monomial_count(degree: int) -> int:
    """MonomialBasis.of_degree(degree).size = (m+1)(m+2)/2 (weights.py:35-68)."""
    return (degree + 1) * (degree + 2) // 2


def _check_spacing(h: float) -> None:
    """geometry.py:222-224."""
    from .errors import ParameterError

    if not (0.0 < h < 0.5):
        raise ParameterError(f"spacing h={h} outside the valid range (0, 0.5)")


def node_count_for_spacing(h: float) -> int:
    """geometry.py:89-95."""
    _check_spacing(h)
    return int(math.floor(math.pi / h**2 + 2.0 * math.pi / h + 0.5))


def spacing_for_node_count(n: int) -> float:
    """geometry.py:98-102 (inverse of node_count_for_spacing)."""
    if n < 30:
        from .errors import ParameterError

        raise ParameterError(f"target node count {n} is too small (need >= 30)")
    return 1.0 / (math.sqrt(1.0 + n / math.pi) - 1.0)


def load_fixture(path) -> tuple[NodeSet, StencilSet, ShapeStore]:
    """Rebuild (nodes, stencils, shapes) from a tests/golden/*.npz fixture."""
    z = np.load(path)
    nodes = NodeSet(positions=z["positions"], is_boundary=z["is_boundary"], h=float(z["h"]))
    neighbors = z["neighbors"].astype(np.int64)
    stencils = StencilSet(n=neighbors.shape[1], neighbors=neighbors)
    shapes = ShapeStore(
        degree=int(z["degree"]),
        interior_nodes=z["interior"].astype(np.int64),
        weights=z["weights"],
        stencils=stencils,
    )
    return nodes, stencils, shapes


def save_problem(path, nodes: NodeSet, stencils: StencilSet, shapes: ShapeStore) -> None:
    """Binary problem cache: one .npy per array in a
    directory, replacing the reference's 17-digit CSV files for large runs
    (geometry.py:201-220, neighborhoods.py:104-122, weights.py:209-215).
    Node ids are stored as int32 when N < 2^31 (half the reference's int64)."""
    import json
    from pathlib import Path

    d = Path(path)
    d.mkdir(parents=True, exist_ok=True)
    idt = np.int32 if nodes.n_total < 2**31 else np.int64
    np.save(d / "positions.npy", np.ascontiguousarray(nodes.positions, dtype=np.float64))
    np.save(d / "is_boundary.npy", np.ascontiguousarray(nodes.is_boundary, dtype=bool))
    np.save(d / "neighbors.npy", np.ascontiguousarray(stencils.neighbors, dtype=idt))
    np.save(d / "interior.npy", np.ascontiguousarray(shapes.interior_nodes, dtype=idt))
    np.save(d / "weights.npy", np.ascontiguousarray(shapes.weights, dtype=np.float64))
    (d / "meta.json").write_text(json.dumps({"h": float(nodes.h), "n": int(stencils.n),
                                             "degree": int(shapes.degree), "version": 1}))


def load_problem(path, mmap: bool = True):
    """(nodes, stencils, shapes) from ``save_problem``; the large arrays are
    memory-mapped (read lazily, straight from the page cache)."""
    import json
    from pathlib import Path

    d = Path(path)
    meta = json.loads((d / "meta.json").read_text())
    mode = "r" if mmap else None
    positions = np.load(d / "positions.npy", mmap_mode=mode)
    is_boundary = np.load(d / "is_boundary.npy")
    neighbors = np.load(d / "neighbors.npy", mmap_mode=mode)
    interior = np.load(d / "interior.npy").astype(np.int64)
    weights = np.load(d / "weights.npy", mmap_mode=mode)
    nodes = NodeSet(positions=positions, is_boundary=is_boundary, h=float(meta["h"]))
    stencils = StencilSet(n=int(meta["n"]), neighbors=neighbors)
    shapes = ShapeStore(degree=int(meta["degree"]), interior_nodes=interior, weights=weights,
                        stencils=stencils)
    return nodes, stencils, shapes
