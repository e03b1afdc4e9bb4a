"""GPU assembly of the Laplacian weight rows.

Mirrors the reference API of pkg/src/rbffd/weights.py -- ``assemble_shapes``
(:143-206) and ``compute_laplacian_weights`` (:99-140) -- over the C ABI
``rbf_assemble_weights``: one warp per (n+M)^2 saddle system on the device.
Results agree with the reference's LAPACK solve to rounding (the reference
pins weights by polynomial reproduction, test_weights.py:51-104), not bit for
bit; the time loop's bitwise parity is always stated on identical weights.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import DeviceError, ParameterError
from .problem import ShapeStore, monomial_count


class DegenerateStencilError(RuntimeError):
    """Mirror of rbffd.errors.DegenerateStencilError (errors.py:8-18)."""

    def __init__(self, message, node_index=None, position=None):
        super().__init__(message)
        self.node_index = node_index
        self.position = position


def _assemble(positions: np.ndarray, rows: np.ndarray, degree: int, device: int = 0) -> np.ndarray:
    lib = _lib.load()
    positions = np.ascontiguousarray(positions, dtype=np.float64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    n_rows, n = rows.shape
    out = np.empty((n_rows, n), dtype=np.float64)
    bad = ctypes.c_int64(-1)
    rc = lib.rbf_assemble_weights(positions.ctypes.data, positions.shape[0], rows.ctypes.data, n_rows,
                                  n, int(degree), out.ctypes.data, ctypes.byref(bad), int(device))
    if rc == _lib.RBF_ERR_PARAM and bad.value >= 0:
        raise DegenerateStencilError(_lib.last_error(lib), node_index=int(bad.value))
    if rc == _lib.RBF_ERR_PARAM:
        raise ParameterError(_lib.last_error(lib))
    if rc != _lib.RBF_OK:
        raise DeviceError(_lib.last_error(lib))
    return out


def compute_laplacian_weights(center, support, degree: int, device: int = 0) -> np.ndarray:
    """Weights approximating the Laplacian at `center` = support[0] (weights.py:99-140)."""
    support = np.asarray(support, dtype=float)
    center = np.asarray(center, dtype=float)
    if support.shape[0] < monomial_count(degree):
        raise ParameterError(f"support size {support.shape[0]} below the "
                             f"{monomial_count(degree)} monomials of degree {degree}")
    if not np.array_equal(support[0], center):
        raise ParameterError("support[0] must be the stencil center")
    rows = np.arange(support.shape[0], dtype=np.int64)[None, :]
    return _assemble(support, rows, degree, device)[0]


def assemble_shapes(nodes, stencils, degree: int, workers: int = 1, device: int = 0) -> ShapeStore:
    """Weight rows for every interior node, on the GPU (weights.py:143-206).

    ``workers`` is the reference's CPU thread-pool knob, accepted and ignored.
    """
    n = stencils.n
    if n < monomial_count(degree):
        raise ParameterError(f"support size {n} below the {monomial_count(degree)} monomials "
                             f"of degree {degree}")
    interior = nodes.interior_indices.astype(np.int64)
    rows = stencils.neighbors[interior]
    try:
        weights = _assemble(nodes.positions, rows, degree, device)
    except DegenerateStencilError as exc:
        k = exc.node_index
        node = int(interior[k])
        x, y = nodes.positions[node]
        raise DegenerateStencilError(
            f"degenerate stencil at node {node} ({x:.6g}, {y:.6g})", node_index=node,
            position=(float(x), float(y))) from None
    return ShapeStore(degree=degree, interior_nodes=interior, weights=weights, stencils=stencils)
