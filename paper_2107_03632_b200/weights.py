"""GPU assembly of the Laplacian weight rows.

Mirrors the reference API of pkg/src/rbffd/weights.py -- ``assemble_shapes``
(:143-206) and ``compute_laplacian_weights`` (:99-140) -- over the C ABI
``rbf_assemble_weights``: one warp per (n+M)^2 saddle system on the device.
Results agree with the reference's LAPACK solve to rounding (the reference
pins weights by polynomial reproduction, test_weights.py:51-104), not bit for
bit; the time loop's bitwise parity is always stated on identical weights.

Condition guard (weights.py:29, :183-192, :250-258).  The reference rejects a
stencil whose np.linalg.cond (2-norm) exceeds COND_LIMIT = 1e14.  The device
estimates the 1-norm condition from its LU factors and flags rows (see
include/rbffd_b200.h, rbf_assemble_weights); only the flagged rows -- none
in well-shaped node sets, whose conditions are 1e3-1e7 -- get the exact
2-norm test here, on the reference's own matrix (same construction, same
np.linalg.cond), in row order, so the first offending node is the one the
reference names.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import DegenerateStencilError, DeviceError, ParameterError
from .problem import ShapeStore, monomial_count

COND_LIMIT = 1e14  # weights.py:29

__all__ = ["COND_LIMIT", "DegenerateStencilError", "assemble_shapes", "compute_laplacian_weights",
           "saddle_condition"]


def _exponents(degree: int) -> np.ndarray:
    return np.asarray([(a, t - a) for t in range(degree + 1) for a in range(t, -1, -1)], dtype=np.int64)


def saddle_condition(supports: np.ndarray, degree: int) -> np.ndarray:
    """np.linalg.cond of the reference's saddle matrices for a (C, n, 2)
    stack of supports (the matrix of weights.py:228-245, the test of :250)."""
    supports = np.asarray(supports, dtype=float)
    count, n, _ = supports.shape
    expo = _exponents(degree)
    size = n + expo.shape[0]
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
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.linalg.cond(mat)


def _resolve_flagged(status: np.ndarray, supports_of, degree: int):
    """First flagged row that fails the reference's test, in row order:
    (k, cond) or None.  status 1 rows get the exact check; status 2 rows
    (zero pivot / non-finite / certain kappa_2 > 1e14) always fail."""
    for k in np.flatnonzero(status):
        k = int(k)
        cond = float(saddle_condition(supports_of(k)[None], degree)[0])
        if status[k] == 2 or not cond <= COND_LIMIT:
            return k, cond
    return None


def _assemble(positions: np.ndarray, rows: np.ndarray, degree: int, device: int = 0):
    """(weights, status) from the device; status is None when no row was flagged."""
    lib = _lib.load()
    positions = np.ascontiguousarray(positions, dtype=np.float64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    n_rows, n = rows.shape
    out = np.empty((n_rows, n), dtype=np.float64)
    status = np.zeros(n_rows, dtype=np.uint8)
    bad = ctypes.c_int64(-1)
    rc = lib.rbf_assemble_weights(positions.ctypes.data, positions.shape[0], rows.ctypes.data, n_rows,
                                  n, int(degree), out.ctypes.data, ctypes.byref(bad), status.ctypes.data,
                                  int(device))
    if rc == _lib.RBF_ERR_ILLCOND:
        return out, status
    if rc == _lib.RBF_ERR_PARAM:
        raise ParameterError(_lib.last_error(lib))
    if rc != _lib.RBF_OK:
        raise DeviceError(_lib.last_error(lib))
    return out, None


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
    w, status = _assemble(support, rows, degree, device)
    if status is not None:
        hit = _resolve_flagged(status, lambda k: support, degree)
        if hit is not None:
            raise DegenerateStencilError(
                f"degenerate stencil at ({center[0]:.6g}, {center[1]:.6g}): "
                f"condition estimate {hit[1]:.3e}",
                position=(float(center[0]), float(center[1])))
    return w[0]


def _raise_for_node(nodes, interior, k, cond):
    node = int(interior[k])
    x, y = nodes.positions[node]
    raise DegenerateStencilError(
        f"degenerate stencil at node {node} ({x:.6g}, {y:.6g}): condition estimate {cond:.3e}",
        node_index=node, position=(float(x), float(y)))


def assemble_shapes(nodes, stencils, degree: int, workers: int = 1, device: int = 0) -> ShapeStore:
    """Weight rows for every interior node, on the GPU (weights.py:143-206).

    ``workers`` is the reference's CPU thread-pool knob, accepted and ignored.
    Raises DegenerateStencilError naming the first offending node, like the
    reference.
    """
    n = stencils.n
    if n < monomial_count(degree):
        raise ParameterError(f"support size {n} below the {monomial_count(degree)} monomials "
                             f"of degree {degree}")
    interior = nodes.interior_indices.astype(np.int64)
    from .solver import _interior_rows

    rows = _interior_rows(stencils.neighbors, interior)  # a view when interior = [B, N): no 8n B/row copy
    weights, status = _assemble(nodes.positions, rows, degree, device)
    if status is not None:
        hit = _resolve_flagged(status, lambda k: nodes.positions[rows[k]], degree)
        if hit is not None:
            _raise_for_node(nodes, interior, *hit)
    return ShapeStore(degree=degree, interior_nodes=interior, weights=weights, stencils=stencils)
