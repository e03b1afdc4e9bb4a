"""Scattered-node unit-disk domains for the benchmark configs.

Nodes (``nodes=``):

* ``"reference"`` (default): the reference's own advancing-front node set
  (geometry.py:105-198) for (spacing_for_node_count(target), seed), produced
  bit-identically by the native generator (geometry.generate_unit_disk_nodes,
  csrc/nodes.cpp) -- ~1 s per 1e6 nodes instead of the Python original's
  ~1 min, so C2..C5 run on the exact node sets SURVEY.md 8(d) prefers;
* ``"hex"``: the faster fallback SURVEY.md 8(d) also accepts, a seeded jittered
  hexagonal fill (disk_nodes below):

* boundary: the reference's equidistant ring, same formula
  (n_b = floor(2 pi / h + 0.5), theta_k = 2 pi k / n_b; geometry.py:135-141);
* interior: a seeded, jittered hexagonal fill of the disk at the spacing that
  hits the target node count, ordered ring-by-ring from the boundary inwards
  like the reference's advancing front (interior ids = [n_b, N), row k updates
  node n_b + k, stencil entry 0 = self, as in generated reference sets);
* supports: exact kNN with scipy's cKDTree (neighborhoods.py:51-94 uses the
  same tree), ties ordered by (distance, index);
* weights: the reference's PHS r^3 + monomial saddle system, restated from
  weights.py:218-259 (shift to the centre, scale by the support radius,
  solve, rescale by 1/r^2), batched with numpy/LAPACK over a thread pool.

The time loop is insensitive to how nodes were placed; what matters for
throughput is N, n and the index locality, and for stability the weights'
Gershgorin bound, which these are (same operator, same scaling).
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .problem import NodeSet, ShapeStore, StencilSet, monomial_count, spacing_for_node_count


def _exponents(degree: int) -> np.ndarray:
    """Graded-lex monomial exponents, x-exponent descending (weights.py:46-57)."""
    return np.asarray([(a, t - a) for t in range(degree + 1) for a in range(t, -1, -1)],
                      dtype=np.int64)


def disk_nodes(target: int, seed: int = 1) -> NodeSet:
    """Jittered-hex scattered node set on the unit disk with ~`target` nodes."""
    h = spacing_for_node_count(target)
    n_b = int(math.floor(2.0 * math.pi / h + 0.5))
    theta = 2.0 * math.pi * np.arange(n_b) / n_b
    bx, by = np.cos(theta), np.sin(theta)
    rng = np.random.default_rng(seed)
    r_in = 1.0 - 0.5 * h
    want = max(1, target - n_b)
    # hexagonal lattice spacing a for `want` points in the disk of radius r_in
    a = math.sqrt(2.0 * math.pi * r_in * r_in / (math.sqrt(3.0) * want))
    ny = int(math.ceil(r_in / (a * math.sqrt(3.0) / 2.0))) + 1
    nx = int(math.ceil(r_in / a)) + 2
    jj, ii = np.meshgrid(np.arange(-ny, ny + 1), np.arange(-nx, nx + 1), indexing="ij")
    x = (ii + 0.5 * (jj & 1)) * a
    y = jj * (a * math.sqrt(3.0) / 2.0)
    x = x.ravel() + rng.uniform(-0.15 * a, 0.15 * a, x.size)
    y = y.ravel() + rng.uniform(-0.15 * a, 0.15 * a, y.size)
    r = np.hypot(x, y)
    keep = r < r_in
    x, y, r = x[keep], y[keep], r[keep]
    # advancing-front-like order: rings of width ~h from the boundary inwards,
    # counter-clockwise within a ring
    ring = np.floor((1.0 - r) / h).astype(np.int64)
    ang = np.arctan2(y, x)
    order = np.lexsort((ang, ring))
    positions = np.empty((n_b + order.size, 2))
    positions[:n_b, 0], positions[:n_b, 1] = bx, by
    positions[n_b:, 0], positions[n_b:, 1] = x[order], y[order]
    is_boundary = np.zeros(positions.shape[0], dtype=bool)
    is_boundary[:n_b] = True
    return NodeSet(positions=positions, is_boundary=is_boundary, h=h)


def knn_stencils(nodes: NodeSet, n: int, workers: int = -1) -> StencilSet:
    """Exact n nearest neighbours, self first, ties by (distance, index):
    neighborhoods.py:51-94 restated (cKDTree with the reference's 8-entry
    tie look-ahead; rows whose cutoff tie group reaches the look-ahead are
    resolved by an exact scan)."""
    from scipy.spatial import cKDTree

    total = nodes.positions.shape[0]
    positions = nodes.positions
    tree = cKDTree(positions)
    k_query = min(total, n + 8)  # neighborhoods.py:22 _TIE_PAD
    dist, idx = tree.query(positions, k=k_query, workers=workers)
    if dist.ndim == 1:
        dist, idx = dist[:, None], idx[:, None]
    order = np.lexsort((idx, dist))
    dist = np.take_along_axis(dist, order, axis=1)
    idx = np.take_along_axis(idx, order, axis=1)
    if k_query < total:
        for i in np.flatnonzero(dist[:, n - 1] == dist[:, k_query - 1]):
            d = positions - positions[i]
            di = np.sqrt(d[:, 0] ** 2 + d[:, 1] ** 2)
            idx[i, :n] = np.lexsort((np.arange(total), di))[:n]
    return StencilSet(n=n, neighbors=np.ascontiguousarray(idx[:, :n], dtype=np.int64))


def _weights_batch(supports: np.ndarray, expo: np.ndarray) -> np.ndarray:
    """PHS r^3 + monomials saddle solve for a (C, n, 2) stack (weights.py:218-259)."""
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
    for k, (ea, eb) in enumerate(expo):
        if (ea, eb) in ((2, 0), (0, 2)):
            lap0[k] = 2.0
    rhs[:, n:] = lap0
    sol = np.linalg.solve(mat, rhs[:, :, None])[:, :, 0]
    return sol[:, :n] / radius[:, None] ** 2


def laplacian_weights(nodes: NodeSet, stencils: StencilSet, degree: int,
                      workers: int | None = None) -> ShapeStore:
    n = stencils.n
    if n < monomial_count(degree):
        raise ValueError(f"support size {n} below the monomials of degree {degree}")
    expo = _exponents(degree)
    interior = nodes.interior_indices.astype(np.int64)
    n_rows = interior.size
    weights = np.empty((n_rows, n))
    size = n + expo.shape[0]
    chunk = max(32, min(8192, 4_000_000 // (size * size)))
    spans = [(lo, min(lo + chunk, n_rows)) for lo in range(0, n_rows, chunk)]

    def run(span):
        lo, hi = span
        sup = nodes.positions[stencils.neighbors[interior[lo:hi]]]
        weights[lo:hi] = _weights_batch(sup, expo)

    workers = workers or min(32, os.cpu_count() or 1)
    if workers > 1 and len(spans) > 1:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            list(pool.map(run, spans))
    else:
        for s in spans:
            run(s)
    return ShapeStore(degree=degree, interior_nodes=interior, weights=weights, stencils=stencils)


def synthetic_problem(target: int, n: int, degree: int, seed: int = 1, weights: str = "cpu",
                      knn: str | None = None, nodes: str = "reference"):
    """(nodes, stencils, shapes) of a synthetic scattered-node disk.

    weights="cpu": numpy/LAPACK restatement above; "gpu": the device assembly
    (paper_2107_03632_b200.weights, minutes -> seconds at 1e7 rows).
    knn="cpu": scipy cKDTree; "gpu": the exact device kNN (default when the
    weights are assembled on the GPU).  nodes="reference": the reference's
    advancing-front set (native, bit-identical); "hex": jittered hex fill."""
    if nodes == "reference":
        from .geometry import generate_unit_disk_nodes

        nodes = generate_unit_disk_nodes(spacing_for_node_count(target), seed)
    elif nodes == "hex":
        nodes = disk_nodes(target, seed)
    else:
        raise ValueError(f"nodes must be 'reference' or 'hex', got {nodes!r}")
    knn = knn or ("gpu" if weights == "gpu" else "cpu")
    if knn == "gpu":
        from .neighborhoods import build_stencils

        stencils = build_stencils(nodes, n)
    else:
        stencils = knn_stencils(nodes, n)
    if weights == "gpu":
        from .weights import assemble_shapes

        shapes = assemble_shapes(nodes, stencils, degree)
    else:
        shapes = laplacian_weights(nodes, stencils, degree)
    return nodes, stencils, shapes
