"""Unit-disk node sets: mirror of rbffd.geometry (pkg/src/rbffd/geometry.py).

``generate_unit_disk_nodes`` runs the reference's advancing-front generator
(geometry.py:105-198) natively (csrc/nodes.cpp behind
``rbf_generate_unit_disk_nodes``) and returns the same node set bit for bit:
same count, same order, same coordinates, for every (h, seed).  The
algorithm accepts candidates in a fixed sequential order, so it runs on the
host; the Python original's cost is interpretation (~59 s at N=1e6 here), the
native one's is ~1 s.  The remaining names are re-exported from
``problem`` (the manufactured solution and the spacing helpers,
geometry.py:74-102).
"""

from __future__ import annotations

import csv
import ctypes
import operator

import numpy as np

from . import _lib
from .errors import ParameterError
from .problem import (
    NodeSet,
    _check_spacing,
    closed_form_solution,
    forcing,
    node_count_for_spacing,
    spacing_for_node_count,
)

__all__ = [
    "NodeSet",
    "closed_form_solution",
    "forcing",
    "BOUNDARY_TOL",
    "generate_unit_disk_nodes",
    "load_nodes_csv",
    "node_count_for_spacing",
    "save_nodes_csv",
    "seed_key",
    "spacing_for_node_count",
]


BOUNDARY_TOL = 1e-12  # geometry.py:23: | ||p|| - 1 | tolerance of boundary nodes


def seed_key(seed: int) -> np.ndarray:
    """32-bit little-endian words of |seed|: the init_by_array key CPython's
    random.seed(int) builds (Modules/_randommodule.c random_seed; one zero
    word for 0)."""
    n = abs(operator.index(seed))
    words = []
    while n:
        words.append(n & 0xFFFFFFFF)
        n >>= 32
    return np.asarray(words or [0], dtype=np.uint32)


def generate_unit_disk_nodes(h: float, seed: int = 0) -> NodeSet:
    """Scattered node set on the unit disk with spacing ``h`` (geometry.py:105-198).

    Boundary ring of round(2*pi/h) equidistant nodes first, then the
    advancing-front interior in acceptance order.  Raises ParameterError for
    h outside (0, 0.5) and for degenerate sets, as the reference does.
    """
    _check_spacing(h)
    h = float(h)
    key = seed_key(seed)
    lib = _lib.load()
    ptr = ctypes.c_void_p()
    n_total = ctypes.c_int64()
    n_boundary = ctypes.c_int64()
    rc = lib.rbf_generate_unit_disk_nodes(h, key.ctypes.data, int(key.size), ctypes.byref(ptr),
                                          ctypes.byref(n_total), ctypes.byref(n_boundary))
    if rc != 0:
        msg = _lib.last_error(lib)
        if msg.startswith("degenerate node set"):
            raise ParameterError(f"degenerate node set for h={h}: " + msg.split(": ", 1)[1])
        raise ParameterError(msg)
    try:
        N = n_total.value
        buf = (ctypes.c_double * (2 * N)).from_address(ptr.value)
        positions = np.frombuffer(buf, dtype=np.float64).reshape(N, 2).copy()
    finally:
        lib.rbf_free_host(ptr)
    is_boundary = np.zeros(N, dtype=bool)
    is_boundary[: n_boundary.value] = True
    return NodeSet(positions=positions, is_boundary=is_boundary, h=h)


def save_nodes_csv(nodes: NodeSet, path) -> None:
    """CSV with header x,y,kind, %.17g coordinates (geometry.py:200-206)."""
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(["x", "y", "kind"])
        for (x, y), b in zip(nodes.positions, nodes.is_boundary):
            writer.writerow([f"{x:.17g}", f"{y:.17g}", "boundary" if b else "interior"])


def load_nodes_csv(path, h: float = float("nan")) -> NodeSet:
    """Read a node set written by save_nodes_csv (geometry.py:209-219)."""
    xs, ys, kinds = [], [], []
    with open(path, newline="") as fh:
        for row in csv.DictReader(fh):
            xs.append(float(row["x"]))
            ys.append(float(row["y"]))
            kinds.append(row["kind"] == "boundary")
    positions = np.column_stack([np.asarray(xs, dtype=float), np.asarray(ys, dtype=float)])
    return NodeSet(positions=positions.reshape(-1, 2), is_boundary=np.asarray(kinds, dtype=bool), h=h)
