"""CPU oracle for the explicit RBF-FD time loop -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker or the CPU
baseline; the product path (paper_2107_03632_b200) never does.

Restates /root/reference/pkg:
  * ``run_time_loop``   <- src/rbffd/solver.py:168-236 (the loop lives in C:
                           rbffd_oracle.c orc_run_time_loop, solver.py:190-225)
  * ``step_kernel``     <- src/rbffd/solver.py:294-311 (C: orc_step_kernel)
  * ``python_explicit_step`` <- tests/oracles.py:66-74 (pure Python, tiny cases)
  * ``apply_dirichlet`` / ``forcing`` / ``stability_bound`` / ``error_norms``
                        <- solver.py:130-138, geometry.py:74-86, solver.py:249-254,
                           solver.py:239-246 (same numpy expressions)

Parity is PINNED: tests/test_oracle.py checks every output here bit-for-bit
against tests/golden/*.npz, which tests/golden/make_golden.py recorded from the
unmodified reference.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liborc.so"

ORC_OK, ORC_INSTABILITY, ORC_TIMEOUT = 0, 4, 5

_lib = None


def build() -> Path:
    subprocess.run(["make", "-C", str(HERE), "-s"], check=True)
    return LIB


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(str(LIB))
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        P = ctypes.POINTER
        L.orc_step_kernel.argtypes = [vp, vp, vp, vp, vp, vp, dbl, i64, i32, i64, vp, i32]
        L.orc_step_kernel.restype = None
        L.orc_run_time_loop.argtypes = [
            i64, i64, i32, vp, vp, vp, vp, vp, dbl, i64, i32, dbl, i64, i32, i64, i32,
            vp, P(i64), P(dbl), P(i32), P(i64), P(dbl), P(dbl),
        ]
        L.orc_run_time_loop.restype = i32
        L.orc_max_threads.restype = i32
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().orc_max_threads())


def _c(a, dtype):
    return np.ascontiguousarray(np.asarray(a), dtype=dtype)


# ---- host prep, restated ---------------------------------------------------
def closed_form_solution(points):  # geometry.py:74-81
    p = np.asarray(points, dtype=float)
    return np.sin(np.pi * p[..., 0]) * np.sin(np.pi * p[..., 1])


def forcing(points):  # geometry.py:84-86
    return 2.0 * np.pi**2 * closed_form_solution(points)


def apply_dirichlet(nodes, values):  # solver.py:130-138
    out = np.asarray(values, dtype=float).copy()
    bidx = np.flatnonzero(nodes.is_boundary)
    out[bidx] = closed_form_solution(nodes.positions[bidx])
    return out


def stability_bound(weights) -> float:  # solver.py:249-254
    return float(2.0 / np.abs(weights).sum(axis=1).max())


def error_norms(values, positions):  # solver.py:239-246
    diff = np.asarray(values, dtype=float) - closed_form_solution(positions)
    return float(np.max(np.abs(diff))), float(math.sqrt(float((diff**2).mean())))


# ---- the update -------------------------------------------------------------
def python_explicit_step(u1, interior, neighbor_rows, weights, f_interior, dt):
    """tests/oracles.py:66-74: plain-Python loop, same summation order."""
    u2 = np.array(u1, dtype=float, copy=True)
    for k in range(len(interior)):
        acc = 0.0
        for j in range(neighbor_rows.shape[1]):
            acc += weights[k, j] * u1[neighbor_rows[k, j]]
        u2[interior[k]] = u1[interior[k]] + dt * (f_interior[k] + acc)
    return u2


def step_kernel(u1, u2, interior, rows, weights, f_int, dt, chunk=1024, threads=1):
    """solver.py:294-311 in C; writes u2[interior] in place, returns flags."""
    interior = _c(interior, np.int64)
    rows = _c(rows, np.int64)
    weights = _c(weights, np.float64)
    f_int = _c(f_int, np.float64)
    u1 = _c(u1, np.float64)
    assert u2.dtype == np.float64 and u2.flags.c_contiguous
    n_rows, width = weights.shape
    flags = np.zeros(max(1, (n_rows + chunk - 1) // chunk), dtype=np.uint8)
    lib().orc_step_kernel(
        u1.ctypes.data, u2.ctypes.data, interior.ctypes.data, rows.ctypes.data,
        weights.ctypes.data, f_int.ctypes.data, float(dt), int(n_rows), int(width),
        int(chunk), flags.ctypes.data, int(threads),
    )
    return flags


def explicit_step(u1, shapes, f, dt, threads=1):
    """solver.py:141-165 through the C kernel; returns (u2, bad)."""
    u1 = np.asarray(u1, dtype=float)
    u2 = u1.copy()
    interior = shapes.interior_nodes
    rows = np.ascontiguousarray(shapes.stencils.neighbors[interior])
    f_int = np.ascontiguousarray(np.asarray(f, dtype=float)[interior])
    flags = step_kernel(u1, u2, interior, rows, shapes.weights, f_int, dt, threads=threads)
    return u2, bool(flags.any())


def run_arrays(N, interior, rows, weights, f_int, u0, dt, *, steps=0, steady=False, tol=1e-9,
               max_steps=1_000_000, copy_back=False, chunk=1024, threads=None):
    """The loop of solver.py:190-225 over raw arrays. Returns a dict."""
    threads = max_threads() if threads is None else threads
    interior = _c(interior, np.int64)
    rows = _c(rows, np.int64)
    weights = _c(weights, np.float64)
    f_int = _c(f_int, np.float64)
    u0 = _c(u0, np.float64)
    field = np.empty(int(N), dtype=np.float64)
    sd, res, hr, bad, mx, sec = (ctypes.c_int64(), ctypes.c_double(), ctypes.c_int32(),
                                 ctypes.c_int64(), ctypes.c_double(), ctypes.c_double())
    n_rows, width = weights.shape
    rc = lib().orc_run_time_loop(
        int(N), int(n_rows), int(width), interior.ctypes.data, rows.ctypes.data,
        weights.ctypes.data, f_int.ctypes.data, u0.ctypes.data, float(dt), int(steps),
        int(bool(steady)), float(tol), int(max_steps), int(bool(copy_back)), int(chunk),
        int(threads), field.ctypes.data, ctypes.byref(sd), ctypes.byref(res), ctypes.byref(hr),
        ctypes.byref(bad), ctypes.byref(mx), ctypes.byref(sec),
    )
    if rc < 0:
        raise MemoryError("oracle allocation failed")
    out = dict(status=rc, field=field, steps=sd.value, residual=res.value if hr.value else None,
               seconds=sec.value, threads=threads)
    if rc == ORC_INSTABILITY:
        out.update(step=bad.value, max_abs=mx.value)
    return out


def run_time_loop(nodes, shapes, *, dt=None, steps=0, mode="fixed", tol=1e-9,
                  max_steps=1_000_000, copy_back=False, threads=None):
    """solver.py:168-236 end to end (host prep + C loop + norms)."""
    interior = shapes.interior_nodes
    rows = np.ascontiguousarray(shapes.stencils.neighbors[interior])
    f_int = np.ascontiguousarray(forcing(nodes.positions[interior]))
    u0 = apply_dirichlet(nodes, np.zeros(nodes.positions.shape[0]))
    dt = dt if dt is not None else 0.5 * stability_bound(shapes.weights)
    out = run_arrays(nodes.positions.shape[0], interior, rows, shapes.weights, f_int, u0, dt,
                     steps=steps, steady=(mode == "steady"), tol=tol, max_steps=max_steps,
                     copy_back=copy_back, threads=threads)
    out["dt"] = dt
    if out["status"] == ORC_OK:
        out["linf"], out["l2"] = error_norms(out["field"], nodes.positions)
    return out


if os.environ.get("RBFFD_ORACLE_BUILD"):  # pragma: no cover
    build()
