"""Generate the golden fixtures for the parity suite from the UNMODIFIED reference.

Test infrastructure only. Run in the build container (where /root/reference
exists); the GPU box never runs this script, it only reads the committed
``*.npz`` files it writes.

    python tests/golden/make_golden.py

Every fixture stores one problem exactly as the reference builds it
(``generate_unit_disk_nodes`` -> ``build_stencils`` -> ``assemble_shapes``,
``pkg/src/rbffd/solver.py:122-127``) together with the reference's own outputs
on that problem: fields from ``explicit_step`` (solver.py:141-165) and
``run_time_loop`` (solver.py:168-236), step counts, residuals, error norms and
exception payloads (errors.py:21-36).  The configurations are the ones the
reference tests use:

* ``hand``    -- the 5-node hand problem, test_solver.py:45-64 / :112-123 (KAT)
* ``small``   -- N~300, seed 2, n=12, m=2 (test_solver.py:31-36)
* ``dome``    -- the paper's Fig. 1 case, N=1025, seed 1, n=15, m=2
                 (test_acceptance.py:43-49): 1e5 steps at dt=1e-6 and steady 1e-9
* ``crit6``   -- acceptance criterion 6, N~2000, seed 6, n=15, dt=1e-5, 100 steps
                 (test_acceptance.py:181-205)
* ``m4``/``m6`` -- wider stencils (n=30 / n=56, degrees 4 / 6) at N~3000
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/rbffd_numba_cache")
sys.path[:0] = [str(REF / "src"), str(REF / "tests")]

from rbffd.errors import InstabilityError, SteadyStateTimeout  # noqa: E402
from rbffd.geometry import (  # noqa: E402
    NodeSet,
    forcing,
    generate_unit_disk_nodes,
    spacing_for_node_count,
)
from rbffd.neighborhoods import StencilSet, build_stencils  # noqa: E402
from rbffd.solver import (  # noqa: E402
    SolveConfig,
    apply_dirichlet,
    explicit_step,
    run_time_loop,
    stability_bound,
)
from rbffd.weights import ShapeStore, assemble_shapes  # noqa: E402

OUT = Path(__file__).resolve().parent


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def problem_arrays(nodes, stencils, shapes):
    return dict(
        positions=nodes.positions,
        is_boundary=nodes.is_boundary,
        h=np.float64(nodes.h),
        neighbors=stencils.neighbors.astype(np.int32),
        interior=shapes.interior_nodes.astype(np.int64),
        weights=shapes.weights,
        degree=np.int64(shapes.degree),
    )


def pipeline(target, seed, n, m):
    nodes = generate_unit_disk_nodes(spacing_for_node_count(target), seed=seed)
    stencils = build_stencils(nodes, n)
    shapes = assemble_shapes(nodes, stencils, m, workers=8)
    return nodes, stencils, shapes


def record_run(arrays, meta, key, config, nodes, shapes, copy_back=False):
    """Run the reference time loop and record field + scalars under `key`."""
    try:
        rep = run_time_loop(config, nodes, shapes, copy_back=copy_back)
    except InstabilityError as exc:
        meta[key] = dict(error="InstabilityError", step=exc.step, max_abs=exc.max_abs)
        return
    except SteadyStateTimeout as exc:
        meta[key] = dict(error="SteadyStateTimeout", steps=exc.steps, residual=exc.residual)
        return
    arrays[f"{key}__field"] = rep.field
    meta[key] = dict(
        steps=rep.steps,
        residual=rep.residual,
        linf=rep.linf,
        l2=rep.l2,
        dt=rep.config["dt"],
        mode=config.mode,
        tol=config.tol,
        max_steps=config.max_steps,
        config_steps=config.steps,
        copy_back=copy_back,
        digest=digest(rep.field),
        ref_wall_time_s=rep.wall_time_s,
    )


def hand_fixture():
    # test_solver.py:45-64 -- 4 boundary corners, 1 interior center
    positions = np.array([[0.6, 0.0], [0.0, 0.6], [-0.6, 0.0], [0.0, -0.6], [0.05, 0.02]])
    boundary = np.array([True, True, True, True, False])
    nodes = NodeSet(positions=positions, is_boundary=boundary, h=0.6)
    neighbors = np.array(
        [[0, 1, 2, 3, 4], [1, 0, 2, 3, 4], [2, 0, 1, 3, 4], [3, 0, 1, 2, 4], [4, 0, 1, 2, 3]],
        dtype=np.int64,
    )
    stencils = StencilSet(n=5, neighbors=neighbors)
    shapes = ShapeStore(
        degree=2,
        interior_nodes=np.array([4], dtype=np.int64),
        weights=np.array([[-11.0, 2.5, 2.5, 3.0, 3.0]]),
        stencils=stencils,
    )
    arrays = problem_arrays(nodes, stencils, shapes)
    meta = {}
    u1 = np.array([0.1, -0.2, 0.3, 0.4, 0.25])
    f = forcing(nodes.positions)
    arrays["kat__u1"] = u1
    arrays["kat__u2"] = explicit_step(u1, shapes, f, 3e-3)
    meta["kat"] = dict(dt=3e-3)
    return arrays, meta


def small_fixture():
    nodes, stencils, shapes = pipeline(300, 2, 12, 2)
    arrays = problem_arrays(nodes, stencils, shapes)
    meta = {"stability_bound": stability_bound(shapes)}
    f = forcing(nodes.positions)
    rng = np.random.default_rng(0)
    u1 = apply_dirichlet(nodes, rng.normal(size=nodes.n_total))
    arrays["step_rand__u1"] = u1
    arrays["step_rand__u2"] = explicit_step(u1, shapes, f, 1e-4)
    meta["step_rand"] = dict(dt=1e-4)
    # explicit blow-up (test_solver.py:162-168)
    huge = np.full(nodes.n_total, 1e308)
    try:
        explicit_step(huge, shapes, f, 1.0)
    except InstabilityError as exc:
        meta["step_blowup"] = dict(dt=1.0, fill=1e308, max_abs=exc.max_abs)
    base = dict(degree=2, support_size=12, nodes=300, tol=1e-9, seed=2)
    record_run(arrays, meta, "fixed50", SolveConfig(mode="fixed", steps=50, dt=1e-4, **base), nodes, shapes)
    record_run(arrays, meta, "fixed120", SolveConfig(mode="fixed", steps=120, dt=1e-4, **base), nodes, shapes)
    record_run(arrays, meta, "fixed120_copy", SolveConfig(mode="fixed", steps=120, dt=1e-4, **base), nodes, shapes, copy_back=True)
    record_run(arrays, meta, "steady", SolveConfig(mode="steady", **base), nodes, shapes)
    record_run(arrays, meta, "timeout", SolveConfig(mode="steady", max_steps=5, **base), nodes, shapes)
    record_run(arrays, meta, "unstable", SolveConfig(mode="fixed", steps=500, dt=1.0, **base), nodes, shapes)
    record_run(arrays, meta, "zero", SolveConfig(mode="fixed", steps=0, dt=1e-5, **base), nodes, shapes)
    return arrays, meta


def dome_fixture():
    nodes, stencils, shapes = pipeline(1027, 1, 15, 2)
    arrays = problem_arrays(nodes, stencils, shapes)
    meta = {"stability_bound": stability_bound(shapes)}
    base = dict(degree=2, support_size=15, nodes=1027, seed=1)
    record_run(arrays, meta, "paper", SolveConfig(mode="fixed", steps=100_000, dt=1e-6, **base), nodes, shapes)
    record_run(arrays, meta, "steady", SolveConfig(mode="steady", tol=1e-9, **base), nodes, shapes)
    return arrays, meta


def crit6_fixture():
    nodes, stencils, shapes = pipeline(2000, 6, 15, 2)
    arrays = problem_arrays(nodes, stencils, shapes)
    meta = {"stability_bound": stability_bound(shapes)}
    cfg = SolveConfig(degree=2, support_size=15, nodes=2000, dt=1e-5, steps=100, seed=6)
    record_run(arrays, meta, "fixed100", cfg, nodes, shapes)
    record_run(arrays, meta, "fixed100_copy", cfg, nodes, shapes, copy_back=True)
    return arrays, meta


def wide_fixture(target, seed, n, m, steps):
    nodes, stencils, shapes = pipeline(target, seed, n, m)
    arrays = problem_arrays(nodes, stencils, shapes)
    meta = {"stability_bound": stability_bound(shapes)}
    cfg = SolveConfig(degree=m, support_size=n, nodes=target, dt=None, steps=steps, seed=seed)
    record_run(arrays, meta, f"fixed{steps}", cfg, nodes, shapes)
    return arrays, meta


def main():
    fixtures = {
        "hand": hand_fixture,
        "small": small_fixture,
        "dome": dome_fixture,
        "crit6": crit6_fixture,
        "m4": lambda: wide_fixture(3000, 4, 30, 4, 200),
        "m6": lambda: wide_fixture(3000, 5, 56, 6, 100),
    }
    manifest = {}
    for name, fn in fixtures.items():
        t0 = time.perf_counter()
        arrays, meta = fn()
        np.savez_compressed(OUT / f"{name}.npz", **arrays)
        manifest[name] = meta
        print(f"{name}: N={arrays['positions'].shape[0]} N_i={arrays['interior'].size} "
              f"n={arrays['weights'].shape[1]} ({time.perf_counter() - t0:.1f}s)")
    import numba
    import scipy

    manifest["_provenance"] = dict(
        reference="/root/reference/pkg (rbffd 0.1.0), unmodified",
        numpy=np.__version__,
        scipy=scipy.__version__,
        numba=numba.__version__,
        script="tests/golden/make_golden.py",
    )
    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
