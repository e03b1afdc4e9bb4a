"""Host-side mirror of the reference solver API (CPU only, no device calls):
config validation, Dirichlet values, forcing, norms, stability bound -- each
checked against the reference's expressions / golden values."""

import csv

import numpy as np
import pytest

import paper_2107_03632_b200 as rb
from paper_2107_03632_b200 import problem
from oracle import oracle as orc


def test_config_validation_mirrors_reference():
    """test_solver.py:67-79."""
    with pytest.raises(rb.ParameterError):
        rb.SolveConfig(nodes=300, h=0.1)
    with pytest.raises(rb.ParameterError):
        rb.SolveConfig()
    with pytest.raises(rb.ParameterError):
        rb.SolveConfig(nodes=300, dt=-1e-6)
    with pytest.raises(rb.ParameterError):
        rb.SolveConfig(nodes=300, steps=-1)
    with pytest.raises(rb.ParameterError):
        rb.SolveConfig(nodes=300, mode="implicit")
    with pytest.raises(rb.ParameterError):
        rb.SolveConfig(nodes=300, degree=2, support_size=5)
    cfg = rb.SolveConfig(nodes=300, dt=1e-5, steps=3)
    assert cfg.as_dict(2e-5)["dt"] == 2e-5 and cfg.as_dict()["m"] == 2


def test_errors_are_catchable_as_reference_errors():
    try:
        from rbffd import errors as ref  # type: ignore
    except Exception:
        pytest.skip("reference package not importable here")
    assert issubclass(rb.InstabilityError, ref.InstabilityError)
    assert issubclass(rb.SteadyStateTimeout, ref.SteadyStateTimeout)
    assert issubclass(rb.ParameterError, ref.ParameterError)


@pytest.mark.parametrize("name", ["small", "dome", "m6"])
def test_host_prep_matches_oracle_bits(golden, manifest, name):
    nodes, _, shapes, z = golden(name)
    assert np.array_equal(rb.forcing(nodes.positions), orc.forcing(nodes.positions))
    u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    assert np.array_equal(u0, orc.apply_dirichlet(nodes, np.zeros(nodes.n_total)))
    assert rb.stability_bound(shapes) == manifest[name]["stability_bound"]
    for case, meta in manifest[name].items():
        if isinstance(meta, dict) and f"{case}__field" in z:
            assert rb.error_norms(z[f"{case}__field"], nodes) == (meta["linf"], meta["l2"])


@pytest.mark.parametrize("n_points", [problem._PAR_MIN, problem._PAR_MIN + 12345, 1_000_003])
def test_parallel_closed_form_is_bitwise(n_points):
    rng = np.random.default_rng(n_points)
    pts = rng.uniform(-1, 1, (n_points, 2))
    assert np.array_equal(problem.closed_form_solution(pts), problem._closed_form_serial(pts))
    assert np.array_equal(rb.forcing(pts), 2.0 * np.pi**2 * problem._closed_form_serial(pts))


def test_interior_rows_view_matches_gather():
    from paper_2107_03632_b200.solver import _interior_rows

    nb = np.arange(40, dtype=np.int64).reshape(10, 4)
    assert np.array_equal(_interior_rows(nb, np.arange(3, 10)), nb[np.arange(3, 10)])
    perm = np.array([9, 3, 5])
    assert np.array_equal(_interior_rows(nb, perm), nb[perm])


def test_synthetic_domain_shape():
    from paper_2107_03632_b200 import synth

    nodes, st, sh = synth.synthetic_problem(5000, 15, 2, seed=2)
    assert abs(nodes.n_total - 5000) < 150
    assert np.array_equal(sh.interior_nodes, np.arange(nodes.n_boundary, nodes.n_total))
    assert np.array_equal(st.neighbors[:, 0], np.arange(nodes.n_total))
    assert np.all(np.hypot(*nodes.positions[nodes.is_boundary].T) == pytest.approx(1.0))
    # Laplacian weights reproduce x^2 + y^2 -> 4 on every row
    rows = st.neighbors[sh.interior_nodes]
    vals = (nodes.positions[:, 0] ** 2 + nodes.positions[:, 1] ** 2)[rows]
    assert np.allclose(np.einsum("ij,ij->i", sh.weights, vals), 4.0, rtol=1e-6)


def test_benchmark_csv_and_speedup(tmp_path):
    """perf.py:110-114, :160-170 (test_perf.py:82-89, :134-142)."""
    from paper_2107_03632_b200 import perf

    r = perf.TimingReport.from_run(1000, 900, 15, 2, 10, 1, 0.5, np.zeros(1000))
    assert r.ns_per_step_node == pytest.approx(1e9 * 0.5 / (10 * 900))
    path = tmp_path / "benchmark.csv"
    perf.save_benchmark_csv([r], path)
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["N", "n", "m", "threads", "steps", "loop_seconds", "ns_per_step_node"]
    assert int(rows[1][0]) == 1000
    assert perf.speedup(10.0, 2.0) == 5.0
    with pytest.raises(rb.ParameterError):
        perf.speedup(0.0, 1.0)


def test_solution_csv_and_report_json(tmp_path, golden):
    """solver.py:262-277 (test_solver.py:321-342) on a recorded golden field."""
    import json

    nodes, _, _, z = golden("small")
    field = z["fixed50__field"]
    linf, l2 = rb.error_norms(field, nodes)
    rep = rb.SolveReport(field=field, steps=50, wall_time_s=0.01, linf=linf, l2=l2,
                         residual=1.5, config=rb.SolveConfig(nodes=300, support_size=12,
                                                             dt=1e-4, steps=50).as_dict())
    path = tmp_path / "solution.csv"
    rb.save_solution_csv(nodes, rep.field, path)
    lines = path.read_text().splitlines()
    assert lines[0] == "x,y,kind,u,exact,abs_error"
    assert len(lines) == nodes.n_total + 1
    cells = lines[1].split(",")
    assert cells[2] in ("interior", "boundary")
    assert float(cells[5]) == abs(float(cells[3]) - float(cells[4]))
    jpath = tmp_path / "report.json"
    rb.save_report_json(rep, jpath)
    loaded = json.loads(jpath.read_text())
    assert set(loaded) == {"steps", "wall_time_s", "linf", "l2", "residual", "config"}
    assert loaded["steps"] == 50 and loaded["config"]["m"] == 2


def test_problem_cache_round_trip(tmp_path, golden):
    """Binary problem cache (save_problem / load_problem, memory-mapped)."""
    nodes, stencils, shapes, _ = golden("m4")
    rb.save_problem(tmp_path / "p", nodes, stencils, shapes)
    n2, s2, sh2 = rb.load_problem(tmp_path / "p")
    assert np.array_equal(n2.positions, nodes.positions)
    assert np.array_equal(n2.is_boundary, nodes.is_boundary) and n2.h == nodes.h
    assert np.array_equal(s2.neighbors, stencils.neighbors) and s2.n == stencils.n
    assert np.array_equal(sh2.interior_nodes, shapes.interior_nodes)
    assert np.array_equal(sh2.weights, shapes.weights) and sh2.degree == shapes.degree
    # host prep is unchanged on memory-mapped arrays
    assert rb.stability_bound(sh2) == rb.stability_bound(shapes)
    assert np.array_equal(rb.forcing(n2.positions), rb.forcing(nodes.positions))


def test_parallel_host_reductions_have_numpy_bits():
    """_par: the chunked / tree-split versions of the host pieces of the solve
    path (forcing gather, error norms) equal numpy's single calls bit for bit."""
    import math

    from paper_2107_03632_b200 import _par

    rng = np.random.default_rng(7)
    for n in (17, 1000, 300_001, 2_000_003):
        v = rng.standard_normal(n)
        e = rng.standard_normal(n) * 0.25
        diff = v - e
        assert _par.error_norms(v, e) == (float(np.max(np.abs(diff))), math.sqrt(float((diff ** 2).mean())))
        x = rng.random(n) ** 2
        assert _par.pairwise_sum(x) == float(np.add.reduce(x))
        idx = rng.integers(0, n, n // 2 + 1)
        assert np.array_equal(_par.scaled_gather(2.0 * np.pi**2, x, idx), 2.0 * np.pi**2 * x[idx])


def test_parallel_stability_bound_has_numpys_bits():
    """solver.stability_bound splits rows over the pool: same bits as
    2 / np.abs(w).sum(axis=1).max() (solver.py:249-254)."""
    from paper_2107_03632_b200.problem import ShapeStore, StencilSet
    from paper_2107_03632_b200.solver import stability_bound

    rng = np.random.default_rng(5)
    for rows, n in ((10, 15), (100_000, 15), (70_001, 56)):
        w = rng.normal(size=(rows, n)) * rng.uniform(0.1, 10.0, size=(rows, 1))
        shapes = ShapeStore(degree=2, interior_nodes=np.arange(rows), weights=w,
                            stencils=StencilSet(n=n, neighbors=np.zeros((rows, n), dtype=np.int64)))
        assert stability_bound(shapes) == float(2.0 / np.abs(w).sum(axis=1).max())


def test_closed_form_and_gather_into_out_have_the_same_bits():
    """run_time_loop evaluates into page-locked scratch arrays (out=): same
    values as the allocating calls."""
    from paper_2107_03632_b200 import _par
    from paper_2107_03632_b200.problem import closed_form_solution

    rng = np.random.default_rng(3)
    for n in (10, 300_000):
        pts = rng.uniform(-1, 1, size=(n, 2))
        want = np.sin(np.pi * pts[:, 0]) * np.sin(np.pi * pts[:, 1])
        out = np.full(n, np.nan)
        assert closed_form_solution(pts, out=out) is out
        assert np.array_equal(out, want)
        idx = rng.integers(0, n, size=n // 2)
        g = np.full(idx.size, np.nan)
        _par.scaled_gather(2.0 * np.pi**2, want, idx, out=g)
        assert np.array_equal(g, 2.0 * np.pi**2 * want[idx])
