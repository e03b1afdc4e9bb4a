"""GPU weight assembly against the reference's own
weight tests (pkg/tests/test_weights.py:49-104) and the reference's weights
recorded in tests/golden (assembled by LAPACK; agreement to rounding)."""

import math

import numpy as np
import pytest

import paper_2107_03632_b200 as rb
from paper_2107_03632_b200 import weights as gw
from paper_2107_03632_b200.solver import Plan
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def scattered_stencil(rng, n, min_sep=None):
    """tests/oracles.py:87-98: n well-separated points in the unit disk, centre first."""
    if min_sep is None:
        min_sep = 0.7 / np.sqrt(n)
    points = [np.zeros(2)]
    while len(points) < n:
        c = rng.uniform(-1.0, 1.0, 2)
        if c @ c > 1.0:
            continue
        if all(np.hypot(*(c - q)) >= min_sep for q in points):
            points.append(c)
    return np.asarray(points)


def monomial_laplacian(a, b, x, y):  # tests/oracles.py:77-84
    out = 0.0
    if a >= 2:
        out += a * (a - 1) * x ** (a - 2) * y**b
    if b >= 2:
        out += b * (b - 1) * x**a * y ** (b - 2)
    return out


@pytest.fixture
def rng():
    return np.random.default_rng(20240811)


def test_weights_sum_to_zero(rng):
    for _ in range(10):
        s = scattered_stencil(rng, 12)
        w = gw.compute_laplacian_weights(s[0], s, 2)
        assert abs(w.sum()) <= 1e-9 * np.abs(w).max()


def test_reproduces_laplacian_of_quadratic(rng):
    for _ in range(10):
        s = scattered_stencil(rng, 12)
        w = gw.compute_laplacian_weights(s[0], s, 2)
        assert w @ (s[:, 0] ** 2 + s[:, 1] ** 2) == pytest.approx(4.0, rel=1e-7)


@pytest.mark.parametrize("degree", [2, 4, 6])
def test_polynomial_reproduction_at_higher_degrees(rng, degree):
    n = 2 * math.comb(degree + 2, 2)
    expo = [(a, t - a) for t in range(degree + 1) for a in range(t, -1, -1)]
    for _ in range(5):
        centre = rng.uniform(-0.3, 0.3, 2)
        s = centre + scattered_stencil(rng, n)
        w = gw.compute_laplacian_weights(s[0], s, degree)
        local = s - s[0]
        for a, b in expo:
            target = monomial_laplacian(a, b, 0.0, 0.0)
            assert abs(w @ (local[:, 0] ** a * local[:, 1] ** b) - target) <= 1e-7 * max(1.0, abs(target))


@pytest.mark.parametrize("scale", [0.1, 10.0])
def test_scaling_covariance(rng, scale):
    s = scattered_stencil(rng, 15)
    w = gw.compute_laplacian_weights(s[0], s, 2)
    ws = gw.compute_laplacian_weights(scale * s[0], scale * s, 2)
    assert np.max(np.abs(ws - w / scale**2)) <= 1e-9 * np.abs(w / scale**2).max()


def test_degenerate_stencil_is_reported():
    s = np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0], [3.0, 0.0], [4.0, 0.0], [5.0, 0.0], [6.0, 0.0]])
    with pytest.raises(gw.DegenerateStencilError):
        gw.compute_laplacian_weights(s[0], s, 2)  # collinear: the y monomials vanish


@pytest.mark.parametrize("name", ["small", "dome", "crit6", "m4", "m6"])
def test_assembled_shapes_match_reference_weights(golden, name):
    nodes, stencils, shapes, _ = golden(name)
    got = gw.assemble_shapes(nodes, stencils, shapes.degree)
    assert np.array_equal(got.interior_nodes, shapes.interior_nodes)
    ref = shapes.weights
    scale = np.abs(ref).max(axis=1, keepdims=True)
    err = float(np.max(np.abs(got.weights - ref) / scale))
    assert err <= 1e-7, err
    # the derived time step agrees to rounding as well
    assert rb.stability_bound(got) == pytest.approx(rb.stability_bound(shapes), rel=1e-9)


def test_plan_with_device_assembled_weights_is_bitwise(golden):
    """Weights assembled inside the plan (never on the host) give the same
    loop bits as a plan built from the same weights downloaded to the host."""
    nodes, stencils, shapes, _ = golden("m4")
    host = gw.assemble_shapes(nodes, stencils, shapes.degree)
    interior = shapes.interior_nodes
    rows = stencils.neighbors[interior]
    f_int = rb.forcing(nodes.positions[interior])
    u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    a = Plan.assembled(nodes.n_total, interior, rows, nodes.positions, f_int, shapes.degree)
    assert 2.0 / a.weight_row_sum_max() == rb.stability_bound(host)  # numpy's row-sum bits
    dt = rb.stability_bound(host) * 0.5
    a.set_field(u0)
    ra = a.run(dt, steps=150)
    want = orc.run_time_loop(nodes, host, dt=dt, steps=150)
    assert np.array_equal(a.get_field(), want["field"]) and ra.residual == want["residual"]


def _wavy_line(eps, n=12):
    """n points on a line bent by eps * sin: the saddle matrix's y columns
    shrink with eps, so its 2-norm condition grows like eps^-4 without any
    exact zero pivot (1e-4 -> 1.39e14, just above COND_LIMIT)."""
    x = np.linspace(0.0, 1.0, n)
    s = np.column_stack([x, eps * np.sin(7.0 * x + 1.0)])
    s[0] = 0.0
    return s


@pytest.mark.parametrize("eps", [1e-4, 1e-6, 0.0])
def test_ill_conditioned_stencil_is_rejected(eps):
    """weights.py:29, :183-192: cond > 1e14 raises DegenerateStencilError even
    when elimination meets no zero pivot (eps=1e-4: host re-check of a
    flagged row; 1e-6: certain on the device; 0: exactly collinear)."""
    s = _wavy_line(eps)
    cond = gw.saddle_condition(s[None], 2)[0]
    assert not cond <= gw.COND_LIMIT
    with pytest.raises(gw.DegenerateStencilError) as ei:
        gw.compute_laplacian_weights(s[0], s, 2)
    assert ei.value.position == (0.0, 0.0)
    assert issubclass(gw.DegenerateStencilError, RuntimeError)


def test_flagged_but_acceptable_stencil_is_kept():
    """kappa_2 ~ 9e12 < 1e14: the device flags it (1-norm estimate above 1e10),
    the exact check accepts it, and the weights are the reference's to
    rounding (polynomial reproduction of the quadratic)."""
    s = _wavy_line(2e-4)
    cond = gw.saddle_condition(s[None], 2)[0]
    assert 1e12 < cond <= gw.COND_LIMIT
    w = gw.compute_laplacian_weights(s[0], s, 2)
    assert np.all(np.isfinite(w))
    assert abs(w.sum()) <= 1e-6 * np.abs(w).max()


def test_assemble_names_degenerate_node():
    """pkg/tests/test_weights.py:128-141 on the device path: a line of nodes
    (every stencil collinear); the error names the node and its position,
    through assemble_shapes and through a plan that assembles on the device."""
    from paper_2107_03632_b200.neighborhoods import build_stencils
    from paper_2107_03632_b200.problem import NodeSet

    positions = np.column_stack([np.linspace(-1, 1, 9), np.zeros(9)])
    boundary = np.zeros(9, dtype=bool)
    boundary[[0, 1, 2, 8]] = True
    nodes = NodeSet(positions=positions, is_boundary=boundary, h=0.25)
    stencils = build_stencils(nodes, 7)
    with pytest.raises(gw.DegenerateStencilError) as excinfo:
        gw.assemble_shapes(nodes, stencils, 2)
    err = excinfo.value
    assert err.node_index is not None
    assert str(err.node_index) in str(err)
    assert err.position is not None
    assert err.node_index == int(nodes.interior_indices[0])  # the first one, like the reference
    interior = nodes.interior_indices.astype(np.int64)
    with pytest.raises(gw.DegenerateStencilError) as excinfo:
        Plan.assembled(nodes.n_total, interior, stencils.neighbors[interior], positions,
                       rb.forcing(positions[interior]), 2)
    assert excinfo.value.node_index == err.node_index


def test_assembled_plan_accepts_flagged_rows_after_the_exact_check(golden):
    """A node set with one slightly ill-conditioned (but acceptable) stencil:
    the plan assembles, the flagged row passes the host's exact test, and the
    loop equals the oracle on the host-assembled weights."""
    nodes, stencils, shapes, _ = golden("small")
    interior = shapes.interior_nodes.astype(np.int64)
    pos = nodes.positions.copy()
    # squeeze the first interior stencil towards a wavy line around its centre
    nb = stencils.neighbors[interior[0]]
    c = pos[nb[0]].copy()
    line = _wavy_line(2e-4, nb.size) * 0.05
    pos[nb] = c + line
    from paper_2107_03632_b200.problem import NodeSet

    nodes2 = NodeSet(positions=pos, is_boundary=nodes.is_boundary, h=nodes.h)
    cond = gw.saddle_condition(pos[nb][None], shapes.degree)[0]
    assert 1e10 < cond <= gw.COND_LIMIT
    host = gw.assemble_shapes(nodes2, stencils, shapes.degree)
    plan = Plan.assembled(nodes2.n_total, interior, stencils.neighbors[interior], pos,
                          rb.forcing(pos[interior]), shapes.degree)
    dt = 0.5 * rb.stability_bound(host)
    plan.set_field(rb.apply_dirichlet(nodes2, np.zeros(nodes2.n_total)))
    res = plan.run(dt, steps=40)
    want = orc.run_time_loop(nodes2, host, dt=dt, steps=40)
    assert np.array_equal(plan.get_field(), want["field"]) and res.residual == want["residual"]
