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
    assert 2.0 / a.weight_row_sum_max() == pytest.approx(rb.stability_bound(host), rel=1e-12)
    dt = rb.stability_bound(host) * 0.5
    a.set_field(u0)
    ra = a.run(dt, steps=150)
    want = orc.run_time_loop(nodes, host, dt=dt, steps=150)
    assert np.array_equal(a.get_field(), want["field"]) and ra.residual == want["residual"]
