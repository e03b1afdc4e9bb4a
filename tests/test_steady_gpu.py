"""Steady-state accuracy on the GPU against an independent direct solve.

Mirrors the reference's test_steady_state_matches_direct_solve
(pkg/tests/test_solver.py:246-252) and acceptance criterion 5
(pkg/tests/test_acceptance.py:162-178): the pseudo-time loop run to steady
state (tol 1e-9) must agree with a sparse LU solve of the same stencil system
sum_j w_ij u_j = -f_i (restated from pkg/tests/oracles.py:36-63) to 1e-6.
The loop itself is bitwise the reference's (test_parity_gpu.py); this checks
the physics end to end, on the device path.
"""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import paper_2107_03632_b200 as rb
from paper_2107_03632_b200 import synth

pytestmark = pytest.mark.gpu


def direct_steady_solution(nodes, shapes):
    interior = shapes.interior_nodes
    n_int = interior.size
    col_of = -np.ones(nodes.n_total, dtype=np.int64)
    col_of[interior] = np.arange(n_int)
    exact = rb.closed_form_solution(nodes.positions)
    rhs = -rb.forcing(nodes.positions[interior])
    nb = shapes.stencils.neighbors[interior]
    w = shapes.weights
    bnd = nodes.is_boundary[nb]
    rhs -= np.where(bnd, w * exact[nb], 0.0).sum(axis=1)
    r, c = np.nonzero(~bnd)
    matrix = sp.csr_matrix((w[r, c], (r, col_of[nb[r, c]])), shape=(n_int, n_int))
    solution = exact.copy()
    solution[interior] = spla.spsolve(matrix, rhs)
    return solution


@pytest.mark.parametrize("name,linf_bound", [("small", 0.1), ("dome", 5e-2)])
def test_steady_state_matches_direct_solve(golden, name, linf_bound):
    nodes, _, shapes, _ = golden(name)
    cfg = rb.SolveConfig(degree=int(shapes.degree), support_size=shapes.weights.shape[1],
                         nodes=nodes.n_total, mode="steady", tol=1e-9)
    report = rb.run_time_loop(cfg, nodes, shapes)
    direct = direct_steady_solution(nodes, shapes)
    assert np.abs(report.field - direct).max() <= 1e-6
    assert report.residual <= 1e-9
    assert report.linf <= linf_bound


def test_steady_state_streaming_path_matches_direct_solve():
    """A 2e4-node reference set through the TMA streaming step (no on-chip
    loop), GPU kNN + GPU weights, steady mode with the device-side decision."""
    nodes, st, shapes = synth.synthetic_problem(20_000, 15, 2, seed=4, weights="gpu")
    interior = shapes.interior_nodes
    plan = rb.Plan(nodes.n_total, interior, st.neighbors[interior], shapes.weights,
                   rb.forcing(nodes.positions[interior]), nodes.positions, renumber=True,
                   resident=False, cluster=False)
    plan.set_field(rb.apply_dirichlet(nodes, np.zeros(nodes.n_total)))
    res = plan.run(0.5 * rb.stability_bound(shapes), mode="steady", tol=1e-9, max_steps=3_000_000)
    assert res.status == 0 and res.residual <= 1e-9
    field = plan.get_field()
    direct = direct_steady_solution(nodes, shapes)
    assert np.abs(field - direct).max() <= 1e-6
