"""Per-rank device setup of the partitioned loop (paper_2107_03632_b200.dsetup):
every rank's part equals the host partitioner's part for the same rank, and
a group of parts whose weights were assembled on the device per part runs
bit for bit like one plan over the whole problem (solver.py:198-217)."""

import numpy as np
import pytest

import paper_2107_03632_b200 as rb
from paper_2107_03632_b200 import synth
from paper_2107_03632_b200.dsetup import build_parts_in_process
from paper_2107_03632_b200.multigpu import LocalGroup, assembled_plan, partition
from paper_2107_03632_b200.solver import Plan

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def problem():
    return synth.synthetic_problem(200_000, 15, 2, seed=3, weights="gpu", knn="gpu")


@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_rank_setup_equals_host_partition(problem, P):
    nodes, st, shapes = problem
    interior = shapes.interior_nodes
    want = partition(nodes.n_total, interior, st.neighbors[interior], None,
                     rb.forcing(nodes.positions[interior]), nodes.positions, P)
    _, got = build_parts_in_process(nodes.positions, nodes.is_boundary, 15, P)
    for a, b in zip(got, want):
        assert (a.n_local, a.n_boundary, a.n_halo) == (b.n_local, b.n_boundary, b.n_halo)
        assert np.array_equal(a.rows_ref, b.rows_ref)
        assert np.array_equal(a.local_to_global, b.local_to_global)
        assert np.array_equal(a.interior, b.interior)
        assert np.array_equal(a.rows, b.rows)
        assert np.array_equal(a.f_int, b.f_int)
        assert a.peers == b.peers and a.recv_offset == b.recv_offset and a.recv_count == b.recv_count
        for x, y in zip(a.send_idx, b.send_idx):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("P", [2, 4])
def test_device_assembled_parts_run_like_one_plan(problem, P):
    """Parts built per rank (own kNN rows, weights assembled inside each
    part's plan) in push mode: field and residual equal one plan assembled on
    the device over the whole problem; the auto dt (2 / max row sum, numpy's
    row-sum order) is the same on the parts and on the whole."""
    nodes, st, shapes = problem
    interior = shapes.interior_nodes
    full = Plan.assembled(nodes.n_total, interior, st.neighbors[interior], nodes.positions,
                          rb.forcing(nodes.positions[interior]), 2, renumber=True, resident=False)
    dt_full = 2.0 / full.weight_row_sum_max() * 0.5
    setups, parts = build_parts_in_process(nodes.positions, nodes.is_boundary, 15, P)
    plans = [assembled_plan(s, 2) for s in setups]
    dt_parts = 2.0 / max(p.weight_row_sum_max() for p in plans) * 0.5
    assert dt_parts == dt_full
    group = LocalGroup(parts, plans=plans)
    assert group.push_mode
    u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    for steps in (70, 3):
        full.set_field(u0)
        ref = full.run(dt_full, steps=steps)
        for part, plan in zip(parts, plans):
            plan.set_field(part.local_field(u0))
        rc, done, residual, _, _ = group.run(dt_full, steps=steps)
        from paper_2107_03632_b200.multigpu import assemble_field

        field = assemble_field(parts, [p.get_field() for p in plans], u0)
        assert done == steps and residual == ref.residual
        assert np.array_equal(field, full.get_field())
    group.close()
