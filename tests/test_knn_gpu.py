"""Exact GPU kNN against the reference's supports in the
golden fixtures and the reference's brute-force oracle (tests/oracles.py:16-24,
acceptance criterion 7 pattern, test_acceptance.py:208-230)."""

import numpy as np
import pytest

import paper_2107_03632_b200 as rb
from paper_2107_03632_b200.neighborhoods import build_stencils, recommended_support_size

pytestmark = pytest.mark.gpu


def brute_force_knn(positions, n):
    """tests/oracles.py:16-24: full scan, ties broken by lower index."""
    positions = np.asarray(positions, dtype=float)
    count = len(positions)
    diff = positions[:, None, :] - positions[None, :, :]
    dist = np.sqrt((diff**2).sum(-1))
    idx = np.broadcast_to(np.arange(count), dist.shape)
    order = np.lexsort((idx, dist))
    return order[:, :n]


@pytest.mark.parametrize("name", ["small", "dome", "crit6", "m4", "m6"])
def test_knn_matches_reference_supports(golden, name):
    nodes, stencils, _, _ = golden(name)
    got = build_stencils(nodes, stencils.n)
    assert np.array_equal(got.neighbors, stencils.neighbors)


def _node_sets(rng):
    sets = []
    for case in range(30):
        kind = case % 3
        if kind == 0:  # scattered
            pts = rng.uniform(-1, 1, (int(rng.integers(50, 1500)), 2))
        elif kind == 1:  # lattice: many exact distance ties
            m = int(rng.integers(5, 35))
            g = np.arange(m) * 0.1
            pts = np.stack(np.meshgrid(g, g), -1).reshape(-1, 2)
        else:  # clustered + anisotropic spread
            pts = rng.normal(size=(int(rng.integers(50, 1200)), 2)) * [3.0, 0.01]
        sets.append(pts)
    return sets


def test_knn_matches_brute_force_oracle_with_ties():
    rng = np.random.default_rng(7)
    for pts in _node_sets(rng):
        nodes = rb.NodeSet(positions=pts, is_boundary=np.zeros(len(pts), bool), h=0.1)
        n = int(rng.integers(1, min(60, len(pts)) + 1))
        got = build_stencils(nodes, n).neighbors
        want = brute_force_knn(pts, n)
        assert np.array_equal(got, want), (len(pts), n)


def test_knn_parameter_errors():
    pts = np.random.default_rng(1).uniform(size=(20, 2))
    nodes = rb.NodeSet(positions=pts, is_boundary=np.zeros(20, bool), h=0.1)
    with pytest.raises(rb.ParameterError):
        build_stencils(nodes, 0)
    with pytest.raises(rb.ParameterError):
        build_stencils(nodes, 21)
    assert build_stencils(nodes, 20).neighbors.shape == (20, 20)
    assert recommended_support_size(2) == 6 and recommended_support_size(4, safety=2) == 30


def test_knn_matches_ckdtree_at_scale():
    from paper_2107_03632_b200 import synth

    nodes = synth.disk_nodes(300_000, seed=2)
    for n in (15, 56):
        got = build_stencils(nodes, n).neighbors
        want = synth.knn_stencils(nodes, n).neighbors
        assert np.array_equal(got, want)
