"""Native advancing-front node generator vs the reference's.

``paper_2107_03632_b200.geometry.generate_unit_disk_nodes`` (csrc/nodes.cpp)
must return exactly the node set of rbffd.geometry.generate_unit_disk_nodes
(pkg/src/rbffd/geometry.py:105-198): tests/golden/nodes.json holds the
reference's counts and position digests (tests/golden/make_nodes_golden.py).
Host code only -- no device is touched.
"""

import hashlib
import json
import math
from pathlib import Path

import numpy as np
import pytest

import paper_2107_03632_b200 as rb
from paper_2107_03632_b200 import geometry

GOLDEN = json.loads((Path(__file__).parent / "golden" / "nodes.json").read_text())


@pytest.mark.parametrize("case", GOLDEN["cases"], ids=lambda c: f"N{c.get('target', c['h'])}-s{c['seed']}")
def test_nodes_bitwise_equal_reference(case):
    ns = geometry.generate_unit_disk_nodes(case["h"], int(case["seed"]))
    assert ns.n_total == case["n_total"]
    assert ns.n_boundary == case["n_boundary"]
    assert ns.is_boundary[: case["n_boundary"]].all() and not ns.is_boundary[case["n_boundary"]:].any()
    assert ns.positions[:3].tolist() == case["head"]
    assert ns.positions[-3:].tolist() == case["tail"]
    assert hashlib.sha256(ns.positions.tobytes()).hexdigest() == case["sha256"]


def test_nodes_match_golden_fixtures(golden):
    """The fixtures' node sets (made by the reference pipeline) regenerate exactly."""
    for name, target, seed in (("dome", 1027, 1), ("crit6", 2000, 6)):
        nodes, _, _, _ = golden(name)
        ns = geometry.generate_unit_disk_nodes(rb.spacing_for_node_count(target), seed)
        assert np.array_equal(ns.positions, nodes.positions)
        assert np.array_equal(ns.is_boundary, nodes.is_boundary)


def test_error_messages_match_reference():
    errs = GOLDEN["errors"]
    for h in (0.0, 0.5, 0.7, -1.0):
        with pytest.raises(rb.ParameterError) as ei:
            geometry.generate_unit_disk_nodes(h, 0)
        assert str(ei.value) == errs[repr(h)]
    with pytest.raises(rb.ParameterError) as ei:
        rb.spacing_for_node_count(29)
    assert str(ei.value) == errs["spacing_for_node_count(29)"]


def test_seed_key_matches_cpython():
    """random.seed(int) keys init_by_array with |seed|'s 32-bit words."""
    import random

    for seed in (0, 1, -1, 2**32 - 1, 2**32, 2**70 + 3):
        key = geometry.seed_key(seed)
        assert int(sum(int(w) << (32 * i) for i, w in enumerate(key))) == abs(seed)
        # same stream: the first draw of random.Random(seed) vs random.Random(|seed|)
        assert random.Random(seed).random() == random.Random(abs(seed)).random()


def test_determinism_and_spacing():
    """Same (h, seed) -> same set; minimum interior separation >= 0.8 h
    (geometry.py:26-31 acceptance rule); all nodes in the closed disk."""
    h = rb.spacing_for_node_count(4000)
    a = geometry.generate_unit_disk_nodes(h, 5)
    b = geometry.generate_unit_disk_nodes(h, 5)
    assert a.positions.tobytes() == b.positions.tobytes()
    r = np.hypot(a.positions[:, 0], a.positions[:, 1])
    assert np.all(r <= 1.0 + 1e-12)
    assert np.all(np.abs(r[a.is_boundary] - 1.0) < 1e-12)
    from scipy.spatial import cKDTree

    interior = a.positions[~a.is_boundary]
    d, _ = cKDTree(interior).query(interior, k=2)
    assert d[:, 1].min() >= 0.8 * h * (1 - 1e-12)
    assert abs(a.n_total - rb.node_count_for_spacing(h)) < 0.1 * a.n_total
    assert math.isclose(a.h, h)


# ---- the reference's own geometry tests (pkg/tests/test_geometry.py:53-129) ----
def test_node_count_for_spacing_values():
    assert rb.node_count_for_spacing(0.055) == 1153
    assert rb.node_count_for_spacing(0.1) == 377
    assert rb.node_count_for_spacing(0.01) / rb.node_count_for_spacing(0.02) == pytest.approx(4.0, rel=0.05)


@pytest.mark.parametrize("h", [0.6, 0.5, 0.0, -0.1])
def test_node_count_rejects_bad_spacing(h):
    with pytest.raises(rb.ParameterError):
        rb.node_count_for_spacing(h)


def test_spacing_for_node_count_inverts_estimate():
    for target in (100, 500, 1027, 10_000):
        assert rb.node_count_for_spacing(rb.spacing_for_node_count(target)) == pytest.approx(target, abs=1)


def test_generate_counts_classification_and_separation():
    h = 0.1
    nodes = geometry.generate_unit_disk_nodes(h, seed=1)
    assert nodes.n_total == nodes.n_interior + nodes.n_boundary and nodes.n_interior >= 1
    assert nodes.n_boundary == round(2 * math.pi / h)
    radii = np.linalg.norm(nodes.positions, axis=1)
    assert np.all(np.abs(radii[nodes.is_boundary] - 1.0) <= geometry.BOUNDARY_TOL)
    assert np.all(radii[~nodes.is_boundary] < 1.0 - geometry.BOUNDARY_TOL)
    c = geometry.generate_unit_disk_nodes(h, seed=8)
    assert not np.array_equal(nodes.positions[:50], c.positions[:50]) or nodes.n_total != c.n_total
    pts = geometry.generate_unit_disk_nodes(0.12, seed=2).positions
    dist = np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1))
    dist[np.diag_indices_from(dist)] = np.inf
    assert dist.min() >= 0.5 * 0.12


def test_nodes_csv_roundtrip(tmp_path):
    nodes = geometry.generate_unit_disk_nodes(0.15, seed=4)
    path = tmp_path / "nodes.csv"
    geometry.save_nodes_csv(nodes, path)
    assert path.read_text().splitlines()[0] == "x,y,kind"
    loaded = geometry.load_nodes_csv(path)
    assert np.array_equal(loaded.positions, nodes.positions)
    assert np.array_equal(loaded.is_boundary, nodes.is_boundary)
