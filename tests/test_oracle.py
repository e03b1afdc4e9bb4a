"""The CPU oracle (oracle/) against the golden vectors recorded from the
unmodified reference (tests/golden/make_golden.py).  CPU only.

Pins the oracle: every field must match the reference bit for bit, every
scalar exactly (same IEEE operations in the same order)."""

import numpy as np
import pytest

from oracle import oracle as orc

FIXED_CASES = [
    ("small", "fixed50"),
    ("small", "fixed120"),
    ("small", "fixed120_copy"),
    ("small", "steady"),
    ("small", "zero"),
    ("dome", "paper"),
    ("dome", "steady"),
    ("crit6", "fixed100"),
    ("crit6", "fixed100_copy"),
    ("m4", "fixed200"),
    ("m6", "fixed100"),
]


def _run(nodes, shapes, meta, threads):
    return orc.run_time_loop(
        nodes, shapes, dt=meta["dt"], steps=meta["config_steps"], mode=meta["mode"],
        tol=meta["tol"], max_steps=meta["max_steps"], copy_back=meta["copy_back"],
        threads=threads,
    )


@pytest.mark.parametrize("name,case", FIXED_CASES)
def test_oracle_run_matches_reference(golden, manifest, name, case):
    nodes, _, shapes, z = golden(name)
    meta = manifest[name][case]
    out = _run(nodes, shapes, meta, threads=1 if name == "dome" else 2)
    assert out["status"] == orc.ORC_OK
    assert np.array_equal(out["field"], z[f"{case}__field"])
    assert out["steps"] == meta["steps"]
    assert out["residual"] == meta["residual"]
    assert (out["linf"], out["l2"]) == (meta["linf"], meta["l2"])


def test_oracle_auto_dt_matches_reference(golden, manifest):
    for name in ("small", "dome", "m4", "m6"):
        _, _, shapes, _ = golden(name)
        assert orc.stability_bound(shapes.weights) == manifest[name]["stability_bound"]


def test_oracle_kat_hand_problem(golden):
    """test_solver.py:112-123 -- hand-evaluated single-node update."""
    nodes, _, shapes, z = golden("hand")
    u1 = z["kat__u1"]
    f = orc.forcing(nodes.positions)
    u2, bad = orc.explicit_step(u1, shapes, f, 3e-3)
    assert not bad
    assert np.array_equal(u2, z["kat__u2"])
    acc = -11.0 * u1[4] + 2.5 * u1[0] + 2.5 * u1[1] + 3.0 * u1[2] + 3.0 * u1[3]
    assert u2[4] == pytest.approx(u1[4] + 3e-3 * (f[4] + acc), rel=1e-15)


def test_oracle_step_matches_reference_and_python_loop(golden):
    """test_solver.py:134-145 -- numba vs plain-Python loop, bitwise."""
    nodes, stencils, shapes, z = golden("small")
    u1 = z["step_rand__u1"]
    f = orc.forcing(nodes.positions)
    u2, bad = orc.explicit_step(u1, shapes, f, 1e-4, threads=4)
    assert not bad
    assert np.array_equal(u2, z["step_rand__u2"])
    interior = shapes.interior_nodes
    py = orc.python_explicit_step(u1, interior, stencils.neighbors[interior], shapes.weights,
                                  f[interior], 1e-4)
    assert np.array_equal(py, z["step_rand__u2"])


def test_oracle_blowup_and_timeout(golden, manifest):
    nodes, _, shapes, _ = golden("small")
    m = manifest["small"]
    u2, bad = orc.explicit_step(np.full(nodes.n_total, 1e308), shapes,
                                orc.forcing(nodes.positions), 1.0)
    assert bad and np.isnan(np.max(np.abs(u2))) == np.isnan(m["step_blowup"]["max_abs"])
    un = orc.run_time_loop(nodes, shapes, dt=1.0, steps=500)
    assert un["status"] == orc.ORC_INSTABILITY
    assert un["step"] == m["unstable"]["step"]
    assert np.isnan(un["max_abs"]) and np.isnan(m["unstable"]["max_abs"])
    to = orc.run_time_loop(nodes, shapes, mode="steady", tol=1e-9, max_steps=5)
    assert to["status"] == orc.ORC_TIMEOUT
    assert to["steps"] == m["timeout"]["steps"] == 5
    assert to["residual"] == m["timeout"]["residual"]


def test_oracle_thread_count_does_not_change_bits(golden):
    """test_solver.py:211-218 / acceptance criterion 6 pattern."""
    nodes, _, shapes, _ = golden("crit6")
    fields = [orc.run_time_loop(nodes, shapes, dt=1e-5, steps=100, threads=t)["field"]
              for t in (1, 2, 8)]
    assert all(np.array_equal(fields[0], f) for f in fields[1:])
