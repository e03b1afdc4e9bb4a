"""Parity of the CUDA path against the reference's golden vectors and the CPU
oracle.  Every test runs the sm_100a library through the C ABI; the bar is
bitwise equality (np.array_equal on fields, == on scalars) -- the reference's
own tests demand exactly that (test_solver.py:134-145, :189-198).

Mirrors pkg/tests/test_solver.py and acceptance criterion 6; adds the
device-only variants (streaming vs resident loop, Morton renumbering, graph
chunking in steady mode) and full-size (BASELINE config 2) parity.
"""

import numpy as np
import pytest

import paper_2107_03632_b200 as rb
from paper_2107_03632_b200 import _lib, synth
from paper_2107_03632_b200.solver import Plan
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

CASES = [
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


def config_for(nodes, shapes, meta, **over):
    auto = meta["dt"] == 0.5 * rb.stability_bound(shapes)
    kw = dict(
        degree=shapes.degree, support_size=shapes.weights.shape[1], nodes=nodes.n_total,
        dt=None if auto else meta["dt"], steps=meta["config_steps"], mode=meta["mode"],
        tol=meta["tol"], max_steps=meta["max_steps"],
    )
    kw.update(over)
    return rb.SolveConfig(**kw)


def check_report(rep, meta, field):
    assert np.array_equal(rep.field, field)
    assert rep.steps == meta["steps"]
    assert rep.residual == meta["residual"]
    assert (rep.linf, rep.l2) == (meta["linf"], meta["l2"])
    assert rep.config["dt"] == meta["dt"]


@pytest.mark.parametrize("name,case", [("small", "steady"), ("crit6", "fixed100"), ("m4", "fixed200"),
                                       ("m6", "fixed100"), ("dome", "steady"), ("small", "fixed120")])
@pytest.mark.parametrize("q", ["2", "5", "8", "16"])
def test_cluster_loop_sizes_match_reference(golden, manifest, name, case, q, monkeypatch):
    """Cluster-resident loop for 2..16 CTAs per cluster (RBFFD_CLUSTER)."""
    monkeypatch.setenv("RBFFD_CLUSTER", q)
    nodes, _, shapes, z = golden(name)
    meta = manifest[name][case]
    interior = shapes.interior_nodes
    plan = Plan(nodes.n_total, interior, shapes.stencils.neighbors[interior], shapes.weights,
                rb.forcing(nodes.positions[interior]))
    info = plan.info()
    if info["variant"] != 3:
        pytest.skip(f"{name} does not fit the cluster loop")
    plan.set_field(rb.apply_dirichlet(nodes, np.zeros(nodes.n_total)))
    res = plan.run(meta["dt"], steps=meta["config_steps"], mode=meta["mode"], tol=meta["tol"],
                   max_steps=meta["max_steps"])
    assert res.steps_done == meta["steps"] and res.residual == meta["residual"]
    assert np.array_equal(plan.get_field(), z[f"{case}__field"])
    plan.close()


def test_interleaved_plans_of_different_sizes(golden, manifest):
    """Kernel attributes are process-global: building a smaller plan must not
    break launches of an earlier, larger one (each loop kind)."""
    runs = []
    for name, case in (("m6", "fixed100"), ("crit6", "fixed100"), ("dome", "paper"), ("small", "fixed50")):
        nodes, _, shapes, z = golden(name)
        interior = shapes.interior_nodes
        for kw in (dict(), dict(cluster=False), dict(resident=False)):
            plan = Plan(nodes.n_total, interior, shapes.stencils.neighbors[interior], shapes.weights,
                        rb.forcing(nodes.positions[interior]), **kw)
            runs.append((plan, nodes, manifest[name][case], z[f"{case}__field"]))
    for plan, nodes, meta, field in reversed(runs):
        plan.set_field(rb.apply_dirichlet(nodes, np.zeros(nodes.n_total)))
        res = plan.run(meta["dt"], steps=meta["config_steps"])
        assert res.residual == meta["residual"]
        assert np.array_equal(plan.get_field(), field)


@pytest.mark.parametrize("renumber", [False, True], ids=["native", "morton"])
@pytest.mark.parametrize("name,case", CASES)
def test_run_time_loop_matches_reference(golden, manifest, name, case, renumber):
    nodes, _, shapes, z = golden(name)
    meta = manifest[name][case]
    rep = rb.run_time_loop(config_for(nodes, shapes, meta), nodes, shapes,
                           copy_back=meta["copy_back"], renumber=renumber)
    check_report(rep, meta, z[f"{case}__field"])


@pytest.mark.parametrize("case", ["paper", "steady"])
def test_streaming_loop_matches_resident_loop(golden, manifest, case):
    """The Fig. 1 case normally runs on-chip (cluster loop); force the
    single-CTA loop and the streaming graph/PDL paths (and their fused
    steady-state stop) and demand the same bits from every one."""
    nodes, _, shapes, z = golden("dome")
    meta = manifest["dome"][case]
    interior = shapes.interior_nodes
    rows = shapes.stencils.neighbors[interior]
    f_int = rb.forcing(nodes.positions[interior])
    u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    for resident, cluster, pdl, tma, variant in (
            (True, True, True, True, 3), (True, False, True, True, 0), (False, True, True, True, 2),
            (False, True, False, True, 2), (False, True, True, False, 1), (False, True, False, False, 1)):
        plan = Plan(nodes.n_total, interior, rows, shapes.weights, f_int, resident=resident,
                    pdl=pdl, tma=tma, cluster=cluster)
        info = plan.info()
        assert info["variant"] == variant
        plan.set_field(u0)
        res = plan.run(meta["dt"], steps=meta["config_steps"], mode=meta["mode"], tol=meta["tol"],
                       max_steps=meta["max_steps"])
        assert res.status == _lib.RBF_OK
        assert res.steps_done == meta["steps"]
        assert res.residual == meta["residual"]
        assert np.array_equal(plan.get_field(), z[f"{case}__field"])
        plan.close()


def test_explicit_step_kat_hand_problem(golden):
    """test_solver.py:112-123."""
    nodes, _, shapes, z = golden("hand")
    u1 = z["kat__u1"]
    f = rb.forcing(nodes.positions)
    u2 = rb.explicit_step(u1, shapes, f, 3e-3)
    acc = -11.0 * u1[4] + 2.5 * u1[0] + 2.5 * u1[1] + 3.0 * u1[2] + 3.0 * u1[3]
    assert u2[4] == pytest.approx(u1[4] + 3e-3 * (f[4] + acc), rel=1e-15)
    assert np.array_equal(u2, z["kat__u2"])
    assert np.array_equal(u2[:4], u1[:4])


def test_explicit_step_matches_reference_loop(golden):
    """test_solver.py:134-145 (bitwise vs the numba kernel and the Python loop)."""
    nodes, stencils, shapes, z = golden("small")
    u1 = z["step_rand__u1"]
    snapshot = u1.copy()
    got = rb.explicit_step(u1, shapes, rb.forcing(nodes.positions), 1e-4)
    assert np.array_equal(got, z["step_rand__u2"])
    assert np.array_equal(u1, snapshot)  # test_solver.py:126-131


def test_plan_cache_sees_in_place_edits(golden):
    """explicit_step caches the packed plan per ShapeStore; editing the
    weights or stencils in place must not reuse stale device data (the
    reference always reads the current arrays)."""
    import copy

    nodes, _, shapes0, z = golden("small")
    shapes = copy.deepcopy(shapes0)
    u1 = z["step_rand__u1"]
    f = rb.forcing(nodes.positions)
    a = rb.explicit_step(u1, shapes, f, 1e-4)
    assert np.array_equal(a, orc.explicit_step(u1, shapes, f, 1e-4)[0])
    shapes.weights[...] *= 1.5  # in place: same buffer, same id(shapes)
    b = rb.explicit_step(u1, shapes, f, 1e-4)
    assert np.array_equal(b, orc.explicit_step(u1, shapes, f, 1e-4)[0])
    assert not np.array_equal(a, b)
    nb = shapes.stencils.neighbors
    nb[shapes.interior_nodes[0], [1, 2]] = nb[shapes.interior_nodes[0], [2, 1]]
    c = rb.explicit_step(u1, shapes, f, 1e-4)
    assert np.array_equal(c, orc.explicit_step(u1, shapes, f, 1e-4)[0])


def test_explicit_step_dt_zero_is_identity(golden):
    nodes, _, shapes, _ = golden("small")
    u1 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    assert np.array_equal(rb.explicit_step(u1, shapes, rb.forcing(nodes.positions), 0.0), u1)


def test_exact_solution_is_near_fixed_point(golden):
    """test_solver.py:148-159."""
    nodes, stencils, shapes, _ = golden("small")
    u_exact = rb.closed_form_solution(nodes.positions)
    f = rb.forcing(nodes.positions)
    u2 = rb.explicit_step(u_exact, shapes, f, 1e-5)
    interior = shapes.interior_nodes
    residual = f[interior] + np.einsum("ij,ij->i", shapes.weights, u_exact[stencils.neighbors[interior]])
    assert np.abs(u2 - u_exact).max() <= 1e-5 * np.abs(residual).max() * (1 + 1e-12)


def test_explicit_step_detects_blowup(golden, manifest):
    nodes, _, shapes, _ = golden("small")
    with pytest.raises(rb.InstabilityError) as ei:
        rb.explicit_step(np.full(nodes.n_total, 1e308), shapes, rb.forcing(nodes.positions), 1.0)
    assert ei.value.max_abs is not None
    assert np.isnan(ei.value.max_abs) == np.isnan(manifest["small"]["step_blowup"]["max_abs"])


@pytest.mark.parametrize("name", ["small", "crit6"])
def test_unstable_dt_raises_at_the_reference_step(golden, manifest, name):
    """test_solver.py:170-175; the failing step and max|u2| match the oracle."""
    nodes, _, shapes, _ = golden(name)
    cfg = rb.SolveConfig(degree=2, support_size=shapes.weights.shape[1], nodes=nodes.n_total,
                         mode="fixed", steps=500, dt=1.0)
    want = orc.run_time_loop(nodes, shapes, dt=1.0, steps=500)
    assert want["status"] == orc.ORC_INSTABILITY
    if name == "small":
        assert want["step"] == manifest["small"]["unstable"]["step"]
    with pytest.raises(rb.InstabilityError) as ei:
        rb.run_time_loop(cfg, nodes, shapes)
    assert "step" in str(ei.value)
    assert ei.value.step == want["step"]
    assert np.array_equal(np.float64(ei.value.max_abs), np.float64(want["max_abs"]), equal_nan=True)


def test_steady_timeout(golden, manifest):
    nodes, _, shapes, _ = golden("small")
    cfg = rb.SolveConfig(degree=2, support_size=12, nodes=300, mode="steady", tol=1e-9,
                         seed=2, max_steps=5)
    with pytest.raises(rb.SteadyStateTimeout) as ei:
        rb.run_time_loop(cfg, nodes, shapes)
    assert ei.value.steps == 5
    assert ei.value.residual == manifest["small"]["timeout"]["residual"]


def test_zero_steps(golden):
    nodes, _, shapes, _ = golden("small")
    cfg = rb.SolveConfig(degree=2, support_size=12, nodes=300, steps=0, dt=1e-5)
    rep = rb.run_time_loop(cfg, nodes, shapes)
    assert rep.steps == 0 and rep.residual is None
    assert (rep.linf, rep.l2) == rb.error_norms(rb.apply_dirichlet(nodes, np.zeros(nodes.n_total)), nodes)


def test_run_time_loop_matches_step_composition(golden):
    """test_solver.py:189-198."""
    nodes, _, shapes, _ = golden("small")
    cfg = rb.SolveConfig(degree=2, support_size=12, nodes=300, steps=50, dt=1e-4)
    rep = rb.run_time_loop(cfg, nodes, shapes)
    u = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    f = rb.forcing(nodes.positions)
    for _ in range(50):
        u = rb.explicit_step(u, shapes, f, 1e-4)
    assert np.array_equal(rep.field, u)


def test_boundary_held_fixed_and_determinism(golden):
    """test_solver.py:221-228, :264-273."""
    nodes, _, shapes, _ = golden("crit6")
    cfg = rb.SolveConfig(degree=2, support_size=15, nodes=2000, steps=300, dt=1e-5)
    a = rb.run_time_loop(cfg, nodes, shapes)
    b = rb.run_time_loop(cfg, nodes, shapes, cache=False)
    bidx = nodes.boundary_indices
    assert np.array_equal(a.field[bidx], rb.closed_form_solution(nodes.positions[bidx]))
    assert np.array_equal(a.field, b.field)
    assert (a.steps, a.linf, a.l2, a.residual) == (b.steps, b.linf, b.l2, b.residual)


def test_residual_monotone_after_startup(golden):
    """test_solver.py:231-243 through explicit_step on the device."""
    nodes, _, shapes, _ = golden("small")
    dt = 0.5 * rb.stability_bound(shapes)
    u = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    f = rb.forcing(nodes.positions)
    updates = []
    for _ in range(3000):
        new = rb.explicit_step(u, shapes, f, dt)
        updates.append(np.abs(new - u).max())
        u = new
    tail = np.asarray(updates[30:])
    assert np.all(np.diff(tail) <= 1e-12 * tail[:-1])


def test_literal_step_kernel_dropin(golden):
    """rbf_step_kernel has the numba kernel's signature (solver.py:294-311)."""
    import ctypes

    nodes, _, shapes, z = golden("crit6")
    lib = _lib.load()
    interior = np.ascontiguousarray(shapes.interior_nodes, dtype=np.int64)
    rows = np.ascontiguousarray(shapes.stencils.neighbors[interior], dtype=np.int64)
    f_int = np.ascontiguousarray(rb.forcing(nodes.positions[interior]))
    rng = np.random.default_rng(5)
    u1 = rb.apply_dirichlet(nodes, rng.normal(size=nodes.n_total))
    for dt in (1e-5, 1.0e3):
        u2 = np.full(nodes.n_total, -7.0)
        want = u2.copy()
        wflags = orc.step_kernel(u1, want, interior, rows, shapes.weights, f_int, dt, chunk=100)
        flags = np.zeros_like(wflags)
        rc = lib.rbf_step_kernel(u1.ctypes.data, u2.ctypes.data, nodes.n_total, interior.ctypes.data,
                                 rows.ctypes.data, shapes.weights.ctypes.data, f_int.ctypes.data,
                                 interior.size, rows.shape[1], dt, 100, flags.ctypes.data, 0)
        assert rc == _lib.RBF_OK
        assert np.array_equal(u2, want)
        assert np.array_equal(flags, wflags)


def test_no_interior_rows():
    nodes = rb.NodeSet(positions=np.array([[1.0, 0.0], [0.0, 1.0], [-1.0, 0.0]]),
                       is_boundary=np.array([True, True, True]), h=0.5)
    st = rb.StencilSet(n=3, neighbors=np.array([[0, 1, 2], [1, 0, 2], [2, 0, 1]]))
    shapes = rb.ShapeStore(degree=0, interior_nodes=np.zeros(0, dtype=np.int64),
                           weights=np.zeros((0, 3)), stencils=st)
    cfg = rb.SolveConfig(degree=0, support_size=3, nodes=300, steps=3, dt=1e-3)
    rep = rb.run_time_loop(cfg, nodes, shapes)
    assert rep.steps == 3 and rep.residual == 0.0


# ---- larger synthetic domains: device vs oracle, bitwise ---------------------
@pytest.fixture(scope="module")
def synth_cache():
    return {}


def _synth(synth_cache, target, n, m):
    key = (target, n, m)
    if key not in synth_cache:
        synth_cache[key] = synth.synthetic_problem(target, n, m, seed=3)
    return synth_cache[key]


@pytest.mark.parametrize("target,n,m,steps", [
    (200_000, 15, 2, 40),
    (100_000, 30, 4, 25),
    (40_000, 56, 6, 20),
    (30_000, 19, 2, 33),   # width without a specialised kernel (generic loop)
])
@pytest.mark.parametrize("renumber", [False, True], ids=["native", "morton"])
def test_synthetic_fixed_matches_oracle(synth_cache, target, n, m, steps, renumber):
    nodes, _, shapes = _synth(synth_cache, target, n, m)
    want = orc.run_time_loop(nodes, shapes, steps=steps)
    cfg = rb.SolveConfig(degree=m, support_size=n, nodes=target, steps=steps)
    rep = rb.run_time_loop(cfg, nodes, shapes, renumber=renumber)
    assert np.array_equal(rep.field, want["field"])
    assert rep.residual == want["residual"]
    assert rep.steps == steps


@pytest.mark.parametrize("target,n,m", [(200_000, 15, 2), (60_000, 30, 4), (40_000, 56, 6)])
def test_tma_and_ldg_step_variants_agree_with_oracle(synth_cache, target, n, m):
    """Both streaming kernels (TMA ring / plain loads), with and without PDL."""
    nodes, _, shapes = _synth(synth_cache, target, n, m)
    interior = shapes.interior_nodes
    rows = shapes.stencils.neighbors[interior]
    f_int = rb.forcing(nodes.positions[interior])
    u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    dt = 0.5 * rb.stability_bound(shapes)
    want = orc.run_time_loop(nodes, shapes, steps=70)
    for tma, pdl, idx16 in ((True, True, True), (True, False, True), (True, True, False),
                            (False, True, True)):
        plan = Plan(nodes.n_total, interior, rows, shapes.weights, f_int, nodes.positions,
                    renumber=True, tma=tma, pdl=pdl, idx16=idx16, resident=False, pair=False)
        info = plan.info()
        assert info["variant"] == (2 if tma else 1)
        assert info["index_bits"] == (16 if (tma and idx16 and n <= 32) else 32)
        plan.set_field(u0)
        res = plan.run(dt, steps=70)
        assert res.residual == want["residual"]
        assert np.array_equal(plan.get_field(), want["field"])
        plan.close()


@pytest.mark.parametrize("target,n,m", [(1_000_000, 15, 2), (400_000, 30, 4), (200_000, 56, 6)])
def test_tma_ring_many_laps_matches_ldg(synth_cache, target, n, m):
    """Hundreds of steps, each wrapping every CTA's ring many times: the TMA
    ring (producer/consumer mbarrier pipeline) must stay bit-identical to the
    plain-load kernel (no phase aliasing, no lost or duplicated slices)."""
    nodes, _, shapes = _synth(synth_cache, target, n, m)
    interior = shapes.interior_nodes
    rows = shapes.stencils.neighbors[interior]
    f_int = rb.forcing(nodes.positions[interior])
    u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    dt = 0.5 * rb.stability_bound(shapes)
    out = []
    for tma, idx16, renumber in ((True, True, True), (True, False, True), (False, False, False),
                                 (True, True, False)):
        plan = Plan(nodes.n_total, interior, rows, shapes.weights, f_int, nodes.positions,
                    renumber=renumber, tma=tma, idx16=idx16)
        plan.set_field(u0)
        res = plan.run(dt, steps=300)
        out.append((plan.get_field(), res.residual, plan.info()["index_bits"]))
        plan.close()
    # Morton order: nearly every slice fits the 16-bit windows (used for n <= 32)
    assert out[0][2] == (16 if n <= 32 else 32)
    for f, r, _ in out[1:]:
        assert np.array_equal(out[0][0], f) and out[0][1] == r


@pytest.mark.parametrize("steps", [2, 3, 64, 65, 129])
def test_streaming_graph_chunk_step_counts(synth_cache, steps):
    """Step counts either side of the 64-step graph chunk on the streaming
    (TMA ring) path: graphs + direct tail launches, residual on the last."""
    nodes, _, shapes = _synth(synth_cache, 200_000, 15, 2)
    interior = shapes.interior_nodes
    want = orc.run_time_loop(nodes, shapes, steps=steps)
    for idx16, persist in ((True, False), (False, False), (True, True), (False, True)):
        plan = Plan(nodes.n_total, interior, shapes.stencils.neighbors[interior], shapes.weights,
                    rb.forcing(nodes.positions[interior]), nodes.positions, renumber=True,
                    idx16=idx16, resident=False, pair=False, persist=persist)
        assert plan.info()["variant"] == 2
        plan.set_field(rb.apply_dirichlet(nodes, np.zeros(nodes.n_total)))
        res = plan.run(0.5 * rb.stability_bound(shapes), steps=steps)
        assert np.array_equal(plan.get_field(), want["field"]) and res.residual == want["residual"]
        assert res.steps_done == steps
        plan.close()


# ---- every specialised stencil width (and two generic ones) -----------------
WIDTHS = [4, 5, 6, 7, 8, 9, 10, 11, 12, 15, 16, 20, 21, 24, 28, 30, 32, 33, 36, 40, 42, 45, 48, 56, 60, 64]
SPECIALISED = {4, 5, 6, 7, 8, 9, 10, 12, 15, 16, 20, 21, 24, 28, 30, 32, 36, 40, 42, 45, 48, 56, 60, 64}


def _degree_for(n):
    return 1 if n < 12 else (2 if n < 30 else (4 if n < 56 else 6))


@pytest.mark.parametrize("n", WIDTHS)
def test_every_width_matches_oracle(n):
    """All kernel instantiations (single-step TMA ring with 16-bit / int32 ids,
    plain-load streaming, two-step tile kernel, generic runtime-n loop) on a
    scattered disk at each width, bitwise vs the oracle."""
    m = _degree_for(n)
    nodes, st, shapes = synth.synthetic_problem(12_000, n, m, seed=5, weights="gpu")
    interior = shapes.interior_nodes
    rows = st.neighbors[interior]
    f_int = rb.forcing(nodes.positions[interior])
    u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    dt = 0.5 * rb.stability_bound(shapes)
    steps = 24
    want = orc.run_time_loop(nodes, shapes, steps=steps)
    stream = dict(resident=False, cluster=False)
    variants = [  # (plan flags, expected variant, expected pair)
        (dict(renumber=True), None, None),                                  # default choice
        (dict(renumber=True, pair=False, **stream), 2, 0),                  # TMA ring, 16-bit ids (n <= 32)
        (dict(renumber=True, pair=True, **stream), 2, 1 if n <= 32 and n in SPECIALISED else 0),
        (dict(renumber=True, idx16=False, pair=False, **stream), 2, 0),     # TMA ring, int32 ids
        (dict(renumber=False, tma=False, pair=False, **stream), 1, 0),      # plain-load streaming
        (dict(renumber=True, cluster=False), None, None),                   # single-CTA resident loop
    ]
    for kw, variant, pair in variants:
        plan = Plan(nodes.n_total, interior, rows, shapes.weights, f_int, nodes.positions, **kw)
        info = plan.info()
        if variant is not None and n in SPECIALISED:
            assert info["variant"] == variant, (n, kw, info)
        if pair is not None:
            assert info["pair"] == pair, (n, kw, info)
        plan.set_field(u0)
        res = plan.run(dt, steps=steps)
        assert res.residual == want["residual"], (n, kw)
        assert np.array_equal(plan.get_field(), want["field"]), (n, kw)
        plan.close()


# ---- grid-resident loop (rows in every SM's shared memory) -------------------
@pytest.mark.parametrize("target,n,m", [(20_000, 15, 2), (150_000, 15, 2), (60_000, 30, 4), (20_000, 56, 6),
                                         (400_000, 15, 2), (250_000, 30, 4)])  # last two: rows partly in L2
def test_grid_loop_matches_oracle(synth_cache, target, n, m):
    """One cooperative launch for all steps: fixed runs of every length, swap
    and copy-back, continued runs, steady mode, and the failure step."""
    nodes, _, shapes = _synth(synth_cache, target, n, m)
    interior = shapes.interior_nodes
    plan = Plan(nodes.n_total, interior, shapes.stencils.neighbors[interior], shapes.weights,
                rb.forcing(nodes.positions[interior]), nodes.positions, renumber=True)
    assert plan.info()["variant"] == 4 and plan.info()["resident"] == 1
    u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    dt = 0.5 * rb.stability_bound(shapes)
    for steps in (1, 2, 3, 130):
        want = orc.run_time_loop(nodes, shapes, steps=steps)
        for copy_back in (False, True):
            plan.set_field(u0)
            res = plan.run(dt, steps=steps, copy_back=copy_back)
            assert res.steps_done == steps and res.residual == want["residual"], (steps, copy_back)
            assert np.array_equal(plan.get_field(), want["field"]), (steps, copy_back)
    plan.set_field(u0)
    plan.run(dt, steps=20)
    plan.run(dt, steps=21)
    want = orc.run_time_loop(nodes, shapes, steps=41)
    assert np.array_equal(plan.get_field(), want["field"])
    # steady: stop step, residual and field are the oracle's
    want = orc.run_time_loop(nodes, shapes, mode="steady", tol=5e-2, max_steps=20_000)
    plan.set_field(u0)
    res = plan.run(dt, mode="steady", tol=5e-2, max_steps=20_000)
    assert res.steps_done == want["steps"] and res.residual == want["residual"]
    assert np.array_equal(plan.get_field(), want["field"])
    # instability: the reference's failing step and its field
    dtb = 40.0 * dt
    want = orc.run_time_loop(nodes, shapes, dt=dtb, steps=400)
    assert want["status"] == orc.ORC_INSTABILITY
    plan.set_field(u0)
    res = plan.run(dtb, steps=400)
    assert res.status == _lib.RBF_ERR_INSTABILITY and res.bad_step == want["step"]
    assert np.array_equal(plan.get_field(), want["field"], equal_nan=True)
    plan.close()


# ---- two steps per launch (pair_kernels.cu) ---------------------------------
@pytest.mark.parametrize("target,n,m", [(20_000, 15, 2), (20_000, 30, 4), (200_000, 15, 2), (50_000, 12, 2)])
@pytest.mark.parametrize("renumber", [False, True], ids=["native", "morton"])
def test_pair_kernel_matches_oracle(synth_cache, target, n, m, renumber):
    """Tile-local temporal blocking: every step count (pairs, an odd last
    step, graph-chunked runs), swap and copy-back, bitwise vs the oracle."""
    nodes, _, shapes = _synth(synth_cache, target, n, m)
    interior = shapes.interior_nodes
    plan = Plan(nodes.n_total, interior, shapes.stencils.neighbors[interior], shapes.weights,
                rb.forcing(nodes.positions[interior]), nodes.positions, renumber=renumber, pair=True,
                resident=False)
    info = plan.info()
    assert info["pair"] == 1 and info["pair_tiles"] > 0 and info["pair_halo_rows"] > 0
    u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    dt = 0.5 * rb.stability_bound(shapes)
    for steps in (1, 2, 3, 64, 65, 130, 131):
        want = orc.run_time_loop(nodes, shapes, steps=steps)
        for copy_back in (False, True):
            plan.set_field(u0)
            res = plan.run(dt, steps=steps, copy_back=copy_back)
            assert res.steps_done == steps and res.residual == want["residual"], (steps, copy_back)
            assert np.array_equal(plan.get_field(), want["field"]), (steps, copy_back)
    # a run continuing from the previous field (the plan tracks the buffer)
    plan.set_field(u0)
    plan.run(dt, steps=33)
    plan.run(dt, steps=40)
    want = orc.run_time_loop(nodes, shapes, steps=73)
    assert np.array_equal(plan.get_field(), want["field"])
    plan.close()


def test_pair_kernel_off_and_auto(synth_cache):
    nodes, _, shapes = _synth(synth_cache, 20_000, 15, 2)
    interior = shapes.interior_nodes
    args = (nodes.n_total, interior, shapes.stencils.neighbors[interior], shapes.weights,
            rb.forcing(nodes.positions[interior]), nodes.positions)
    assert Plan(*args, renumber=True, resident=False).info()["pair"] == 1  # small, streaming: on
    assert Plan(*args, renumber=True).info()["pair"] == 0          # the grid-resident loop runs instead
    assert Plan(*args, renumber=True, resident=False, pair=False).info()["pair"] == 0
    nodes, _, shapes = _synth(synth_cache, 200_000, 15, 2)
    interior = shapes.interior_nodes
    big = Plan(nodes.n_total, interior, shapes.stencils.neighbors[interior], shapes.weights,
               rb.forcing(nodes.positions[interior]), nodes.positions, renumber=True)
    assert big.info()["pair"] == 0                                  # N_i*n > 1e6: single step


def test_pair_kernel_failure_replays_the_exact_step(synth_cache):
    """A non-finite value inside a pair is replayed on the single-step path:
    the failing step and field are the reference's (solver.py:200-206)."""
    nodes, _, shapes = _synth(synth_cache, 20_000, 15, 2)
    interior = shapes.interior_nodes
    plan = Plan(nodes.n_total, interior, shapes.stencils.neighbors[interior], shapes.weights,
                rb.forcing(nodes.positions[interior]), nodes.positions, renumber=True, pair=True,
                resident=False)
    dt = 40.0 * rb.stability_bound(shapes)
    want = orc.run_time_loop(nodes, shapes, dt=dt, steps=400)
    assert want["status"] == orc.ORC_INSTABILITY
    plan.set_field(rb.apply_dirichlet(nodes, np.zeros(nodes.n_total)))
    res = plan.run(dt, steps=400)
    assert res.status == _lib.RBF_ERR_INSTABILITY and res.bad_step == want["step"]
    assert np.array_equal(plan.get_field(), want["field"], equal_nan=True)
    plan.set_field(rb.apply_dirichlet(nodes, np.zeros(nodes.n_total)))
    res = plan.run(0.5 * rb.stability_bound(shapes), steps=77)
    want = orc.run_time_loop(nodes, shapes, steps=77)
    assert np.array_equal(plan.get_field(), want["field"]) and res.residual == want["residual"]


def test_idx16_overflow_slices_path(synth_cache, monkeypatch):
    """Force 16-bit ids on the native (non-Morton) order, where many slices
    overflow the two windows and read int32 ids from HBM instead."""
    monkeypatch.setenv("RBFFD_IDX16", "2")
    nodes, _, shapes = _synth(synth_cache, 200_000, 15, 2)
    interior = shapes.interior_nodes
    plan = Plan(nodes.n_total, interior, shapes.stencils.neighbors[interior], shapes.weights,
                rb.forcing(nodes.positions[interior]))
    info = plan.info()
    assert info["index_bits"] == 16
    assert info["stream_bytes_per_step"] > info["N_i"] * (10 * 15 + 24)  # some overflow slices
    plan.set_field(rb.apply_dirichlet(nodes, np.zeros(nodes.n_total)))
    res = plan.run(0.5 * rb.stability_bound(shapes), steps=60)
    want = orc.run_time_loop(nodes, shapes, steps=60)
    assert np.array_equal(plan.get_field(), want["field"]) and res.residual == want["residual"]


def test_synthetic_steady_streaming_matches_oracle(synth_cache):
    """Steady mode through the graph-chunked streaming path (forced: at 30k
    nodes the plan would pick the grid-resident loop) and through the default
    path; the stop step, the residual and the field must equal the oracle's."""
    nodes, _, shapes = _synth(synth_cache, 30_000, 15, 2)
    cfg = rb.SolveConfig(degree=2, support_size=15, nodes=30_000, mode="steady", tol=1e-2,
                         max_steps=200_000)
    want = orc.run_time_loop(nodes, shapes, mode="steady", tol=1e-2, max_steps=200_000)
    assert want["status"] == orc.ORC_OK
    rep = rb.run_time_loop(cfg, nodes, shapes)
    assert rep.steps == want["steps"]
    assert rep.residual == want["residual"]
    assert np.array_equal(rep.field, want["field"])
    interior = shapes.interior_nodes
    for renumber, persist in ((False, False), (True, False), (True, True)):
        plan = Plan(nodes.n_total, interior, shapes.stencils.neighbors[interior], shapes.weights,
                    rb.forcing(nodes.positions[interior]), nodes.positions, renumber=renumber,
                    resident=False, pair=False, persist=persist)
        assert plan.info()["variant"] == 2 and plan.info()["resident"] == 0
        plan.set_field(rb.apply_dirichlet(nodes, np.zeros(nodes.n_total)))
        res = plan.run(0.5 * rb.stability_bound(shapes), mode="steady", tol=1e-2, max_steps=200_000)
        assert res.steps_done == want["steps"] and res.residual == want["residual"]
        assert np.array_equal(plan.get_field(), want["field"])
        plan.close()


def test_full_size_config2_matches_oracle(synth_cache):
    """BASELINE config 2 (m=2, n=15, N=1e6) at full size: bitwise vs the oracle
    over 12 steps, plus swap == copy-back on the device."""
    nodes, _, shapes = _synth(synth_cache, 1_000_000, 15, 2)
    want = orc.run_time_loop(nodes, shapes, steps=12)
    cfg = rb.SolveConfig(degree=2, support_size=15, nodes=1_000_000, steps=12)
    rep = rb.run_time_loop(cfg, nodes, shapes)
    assert np.array_equal(rep.field, want["field"])
    assert rep.residual == want["residual"]
    cb = rb.run_time_loop(cfg, nodes, shapes, copy_back=True)
    assert np.array_equal(cb.field, rep.field) and cb.residual == rep.residual


@pytest.mark.parametrize("target,n,m,steps", [(10_000_000, 30, 4, 70), (25_000_000, 56, 6, 70)],
                         ids=["C3", "C4"])
def test_full_size_configs_3_4_match_oracle(target, n, m, steps):
    """BASELINE configs 3 and 4 at full size (the bench's own problems: the
    reference's node set for seed 1, device kNN + weights): the kernels the
    bench selects there (16-bit-id / int32-id TMA rings, Morton order) are
    bitwise equal to the oracle over 70 steps -- a full 64-step graph chunk
    plus direct tail launches, the L2-resident ring fill reused across many
    steps -- fields, residual and error norms."""
    nodes, _, shapes = synth.synthetic_problem(target, n, m, seed=1, weights="gpu")
    want = orc.run_time_loop(nodes, shapes, steps=steps)
    cfg = rb.SolveConfig(degree=m, support_size=n, nodes=target, steps=steps)
    rep = rb.run_time_loop(cfg, nodes, shapes, cache=False)
    assert np.array_equal(rep.field, want["field"])
    assert rep.residual == want["residual"]
    assert (rep.linf, rep.l2) == (want["linf"], want["l2"])


def test_full_size_config5_matches_oracle():
    """BASELINE config 5 on one B200 (N=1.05e8, n=56, m=6, seed 1): the only
    config whose SELL arrays exceed 2^31 entries (N_i * n = 5.9e9), so every
    64-bit offset of the packing, the TMA ring and the field transfers is
    exercised.  Field, residual and norms bitwise vs the oracle after 3 steps
    (solver.py:294-311).  Host peak ~100 GB (positions, int64 stencils,
    weights; the interior rows are a view of the stencil array)."""
    nodes, st, shapes = synth.synthetic_problem(100_000_000, 56, 6, seed=1, weights="gpu")
    N, N_i = nodes.n_total, shapes.n_rows
    assert N_i * 56 > 2**31
    interior = shapes.interior_nodes
    B = N - N_i
    assert interior[0] == B and interior[-1] == N - 1  # generated set: interior is the tail
    rows = st.neighbors[B:]  # view, no 47 GB copy
    dt = 0.5 * rb.stability_bound(shapes)
    f_int = orc.forcing(nodes.positions[interior])
    u0 = orc.apply_dirichlet(nodes, np.zeros(N))
    want = orc.run_arrays(N, interior, rows, shapes.weights, f_int, u0, dt, steps=3)
    del f_int, u0
    cfg = rb.SolveConfig(degree=6, support_size=56, nodes=100_000_000, dt=dt, steps=3)
    rep = rb.run_time_loop(cfg, nodes, shapes)
    assert rep.residual == want["residual"]
    assert np.array_equal(rep.field, want["field"])
    assert (rep.linf, rep.l2) == orc.error_norms(want["field"], nodes.positions)


# ---- node-partitioned loop on one device (multigpu.LocalGroup) ---------------
@pytest.mark.parametrize("name,case,P", [
    ("crit6", "fixed100", 1), ("crit6", "fixed100", 2), ("crit6", "fixed100", 3),
    ("m6", "fixed100", 4), ("dome", "paper", 2), ("small", "steady", 2), ("dome", "steady", 3),
])
def test_partitioned_group_matches_reference(golden, manifest, name, case, P):
    """The pack / exchange / step / all-reduce / decide sequence of the
    multi-GPU path, all parts on one GPU: same bits as the reference."""
    from paper_2107_03632_b200.multigpu import LocalGroup, partition, run_partitioned

    nodes, _, shapes, z = golden(name)
    meta = manifest[name][case]
    interior = shapes.interior_nodes
    rows = shapes.stencils.neighbors[interior]
    parts = partition(nodes.n_total, interior, rows, shapes.weights,
                      rb.forcing(nodes.positions[interior]), nodes.positions, P)
    group = LocalGroup(parts)
    cfg = config_for(nodes, shapes, meta)
    field, steps, residual, _, dt = run_partitioned(group, nodes, shapes, cfg)
    assert np.array_equal(field, z[f"{case}__field"])
    assert steps == meta["steps"] and residual == meta["residual"] and dt == meta["dt"]
    group.close()


@pytest.mark.parametrize("exact", [False, True], ids=["fast", "per-step-reduce"])
def test_partitioned_group_paths(golden, manifest, monkeypatch, exact):
    """Fixed mode runs without per-step reductions (one reduction at the end,
    exact replay on failure); RBFFD_GROUP_EXACT forces the per-step path."""
    from paper_2107_03632_b200.multigpu import LocalGroup, partition, run_partitioned

    if exact:
        monkeypatch.setenv("RBFFD_GROUP_EXACT", "1")
    for name, case, P in (("m4", "fixed200", 3), ("crit6", "fixed100", 4)):
        nodes, _, shapes, z = golden(name)
        meta = manifest[name][case]
        interior = shapes.interior_nodes
        parts = partition(nodes.n_total, interior, shapes.stencils.neighbors[interior], shapes.weights,
                          rb.forcing(nodes.positions[interior]), nodes.positions, P)
        group = LocalGroup(parts)
        field, steps, residual, _, _ = run_partitioned(group, nodes, shapes, config_for(nodes, shapes, meta))
        assert np.array_equal(field, z[f"{case}__field"]) and residual == meta["residual"]
        group.close()


def test_partitioned_group_instability_and_synthetic(golden, synth_cache):
    from paper_2107_03632_b200.multigpu import LocalGroup, partition, run_partitioned

    nodes, _, shapes, _ = golden("crit6")
    interior = shapes.interior_nodes
    rows = shapes.stencils.neighbors[interior]
    parts = partition(nodes.n_total, interior, rows, shapes.weights,
                      rb.forcing(nodes.positions[interior]), nodes.positions, 3)
    group = LocalGroup(parts)
    want = orc.run_time_loop(nodes, shapes, dt=1.0, steps=500)
    cfg = rb.SolveConfig(degree=2, support_size=15, nodes=2000, steps=500, dt=1.0)
    with pytest.raises(rb.InstabilityError) as ei:
        run_partitioned(group, nodes, shapes, cfg)
    assert ei.value.step == want["step"]
    # max|u2| of the failing step, like solver.py:200-206
    assert np.array_equal(np.float64(ei.value.max_abs), np.float64(want["max_abs"]),
                          equal_nan=True)
    group.close()

    nodes, _, shapes = _synth(synth_cache, 200_000, 15, 2)
    interior = shapes.interior_nodes
    rows = shapes.stencils.neighbors[interior]
    parts = partition(nodes.n_total, interior, rows, shapes.weights,
                      rb.forcing(nodes.positions[interior]), nodes.positions, 4)
    group = LocalGroup(parts)
    cfg = rb.SolveConfig(degree=2, support_size=15, nodes=200_000, steps=50)
    field, steps, residual, _, _ = run_partitioned(group, nodes, shapes, cfg)
    want = orc.run_time_loop(nodes, shapes, steps=50)
    assert np.array_equal(field, want["field"]) and residual == want["residual"]
    group.close()


@pytest.mark.parametrize("push,fused", [(True, True), (True, False), (False, False)],
                         ids=["fused-part-loop", "p2p-push-kernels", "copy-exchange"])
@pytest.mark.parametrize("P", [2, 5])
def test_partitioned_push_mode_runs(synth_cache, monkeypatch, push, fused, P):
    """Push-mode halos against the copy exchange and the oracle, over
    repeated runs (the arrival counters keep counting across runs), odd step
    counts and graph-chunked runs: the fused partitioned persistent loop (all
    parts in one launch, pushes from the lanes that compute the sent rows)
    and the step + push_halo_kernel graph path."""
    from paper_2107_03632_b200.multigpu import LocalGroup, partition, run_partitioned

    monkeypatch.setenv("RBFFD_PART_LOOP", "1" if fused else "0")
    nodes, _, shapes = _synth(synth_cache, 200_000, 15, 2)
    interior = shapes.interior_nodes
    parts = partition(nodes.n_total, interior, shapes.stencils.neighbors[interior], shapes.weights,
                      rb.forcing(nodes.positions[interior]), nodes.positions, P)
    group = LocalGroup(parts, push=push)
    assert group.push_mode == push
    for steps in (50, 37, 131, 2):
        cfg = rb.SolveConfig(degree=2, support_size=15, nodes=200_000, steps=steps)
        field, done, residual, _, _ = run_partitioned(group, nodes, shapes, cfg)
        want = orc.run_time_loop(nodes, shapes, steps=steps)
        assert done == steps and residual == want["residual"], steps
        assert np.array_equal(field, want["field"]), steps
        assert group.fused == fused, steps
    # a failure inside a pushed run replays on the exact path (same step as the oracle)
    cfg = rb.SolveConfig(degree=2, support_size=15, nodes=200_000, steps=300, dt=40.0 * rb.stability_bound(shapes))
    want = orc.run_time_loop(nodes, shapes, dt=cfg.dt, steps=300)
    with pytest.raises(rb.InstabilityError) as ei:
        run_partitioned(group, nodes, shapes, cfg)
    assert ei.value.step == want["step"]
    assert np.array_equal(np.float64(ei.value.max_abs), np.float64(want["max_abs"]),
                          equal_nan=True)
    # and the group keeps working (pushing) afterwards
    cfg = rb.SolveConfig(degree=2, support_size=15, nodes=200_000, steps=65)
    field, _, residual, _, _ = run_partitioned(group, nodes, shapes, cfg)
    want = orc.run_time_loop(nodes, shapes, steps=65)
    assert np.array_equal(field, want["field"]) and residual == want["residual"]
    assert group.push_mode == push
    # switching a pushing group back to the copy exchange (rbf_group_push_off)
    group.plans[0]._check(group._lib.rbf_group_push_off(group._h))
    assert not group.push_mode
    field, _, residual, _, _ = run_partitioned(group, nodes, shapes, cfg)
    assert np.array_equal(field, want["field"]) and residual == want["residual"]
    group.close()


@pytest.mark.parametrize("n_rows", [1, 33, 100])
def test_streaming_variants_on_tiny_row_counts(n_rows):
    """Partial last slices and single-row problems through every loop variant."""
    rng = np.random.default_rng(n_rows)
    N = n_rows + 40
    n = 15
    interior = np.arange(40, N, dtype=np.int64)
    rows = np.empty((n_rows, n), dtype=np.int64)
    rows[:, 0] = interior
    rows[:, 1:] = rng.integers(0, N, size=(n_rows, n - 1))
    weights = rng.normal(size=(n_rows, n)) * 1e-2
    f = rng.normal(size=n_rows)
    u0 = rng.normal(size=N)
    u2 = u0.copy()
    want = u0.copy()
    for _ in range(7):
        step = want.copy()
        orc.step_kernel(want, step, interior, rows, weights, f, 0.3)
        want = step
    for kw in (dict(), dict(cluster=False), dict(resident=False), dict(resident=False, tma=False),
               dict(resident=False, pdl=False)):
        plan = Plan(N, interior, rows, weights, f, **kw)
        plan.set_field(u0)
        res = plan.run(0.3, steps=7)
        assert res.steps_done == 7
        assert np.array_equal(plan.get_field(), want), kw
        plan.close()
    del u2



@pytest.mark.parametrize("which", ["dome", "crit6", "synthetic"])
def test_plan_file_round_trip_is_bitwise(golden, synth_cache, tmp_path, which):
    """rbf_plan_save / rbf_plan_load: the loaded plan (no packing, renumbering
    or id compression at load) runs bit-identically to the saved one."""
    if which == "synthetic":
        nodes, _, shapes = _synth(synth_cache, 200_000, 15, 2)
    else:
        nodes, _, shapes, _ = golden(which)
    interior = shapes.interior_nodes
    plan = Plan(nodes.n_total, interior, shapes.stencils.neighbors[interior], shapes.weights,
                rb.forcing(nodes.positions[interior]), nodes.positions, renumber=True)
    path = tmp_path / "plan.rbf"
    plan.save(path)
    loaded = Plan.load(path)
    a, b = plan.info(), loaded.info()
    for k in ("N", "N_i", "n", "variant", "index_bits", "renumbered"):
        assert a[k] == b[k], k
    u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    dt = 0.5 * rb.stability_bound(shapes)
    out = []
    for p in (plan, loaded):
        p.set_field(u0)
        r = p.run(dt, steps=130)
        out.append((p.get_field(), r.residual))
    assert np.array_equal(out[0][0], out[1][0]) and out[0][1] == out[1][1]
    want = orc.run_time_loop(nodes, shapes, steps=130)
    assert np.array_equal(out[1][0], want["field"])
    bad = tmp_path / "bad.rbf"
    bad.write_bytes(b"not a plan" * 10)
    with pytest.raises(rb.ParameterError):
        Plan.load(bad)
    trunc = tmp_path / "trunc.rbf"
    trunc.write_bytes(path.read_bytes()[:200])
    with pytest.raises(rb.ParameterError):
        Plan.load(trunc)
    # payload checks: trailing bytes, a node id out of range, a 16-bit id that
    # does not decode to its int32 id (header 96 B, then W, C, F, C16, meta, ...)
    raw = path.read_bytes()
    longer = tmp_path / "longer.rbf"
    longer.write_bytes(raw + b"\0")
    with pytest.raises(rb.ParameterError, match="trailing"):
        Plan.load(longer)
    S, n = (a["N_i"] + 31) // 32, a["n"]
    c_off = 96 + S * 32 * n * 8
    corrupt = bytearray(raw)
    corrupt[c_off:c_off + 4] = np.int32(a["N"] + 5).tobytes()
    cpath = tmp_path / "corrupt.rbf"
    cpath.write_bytes(bytes(corrupt))
    with pytest.raises(rb.ParameterError, match="corrupt"):
        Plan.load(cpath)
    if a["index_bits"] == 16:
        c16_off = c_off + S * 32 * n * 4 + S * 32 * 8
        corrupt = bytearray(raw)
        corrupt[c16_off:c16_off + 2] = np.uint16(np.frombuffer(raw[c16_off:c16_off + 2], np.uint16)[0] ^ 1).tobytes()
        cpath.write_bytes(bytes(corrupt))
        with pytest.raises(rb.ParameterError, match="corrupt"):
            Plan.load(cpath)


def test_device_morton_renumbering_is_the_z_order(synth_cache, tmp_path):
    """The plan's row order must be the (Morton code, k) order over the
    bounding box of all nodes (a wrong order keeps bitwise parity but loses
    the locality the 16-bit ids and the gathers rely on)."""
    import struct

    from paper_2107_03632_b200.multigpu import morton_codes

    nodes, _, shapes = _synth(synth_cache, 30_000, 15, 2)
    interior = shapes.interior_nodes
    plan = Plan(nodes.n_total, interior, shapes.stencils.neighbors[interior], shapes.weights,
                rb.forcing(nodes.positions[interior]), nodes.positions, renumber=True)
    path = tmp_path / "p.rbf"
    plan.save(path)
    raw = path.read_bytes()
    fmt = "<8sii4qii5q"
    _, _, n, N, N_i, B, S, ib, ren, _ = struct.unpack(fmt, raw[:struct.calcsize(fmt)])[:10]
    off = struct.calcsize(fmt) + S * 32 * n * 12 + S * 32 * 8 + (S * 32 * n * 2 + S * 16 if ib == 16 else 0)
    new_id = np.frombuffer(raw, dtype=np.int32, count=N, offset=off)
    row_of_k = np.frombuffer(raw, dtype=np.int64, count=N_i, offset=off + 4 * N)
    xy = nodes.positions
    lo, span = xy.min(0), xy.max(0) - xy.min(0)
    codes = morton_codes(np.vstack([xy[interior], lo, lo + span]))[:-2]  # same box as the library
    order = np.lexsort((np.arange(N_i), codes))
    want = np.empty(N_i, np.int64)
    want[order] = np.arange(N_i)
    assert ren == 1 and np.array_equal(row_of_k, want)
    assert np.array_equal(new_id[interior], B + want)
    assert np.array_equal(np.sort(new_id[~np.isin(np.arange(N), interior)]), np.arange(B))


@pytest.mark.parametrize("N", [1, 5, 8, 100, 128, 129, 1000, 100_003, 1_048_583])
@pytest.mark.parametrize("renumber", [False, True], ids=["native", "morton"])
def test_device_error_norms_have_numpys_bits(N, renumber):
    """rbf_error_norms: linf and l2 of (u - exact) equal numpy's
    (solver.py:239-246: np.max(np.abs(d)), math.sqrt((d**2).mean())) bit for
    bit -- the block sums follow numpy's pairwise tree."""
    import math

    rng = np.random.default_rng(N)
    n_rows = 1 if N < 40 else 33
    B = N - n_rows
    interior = np.arange(B, N, dtype=np.int64)
    rows = rng.integers(0, N, size=(n_rows, 4)).astype(np.int64)
    rows[:, 0] = interior
    pos = rng.uniform(-1, 1, size=(N, 2))
    plan = Plan(N, interior, rows, rng.normal(size=(n_rows, 4)), np.zeros(n_rows), pos if renumber else None,
                renumber=renumber and n_rows > 1)
    for scale in (1.0, 1e-12, 1e150):
        u = rng.normal(size=N) * scale
        exact = rng.normal(size=N) * scale
        plan.set_field(u)
        linf, l2 = plan.error_norms(exact)
        d = u - exact
        assert linf == float(np.max(np.abs(d)))
        assert l2 == math.sqrt(float((d**2).mean())), (N, scale)
    plan.close()


@pytest.mark.parametrize("n", [5, 8, 12, 15, 30, 56, 64, 130])
def test_device_stability_bound_has_numpys_bits(n):
    """rbf_plan_weight_row_sum_max sums each row in numpy's pairwise order:
    2 / it == stability_bound (solver.py:249-254) bit for bit."""
    rng = np.random.default_rng(n)
    n_rows, N = 2000, 5000
    interior = np.arange(N - n_rows, N, dtype=np.int64)
    rows = rng.integers(0, N, size=(n_rows, n)).astype(np.int64)
    w = rng.normal(size=(n_rows, n)) * np.exp(rng.normal(size=(n_rows, n)) * 4)
    plan = Plan(N, interior, rows, w, np.zeros(n_rows))
    shapes = rb.ShapeStore(degree=2, interior_nodes=interior, weights=w,
                           stencils=rb.StencilSet(n=n, neighbors=np.zeros((N, n), dtype=np.int64)))
    assert 2.0 / plan.weight_row_sum_max() == rb.stability_bound(shapes)
    plan.close()


@pytest.mark.parametrize("persist", [True, False], ids=["persistent-loop", "graph-loop"])
def test_streaming_failure_and_copy_back(synth_cache, persist):
    """Streaming runs (persistent loop: one cooperative launch per run; graph
    loop: one launch per step): a non-finite step stops at the oracle's step
    with its u2 as the field (solver.py:200-206), copy-back equals swap, and
    the plan keeps working after the failure."""
    nodes, _, shapes = _synth(synth_cache, 1_000_000, 15, 2)
    interior = shapes.interior_nodes
    plan = Plan(nodes.n_total, interior, shapes.stencils.neighbors[interior], shapes.weights,
                rb.forcing(nodes.positions[interior]), nodes.positions, renumber=True, resident=False,
                pair=False, persist=persist)
    u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    bad_dt = 40.0 * rb.stability_bound(shapes)
    want = orc.run_time_loop(nodes, shapes, dt=bad_dt, steps=200)
    assert want["status"] == orc.ORC_INSTABILITY
    plan.set_field(u0)
    res = plan.run(bad_dt, steps=200)
    assert res.status == _lib.RBF_ERR_INSTABILITY and res.bad_step == want["step"]
    assert np.array_equal(plan.get_field(), want["field"], equal_nan=True)
    dt = 0.5 * rb.stability_bound(shapes)
    want = orc.run_time_loop(nodes, shapes, dt=dt, steps=67)
    for copy_back in (False, True):
        plan.set_field(u0)
        res = plan.run(dt, steps=67, copy_back=copy_back)
        assert res.steps_done == 67 and res.residual == want["residual"]
        assert np.array_equal(plan.get_field(), want["field"])
    plan.close()

