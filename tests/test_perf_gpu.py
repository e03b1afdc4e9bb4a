"""Benchmark harness mirror (pkg/tests/test_perf.py:91-152) on the GPU path."""

import csv
from dataclasses import replace

import numpy as np
import pytest

import paper_2107_03632_b200 as rb
from paper_2107_03632_b200 import perf, synth
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bench_problem():
    return synth.synthetic_problem(3000, 12, 2, seed=4)


@pytest.fixture(scope="module")
def bench_config():
    return rb.SolveConfig(degree=2, support_size=12, nodes=3000, dt=None, steps=2000, seed=4)


def test_benchmark_zero_steps(bench_config, bench_problem):
    reports = perf.benchmark_time_loop(replace(bench_config, steps=0), [1], repeats=1,
                                       problem=bench_problem)
    assert reports[0].ns_per_step_node is None
    assert reports[0].loop_seconds < 0.05


def test_benchmark_repeats_consistent(bench_config, bench_problem):
    a, b = perf.benchmark_time_loop(bench_config, [1, 1], repeats=3, problem=bench_problem)
    assert abs(a.loop_seconds - b.loop_seconds) <= 0.2 * max(a.loop_seconds, b.loop_seconds)


def test_benchmark_digest_matches_cpu_oracle(bench_config, bench_problem):
    """Digests are identical across thread counts AND equal to the digest of
    the CPU oracle's field (perf.py:75 used as a bitwise check)."""
    import hashlib

    reports = perf.benchmark_time_loop(bench_config, [1, 2], repeats=1, problem=bench_problem)
    assert reports[0].field_digest == reports[1].field_digest
    assert reports[0].threads == 1
    nodes, _, shapes = bench_problem
    want = orc.run_time_loop(nodes, shapes, steps=bench_config.steps)
    assert reports[0].field_digest == hashlib.sha256(want["field"].tobytes()).hexdigest()


def test_benchmark_rate_definition(bench_config, bench_problem):
    (r,) = perf.benchmark_time_loop(bench_config, [1], repeats=1, problem=bench_problem)
    assert r.ns_per_step_node == pytest.approx(1e9 * r.loop_seconds / (r.steps * r.n_interior), rel=1e-12)


def test_benchmark_rejects_bad_arguments(bench_config, bench_problem):
    with pytest.raises(rb.ParameterError):
        perf.benchmark_time_loop(bench_config, [1], repeats=0, problem=bench_problem)
    with pytest.raises(rb.ParameterError):
        perf.benchmark_time_loop(bench_config, [], repeats=1, problem=bench_problem)
    with pytest.raises(rb.ParameterError):
        perf.benchmark_time_loop(replace(bench_config, mode="steady"), [1], repeats=1,
                                 problem=bench_problem)
