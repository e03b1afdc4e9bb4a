"""Both bench arms build their workload on the reference's own arrays.

The GPU arm (paper_2107_03632_b200.synth with knn="cpu", weights="cpu") and
the reference arm (oracle/problem.py, which never maps the product library)
must produce byte-identical positions, stencils and weights, and both must
equal the unmodified reference pipeline (digests recorded by
tests/golden/make_setup_golden.py).  CPU only."""

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN

CASES = json.loads((GOLDEN / "setup.json").read_text())["cases"]


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"N{c['target']}-n{c['n']}-m{c['m']}")
def test_reference_arm_setup_matches_reference(case):
    from oracle import problem as op

    nodes, st, sh = op.reference_problem(case["target"], case["n"], case["m"], seed=case["seed"],
                                         cond_check=True)
    assert nodes.n_total == case["n_total"]
    assert _digest(nodes.positions) == case["positions"]
    assert _digest(st.neighbors) == case["neighbors"]
    assert _digest(sh.interior_nodes) == case["interior"]
    assert _digest(sh.weights) == case["weights"]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"N{c['target']}-n{c['n']}-m{c['m']}")
def test_gpu_arm_cpu_setup_matches_reference(case):
    from paper_2107_03632_b200 import synth

    nodes, st, sh = synth.synthetic_problem(case["target"], case["n"], case["m"], seed=case["seed"],
                                            weights="cpu", knn="cpu")
    assert _digest(nodes.positions) == case["positions"]
    assert _digest(st.neighbors) == case["neighbors"]
    assert _digest(sh.interior_nodes.astype(np.int64)) == case["interior"]
    assert _digest(sh.weights) == case["weights"]


def test_reference_arm_never_maps_the_product_library():
    """oracle/problem.py must not import the package (its __init__ or any
    module that loads librbffd_b200.so)."""
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, '.'); from oracle import problem as op; "
            "op.reference_problem(2000, 15, 2, seed=1); "
            "maps = open('/proc/self/maps').read(); "
            "assert 'librbffd_b200' not in maps, 'product library mapped'; "
            "assert 'paper_2107_03632_b200' not in sys.modules; print('ok')")
    from conftest import ROOT

    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr
