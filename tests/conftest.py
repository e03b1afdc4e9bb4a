import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the sm_100a library)")


@pytest.fixture(scope="session")
def manifest():
    return json.loads((GOLDEN / "manifest.json").read_text())


def load_golden(name):
    """(nodes, stencils, shapes, npz) of a committed golden fixture."""
    from paper_2107_03632_b200.problem import load_fixture

    path = GOLDEN / f"{name}.npz"
    nodes, stencils, shapes = load_fixture(path)
    return nodes, stencils, shapes, np.load(path)


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]

    return get
