"""Golden node sets from the UNMODIFIED reference generator (test infrastructure).

Records, for a spread of spacings and seeds, what
``rbffd.geometry.generate_unit_disk_nodes`` (pkg/src/rbffd/geometry.py:105-198)
returns: node counts, boundary counts, the sha256 of the positions' bytes and
a few coordinates.  tests/test_geometry.py checks the native generator
(csrc/nodes.cpp) against them bit for bit.  Run in the build container:

    python tests/golden/make_nodes_golden.py
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
from rbffd import geometry as g  # noqa: E402
from rbffd.errors import ParameterError  # noqa: E402

OUT = Path(__file__).with_name("nodes.json")

# (target node count, seed): the reference tests' sets (test_geometry.py,
# test_acceptance.py: seeds 0/1/2/6), negative and multi-word seeds, and the
# C2 benchmark set (target 1e6, seed 1)
CASES = [(30, 0), (100, 0), (100, 1), (300, 2), (1027, 1), (2000, 6), (3000, 7), (5000, -3),
         (3000, 2**40 + 5), (3000, 2**64 + 7), (20000, 3), (100000, 11), (1_000_000, 1)]
H_CASES = [0.49, 0.3, 0.125, 0.05]


def record(h, seed):
    t = time.time()
    ns = g.generate_unit_disk_nodes(h, seed)
    p = ns.positions
    return {"h": h, "seed": str(seed), "n_total": int(ns.n_total), "n_boundary": int(ns.n_boundary),
            "sha256": hashlib.sha256(p.tobytes()).hexdigest(),
            "head": p[:3].tolist(), "tail": p[-3:].tolist(), "ref_seconds": round(time.time() - t, 3)}


def main():
    cases = []
    for target, seed in CASES:
        rec = record(g.spacing_for_node_count(target), seed)
        rec["target"] = target
        cases.append(rec)
        print(target, seed, rec["n_total"], rec["ref_seconds"], flush=True)
    for h in H_CASES:
        cases.append(record(h, 0))
    errors = {}
    for h in (0.0, 0.5, 0.7, -1.0):
        try:
            g.generate_unit_disk_nodes(h, 0)
        except ParameterError as e:
            errors[repr(h)] = str(e)
    try:
        g.spacing_for_node_count(29)
    except ParameterError as e:
        errors["spacing_for_node_count(29)"] = str(e)
    OUT.write_text(json.dumps({"_provenance": {"reference": "/root/reference/pkg (rbffd 0.1.0), unmodified",
                                               "script": "tests/golden/make_nodes_golden.py"},
                               "cases": cases, "errors": errors}, indent=1) + "\n")


if __name__ == "__main__":
    main()
