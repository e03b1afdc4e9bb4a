"""Record digests of the reference's own benchmark setup (node set ->
build_stencils -> assemble_shapes) for small (target, n, m, seed) cases:
tests/golden/setup.json.  Run in the build container, where the unmodified
reference imports:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb \\
        python tests/golden/make_setup_golden.py

tests/test_bench_setup.py checks oracle/problem.py (the reference arm's
setup) and paper_2107_03632_b200.synth (the GPU arm's CPU setup) against
these digests, so both bench arms time the loop on the reference's arrays."""

import hashlib
import json
from pathlib import Path

import numpy as np
from rbffd.geometry import generate_unit_disk_nodes, spacing_for_node_count
from rbffd.neighborhoods import build_stencils
from rbffd.weights import assemble_shapes

CASES = [(20_000, 15, 2, 1), (20_000, 30, 4, 1), (8_000, 56, 6, 1), (3_000, 12, 2, 5)]


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = {"_provenance": {"reference": "/root/reference/pkg (rbffd 0.1.0), unmodified",
                           "script": "tests/golden/make_setup_golden.py"}, "cases": []}
    for target, n, m, seed in CASES:
        nodes = generate_unit_disk_nodes(spacing_for_node_count(target), seed)
        st = build_stencils(nodes, n)
        sh = assemble_shapes(nodes, st, m)
        out["cases"].append({"target": target, "n": n, "m": m, "seed": seed,
                             "n_total": int(nodes.n_total), "positions": digest(nodes.positions),
                             "neighbors": digest(st.neighbors), "weights": digest(sh.weights),
                             "interior": digest(sh.interior_nodes.astype(np.int64))})
        print(out["cases"][-1])
    Path(__file__).with_name("setup.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
