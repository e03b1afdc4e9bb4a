"""RBFFD_TRACE timelines of the fused partitioned loop: P in-process parts
(tools/trace_summary.py reads the file; needs a `make TRACE=1` library via
RBFFD_LIB).

    RBFFD_LIB=exp/lib_trace.so RBFFD_TRACE=/tmp/g.bin python tools/group_trace.py 1e6 2
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_03632_b200 as rb  # noqa: E402
from paper_2107_03632_b200 import synth  # noqa: E402
from paper_2107_03632_b200.multigpu import LocalGroup, partition  # noqa: E402

target = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
P = int(sys.argv[2]) if len(sys.argv) > 2 else 2
nodes, st, sh = synth.synthetic_problem(target, 15, 2, weights="gpu")
interior = sh.interior_nodes
rows = st.neighbors[interior]
f = rb.forcing(nodes.positions[interior])
u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
dt = 0.5 * rb.stability_bound(sh)
parts = partition(nodes.n_total, interior, rows, sh.weights, f, nodes.positions, P)
g = LocalGroup(parts)
for part, p in zip(parts, g.plans):
    p.set_field(part.local_field(u0))
rc, done, res, bad, sec = g.run(dt, steps=200)
print(f"P={P} fused={g.fused}: {1e6 * sec / 200:.2f} us/step", flush=True)
for part, p in zip(parts, g.plans):
    print(f"  part {part.rank}: rows {part.interior.size}, halo_row0 {p.info().get('halo_row0', '?')}")
g.close()
