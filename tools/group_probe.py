"""Partitioned loop on one GPU: per-step cost of the halo exchange modes.

All parts run in order on one device, so a P-part step costs the sum of the
parts' steps plus the exchange: compare against one plan over all rows.
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2107_03632_b200 as rb  # noqa: E402
from paper_2107_03632_b200 import synth  # noqa: E402
from paper_2107_03632_b200.multigpu import LocalGroup, partition  # noqa: E402

target = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
nodes, st, sh = synth.synthetic_problem(target, 15, 2, weights="gpu")
interior = sh.interior_nodes
rows = st.neighbors[interior]
f = rb.forcing(nodes.positions[interior])
u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
dt = 0.5 * rb.stability_bound(sh)
steps = 2000
for persist in (False, True):
    plan = rb.Plan(nodes.n_total, interior, rows, sh.weights, f, nodes.positions, renumber=True, pair=False,
                   persist=persist)
    plan.set_field(u0)
    plan.run(dt, steps=100)
    t = min(plan.run(dt, steps=steps).device_seconds for _ in range(3)) / steps
    print(f"N={nodes.n_total} one plan ({'persistent loop' if persist else 'graph loop'}): "
          f"{1e6 * t:.2f} us/step", flush=True)
    if not persist:
        t1 = t  # the parts run the graph loop: compare like with like
    del plan
for P in (1, 2, 4):
    parts = partition(nodes.n_total, interior, rows, sh.weights, f, nodes.positions, P)
    for label, push, fused in (("fused part loop", True, "1"), ("push kernels", True, "0"), ("copy", False, "0")):
        os.environ["RBFFD_PART_LOOP"] = fused
        g = LocalGroup(parts, push=push)
        for part, p in zip(parts, g.plans):
            p.set_field(part.local_field(u0))
        g.run(dt, steps=100)
        best = 1e9
        for _ in range(3):
            for part, p in zip(parts, g.plans):
                p.set_field(part.local_field(u0))
            rc, done, res, bad, sec = g.run(dt, steps=steps)
            best = min(best, sec / steps)
        halo = sum(pt.halo_bytes_per_step() for pt in parts)
        print(f"  P={P} {label} (fused={g.fused}): {1e6 * best:.2f} us/step for all parts "
              f"(+{1e6 * (best - t1):.2f} us vs one plan; halo {halo / 1e3:.0f} kB/step)", flush=True)
        g.close()
