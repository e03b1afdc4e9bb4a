"""Mid-size problems: single-step graph loop vs the grid-resident loop (us/step)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_03632_b200 as rb  # noqa: E402
from paper_2107_03632_b200 import synth  # noqa: E402

n, m = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (15, 2)
import os
sizes = [int(float(x)) for x in os.environ.get('SIZES', '12000,20000,50000,100000,150000,200000,400000').split(',')]
for target in sizes:
    nodes, st, sh = synth.synthetic_problem(target, n, m, weights="gpu")
    interior = sh.interior_nodes
    f = rb.forcing(nodes.positions[interior])
    u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    dt = 0.5 * rb.stability_bound(sh)
    steps = 4000
    out = {}
    for name, kw in (("single", dict(pair=False, resident=False)), ("grid", dict(resident=True))):
        p = rb.Plan(nodes.n_total, interior, st.neighbors[interior], sh.weights, f, nodes.positions,
                    renumber=True, cluster=False, **kw)
        if name == "grid" and p.info()["variant"] != 4:
            out[name] = float("nan")
            continue
        p.set_field(u0)
        p.run(dt, steps=100)
        out[name] = min(p.run(dt, steps=steps).device_seconds for _ in range(3)) / steps * 1e6
        del p
    print(f"N={nodes.n_total:>8d} n={n} " + "  ".join(f"{k} {v:7.2f}" for k, v in out.items()), flush=True)
