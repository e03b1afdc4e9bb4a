"""Two-step tile kernel vs single-step path: device us/step across problem sizes."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_03632_b200 as rb  # noqa: E402
from paper_2107_03632_b200 import synth  # noqa: E402

n, m = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (15, 2)
for target in (5_000, 20_000, 50_000, 100_000, 200_000, 400_000, 1_000_000):
    nodes, st, sh = synth.synthetic_problem(target, n, m, weights="gpu")
    interior = sh.interior_nodes
    f = rb.forcing(nodes.positions[interior])
    u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
    dt = 0.5 * rb.stability_bound(sh)
    steps = 4000
    res = {}
    for pair in (True, False):
        p = rb.Plan(nodes.n_total, interior, st.neighbors[interior], sh.weights, f, nodes.positions,
                    renumber=True, pair=pair)
        p.set_field(u0)
        p.run(dt, steps=100)
        res[pair] = min(p.run(dt, steps=steps).device_seconds for _ in range(3)) / steps * 1e6
        info = p.info()
        del p
    print(f"N={nodes.n_total:>8d} n={n} variant={info['variant']} pair {res[True]:7.2f} us/step  single {res[False]:7.2f}"
          f"  ratio {res[False] / res[True]:.3f}", flush=True)
