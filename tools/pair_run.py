"""C2 plan with the two-step tile kernel; runs `steps` fixed steps (for ncu / sweeps)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_03632_b200 as rb  # noqa: E402
from paper_2107_03632_b200 import synth  # noqa: E402

target = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
n, m = (15, 2) if len(sys.argv) <= 3 else (int(sys.argv[3]), int(sys.argv[4]))
nodes, st, sh = synth.synthetic_problem(target, n, m, weights="gpu")
interior = sh.interior_nodes
p = rb.Plan(nodes.n_total, interior, st.neighbors[interior], sh.weights, rb.forcing(nodes.positions[interior]),
            nodes.positions, renumber=True)
u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
dt = 0.5 * rb.stability_bound(sh)
p.set_field(u0)
p.run(dt, steps=20)
best = min(p.run(dt, steps=steps).device_seconds for _ in range(3))
print(f"N_i={sh.weights.shape[0]} info={ {k: v for k, v in p.info().items() if k.startswith('pair')} } "
      f"{steps * sh.weights.shape[0] / best:.4e} upd/s {1e6 * best / steps:.2f} us/step", flush=True)
