"""Two-step tile kernel vs the single-step path: bitwise equality and timing."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2107_03632_b200 as rb  # noqa: E402
from paper_2107_03632_b200 import synth  # noqa: E402

target = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
n, m = (15, 2) if len(sys.argv) <= 2 else (int(sys.argv[2]), int(sys.argv[3]))
t0 = time.time()
nodes, st, sh = synth.synthetic_problem(target, n, m, weights="gpu")
interior = sh.interior_nodes
rows = st.neighbors[interior]
f = rb.forcing(nodes.positions[interior])
u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
dt = 0.5 * rb.stability_bound(sh)
print(f"setup {time.time()-t0:.1f}s N={nodes.n_total} n={n}", flush=True)
plans = {}
for pair in (True, False):
    t0 = time.time()
    p = rb.Plan(nodes.n_total, interior, rows, sh.weights, f, nodes.positions, renumber=True, pair=pair)
    print("pair" if pair else "single", f"plan {time.time()-t0:.2f}s", {k: v for k, v in p.info().items()
          if k in ("variant", "index_bits", "pair", "pair_tiles", "pair_halo_rows", "grid")}, flush=True)
    plans[pair] = p
for steps in (1, 2, 3, 64, 101, 130, 1000):
    out = {}
    for pair, p in plans.items():
        p.set_field(u0)
        r = p.run(dt, steps=steps)
        out[pair] = (p.get_field(), r.steps_done, r.residual)
    same = out[True][0].tobytes() == out[False][0].tobytes()
    print(f"steps={steps}: bitwise={same} steps={out[True][1]}/{out[False][1]} res={out[True][2]!r}/{out[False][2]!r}", flush=True)
    if not same:
        d = np.flatnonzero(out[True][0] != out[False][0])
        print("  differing nodes", d.size, d[:10])
for pair, p in plans.items():
    p.set_field(u0)
    p.run(dt, steps=200)
    best = []
    for _ in range(3):
        r = p.run(dt, steps=4000)
        best.append(r.device_seconds)
    t = min(best)
    print(("pair  " if pair else "single"), f"{4000 * sh.weights.shape[0] / t:.4e} upd/s  {1e6 * t / 4000:.2f} us/step", flush=True)
