"""Plan build from host arrays vs rbf_plan_save / rbf_plan_load (C3 size)."""
import os, sys, time, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_03632_b200 as rb
from paper_2107_03632_b200 import synth
target, n, m = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (10_000_000, 30, 4)
nodes, st, sh = synth.synthetic_problem(target, n, m, weights="gpu")
interior = sh.interior_nodes
rows = rb.solver._interior_rows(st.neighbors, interior)
f = rb.forcing(nodes.positions[interior])
rb.Plan(nodes.n_total, interior[:1000], rows[:1000], sh.weights[:1000], f[:1000]).close()  # warm
t0 = time.perf_counter()
plan = rb.Plan(nodes.n_total, interior, rows, sh.weights, f, nodes.positions, renumber=True)
t1 = time.perf_counter()
d = tempfile.mkdtemp()
path = os.path.join(d, "c.rbf")
plan.save(path)
t2 = time.perf_counter()
loaded = rb.Plan.load(path)
t3 = time.perf_counter()
u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
dt = 0.5 * rb.stability_bound(sh)
res = []
for p in (plan, loaded):
    p.set_field(u0); r = p.run(dt, steps=50); res.append((p.get_field(), r.residual))
size = os.path.getsize(path)
print(f"N={nodes.n_total} n={n}: build {t1-t0:.2f}s  save {t2-t1:.2f}s  load {t3-t2:.2f}s  file {size/1e9:.2f} GB  "
      f"bitwise {np.array_equal(res[0][0], res[1][0]) and res[0][1] == res[1][1]}")
os.remove(path)
