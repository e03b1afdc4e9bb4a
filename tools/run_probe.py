"""Wall vs device time of consecutive Plan.run calls on one plan."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_03632_b200 as rb
from paper_2107_03632_b200 import synth
nodes, st, sh = synth.synthetic_problem(1_000_000, 15, 2, weights="gpu")
f_int = rb.forcing(nodes.positions[sh.interior_nodes])
u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
rows = rb.solver._interior_rows(st.neighbors, sh.interior_nodes)
dt = 0.5 * rb.stability_bound(sh)
for rep in range(3):
    plan = rb.Plan(nodes.n_total, sh.interior_nodes, rows, sh.weights, f_int, nodes.positions, renumber=True)
    plan.set_field(u0)
    for k in (1000, 1000, 10, 64, 65):
        t0 = time.perf_counter(); res = plan.run(dt, steps=k); t1 = time.perf_counter()
        print(f"plan{rep} steps={k}: wall {1e3*(t1-t0):.2f} ms dev {1e3*res.device_seconds:.2f} ms")
    t0 = time.perf_counter(); plan.close(); print(f"close {1e3*(time.perf_counter()-t0):.1f} ms")
