"""Break down the e2e (public API) time of one run_time_loop call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["RBFFD_VERBOSE"] = "1"
import numpy as np
import paper_2107_03632_b200 as rb
from paper_2107_03632_b200 import synth
target = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
n, m = (15, 2) if len(sys.argv) < 3 else (int(sys.argv[2]), int(sys.argv[3]))
nodes, st, sh = synth.synthetic_problem(target, n, m, weights="gpu")
cfg = rb.SolveConfig(degree=m, support_size=n, nodes=target, steps=1000)
rb.run_time_loop(cfg, nodes, sh, cache=False)
for _ in range(2):
    t0 = time.perf_counter()
    f_int = rb.forcing(nodes.positions[sh.interior_nodes]); t1 = time.perf_counter()
    u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total)); t2 = time.perf_counter()
    rows = rb.solver._interior_rows(st.neighbors, sh.interior_nodes); t3 = time.perf_counter()
    plan = rb.Plan(nodes.n_total, sh.interior_nodes, rows, sh.weights, f_int, nodes.positions, renumber=True); t4 = time.perf_counter()
    plan.set_field(u0); t5 = time.perf_counter()
    res = plan.run(0.5 * rb.stability_bound(sh), steps=1000); t6 = time.perf_counter()
    fld = plan.get_field(); t7 = time.perf_counter()
    rb.error_norms(fld, nodes); t8 = time.perf_counter()
    print(f"forcing {1e3*(t1-t0):.1f} dirichlet {1e3*(t2-t1):.1f} rows {1e3*(t3-t2):.1f} plan {1e3*(t4-t3):.1f} "
          f"set_field {1e3*(t5-t4):.1f} run {1e3*(t6-t5):.1f} (dev {1e3*res.device_seconds:.1f}) get {1e3*(t7-t6):.1f} norms {1e3*(t8-t7):.1f} ms")
    plan.close()
