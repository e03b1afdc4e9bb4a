import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_03632_b200 as rb
from paper_2107_03632_b200.solver import Plan
from paper_2107_03632_b200 import _lib
nodes, st, sh = rb.load_fixture(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "crit6.npz"))
interior = sh.interior_nodes
for cl in (True,):
    plan = Plan(nodes.n_total, interior, st.neighbors[interior], sh.weights, rb.forcing(nodes.positions[interior]), cluster=cl)
    print(plan.info())
    plan.set_field(rb.apply_dirichlet(nodes, np.zeros(nodes.n_total)))
    for dt, steps in ((1e-5, 100), (1.0, 500)):
        try:
            res = plan.run(dt, steps=steps)
            print("dt", dt, res)
        except Exception as e:
            print("dt", dt, "ERR", e)
        try:
            f = plan.get_field(); print("field ok", np.isfinite(f).sum())
        except Exception as e:
            print("get ERR", e)
