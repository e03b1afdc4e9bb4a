import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2107_03632_b200 as rb
from paper_2107_03632_b200 import synth
from oracle import oracle as orc
for target, n, m in ((20_000, 15, 2), (100_000, 15, 2), (50_000, 30, 4), (20_000, 56, 6)):
    nodes, st, sh = synth.synthetic_problem(target, n, m, seed=3, weights="gpu")
    interior = sh.interior_nodes
    p = rb.Plan(nodes.n_total, interior, st.neighbors[interior], sh.weights, rb.forcing(nodes.positions[interior]),
                nodes.positions, renumber=True, cluster=False)
    info = p.info()
    dt = 0.5 * rb.stability_bound(sh)
    for steps in (1, 2, 77, 500):
        want = orc.run_time_loop(nodes, sh, steps=steps)
        p.set_field(rb.apply_dirichlet(nodes, np.zeros(nodes.n_total)))
        r = p.run(dt, steps=steps)
        ok = np.array_equal(p.get_field(), want["field"]) and r.residual == want["residual"]
        print(target, n, "variant", info["variant"], "steps", steps, "bitwise", ok, flush=True)
    # steady
    p.set_field(rb.apply_dirichlet(nodes, np.zeros(nodes.n_total)))
    r = p.run(dt, mode="steady", tol=1e-3, max_steps=200000)
    want = orc.run_time_loop(nodes, sh, steps=0, mode="steady", tol=1e-3, max_steps=200000) if False else None
    print("  steady steps", r.steps_done, r.residual)
