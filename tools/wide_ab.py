"""A/B of the wide-stencil (n=56) TMA step: 15 consumer warps with two gather
halves (default build) vs 8 warps with all gathers in flight (RBFFD_WIDE8)."""
import os, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, numpy as np
sys.path.insert(0, ROOT)
import paper_2107_03632_b200 as rb
from paper_2107_03632_b200 import synth
nodes, st, sh = synth.synthetic_problem(3_000_000, 56, 6, weights="gpu")
interior = sh.interior_nodes
plan = rb.Plan(nodes.n_total, interior, rb.solver._interior_rows(st.neighbors, interior), sh.weights,
               rb.forcing(nodes.positions[interior]), nodes.positions, renumber=True)
plan.set_field(rb.apply_dirichlet(nodes, np.zeros(nodes.n_total)))
dt = 0.5 * rb.stability_bound(sh)
plan.run(dt, steps=20)
r = plan.run(dt, steps=300)
info = plan.info()
print(LABEL, info["block"], f"{300 * info['N_i'] / r.device_seconds:.4e} upd/s",
      f"{info['bytes_per_step'] * 300 / r.device_seconds / 1e9:.0f} GB/s")
'''
for label, lib in (("cw15-halves", None), ("cw8-full", os.path.join(root, "paper_2107_03632_b200", "librbffd_wide8.so"))):
    env = dict(os.environ)
    if lib:
        env["RBFFD_LIB"] = lib
    subprocess.run([sys.executable, "-c", code.replace("ROOT", repr(root)).replace("LABEL", repr(label))], env=env, check=False)
