"""Repeated run_time_loop(cache=False) wall times on C2 (e2e leg of bench.py)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("RBFFD_VERBOSE", "1")
import numpy as np
import paper_2107_03632_b200 as rb
from paper_2107_03632_b200 import synth
T = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
nodes, st, sh = synth.synthetic_problem(T, 15, 2, weights="gpu")
cfg = rb.SolveConfig(degree=2, support_size=15, nodes=T, dt=0.5 * rb.stability_bound(sh), steps=K)
for i in range(4):
    t0 = time.perf_counter()
    rep = rb.run_time_loop(cfg, nodes, sh, cache=False)
    print(f"call {i}: {1e3 * (time.perf_counter() - t0):.1f} ms (loop wall {1e3 * rep.wall_time_s:.1f}, device {1e3 * rep.device_seconds:.1f})", flush=True)
