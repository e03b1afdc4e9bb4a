"""Phase times of run_time_loop (the bench's e2e leg) on C2 at K steps:
python tools/e2e_phases.py [K]   (RBFFD_VERBOSE phase lines on stderr)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("RBFFD_VERBOSE", "1")
import paper_2107_03632_b200 as rb  # noqa: E402
from paper_2107_03632_b200 import synth  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nodes, st, sh = synth.synthetic_problem(1_000_000, 15, 2, seed=1, weights="cpu", knn="cpu")
cfg = rb.SolveConfig(degree=2, support_size=15, nodes=1_000_000, dt=0.5 * rb.stability_bound(sh), steps=K)
for i in range(5):
    t0 = time.perf_counter()
    rep = rb.run_time_loop(cfg, nodes, sh)
    t = time.perf_counter() - t0
    print(f"call {i}: {1e3 * t:.2f} ms (device loop {1e3 * rep.device_seconds:.3f} ms, "
          f"non-loop {1e3 * (t - rep.device_seconds):.2f} ms)", file=sys.stderr, flush=True)
