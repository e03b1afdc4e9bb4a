"""Check the device renumbering (row_of_k / new_id) against numpy via a plan file."""
import os, sys, struct, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2107_03632_b200 as rb
from paper_2107_03632_b200 import synth
from paper_2107_03632_b200.multigpu import morton_codes
nodes, st, sh = synth.synthetic_problem(20000, 15, 2, weights="gpu")
interior = sh.interior_nodes
plan = rb.Plan(nodes.n_total, interior, st.neighbors[interior], sh.weights, rb.forcing(nodes.positions[interior]),
               nodes.positions, renumber=True)
path = os.path.join(tempfile.mkdtemp(), "p.rbf")
plan.save(path)
raw = open(path, "rb").read()
hdr = struct.unpack("<8sii4qii5q", raw[:struct.calcsize("<8sii4qii5q")])
magic, ver, n, N, N_i, B, S, ib, ren, over = hdr[:10]
print("hdr", N, N_i, B, S, ib, ren, over)
off = struct.calcsize("<8sii4qii5q")
sell = S * 32 * n
off += sell * 8 + sell * 4 + S * 32 * 8
if ib == 16:
    off += sell * 2 + S * 16
new_id = np.frombuffer(raw, dtype=np.int32, count=N, offset=off); off += N * 4
row_of_k = np.frombuffer(raw, dtype=np.int64, count=N_i, offset=off)
# the library normalises over the bounding box of ALL nodes
xy = nodes.positions
lo = xy.min(0); span = xy.max(0) - lo
q = ((xy[interior] - lo) * (2097151.0 / span)).astype(np.uint64)
def spread(v):
    v = v & np.uint64(0x1FFFFF)
    for sh, m in ((16, 0x0000FFFF0000FFFF), (8, 0x00FF00FF00FF00FF), (4, 0x0F0F0F0F0F0F0F0F), (2, 0x3333333333333333), (1, 0x5555555555555555)):
        v = (v | (v << np.uint64(sh))) & np.uint64(m)
    return v
codes = spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1))
order = np.lexsort((np.arange(N_i), codes))
want_row = np.empty(N_i, np.int64); want_row[order] = np.arange(N_i)
print("row_of_k equal:", np.array_equal(row_of_k, want_row), row_of_k[:10], want_row[:10])
want_new = np.empty(N, np.int64); nb = ~np.isin(np.arange(N), interior)
want_new[nb] = np.arange(nb.sum()); want_new[interior] = B + want_row
print("new_id equal:", np.array_equal(new_id, want_new))
