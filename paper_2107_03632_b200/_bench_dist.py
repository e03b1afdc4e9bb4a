"""bench.py under torchrun (N > 1 ranks, one GPU each): the node-partitioned
loop with NCCL halo exchange (multigpu.NcclGroup).

Weak scaling: each GPU holds one BASELINE-config-2-sized share (N = 1e6 per
GPU, m=2, n=15) of the reference's advancing-front disk of N x world nodes; value = all ranks'
node-updates / max-over-ranks device time.  Each rank assembles only the
weights of its own rows.  torch.distributed (gloo) is the control plane
(NCCL id broadcast, barriers, max over ranks); the halos and the per-step
all-reduce run on the library's own NCCL communicator.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np


def main(args, metric, workloads):  # pragma: no cover - needs >1 GPU
    import torch
    import torch.distributed as dist

    from . import synth
    from .multigpu import NcclGroup, nccl_unique_id, partition
    from .problem import forcing
    from .solver import apply_dirichlet

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    target_per_gpu, n, m, desc = workloads[args.workload]
    target = target_per_gpu * world
    t0 = time.perf_counter()
    from .geometry import generate_unit_disk_nodes
    from .problem import spacing_for_node_count

    # the reference's advancing-front set, identical on every rank
    nodes = generate_unit_disk_nodes(spacing_for_node_count(target), 1)
    st = synth.knn_stencils(nodes, n, workers=max(1, (os.cpu_count() or 1) // world))
    interior = nodes.interior_indices.astype(np.int64)
    rows = np.ascontiguousarray(st.neighbors[interior])
    f_int = forcing(nodes.positions[interior])
    parts = partition(nodes.n_total, interior, rows, None, f_int, nodes.positions, world)
    me = parts[rank]
    expo = synth._exponents(m)
    w = np.empty((me.n_own, n))
    for lo in range(0, me.n_own, 4096):
        hi = min(lo + 4096, me.n_own)
        sup = nodes.positions[rows[me.rows_ref[lo:hi]]]
        w[lo:hi] = synth._weights_batch(sup, expo)
    me.weights = w
    # dt = 0.5 * stability_bound over ALL rows (solver.py:188, :249-254)
    mx = torch.tensor([float(np.abs(w).sum(axis=1).max())], dtype=torch.float64)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dt = 0.5 * float(2.0 / mx.item())
    t_setup = time.perf_counter() - t0
    uid = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    def allgather(blob: bytes):
        out = [None] * world
        dist.all_gather_object(out, blob)
        return out

    push = os.environ.get("RBFFD_GROUP_PUSH", "1") != "0"
    group = NcclGroup(me, rank, world, local, uid[0], allgather=allgather if push else None)
    dist.barrier()  # every rank mapped its neighbours before any rank pushes
    plan = group.plans[0]
    u0 = apply_dirichlet(nodes, np.zeros(nodes.n_total))
    u_loc = me.local_field(u0)
    plan.set_field(u_loc)
    group.run(dt, steps=args.warmup)
    plan.set_field(u_loc)
    dist.barrier()
    torch.cuda.synchronize()
    rc, steps, residual, bad, sec = group.run(dt, steps=args.steps)
    torch.cuda.synchronize()
    t = torch.tensor([sec], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # end to end: host field in, K steps, host field out
    dist.barrier()
    te = time.perf_counter()
    plan.set_field(u_loc)
    group.run(dt, steps=args.steps)
    plan.get_field()
    te = torch.tensor([time.perf_counter() - te], dtype=torch.float64)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    n_rows_total = int(interior.size)
    peak = 6650.0
    try:
        from pathlib import Path

        peak = float(json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json")
                                .read_text())["hbm_gbs"])
    except Exception:
        pass
    if rank == 0:
        tmax = t.item()
        value = args.steps * n_rows_total / tmax
        bytes_per_step = n_rows_total * (12 * n + 24)
        per_gpu = bytes_per_step / world / (tmax / args.steps) / 1e9
        line = {
            "metric": metric, "value": value, "unit": "node-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tmax / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{desc} per GPU (weak scaling, one disk of {nodes.n_total} nodes)",
                       "N": int(nodes.n_total), "N_i": n_rows_total, "n": n, "m": m, "dt": dt,
                       "parallelism": (f"node-partitioned x{world}, halo exchange: "
                                       + ("P2P push over NVLink (CUDA IPC), fused arrival flags"
                                          if group.push_mode else "NCCL send/recv")),
                       "halo_bytes_per_step_rank0": me.halo_bytes_per_step(),
                       "setup_seconds": t_setup},
            "roofline": {"bound": "hbm", "achieved": per_gpu, "peak": peak, "unit": "GB/s per GPU",
                         "frac": per_gpu / peak, "traffic": None},
            "e2e": {"value": args.steps * n_rows_total / te.item(), "unit": "node-updates/s",
                    "h2d_bytes_per_step": 8 * nodes.n_total / args.steps,
                    "d2h_bytes_per_step": 8 * nodes.n_total / args.steps},
            "gpu_launches": (2 if group.push_mode else 4) * args.steps,
        }
        print(json.dumps(line), flush=True)
    group.close()
    dist.destroy_process_group()
    return 0
