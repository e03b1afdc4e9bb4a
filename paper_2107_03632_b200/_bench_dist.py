"""bench.py under torchrun (N > 1 ranks, one GPU each): the node-partitioned
loop, each rank building only its own part on its GPU (dsetup.RankSetup).

* ``--workload c5`` (BASELINE config 5): strong scaling -- the same
  N = 1e8, m = 6, n = 56 node set split over the ranks;
* the default workload (C2): weak scaling -- N = 1e6 x world nodes, one
  BASELINE-config-2-sized share per GPU (the N = 1 line is the C2 headline).

Setup: rank 0 generates the reference's advancing-front node set (native
generator, bit-identical) and broadcasts it (NCCL); every rank then runs the
exact kNN of its own rows (rbf_knn_subset), its local numbering and halo lists
on its GPU, exchanges halo requests (one all-gather of small dicts), and
assembles its weights inside its plan (rbf_plan_create_assembled).  dt =
0.5 * 2 / (max over ranks of the device row sums, numpy's order) -- the
reference's auto dt for these weights.  The fixed-step loop pushes halos
peer-to-peer over NVLink (CUDA IPC mappings, arrival flags; NCCL for steady
runs).  value = all ranks' node-updates / max-over-ranks device time.
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np


def _log(rank, *a):
    if rank == 0:
        print(*a, file=sys.stderr, flush=True)


def main(args, metric, workloads):  # pragma: no cover - needs >1 GPU (or --force-dist)
    import torch
    import torch.distributed as dist

    from .dsetup import RankSetup
    from .geometry import generate_unit_disk_nodes
    from .multigpu import NcclGroup, assembled_plan, nccl_unique_id
    from .problem import spacing_for_node_count
    from .solver import apply_dirichlet

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("cpu:gloo,cuda:nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", local))
    base_target, n, m, desc = workloads[args.workload]
    strong = args.workload == "c5"
    target = base_target if strong else base_target * world
    t0 = time.perf_counter()
    # ---- the node set: generated once, broadcast
    if rank == 0:
        nodes = generate_unit_disk_nodes(spacing_for_node_count(target), 1)
        meta = torch.tensor([nodes.n_total, int(nodes.is_boundary.sum())], dtype=torch.int64, device="cuda")
        pos_t = torch.from_numpy(nodes.positions).cuda()
    else:
        meta = torch.zeros(2, dtype=torch.int64, device="cuda")
    dist.broadcast(meta, src=0)
    N, nb = int(meta[0]), int(meta[1])
    if rank != 0:
        pos_t = torch.empty((N, 2), dtype=torch.float64, device="cuda")
    dist.broadcast(pos_t, src=0)
    positions = pos_t.cpu().numpy()
    del pos_t
    is_boundary = np.zeros(N, dtype=bool)
    is_boundary[:nb] = True  # generated sets: boundary ring first
    t_nodes = time.perf_counter() - t0
    _log(rank, f"[dist] nodes N={N} in {t_nodes:.1f}s")
    # ---- this rank's part
    setup = RankSetup(positions, is_boundary, n, rank, world, device=local)
    reqs = [None] * world
    dist.all_gather_object(reqs, setup.requests)
    part = setup.finish(reqs)
    plan = assembled_plan(setup, m, device=local)
    mx = torch.tensor([plan.weight_row_sum_max()], dtype=torch.float64)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dt = 0.5 * float(2.0 / mx.item())  # solver.py:188, :249-254
    t_setup = time.perf_counter() - t0
    _log(rank, f"[dist] setup {t_setup:.1f}s (own rows {setup.n_own}, halo {setup.H})")

    uid = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)

    def allgather(blob: bytes):
        out = [None] * world
        dist.all_gather_object(out, blob)
        return out

    push = os.environ.get("RBFFD_GROUP_PUSH", "1") != "0"
    group = NcclGroup(part, rank, world, local, uid[0], allgather=allgather if push else None, plan=plan)
    dist.barrier()  # every rank mapped its neighbours before any rank pushes
    u0 = apply_dirichlet(_Nodes(positions, is_boundary), np.zeros(N))
    u_loc = part.local_field(u0)
    plan.set_field(u_loc)
    group.run(dt, steps=args.warmup)
    plan.set_field(u_loc)
    dist.barrier()
    torch.cuda.synchronize()
    l0 = plan.info()["launches"]
    rc, steps, residual, bad, sec = group.run(dt, steps=args.steps)
    launches = plan.info()["launches"] - l0
    torch.cuda.synchronize()
    t = torch.tensor([sec], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # end to end: host field in, K steps, host field out (per rank, max)
    dist.barrier()
    te = time.perf_counter()
    plan.set_field(u_loc)
    group.run(dt, steps=args.steps)
    plan.get_field()
    te = torch.tensor([time.perf_counter() - te], dtype=torch.float64)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    halo = torch.tensor([8 * sum(part.recv_count)], dtype=torch.int64)
    dist.all_reduce(halo, op=dist.ReduceOp.MAX)
    stream = torch.tensor([float(plan.info()["stream_bytes_per_step"])], dtype=torch.float64)
    dist.all_reduce(stream, op=dist.ReduceOp.SUM)  # bytes all ranks' loops stream per step
    n_rows_total = int(N - nb)
    peak = 6650.0
    try:
        peak = float(json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json")
                                .read_text())["hbm_gbs"])
    except Exception:
        pass
    if rank == 0:
        tmax = t.item()
        value = args.steps * n_rows_total / tmax
        per_gpu = stream.item() / world / (tmax / args.steps) / 1e9
        line = {
            "metric": metric, "value": value, "unit": "node-updates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tmax / args.steps,
            "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic: the reference's advancing-front node set (seed 1), exact GPU kNN, "
                    "GPU-assembled weights per rank",
            "config": {"workload": (f"{desc}, split over {world} GPUs (strong scaling)" if strong else
                                    f"{desc} per GPU (weak scaling: one disk of {N} nodes)"),
                       "N": N, "N_i": n_rows_total, "n": n, "m": m, "dt": dt,
                       "parallelism": (f"node-partitioned x{world}, "
                                       + ("fused partitioned persistent loop (one launch per run; halo "
                                          "values pushed P2P over NVLink through CUDA IPC by the lanes "
                                          "that compute them, release/acquire arrival counters)"
                                          if group.fused and group.push_mode else
                                          "fused partitioned persistent loop (one part: no exchange)"
                                          if group.fused else
                                          "halo exchange: P2P push kernels over NVLink (CUDA IPC)"
                                          if group.push_mode else "halo exchange: NCCL send/recv")),
                       "halo_bytes_per_step_max_rank": int(halo.item()),
                       "setup_seconds": t_setup, "node_generation_seconds": t_nodes},
            "roofline": {"bound": "hbm", "achieved": per_gpu, "peak": peak, "unit": "GB/s per GPU",
                         "frac": per_gpu / peak, "traffic": None,
                         "bytes_formula": "bytes the ranks' loops stream per step (16-bit ids: 10n+24 per "
                                          "row + 16 per slice; int32: 12n+24) / world"},
            "e2e": {"value": args.steps * n_rows_total / te.item(), "unit": "node-updates/s",
                    "h2d_bytes_per_step": 8 * N / args.steps, "d2h_bytes_per_step": 8 * N / args.steps},
            "gpu_launches": launches,
            "residual": residual,
        }
        print(json.dumps(line), flush=True)
    group.close()
    dist.destroy_process_group()
    return 0


class _Nodes:
    """The NodeSet fields apply_dirichlet reads."""

    def __init__(self, positions, is_boundary):
        self.positions = positions
        self.is_boundary = is_boundary

    @property
    def n_total(self):
        return self.positions.shape[0]

    @property
    def boundary_indices(self):
        return np.flatnonzero(self.is_boundary)
