"""The cross-process partitioned loop on the device: two processes, one
part each, halos pushed peer-to-peer through CUDA IPC mappings of each
other's field buffers, arrival flags with system-scope release / acquire
(csrc/group.inc.cuh).  The driver gives one GPU, so both ranks share it:
NCCL refuses two ranks on one device, and kernels that wait on each other
across time-sliced contexts are not guaranteed to be co-scheduled
(B200_PROFILING.md), so the steps are paced by a gloo barrier
(multigpu.HostPacedGroup): every wait a step kernel performs is already
satisfied when it starts.  The assembled field and residual must equal the
oracle's bit for bit (solver.py:198-217)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, target, steps_list, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), RBFFD_WAIT_TIMEOUT_MS="5000")
    import torch.distributed as dist

    import paper_2107_03632_b200 as rb
    from oracle import oracle as orc
    from paper_2107_03632_b200 import synth
    from paper_2107_03632_b200.multigpu import HostPacedGroup, assemble_field, partition

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nodes, st, shapes = synth.synthetic_problem(target, 15, 2, seed=3, weights="cpu", knn="cpu")
        interior = shapes.interior_nodes
        rows = st.neighbors[interior]
        parts = partition(nodes.n_total, interior, rows, shapes.weights,
                          rb.forcing(nodes.positions[interior]), nodes.positions, world)

        def allgather(blob: bytes):
            out = [None] * world
            dist.all_gather_object(out, blob)
            return out

        group = HostPacedGroup(parts[rank], rank, world, 0, allgather, dist.barrier)
        dt = 0.5 * rb.stability_bound(shapes)
        u0 = rb.apply_dirichlet(nodes, np.zeros(nodes.n_total))
        results = []
        for steps in steps_list:
            group.plans[0].set_field(parts[rank].local_field(u0))
            rc, done, residual, bad, _ = group.run(dt, steps=steps)
            loc = group.plans[0].get_field()
            locs = [None] * world
            dist.all_gather_object(locs, loc)
            if rank == 0:
                field = assemble_field(parts, locs, u0)
                want = orc.run_time_loop(nodes, shapes, dt=dt, steps=steps)
                results.append((steps, rc, done, bool(np.array_equal(field, want["field"])),
                                residual == want["residual"], bad))
        group.close()
        if rank == 0:
            q.put(("ok", results, int(sum(len(s) for s in parts[0].send_idx)),
                   int(sum(parts[0].recv_count))))
    except Exception as exc:  # report instead of hanging the peer
        q.put(("error", f"rank {rank}: {type(exc).__name__}: {exc}", 0, 0))
        raise
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_two_process_ipc_push_group_is_bitwise():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    steps_list = [2, 37, 70]
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 100_000, steps_list, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=600)
        if pr.exitcode is None:
            pr.kill()
    status, results, sent, received = q.get(timeout=30)
    assert status == "ok", results
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    assert sent > 0 and received > 0  # a real two-way halo
    for steps, rc, done, field_ok, res_ok, bad in results:
        assert rc == 0 and done == steps and bad == -1, (steps, rc, done, bad)
        assert field_ok and res_ok, steps
