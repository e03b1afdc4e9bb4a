"""Per-rank setup of the partitioned loop (dsetup.RankSetup) on the CPU:
torch CPU tensors for the index arithmetic and a host kNN, so the multi-rank
logic (Morton split, interior-first rows, local numbering, halo requests
exchanged between ranks) runs here; every part must equal the host
partitioner's (multigpu.partition).  The device path is
tests/test_dsetup_gpu.py."""

import os
import socket

import numpy as np
import pytest

from paper_2107_03632_b200 import synth
from paper_2107_03632_b200.dsetup import RankSetup, build_parts_in_process
from paper_2107_03632_b200.multigpu import partition
from paper_2107_03632_b200.problem import forcing


@pytest.fixture(scope="module")
def problem():
    return synth.synthetic_problem(6_000, 15, 2, seed=4, weights="cpu", knn="cpu")


def _assert_same(a, b):
    assert (a.n_local, a.n_boundary, a.n_halo) == (b.n_local, b.n_boundary, b.n_halo)
    for f in ("rows_ref", "local_to_global", "interior", "rows", "f_int"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert a.peers == b.peers and a.recv_offset == b.recv_offset and a.recv_count == b.recv_count
    for x, y in zip(a.send_idx, b.send_idx):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_rank_setups_equal_host_partition(problem, P):
    nodes, st, shapes = problem
    interior = shapes.interior_nodes
    want = partition(nodes.n_total, interior, st.neighbors[interior], None,
                     forcing(nodes.positions[interior]), nodes.positions, P)
    _, got = build_parts_in_process(nodes.positions, nodes.is_boundary, 15, P,
                                    knn=lambda pos, n, q: st.neighbors[q], array_device="cpu")
    for a, b in zip(got, want):
        _assert_same(a, b)
    if P > 1:  # interior-first: no row before the first halo-reading row reads a halo node
        for part in got:
            base = part.n_boundary
            reads = ((part.rows >= base) & (part.rows < base + part.n_halo)).any(axis=1)
            first = np.argmax(reads) if reads.any() else reads.size
            assert not reads[:first].any() and reads[first:].all()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nodes, st, shapes = synth.synthetic_problem(6_000, 15, 2, seed=4, weights="cpu", knn="cpu")
        setup = RankSetup(nodes.positions, nodes.is_boundary, 15, rank, world,
                          knn=lambda pos, n, qq: st.neighbors[qq], array_device="cpu")
        reqs = [None] * world
        dist.all_gather_object(reqs, setup.requests)
        part = setup.finish(reqs)
        interior = shapes.interior_nodes
        want = partition(nodes.n_total, interior, st.neighbors[interior], None,
                         forcing(nodes.positions[interior]), nodes.positions, world)[rank]
        _assert_same(part, want)
        q.put((rank, "ok"))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, f"{type(exc).__name__}: {exc}"))
        raise
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_gloo_world3_rank_setups_exchange_requests():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    results = sorted(q.get(timeout=10) for _ in range(3))
    assert [r[1] for r in results] == ["ok"] * 3, results
    assert all(p.exitcode == 0 for p in procs)
