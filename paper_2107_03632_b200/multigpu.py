"""Node-partitioned multi-GPU time loop -- host side.

The reference has no multi-device code (the paper lists it
as future work); BASELINE.json's north star adds it: partition
the nodes across the GPUs of one box and exchange partition-boundary halos of
u every step.

Partitioning (``partition``):

* interior rows are put in Morton order of their node positions and split
  into P contiguous, row-balanced ranges (bytes balance too: n is constant);
* part p owns its rows' weights / ids / forcing and the u values of its
  interior nodes;
* its halo = the interior nodes owned by other parts that its rows read;
  non-interior (Dirichlet) nodes its rows read are replicated -- they never
  change;
* local numbering: ``[boundary refs | halo (grouped by owner) | owned rows]``,
  so owned row r updates local node ``B_p + H_p + r`` (the plan's canonical
  layout: no renumbering on the device) and the halo of each peer is one
  contiguous slice of u -- received in place;
* owned rows interior-first: rows that read no halo value come before the
  rest (each group in Morton order), so the push-mode step computes them
  while the neighbours' halos are still arriving;
* the per-row j-order is untouched, so a partitioned run is bitwise identical
  to one GPU and to the CPU oracle.

Per step each part packs the owned values its peers read, exchanges them
(NCCL send/recv over NVLink between processes, or device copies between the
parts of one process), runs the step kernel, and all-reduces (max) the
residual bits and the non-finite flag (exact: max of non-negative doubles).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from .errors import InstabilityError, ParameterError, SteadyStateTimeout


def morton_codes(xy: np.ndarray) -> np.ndarray:
    """42-bit Morton codes of 2-D points (21 bits per axis over the bounding box)."""
    xy = np.asarray(xy, dtype=np.float64)
    lo = xy.min(axis=0)
    span = xy.max(axis=0) - lo
    span[span == 0] = 1.0
    q = ((xy - lo) * (2097151.0 / span)).astype(np.uint64)

    def spread(v):  # 2-D bit interleave: bit i -> bit 2i
        v = v & np.uint64(0x1FFFFF)
        v = (v | (v << np.uint64(16))) & np.uint64(0x0000FFFF0000FFFF)
        v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF00FF00FF)
        v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F0F0F0F0F)
        v = (v | (v << np.uint64(2))) & np.uint64(0x3333333333333333)
        v = (v | (v << np.uint64(1))) & np.uint64(0x5555555555555555)
        return v

    return spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1))


@dataclass
class Part:
    """One partition's local problem and its exchange lists (all local ids)."""

    rank: int
    n_local: int
    n_boundary: int  # B_p: replicated non-interior nodes
    n_halo: int  # H_p
    rows_ref: np.ndarray  # reference row ids k owned, in local row order
    local_to_global: np.ndarray  # [n_local] global node id of each local node
    interior: np.ndarray  # [n_own] local ids (= B_p + H_p + r)
    rows: np.ndarray  # [n_own, n] local ids
    weights: Optional[np.ndarray]  # [n_own, n] (None: filled in later by the caller)
    f_int: np.ndarray  # [n_own]
    peers: List[int] = field(default_factory=list)  # sorted peer ranks
    send_idx: List[np.ndarray] = field(default_factory=list)  # per peer: local ids to send
    recv_offset: List[int] = field(default_factory=list)  # per peer: start of its halo slice
    recv_count: List[int] = field(default_factory=list)

    @property
    def n_own(self) -> int:
        return int(self.interior.size)

    def local_field(self, u_global: np.ndarray) -> np.ndarray:
        return np.ascontiguousarray(np.asarray(u_global, dtype=np.float64)[self.local_to_global])

    def halo_bytes_per_step(self) -> int:
        return 8 * int(sum(self.recv_count))


def partition(n_total: int, interior: np.ndarray, rows: np.ndarray, weights: np.ndarray,
              f_int: np.ndarray, positions: Optional[np.ndarray], n_parts: int,
              order: str = "morton") -> List[Part]:
    """Split the problem into `n_parts` row-balanced parts with halo lists.

    `rows` is the reference's ``neighbors[interior]`` (solver.py:182).
    `weights` may be None when each rank assembles only its own rows' weights.
    """
    interior = np.ascontiguousarray(interior, dtype=np.int64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    n_rows = interior.size
    if n_parts < 1:
        raise ParameterError("need at least one part")
    if n_rows < n_parts:
        raise ParameterError(f"{n_rows} interior rows cannot be split into {n_parts} parts")
    if order == "morton":
        if positions is None:
            raise ParameterError("Morton partitioning needs node positions")
        codes = morton_codes(np.asarray(positions)[interior])
        perm = np.lexsort((np.arange(n_rows), codes))
    elif order == "native":
        perm = np.arange(n_rows)
    else:
        raise ParameterError(f"unknown order {order!r}")
    bounds = np.linspace(0, n_rows, n_parts + 1).round().astype(np.int64)

    owner = np.full(n_total, -1, dtype=np.int32)  # part owning each interior node
    mslot = np.full(n_total, -1, dtype=np.int64)  # position of a node in its owner's Morton range
    for p in range(n_parts):
        ks = perm[bounds[p]:bounds[p + 1]]
        owner[interior[ks]] = p
        mslot[interior[ks]] = np.arange(ks.size)
    # each part's rows interior-first, in three groups, each in Morton order:
    # rows that neither read a halo value nor are read by another part, then
    # rows only read by another part (pushed), then rows that read a halo
    # value -- the push-mode step overlaps the first group with the exchange
    # (StepArgs::halo_row0, PartLoop::sync_row0)
    sent = np.zeros(n_total, dtype=bool)  # interior nodes some other part's rows read
    row_owner = owner[interior]
    for lo in range(0, n_rows, 1 << 20):
        r = rows[lo:lo + (1 << 20)]
        of = owner[r]
        cross = (of >= 0) & (of != row_owner[lo:lo + (1 << 20), None])
        sent[r[cross]] = True
    own_ks = []
    slot = np.full(n_total, -1, dtype=np.int64)  # final row position of a node in its owner
    for p in range(n_parts):
        ks = perm[bounds[p]:bounds[p + 1]]
        of = owner[rows[ks]]
        reads_halo = ((of >= 0) & (of != p)).any(axis=1)
        group = np.where(reads_halo, 2, np.where(sent[interior[ks]], 1, 0))
        ks = ks[np.argsort(group, kind="stable")]
        own_ks.append(ks)
        slot[interior[ks]] = np.arange(ks.size)

    parts: List[Part] = []
    halo_from: List[dict] = []
    for p in range(n_parts):
        ks = own_ks[p]
        own_nodes = interior[ks]
        refs = rows[ks]
        uniq = np.unique(refs)
        own_of = owner[uniq]
        bnd = uniq[own_of < 0]
        halo = uniq[(own_of >= 0) & (own_of != p)]
        # group the halo by owner, each group in the owner's Morton order
        hk = np.lexsort((mslot[halo], owner[halo]))
        halo = halo[hk]
        l2g = np.concatenate([bnd, halo, own_nodes]).astype(np.int64)
        g2l = np.full(n_total, -1, dtype=np.int64)
        g2l[l2g] = np.arange(l2g.size)
        local_rows = g2l[refs]
        if (local_rows < 0).any():  # pragma: no cover - construction guarantees coverage
            raise AssertionError("unmapped stencil entry")
        B, H = bnd.size, halo.size
        part = Part(
            rank=p, n_local=int(l2g.size), n_boundary=int(B), n_halo=int(H), rows_ref=ks,
            local_to_global=l2g, interior=np.arange(B + H, B + H + ks.size, dtype=np.int64),
            rows=np.ascontiguousarray(local_rows),
            weights=None if weights is None else np.ascontiguousarray(weights[ks]),
            f_int=np.ascontiguousarray(np.asarray(f_int)[ks]),
        )
        groups = {}
        if H:
            owners_h = owner[halo]
            starts = np.flatnonzero(np.r_[True, owners_h[1:] != owners_h[:-1]])
            ends = np.r_[starts[1:], H]
            for s, e in zip(starts, ends):
                groups[int(owners_h[s])] = (B + int(s), halo[s:e])
        parts.append(part)
        halo_from.append(groups)

    # exchange lists.  kNN stencils are not symmetric, so the peer graph need
    # not be either: a peer may only send, or only receive.
    empty = np.zeros(0, dtype=np.int64)
    for q, part in enumerate(parts):
        base = part.n_boundary + part.n_halo
        recv = halo_from[q]
        send_to = {p: halo_from[p][q][1] for p in range(n_parts) if q in halo_from[p]}
        part.peers = sorted(set(recv) | set(send_to))
        part.recv_offset = [int(recv[pp][0]) if pp in recv else 0 for pp in part.peers]
        part.recv_count = [int(recv[pp][1].size) if pp in recv else 0 for pp in part.peers]
        part.send_idx = [(base + slot[send_to[pp]]).astype(np.int64) if pp in send_to else empty
                         for pp in part.peers]
    return parts


def assemble_field(parts: Sequence[Part], local_fields: Sequence[np.ndarray], u_template: np.ndarray) -> np.ndarray:
    """Global field from each part's owned values (non-interior entries from the template)."""
    out = np.array(u_template, dtype=np.float64, copy=True)
    for part, loc in zip(parts, local_fields):
        own = part.n_boundary + part.n_halo
        out[part.local_to_global[own:]] = loc[own:]
    return out


# ---------------------------------------------------------------------------
# device groups over the C ABI (dist.cu)

class _Group:
    """Partitioned loop on the device: one ``rbf_group`` over local plans."""

    def __init__(self, parts: Sequence[Part], plans, uid: Optional[bytes], rank: int, nranks: int):
        from . import _lib

        self._lib = _lib.load()
        self.parts = list(parts)
        self.plans = list(plans)
        for part, plan in zip(self.parts, self.plans):
            counts_s = np.array([s.size for s in part.send_idx], dtype=np.int64)
            idx = (np.concatenate(part.send_idx) if part.send_idx else np.zeros(0)).astype(np.int64)
            peers = np.array(part.peers, dtype=np.int32)
            roff = np.array(part.recv_offset, dtype=np.int64)
            rcnt = np.array(part.recv_count, dtype=np.int64)
            rc = self._lib.rbf_plan_set_halo(plan._h, peers.size, peers.ctypes.data, counts_s.ctypes.data,
                                             idx.ctypes.data, rcnt.ctypes.data, roff.ctypes.data)
            plan._check(rc)
        arr = (ctypes.c_void_p * len(self.plans))(*[p._h.value for p in self.plans])
        ids = np.array([p.rank for p in self.parts], dtype=np.int32)
        h = ctypes.c_void_p()
        uidbuf = None if uid is None else ctypes.create_string_buffer(uid, 128)
        rc = self._lib.rbf_group_create(ctypes.byref(h), len(self.plans),
                                        ctypes.cast(arr, ctypes.c_void_p), ids.ctypes.data,
                                        uidbuf, rank, nranks)
        self.plans[0]._check(rc)
        self._h = h
        import weakref

        self._fin = weakref.finalize(self, self._lib.rbf_group_destroy, h)

    def close(self):
        self._fin()

    @property
    def push_mode(self) -> bool:
        """True when the fixed-step fast path pushes halos peer-to-peer."""
        return bool(self._lib.rbf_group_push_mode(self._h))

    @property
    def fused(self) -> bool:
        """True when the last fixed-step fast run was one launch of the
        partitioned persistent loop (halo pushes fused into the step)."""
        return bool(self._lib.rbf_group_fused(self._h))

    def _push_local(self):
        self.plans[0]._check(self._lib.rbf_group_push_local(self._h))

    def _push_ipc(self, allgather):
        """Exchange the push-mode blobs through `allgather(bytes) -> [bytes]`
        (every rank's blob, e.g. torch.distributed.all_gather_object) and map
        the neighbours' buffers.  The caller must barrier before running."""
        buf = ctypes.create_string_buffer(1024)
        n = ctypes.c_int64()
        ok = self._lib.rbf_group_push_export(self._h, buf, 1024, ctypes.byref(n)) == 0
        blobs = allgather(buf.raw[: n.value] if ok else b"")
        if ok and all(blobs):
            stride = max(len(b) for b in blobs)
            flat = ctypes.create_string_buffer(b"".join(b.ljust(stride, b"\0") for b in blobs),
                                               stride * len(blobs))
            ok = self._lib.rbf_group_push_import(self._h, len(blobs), flat, stride) == 0
        else:
            ok = False
        # every rank must run the same exchange: push only if all ranks mapped
        verdicts = allgather(b"1" if ok else b"0")
        if not all(v == b"1" for v in verdicts):
            self.plans[0]._check(self._lib.rbf_group_push_off(self._h))

    def run(self, dt, steps=0, mode="fixed", tol=1e-9, max_steps=1_000_000):
        from . import _lib

        sd, res, hr, bad, sec = (ctypes.c_int64(), ctypes.c_double(), ctypes.c_int32(),
                                 ctypes.c_int64(), ctypes.c_double())
        m = _lib.RBF_MODE_STEADY if mode == "steady" else _lib.RBF_MODE_FIXED
        rc = self._lib.rbf_group_run(self._h, float(dt), int(steps), m, float(tol), int(max_steps),
                                     ctypes.byref(sd), ctypes.byref(res), ctypes.byref(hr),
                                     ctypes.byref(bad), ctypes.byref(sec))
        self.plans[0]._check(rc)
        return rc, sd.value, (res.value if hr.value else None), bad.value, sec.value


class LocalGroup(_Group):
    """All parts in this process (one GPU): the single-process form of the
    partitioned loop.  Fixed-step runs push halos straight into the peers'
    buffers after each part's step (push mode, the default); steady runs and
    failure replays use pack / device copy / step / reduce on one stream."""

    def __init__(self, parts: Sequence[Part], devices: Optional[Sequence[int]] = None, push: bool = True,
                 plans=None):
        from .solver import Plan

        devices = list(devices) if devices is not None else [0] * len(parts)
        if plans is None:
            plans = [Plan(pt.n_local, pt.interior, pt.rows, pt.weights, pt.f_int, device=d,
                          resident=False) for pt, d in zip(parts, devices)]
        super().__init__(parts, plans, None, 0, 1)
        if push and len(parts) > 1:
            self._push_local()


class NcclGroup(_Group):
    """One part per process / GPU, launched with torchrun.  With `allgather`
    (bytes -> every rank's bytes) the fixed-step fast path pushes halos over
    NVLink through CUDA IPC mappings of the peers' buffers; steady runs and
    failure replays exchange by NCCL send/recv."""

    def __init__(self, part: Part, rank: int, nranks: int, device: int, uid: bytes, allgather=None,
                 plan=None):
        from .solver import Plan

        if plan is None:
            plan = Plan(part.n_local, part.interior, part.rows, part.weights, part.f_int,
                        device=device, resident=False)
        super().__init__([part], [plan], uid, rank, nranks)
        if allgather is not None and nranks > 1:
            self._push_ipc(allgather)


class HostPacedGroup(_Group):
    """One part per process, halos pushed peer-to-peer through CUDA IPC
    mappings (the NcclGroup fast path), each step followed by a host barrier
    (rbf_group_set_step_barrier): no step kernel waits on a kernel of another
    process.  This is the cross-process push path for ranks that share one
    GPU (NCCL refuses two ranks on one device, and time-sliced contexts do
    not guarantee that waiting kernels are co-scheduled); fixed-step runs
    only.  `allgather(bytes) -> [bytes]` and `barrier()` are the ranks'
    control plane (e.g. torch.distributed with gloo)."""

    def __init__(self, part: Part, rank: int, nranks: int, device: int, allgather, barrier):
        from .solver import Plan

        plan = Plan(part.n_local, part.interior, part.rows, part.weights, part.f_int,
                    device=device, resident=False)
        super().__init__([part], [plan], None, rank, nranks)
        self._allgather = allgather
        self._push_ipc(allgather)
        if not self.push_mode:
            raise RuntimeError("IPC push mode could not be set up on every rank")
        self._barrier_fn = barrier
        self._cb = ctypes.CFUNCTYPE(None, ctypes.c_void_p)(lambda _ctx: self._barrier_fn())
        self.plans[0]._check(self._lib.rbf_group_set_step_barrier(
            self._h, ctypes.cast(self._cb, ctypes.c_void_p), None))

    def run(self, dt, steps=0, mode="fixed", tol=1e-9, max_steps=1_000_000):
        if mode != "fixed" or steps < 2:
            raise ParameterError("host-paced groups run fixed-step runs of >= 2 steps")
        rc, done, residual, bad, sec = super().run(dt, steps=steps)
        # each rank holds its own part's residual / first bad step: reduce
        # (max of non-negative residuals is exact; first bad step = min)
        import struct

        blobs = self._allgather(struct.pack("<qdq", bad, -1.0 if residual is None else residual, rc))
        vals = [struct.unpack("<qdq", b) for b in blobs]
        bads = [v[0] for v in vals if v[0] >= 0]
        res = max(v[1] for v in vals)
        rc = max(v[2] for v in vals)
        return rc, done, (None if res < 0 else res), (min(bads) if bads else -1), sec


def assembled_plan(setup, degree: int, device: int = 0):
    """The plan of a dsetup.RankSetup part with its weights assembled on the
    device (never on the host); streaming loop (groups step every part)."""
    from .solver import Plan

    return Plan.assembled(setup.l2g.size, np.arange(setup.B + setup.H, setup.B + setup.H + setup.n_own,
                                                    dtype=np.int64),
                          setup.rows, setup.positions_local, setup.f_int, degree, device=device,
                          resident=False)


def nccl_unique_id() -> bytes:
    from . import _lib

    lib = _lib.load()
    buf = ctypes.create_string_buffer(128)
    rc = lib.rbf_nccl_unique_id(buf)
    if rc != 0:
        raise RuntimeError(_lib.last_error(lib))
    return buf.raw


def run_partitioned(group: _Group, nodes, shapes, config, u0: Optional[np.ndarray] = None,
                    reduce_max=None):
    """run_time_loop (solver.py:168-236) over a partitioned group; returns
    (field, steps, residual, device_seconds) on every rank's assembled parts.

    On a non-finite step the InstabilityError carries max|u2| of the failing
    step's field (solver.py:200-206), assembled from the parts; with parts in
    other processes ``reduce_max(float) -> float`` (a max over ranks, e.g. a
    torch.distributed all_reduce) completes it."""
    from .solver import _AUTO_DT_SAFETY, apply_dirichlet, stability_bound

    u0 = apply_dirichlet(nodes, np.zeros(nodes.n_total)) if u0 is None else u0
    dt = config.dt if config.dt is not None else _AUTO_DT_SAFETY * stability_bound(shapes)
    for part, plan in zip(group.parts, group.plans):
        plan.set_field(part.local_field(u0))
    rc, steps, residual, bad, sec = group.run(dt, steps=config.steps, mode=config.mode,
                                              tol=config.tol, max_steps=config.max_steps)
    locs = [plan.get_field() for plan in group.plans]
    from . import _lib

    if rc == _lib.RBF_ERR_INSTABILITY:
        # the parts hold the failing step's u2; non-owned entries are Dirichlet
        # values, identical to u2's (solver.py:201: max_abs = max|u2|)
        failed = assemble_field(group.parts, locs, u0)
        max_abs = float(np.max(np.abs(failed)))
        if reduce_max is not None:
            max_abs = float(reduce_max(max_abs))
        raise InstabilityError(f"time loop unstable at step {bad} (max |u| = {max_abs})",
                               step=bad, max_abs=max_abs)
    if rc == _lib.RBF_ERR_TIMEOUT:
        raise SteadyStateTimeout(f"no steady state after {steps} steps (residual {residual})",
                                 steps=steps, residual=residual)
    return assemble_field(group.parts, locs, u0), steps, residual, sec, dt


def bench_main(args, metric, workloads):  # pragma: no cover - needs >1 GPU
    from . import _bench_dist

    return _bench_dist.main(args, metric, workloads)
