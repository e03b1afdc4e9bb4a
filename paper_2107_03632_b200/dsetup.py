"""Per-rank device setup of the node-partitioned loop.

`multigpu.partition` builds every part from the full problem on the host;
at BASELINE config 5 (N=1e8, n=56) that is hours of CPU kNN and weights and
~100 GB of host arrays per rank.  Here each rank builds only its own rows
plus halo, with the heavy array work on its GPU:

1. the node set (positions, boundary mask) is the same on every rank
   (rank 0 generates it and broadcasts, bench's job);
2. interior rows in Morton order of their positions (torch stable sort on
   the device: the (code, index) order of ``multigpu.partition``), split
   into `world` row-balanced ranges; `owner` / `slot` of every interior
   node;
3. exact kNN supports of the rank's own rows only (rbf_knn_subset: all N
   nodes are candidates);
4. local numbering ``[boundary refs | halo by (owner, slot) | owned rows]``
   computed in row chunks on the device: entries owned by this rank map
   straight to B + H + slot; only the rest (boundary and halo references,
   a few % of the entries) are uniqued;
5. own rows interior-first (rows that read no halo value before the rest,
   each group in Morton order), so the push-mode step overlaps them with the
   exchange;
6. halo requests (the global ids this rank reads from each peer, in its
   halo order) go to their owners (one all-gather of small dicts), which turn
   them into send lists of their own row positions;
7. the weights are assembled on the device inside the plan
   (rbf_plan_create_assembled), never on the host.

The Part this produces equals ``multigpu.partition``'s part for the same
rank (tests/test_dsetup_gpu.py), so the exchange and the bitwise-parity
argument are those of the partitioned loop.
"""

from __future__ import annotations

import numpy as np

from .multigpu import Part

_CHUNK = 1 << 24  # stencil entries per device chunk of the local-numbering pass


def _spread(v):  # 2-D bit interleave of 21-bit ints (torch int64): bit i -> bit 2i
    v = v & 0x1FFFFF
    v = (v | (v << 16)) & 0x0000FFFF0000FFFF
    v = (v | (v << 8)) & 0x00FF00FF00FF00FF
    v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0F
    v = (v | (v << 2)) & 0x3333333333333333
    v = (v | (v << 1)) & 0x5555555555555555
    return v


def morton_codes_device(xy):
    """multigpu.morton_codes on a (M, 2) float64 CUDA tensor: same IEEE
    quantisation over the bounding box, same 42-bit codes."""
    import torch

    lo = xy.min(dim=0).values
    span = xy.max(dim=0).values - lo
    span = torch.where(span == 0, torch.ones_like(span), span)
    q = ((xy - lo) * (2097151.0 / span)).to(torch.int64)  # truncation, like astype(uint64)
    return _spread(q[:, 0]) | (_spread(q[:, 1]) << 1)


class RankSetup:
    """Phase 1 of a rank's part (own rows, supports, halo, requests); phase 2
    (``finish``) turns every rank's requests into this rank's send lists."""

    def __init__(self, positions: np.ndarray, is_boundary: np.ndarray, n: int, rank: int, world: int,
                 device: int = 0, knn=None, array_device=None):
        """`knn(positions, n, query_ids) -> (len(query), n) int64` defaults to
        the device kNN (rbf_knn_subset on `device`); `array_device` (a torch
        device, default cuda:`device`) holds the index arithmetic.  The CPU
        tests of the multi-rank logic pass a host kNN and "cpu"."""
        import torch

        from .neighborhoods import build_stencils_subset
        from .problem import forcing

        self.rank, self.world, self.n = rank, world, n
        positions = np.ascontiguousarray(positions, dtype=np.float64)
        N = positions.shape[0]
        dev = torch.device(array_device) if array_device is not None else torch.device("cuda", device)
        if knn is None:
            def knn(pos, nn, query):
                return build_stencils_subset(pos, nn, query, device=device)
        interior = np.flatnonzero(~np.asarray(is_boundary)).astype(np.int64)
        n_rows = interior.size
        if n_rows < world:
            from .errors import ParameterError

            raise ParameterError(f"{n_rows} interior rows cannot be split into {world} parts")
        int_t = torch.from_numpy(interior).to(dev)
        codes = morton_codes_device(torch.from_numpy(positions).to(dev)[int_t])
        perm = torch.sort(codes, stable=True).indices  # (code, row index) order
        del codes
        bounds = np.linspace(0, n_rows, world + 1).round().astype(np.int64)
        owner = torch.full((N,), -1, dtype=torch.int32, device=dev)
        slot = torch.full((N,), -1, dtype=torch.int64, device=dev)
        for p in range(world):
            nodes_p = int_t[perm[bounds[p]:bounds[p + 1]]]
            owner[nodes_p] = p
            slot[nodes_p] = torch.arange(nodes_p.numel(), device=dev)
        ks = perm[bounds[rank]:bounds[rank + 1]]
        own_nodes = int_t[ks]
        rows_ref = ks.cpu().numpy()
        own_nodes_h = own_nodes.cpu().numpy()
        del perm, int_t
        # exact supports of the own rows only (global ids, host)
        rows_g = np.ascontiguousarray(knn(positions, n, own_nodes_h), dtype=np.int64)
        # interior-first row order (multigpu.partition): rows that read no
        # halo value first, each group in Morton order
        reads_halo = np.zeros(rows_g.shape[0], dtype=bool)
        for lo in range(0, rows_g.shape[0], max(1, _CHUNK // max(n, 1))):
            r = torch.from_numpy(rows_g[lo:lo + max(1, _CHUNK // max(n, 1))]).to(dev)
            o = owner[r]
            reads_halo[lo:lo + r.shape[0]] = ((o >= 0) & (o != rank)).any(dim=1).cpu().numpy()
        if reads_halo.any():
            order = np.argsort(reads_halo, kind="stable")
            rows_ref, own_nodes_h, rows_g = rows_ref[order], own_nodes_h[order], rows_g[order]
            reads_halo = reads_halo[order]
            own_nodes = torch.from_numpy(own_nodes_h).to(dev)
        self._reads_halo = reads_halo  # finish() moves the rows peers read before these
        self.rows_ref = rows_ref
        # final row position of the own nodes (slot keeps the Morton position
        # of every interior node: it orders the halo groups on every rank)
        fslot = torch.full((N,), -1, dtype=torch.int64, device=dev)
        fslot[own_nodes] = torch.arange(own_nodes.numel(), device=dev)
        # pass 1: the non-owned references (boundary + halo), uniqued
        ext = []
        for lo in range(0, rows_g.size, _CHUNK):
            r = torch.from_numpy(rows_g.reshape(-1)[lo:lo + _CHUNK]).to(dev)
            e = r[owner[r] != rank]
            if e.numel():
                ext.append(torch.unique(e))
        U = torch.unique(torch.cat(ext)) if ext else torch.zeros(0, dtype=torch.int64, device=dev)
        del ext
        own_of = owner[U]
        mb = own_of < 0
        bnd = U[mb]
        hidx = torch.nonzero(~mb).flatten()
        halo_u = U[hidx]
        horder = torch.sort(owner[halo_u].to(torch.int64) * (1 << 40) + slot[halo_u], stable=True).indices
        halo = halo_u[horder]
        B, H = int(bnd.numel()), int(halo.numel())
        lid_u = torch.empty(U.numel(), dtype=torch.int64, device=dev)
        lid_u[mb] = torch.arange(B, device=dev)
        lid_u[hidx[horder]] = B + torch.arange(H, device=dev)
        # pass 2: local ids of every entry (owned: B + H + slot; others: lookup in U)
        local = np.empty_like(rows_g)
        lf = local.reshape(-1)
        for lo in range(0, rows_g.size, _CHUNK):
            r = torch.from_numpy(rows_g.reshape(-1)[lo:lo + _CHUNK]).to(dev)
            mine = owner[r] == rank
            out = B + H + fslot[r]
            if (~mine).any():
                other = r[~mine]
                out[~mine] = lid_u[torch.searchsorted(U, other)]
            lf[lo:lo + r.numel()] = out.cpu().numpy()
        halo_owner = owner[halo].cpu().numpy()
        halo_h = halo.cpu().numpy()
        self.l2g = np.concatenate([bnd.cpu().numpy(), halo_h, own_nodes_h]).astype(np.int64)
        del owner, slot, fslot, U, lid_u
        if dev.type == "cuda":
            torch.cuda.empty_cache()
        self.B, self.H = B, H
        self.n_own = own_nodes_h.size
        self._own_sorted = np.argsort(own_nodes_h, kind="stable")
        self._own_nodes = own_nodes_h
        self.rows = local
        self.positions_local = np.ascontiguousarray(positions[self.l2g])
        self.f_int = np.ascontiguousarray(forcing(positions[own_nodes_h]))
        # halo groups by owner: this rank's receive slices and its requests
        self.recv = {}
        self.requests = {}
        if H:
            starts = np.flatnonzero(np.r_[True, halo_owner[1:] != halo_owner[:-1]])
            ends = np.r_[starts[1:], H]
            for s0, e0 in zip(starts, ends):
                q = int(halo_owner[s0])
                self.recv[q] = (B + int(s0), int(e0 - s0))
                self.requests[q] = halo_h[s0:e0].astype(np.int64)  # global ids, in this rank's halo order

    def _rows_of(self, ids):  # row positions of own global node ids
        own_sorted = self._own_nodes[self._own_sorted]
        return self._own_sorted[np.searchsorted(own_sorted, ids)]

    def finish(self, requests_by_rank) -> Part:
        """requests_by_rank[p] = rank p's ``requests`` dict (all ranks).

        Rows are put in multigpu.partition's three groups: rows no other rank
        reads and that read no halo value, rows only read by other ranks, rows
        that read a halo value (each in Morton order)."""
        base = self.B + self.H
        sent = np.zeros(self.n_own, dtype=bool)
        for p, req in enumerate(requests_by_rank):
            if p != self.rank and self.rank in req:
                sent[self._rows_of(req[self.rank])] = True
        group = np.where(self._reads_halo, 2, np.where(sent, 1, 0))
        perm = np.argsort(group, kind="stable")
        if not np.array_equal(perm, np.arange(self.n_own)):
            inv = np.empty_like(perm)
            inv[perm] = np.arange(perm.size)
            self.rows_ref = self.rows_ref[perm]
            self._own_nodes = self._own_nodes[perm]
            self._own_sorted = np.argsort(self._own_nodes, kind="stable")
            self.f_int = np.ascontiguousarray(self.f_int[perm])
            rows = self.rows[perm]
            flat = rows.reshape(-1)
            for lo in range(0, flat.size, _CHUNK):
                seg = flat[lo:lo + _CHUNK]
                m = seg >= base
                seg[m] = base + inv[seg[m] - base]
            self.rows = rows
            self.l2g = self.l2g.copy()
            self.l2g[base:] = self._own_nodes
            self.positions_local = np.ascontiguousarray(self.positions_local)
            self.positions_local[base:] = self.positions_local[base:][perm]
            self._reads_halo = self._reads_halo[perm]
        rows_of = self._rows_of

        send_to = {p: rows_of(req[self.rank]) for p, req in enumerate(requests_by_rank)
                   if p != self.rank and self.rank in req}
        peers = sorted(set(self.recv) | set(send_to))
        empty = np.zeros(0, dtype=np.int64)
        part = Part(
            rank=self.rank, n_local=int(self.l2g.size), n_boundary=self.B, n_halo=self.H,
            rows_ref=self.rows_ref, local_to_global=self.l2g,
            interior=np.arange(base, base + self.n_own, dtype=np.int64), rows=self.rows, weights=None,
            f_int=self.f_int,
        )
        part.peers = peers
        part.recv_offset = [self.recv[q][0] if q in self.recv else 0 for q in peers]
        part.recv_count = [self.recv[q][1] if q in self.recv else 0 for q in peers]
        part.send_idx = [(base + send_to[q]).astype(np.int64) if q in send_to else empty for q in peers]
        return part


def build_parts_in_process(positions, is_boundary, n, world, device=0, knn=None, array_device=None):
    """All ranks' parts in one process (tests, and single-process groups):
    phase 1 for every rank, then the request exchange, then phase 2."""
    setups = [RankSetup(positions, is_boundary, n, p, world, device, knn=knn, array_device=array_device)
              for p in range(world)]
    reqs = [s.requests for s in setups]
    return setups, [s.finish(reqs) for s in setups]
