"""Row-sharded Laplacian across the GPUs of one node.

Partition: contiguous node ranges balanced by nonzeros.  Rank r owns rows
[b_r, b_{r+1}) of L, of V and of every polynomial intermediate.  Its local
CSR keeps only its rows; columns are remapped to an extended block

    E = [ own rows (n_own) | halo rows (n_halo) ]

where the halo is the sorted set of off-shard columns its rows reference,
grouped by owner rank.  Per polynomial term the owners send exactly those
rows (grouped NCCL send/recv over NVLink, ``batch_isend_irecv``) straight
into the halo region of E, then the fused SpMM term kernel runs on the local
rows reading E (C1).  With halos, the shard's CSR is split into own-column
and halo-column entries: the own-column pass runs while the halo rows are in
flight (NCCL's stream only waits for the pack kernel), the halo-column pass
adds its partial sums and applies the term epilogue
(``sped_csr_term_split``).  The exchange is deduplicated on purpose: direct
NVLink peer loads inside the term kernel would move every remote nonzero's
row (config 4 at 8 GPUs: ~2.2 GB per GPU per term) instead of each distinct
halo row once (~0.56 GB).  Per solver step the 3 k x k Gram blocks are summed with
one all-reduce (C2; Oja's CholQR2 needs a second one) and every rank applies
the same k x k coefficients to its rows.  No other data crosses ranks.

Construction without the whole graph on any rank
(``plan_shard_edges`` + ``ShardedLaplacian.from_shard_edges``): every rank
starts from its own slice of the canonical edge list.  One all-reduce of the
integer degree counts gives every rank the row lengths (and the same
degree-descending relabelling for power-law graphs), the nnz-balanced row
offsets, and each edge's owners; a grouped send/recv routes every edge to
the owners of its two endpoints; each rank builds ITS rows of the CSR on the
device (``sped_laplacian_build_rows``: bit-identical to those rows of the
single-GPU build) and plans its halo with device sorts.  Normalized weighted
graphs all-gather the shards' fp64 degrees once (the d^-1/2 of the halo
columns).  Memory per rank: O(nnz/P + n) (row lengths and degrees are
n-vectors), never O(m).

Stochastic mode: every rank draws the SAME global edge batch (same PCG64
seed) and keeps only the samples with an endpoint it owns, in sample order
(a device searchsorted of the global ids into its sorted local edge ids),
so its records / sort / row sweep are O(B / P); the row sweep writes only
owned rows and reads the other endpoint's row from the halo, with the global
estimator scale m / B -- the single-GPU arithmetic row for row.

The exchange/partition logic is device-agnostic (it also runs on CPU tensors
under gloo, which is how it is tested without GPUs); the local term on a GPU
is always ``sped_csr_poly_apply``.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib

__all__ = ["partition_rows", "HaloPlan", "ShardEdges", "plan_shard_edges", "ShardedLaplacian",
           "ShardedOperator", "ShardedStochasticOperator", "sharded_mu_eg_step",
           "sharded_oja_step", "exchange_bytes_per_term"]


def partition_rows(indptr, parts: int) -> np.ndarray:
    """Node offsets (parts+1) splitting rows into contiguous ranges with
    about nnz/parts nonzeros each (each range non-empty when n >= parts).
    ``indptr``: numpy or torch (a device indptr is searched on the device)."""
    ip = torch.as_tensor(indptr)
    n = int(ip.numel()) - 1
    nnz = int(ip[-1])
    targets = torch.as_tensor((np.arange(1, parts, dtype=np.int64) * nnz) // parts,
                              dtype=ip.dtype, device=ip.device)
    cuts = (torch.searchsorted(ip[1:].contiguous(), targets, side="left") + 1).cpu().numpy()
    off = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    for i in range(1, parts + 1):  # strictly increasing when possible
        off[i] = max(off[i], min(off[i - 1] + 1, n))
    off[-1] = n
    return off


@dataclass
class HaloPlan:
    """Fields are numpy arrays when the plan was built from numpy columns,
    torch tensors (on the columns' device) otherwise; ``recv_counts`` is
    always numpy (host bookkeeping of the exchange)."""
    rank: int
    world: int
    offsets: np.ndarray          # parts+1 node offsets
    n_own: int
    halo_cols: object            # global ids of halo rows, grouped by owner
    recv_counts: np.ndarray      # per owner
    send_rows: list              # per peer: local row ids this rank sends
    local_indices: object        # local CSR columns remapped into E

    @property
    def n_halo(self) -> int:
        return int(self.halo_cols.shape[0])

    @property
    def send_counts(self) -> np.ndarray:
        return np.array([int(s.shape[0]) for s in self.send_rows], dtype=np.int64)


def _local_view(cols: torch.Tensor, offsets: np.ndarray, rank: int, world: int):
    """Halo of a shard and its columns remapped into E = [own | halo]: one
    device sort (unique) + binary searches, no host work over the nonzeros."""
    b, e = int(offsets[rank]), int(offsets[rank + 1])
    cols = cols.to(torch.int64)
    remote = (cols < b) | (cols >= e)
    halo = torch.unique(cols[remote])                    # sorted => grouped by owner
    off_t = torch.as_tensor(offsets, dtype=torch.int64, device=cols.device)
    owners = torch.searchsorted(off_t, halo, right=True) - 1
    recv_counts = torch.bincount(owners, minlength=world).cpu().numpy().astype(np.int64)
    local = torch.where(remote, (e - b) + torch.searchsorted(halo, cols), cols - b)
    return b, e, halo, recv_counts, local


def _as_torch(x):
    return (torch.from_numpy(np.ascontiguousarray(x)), True) if isinstance(x, np.ndarray) \
        else (x, False)


def build_halo_plans_local(indptr, indices, offsets: np.ndarray) -> list:
    """Every rank's HaloPlan computed in one process (no communication):
    the same result build_halo_plan agrees on collectively.  Used by
    single-device tests of the shard kernels and by planning tools."""
    ip, _ = _as_torch(indptr)
    idx, was_np = _as_torch(indices)
    world = offsets.size - 1
    views = []
    for r in range(world):
        p0, p1 = int(ip[int(offsets[r])]), int(ip[int(offsets[r + 1])])
        views.append(_local_view(idx[p0:p1], offsets, r, world))
    conv = (lambda t: t.cpu().numpy()) if was_np else (lambda t: t)
    off_t = torch.as_tensor(offsets, dtype=torch.int64, device=idx.device)
    plans = []
    for r in range(world):
        b, e, halo, recv_counts, local = views[r]
        send_rows = []
        for q in range(world):
            if q == r:
                send_rows.append(conv(torch.zeros(0, dtype=torch.int64, device=idx.device)))
                continue
            hq = views[q][2]
            oq = torch.searchsorted(off_t, hq, right=True) - 1
            send_rows.append(conv(hq[oq == r] - b))
        plans.append(HaloPlan(r, world, offsets, e - b, conv(halo), recv_counts, send_rows,
                              conv(local)))
    return plans


def _comm_device(group=None) -> torch.device:
    """Tensors for collectives must live where the backend expects them."""
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _exchange(sends: list, recv_counts, group, template: torch.Tensor) -> list:
    """Grouped send/recv: ``sends[q]`` goes to rank q; returns the received
    tensors (``recv_counts[q]`` leading rows each, dtype/trailing shape of
    ``template``).  The own slot is passed through."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    cdev = _comm_device(group)
    tail = tuple(template.shape[1:])
    out = [None] * world
    ops = []
    for q in range(world):
        if q == rank:
            out[q] = sends[q]
            continue
        if sends[q] is not None and sends[q].shape[0]:
            ops.append(dist.P2POp(dist.isend, sends[q].to(cdev).contiguous(), q, group=group))
        buf = torch.empty((int(recv_counts[q]),) + tail, dtype=template.dtype, device=cdev)
        out[q] = buf
        if buf.shape[0]:
            ops.append(dist.P2POp(dist.irecv, buf, q, group=group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    return out


def _all_counts(counts: np.ndarray, group) -> np.ndarray:
    """world x world matrix: row r = rank r's per-destination counts."""
    world = dist.get_world_size(group)
    cdev = _comm_device(group)
    t = torch.as_tensor(counts, dtype=torch.int64).to(cdev)
    parts = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    return torch.stack(parts).cpu().numpy()


def build_halo_plan(indices_global, offsets: np.ndarray, rank: int, world: int,
                    group=None) -> HaloPlan:
    """Remap a rank's CSR columns into [own | halo] and agree on the send
    lists with every peer (collective over ``group``).  Device columns stay
    on the device (the plan is built with device sorts/searches)."""
    cols, was_np = _as_torch(indices_global)
    b, e, halo, recv_counts, local = _local_view(cols, offsets, rank, world)
    conv = (lambda t: t.cpu().numpy()) if was_np else (lambda t: t.to(cols.device))
    if world == 1:  # nothing to agree on (no process group needed)
        return HaloPlan(rank, world, offsets, e - b, conv(halo), recv_counts,
                        [conv(torch.zeros(0, dtype=torch.int64))], conv(local))
    send_counts = _all_counts(recv_counts, group)[:, rank]
    starts = np.concatenate([[0], np.cumsum(recv_counts)])
    reqs = [halo[starts[q]:starts[q + 1]] for q in range(world)]
    reqs[rank] = None
    got = _exchange(reqs, send_counts, group, halo.new_empty((0,)))
    send_rows = []
    for q in range(world):
        if q == rank or got[q] is None:
            send_rows.append(conv(torch.zeros(0, dtype=torch.int64)))
        else:
            send_rows.append(conv(got[q] - b))
    return HaloPlan(rank, world, offsets, e - b, conv(halo), recv_counts, send_rows, conv(local))


def exchange_bytes_per_term(indptr, indices, offsets: np.ndarray, k: int,
                            replicate_rows: int = 0) -> dict:
    """Predicted halo bytes per polynomial term for a row partition (SURVEY
    8e): per rank, the distinct off-shard rows its nonzeros reference x 4k
    bytes (deduplicated send/recv).  ``replicate_rows`` > 0 models hub-prefix
    replication: rows [0, H) of a degree-ordered graph are all-gathered
    every term (each rank receives the H - own part of the prefix) and leave
    the point-to-point halos."""
    plans = build_halo_plans_local(indptr, indices, offsets)
    world = offsets.size - 1
    H = int(replicate_rows)
    per = []
    for r, p in enumerate(plans):
        halo = torch.as_tensor(p.halo_cols)
        b, e = int(offsets[r]), int(offsets[r + 1])
        own_prefix = max(0, min(e, H) - min(b, H))
        p2p = int((halo >= H).sum()) if H else int(halo.numel())
        per.append({"rank": r, "own_rows": e - b, "halo_rows": int(halo.numel()),
                     "p2p_rows": p2p, "allgather_rows": (H - own_prefix) if H else 0})
    for d in per:
        d["bytes"] = 4 * k * (d["p2p_rows"] + d["allgather_rows"])
    return {"world": world, "k": k, "replicate_rows": H,
            "max_bytes_per_rank": max(d["bytes"] for d in per),
            "total_bytes": sum(d["bytes"] for d in per), "ranks": per}


class HaloExchanger:
    """Per-term halo fill of E = [own | halo] (grouped send/recv)."""

    def __init__(self, plan: HaloPlan, k: int, device, group=None):
        self.plan, self.k, self.device, self.group = plan, k, torch.device(device), group
        rows = [torch.as_tensor(r).to(torch.int64) for r in plan.send_rows]
        self.send_idx = (torch.cat(rows) if rows else torch.zeros(0, dtype=torch.int64)).to(
            device=self.device, dtype=torch.int32)
        sc = plan.send_counts
        self.send_off = np.concatenate([[0], np.cumsum(sc)])
        self.recv_off = np.concatenate([[0], np.cumsum(plan.recv_counts)])
        self.send_buf = torch.empty((int(sc.sum()), k), dtype=torch.float32, device=self.device)

    def gather(self, E: torch.Tensor):
        if self.send_buf.shape[0] == 0:
            return
        if E.is_cuda:
            lib = _lib.load()
            rc = lib.sped_gather_rows(self.send_buf.shape[0], self.k, _lib.ptr(self.send_idx),
                                      _lib.ptr(E), _lib.ptr(self.send_buf),
                                      _lib.stream_ptr(E.device))
            _lib.check(rc, "sped_gather_rows")
        else:
            torch.index_select(E, 0, self.send_idx.long(), out=self.send_buf)

    def exchange(self, E: torch.Tensor):
        """E[:n_own] holds this rank's rows; fill E[n_own:] from the owners."""
        self.finish(self.start(E))

    @staticmethod
    def finish(works):
        """Wait for a started exchange (stream-ordered for NCCL)."""
        for r in works:
            r.wait()

    def start(self, E: torch.Tensor) -> list:
        """Pack this rank's send rows and post the grouped send/recv; returns
        the works to ``finish``.  E's own rows may be read meanwhile, its halo
        rows only after ``finish``."""
        p = self.plan
        self.gather(E)
        ops = []
        for q in range(p.world):
            if q == p.rank:
                continue
            s0, s1 = self.send_off[q], self.send_off[q + 1]
            if s1 > s0:
                ops.append(dist.P2POp(dist.isend, self.send_buf[s0:s1], q, group=self.group))
            r0, r1 = self.recv_off[q], self.recv_off[q + 1]
            if r1 > r0:
                ops.append(dist.P2POp(dist.irecv, E[p.n_own + r0:p.n_own + r1], q, group=self.group))
        return dist.batch_isend_irecv(ops) if ops else []


class SplitCSR:
    """One half of a shard's CSR (own-column or halo-column entries): device
    arrays, long-row plan and segment table for ``sped_csr_term_split``."""

    def __init__(self, indptr, indices, values, device, long_threshold: int, chunk_len: int):
        indptr = torch.as_tensor(indptr)
        self.n = self.n_rows = int(indptr.numel() - 1)
        self.nnz = int(indptr[-1])
        self.rowlen = torch.diff(indptr).cpu().numpy()
        self.indptr = indptr.to(device=device, dtype=torch.int32)
        self.indices = torch.as_tensor(indices).to(device=device, dtype=torch.int32).contiguous()
        self.values = torch.as_tensor(values).to(device=device, dtype=torch.float32).contiguous()
        self.long_threshold, self.chunk_len = long_threshold, chunk_len
        self.n_chunks, self.chunk_desc = _plan_chunks(
            self.n, self.nnz, self.indptr, long_threshold, chunk_len, device)
        self._segments = {}

    def segments(self, k):
        from .graph import segment_table
        key = min(k, 128)
        if key not in self._segments:
            self._segments[key] = segment_table(self.rowlen, key, False,
                                                self.long_threshold if self.n_chunks else None)
        return self._segments[key]

    def term(self, E, x_own, partial_in, raw_out, out, alpha, beta, gamma, w0, lam_f, s_final, k,
             row_scale=None, scaled_in=False, scaled_out=False, hot=(0, 0)):
        _shard_term_call(self, E, x_own, partial_in, raw_out, out, alpha, beta, gamma, w0, lam_f,
                         s_final, k, row_scale, scaled_in, scaled_out, hot)


def _shard_term_call(csr, E, x_own, partial_in, raw_out, out, alpha, beta, gamma, w0, lam_f,
                     s_final, k, row_scale, scaled_in, scaled_out, hot):
    """sped_csr_term_shard on one (split or whole) shard CSR."""
    lib = _lib.load()
    nseg, seg = csr.segments(k)
    partials = (torch.empty(csr.n_chunks * min(k, 128), dtype=torch.float32, device=E.device)
                if csr.n_chunks else None)
    tickets = (torch.zeros(csr.n_chunks, dtype=torch.int32, device=E.device)
               if csr.n_chunks else None)
    rc = lib.sped_csr_term_shard(
        csr.n_rows, k, _lib.ptr(csr.indptr), _lib.ptr(csr.indices), _lib.ptr(csr.values),
        csr.long_threshold, csr.chunk_len, _lib.ptr(csr.chunk_desc), csr.n_chunks,
        _lib.ptr(partials), _lib.ptr(tickets), seg, nseg, _lib.ptr(row_scale), int(scaled_in),
        int(scaled_out), int(hot[0]), int(hot[1]),
        _lib.ptr(x_own), _lib.ptr(E), _lib.ptr(partial_in), int(raw_out), _lib.ptr(out),
        float(alpha), float(beta), float(gamma), float(w0), float(lam_f), float(s_final),
        _lib.stream_ptr(E.device))
    _lib.check(rc, "sped_csr_term_shard")


def _plan_chunks(n, nnz, indptr_dev, long_threshold, chunk_len, device):
    """Long-row chunk plan (sped_spmm_plan) of a CSR: (n_chunks, desc).  The
    arrival tickets are allocated zeroed per call (thread safety)."""
    import ctypes as C
    lib = _lib.load()
    maxc = int(lib.sped_spmm_plan_max_chunks(n, nnz, long_threshold, chunk_len))
    desc = torch.empty(max(4 * maxc, 4), dtype=torch.int32, device=device)
    nch, nlong = C.c_int64(0), C.c_int64(0)
    rc = lib.sped_spmm_plan(n, _lib.ptr(indptr_dev), long_threshold, chunk_len, _lib.ptr(desc),
                            maxc, C.byref(nch), C.byref(nlong), _lib.stream_ptr(device))
    _lib.check(rc, "sped_spmm_plan")
    n_chunks = int(nch.value)
    chunk_desc = desc[: max(4 * n_chunks, 4)].clone() if n_chunks else None
    return n_chunks, chunk_desc


def split_local_csr(indptr, local_indices, values, n_own: int):
    """Split a shard's CSR (columns in E numbering) into own-column entries
    (col < n_own, diagonal included) and halo-column entries, keeping each
    row's entry order.  ``values`` None = implicit unit-weight combinatorial
    Laplacian (materialised: -1 off the diagonal, row length - 1 on it, the
    values the implicit kernel synthesises).  Device tensors are split on
    their device; numpy in -> numpy out.  Returns two (indptr, indices,
    values) triples."""
    ip, was_np = _as_torch(indptr)
    cols, _ = _as_torch(local_indices)
    ip = ip.to(torch.int64)
    cols = cols.to(device=ip.device, dtype=torch.int64)
    rowlen = torch.diff(ip)
    rows = torch.repeat_interleave(torch.arange(n_own, dtype=torch.int64, device=ip.device), rowlen)
    if values is None:
        vals = torch.full((cols.numel(),), -1.0, dtype=torch.float32, device=ip.device)
        diag = cols == rows
        vals[diag] = (rowlen[rows[diag]] - 1).to(torch.float32)
    else:
        vals = torch.as_tensor(values).to(device=ip.device, dtype=torch.float32)
    out = []
    for mask in (cols < n_own, cols >= n_own):
        p = torch.zeros(n_own + 1, dtype=torch.int64, device=ip.device)
        torch.cumsum(torch.bincount(rows[mask], minlength=n_own), 0, out=p[1:])
        part = (p, cols[mask], vals[mask])
        out.append(tuple(t.cpu().numpy() for t in part) if was_np else part)
    return out


# -- construction from edge slices (no whole graph on any rank) ---------------

@dataclass
class ShardEdges:
    """One rank's share of a row-partitioned graph, before the CSR build:
    the edges incident to its rows (internal labels lo < hi, lexsorted, with
    their ORIGINAL global edge ids and raw weights), the row offsets, and the
    relabelling every rank agreed on (None = original order)."""
    n: int
    m: int                       # global edge count (the sampler's range)
    rank: int
    world: int
    offsets: np.ndarray
    lo: torch.Tensor
    hi: torch.Tensor
    w: torch.Tensor              # fp64
    eid: torch.Tensor            # int64 original edge ids
    rowlen: torch.Tensor         # int64[n] global row lengths (internal order)
    perm: torch.Tensor | None    # internal row -> original node (None: identity)
    unit_weight: bool

    @property
    def row_range(self):
        return int(self.offsets[self.rank]), int(self.offsets[self.rank + 1])


def _degree_order(rowlen: torch.Tensor):
    """perm (internal -> original) by descending row length, stable: the
    order sped_degree_order gives the single-GPU operator."""
    _, perm = torch.sort(rowlen, descending=True, stable=True)
    iperm = torch.empty_like(perm)
    iperm[perm] = torch.arange(perm.numel(), dtype=perm.dtype, device=perm.device)
    return perm, iperm


def plan_shard_edges(n: int, u, v, w, eid, rank: int, world: int, group=None,
                     reorder: str | None = "auto") -> ShardEdges:
    """Route this rank's slice of the canonical edge list (``u < v``, any
    subset; ``eid`` = the edges' global ids) so that every rank ends up with
    the edges incident to its rows.  Collective over ``group``: one
    all-reduce of the n degree counts, one all-gather of the P x P routing
    counts, one grouped send/recv of the edges.  Device-agnostic (gloo on
    CPU tensors, NCCL on device tensors)."""
    from .graph import SKEW_REORDER
    dev = torch.as_tensor(u).device
    u = torch.as_tensor(u, dtype=torch.int64, device=dev)
    v = torch.as_tensor(v, dtype=torch.int64, device=dev)
    w = torch.as_tensor(w, dtype=torch.float64, device=dev)
    eid = torch.as_tensor(eid, dtype=torch.int64, device=dev)
    cdev = _comm_device(group)
    cnt = (torch.bincount(u, minlength=n) + torch.bincount(v, minlength=n)).to(cdev)
    stats = torch.tensor([u.numel(), int((w != 1.0).sum())], dtype=torch.int64, device=cdev)
    dist.all_reduce(cnt, group=group)
    dist.all_reduce(stats, group=group)
    m, nonunit = int(stats[0]), int(stats[1])
    cnt = cnt.to(dev)
    rowlen = cnt + (cnt > 0).to(cnt.dtype)
    perm = None
    mean = float(rowlen.sum()) / n if n else 0.0
    skewed = n > 0 and mean > 0 and float(rowlen.max()) > SKEW_REORDER * mean
    if reorder == "degree" or (reorder == "auto" and skewed and n >= 4096):
        perm, iperm = _degree_order(rowlen)
        rowlen = rowlen[perm]
        a, b = iperm[u], iperm[v]
        u, v = torch.minimum(a, b), torch.maximum(a, b)
    indptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(rowlen, 0, out=indptr[1:])
    offsets = partition_rows(indptr, world)
    off_t = torch.as_tensor(offsets, device=dev)
    o_lo = torch.searchsorted(off_t, u, right=True) - 1
    o_hi = torch.searchsorted(off_t, v, right=True) - 1
    # each edge to the owner of lo, and to the owner of hi when different
    dest = torch.cat([o_lo, o_hi[o_hi != o_lo]])
    sel = torch.cat([torch.arange(u.numel(), device=dev), torch.nonzero(o_hi != o_lo).flatten()])
    order = torch.argsort(dest, stable=True)
    dest, sel = dest[order], sel[order]
    counts = torch.bincount(dest, minlength=world).cpu().numpy().astype(np.int64)
    recv = _all_counts(counts, group)[:, rank]
    starts = np.concatenate([[0], np.cumsum(counts)])
    ints = torch.stack([u[sel], v[sel], eid[sel]], 1)
    wts = w[sel]
    sends_i = [ints[starts[q]:starts[q + 1]] for q in range(world)]
    sends_w = [wts[starts[q]:starts[q + 1]] for q in range(world)]
    got_i = _exchange(sends_i, recv, group, ints.new_empty((0, 3)))
    got_w = _exchange(sends_w, recv, group, wts.new_empty((0,)))
    ints = torch.cat([t.to(dev) for t in got_i])
    wts = torch.cat([t.to(dev) for t in got_w])
    key = ints[:, 0] * n + ints[:, 1]           # unique per edge: the lexsort
    order = torch.argsort(key)
    ints, wts = ints[order], wts[order]
    return ShardEdges(n, m, rank, world, offsets, ints[:, 0].contiguous(), ints[:, 1].contiguous(),
                      wts.contiguous(), ints[:, 2].contiguous(), rowlen, perm, nonunit == 0)


class ShardedLaplacian:
    """This rank's rows of L on its GPU, plus the halo plan.

    ``ShardedLaplacian(full_laplacian, rank, world)`` slices an operator
    that exists whole (tests, one-GPU multi-shard runs);
    ``ShardedLaplacian.from_shard_edges(plan_shard_edges(...), mode)`` builds
    the shard from routed edges without the whole graph (multi-GPU runs)."""

    def __init__(self, full_laplacian, rank: int, world: int, group=None,
                 offsets: np.ndarray | None = None, plan: HaloPlan | None = None):
        lap = full_laplacian
        self.device = lap.device
        indptr_d = lap.indptr.to(torch.int64)
        offsets = partition_rows(indptr_d, world) if offsets is None else offsets
        b, e = int(offsets[rank]), int(offsets[rank + 1])
        p0, p1 = int(indptr_d[b]), int(indptr_d[e])
        cols = lap.indices[p0:p1]
        # the shard's edges: those with an entry in its rows (the global
        # epos table is indexed by original edge id)
        ep = lap.epos[: 2 * lap.graph.m].view(-1, 2).long() if lap.graph.m else \
            torch.zeros((0, 2), dtype=torch.int64, device=self.device)
        own = (ep >= p0) & (ep < p1)
        eids = torch.nonzero(own.any(1)).flatten()
        epos_l = torch.where(own[eids], ep[eids] - p0, torch.full_like(ep[eids], -1))
        ew = None if lap.edge_w is None else lap.edge_w[eids]
        self._setup(offsets, rank, world, group, plan, lap.n, lap.nnz, lap.graph.m,
                    (indptr_d[b:e + 1] - p0).to(torch.int32), cols,
                    None if lap.values is None else lap.values[p0:p1].contiguous(),
                    lap.long_threshold, lap.chunk_len, lap.reordered, eids, epos_l, ew)
        if lap.row_scale is not None and os.environ.get("SPED_SHARD_SCALED", "1") != "0":
            self.row_scale = lap.row_scale[b:e].contiguous()

    @classmethod
    def from_shard_edges(cls, se: ShardEdges, mode: str = "unnormalized", device=None,
                         group=None, long_threshold: int | None = None,
                         chunk_len: int | None = None, implicit: bool | None = None,
                         col_degrees: torch.Tensor | None = None, plan: HaloPlan | None = None):
        """Build this rank's rows on the device from routed edges
        (``sped_laplacian_build_rows``; bit-identical to the same rows of
        the single-GPU operator in the same internal order).  Collective over
        ``group`` (the degree all-gather of normalized mode, the halo plan)
        unless ``col_degrees`` / ``plan`` are given (one-process multi-shard
        runs)."""
        import ctypes as C
        from .graph import long_row_plan
        if mode not in ("unnormalized", "normalized"):
            raise ValueError(f"unknown Laplacian mode: {mode!r}")
        dev = _lib.require_cuda(device)
        lib = _lib.load()
        self = cls.__new__(cls)
        self.device = dev
        b, e = se.row_range
        nr = e - b
        lo, hi, w = se.lo.to(dev), se.hi.to(dev), se.w.to(dev)
        ml = int(lo.numel())
        if implicit is None:
            implicit = mode == "unnormalized" and se.unit_weight
        normalized = mode == "normalized"
        cap = 2 * ml + nr
        indptr = torch.empty(nr + 1, dtype=torch.int32, device=dev)
        indices = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        vals = None if implicit else torch.empty(max(cap, 1), dtype=torch.float32, device=dev)
        deg = torch.empty(max(nr, 1), dtype=torch.float64, device=dev)
        epos = torch.empty(max(2 * ml, 1), dtype=torch.int32, device=dev)
        nnz = C.c_int64(0)
        col_deg = None
        stream = _lib.stream_ptr(dev)
        if normalized:
            # own fp64 degrees first (bincount order), then every node's
            # degree for the halo columns' d^-1/2
            with torch.cuda.device(dev):
                rc = lib.sped_laplacian_build_rows(se.n, b, e, ml, _lib.ptr(lo), _lib.ptr(hi),
                                                   _lib.ptr(w), None, 0, 0, _lib.ptr(indptr),
                                                   _lib.ptr(indices), None, _lib.ptr(deg),
                                                   _lib.ptr(epos), C.byref(nnz), stream)
            _lib.check(rc, "sped_laplacian_build_rows")
            col_deg = (_all_gather_rows(deg[:nr], se.offsets, group) if col_degrees is None
                       else col_degrees).to(device=dev, dtype=torch.float64).contiguous()
            if bool((col_deg == 0).any()):
                raise ValueError("normalized Laplacian requires all degrees > 0")
        with torch.cuda.device(dev):
            rc = lib.sped_laplacian_build_rows(se.n, b, e, ml, _lib.ptr(lo), _lib.ptr(hi),
                                               _lib.ptr(w), _lib.ptr(col_deg),
                                               1 if normalized else 0, 0 if implicit else 1,
                                               _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(vals),
                                               _lib.ptr(deg), _lib.ptr(epos), C.byref(nnz), stream)
        _lib.check(rc, "sped_laplacian_build_rows")
        nnz_l = int(nnz.value)
        nnz_g = int(se.rowlen.sum())
        thr, cl = long_row_plan(nnz_g)
        epos_l = epos[: 2 * ml].view(-1, 2).long()
        self._setup(se.offsets, se.rank, se.world, group, plan, se.n, nnz_g, se.m, indptr,
                    indices[:nnz_l], None if vals is None else vals[:nnz_l],
                    int(long_threshold if long_threshold is not None else thr),
                    int(chunk_len if chunk_len is not None else cl), se.perm is not None,
                    se.eid.to(dev), epos_l,
                    None if se.unit_weight else w.to(torch.float32))
        self.perm = None if se.perm is None else se.perm.to(dev)
        self.degrees_own = deg[:nr]
        if (normalized and se.unit_weight and vals is not None
                and os.environ.get("SPED_SHARD_SCALED", "1") != "0"):
            # the single-GPU row_scale: fp32(rsqrt(fp64 degree))
            self.row_scale = torch.rsqrt(deg[:nr].double()).float().contiguous()
        return self

    def lambda_upper(self, mode: str) -> float:
        """The reference's degree bound (graph.py:351-362, transforms.py:
        280-288) over all shards: 2.0 normalized, else 2 max_i d_i (one MAX
        all-reduce of the shards' own fp64 degrees)."""
        if mode == "normalized":
            return 2.0
        if self.m_global == 0:
            return 0.0
        d = getattr(self, "degrees_own", None)
        loc = float(d.max()) if d is not None and d.numel() and self.n_own else 0.0
        if self.world > 1:
            t = torch.tensor([loc], dtype=torch.float64, device=_comm_device(self.group))
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
            loc = float(t.item())
        return 2.0 * loc

    def _setup(self, offsets, rank, world, group, plan, n_global, nnz_global, m_global, indptr,
               cols_global, values, long_threshold, chunk_len, sorted_rows, eids, epos_l, edge_w):
        self.offsets = offsets
        b, e = int(offsets[rank]), int(offsets[rank + 1])
        if plan is None:
            plan = build_halo_plan(cols_global, offsets, rank, world, group)
        self.plan = plan
        self.group = group
        self.rank, self.world = rank, world
        self.n_own = e - b
        self.row0 = b
        self.n_global = n_global
        self.nnz_global = nnz_global
        self.m_global = m_global
        self.indptr = indptr.to(self.device)
        self.nnz_local = int(self.indptr[-1]) if self.n_own else 0
        self.indices = torch.as_tensor(plan.local_indices).to(device=self.device,
                                                             dtype=torch.int32)
        self.values = values
        self.implicit = values is None
        self.long_threshold, self.chunk_len = long_threshold, chunk_len
        self.rowlen = torch.diff(self.indptr.long()).cpu().numpy()
        self.sorted_rows = sorted_rows
        self._segments = {}
        self._bws = None
        self._split = None
        # the shard's edges (local index j): original global id, the local
        # CSR positions of its two entries (-1: row not owned), their local
        # rows, raw weight (None: unit)
        self.edge_ids = eids
        self.epos_l = epos_l.to(torch.int32).contiguous().view(-1)
        rows = torch.searchsorted(self.indptr.long(), epos_l.clamp_min(0), right=True) - 1
        self.erow_l = torch.where(epos_l >= 0, rows, torch.full_like(rows, -1)).to(
            torch.int32).contiguous().view(-1)
        self.edge_w_l = edge_w
        self._eid_sorted, self._eid_order = torch.sort(eids)
        self.row_scale = None       # d^-1/2 of the own rows: scaled-normalized terms
        self._plan_chunks()

    @property
    def n_rows(self) -> int:
        return self.n_own

    def scaled_terms(self, k: int) -> bool:
        """Terms after the first run on u = D^-1/2 w without values (the
        single-GPU VM 2 form; unit-weight normalized Laplacians)."""
        return self.row_scale is not None and k in (4, 8, 16, 32, 64, 128)

    def hot_range(self, k: int):
        """Rows of E = [own | halo] holding the hub prefix of a
        degree-ordered graph (the single-GPU operator's persisting window):
        the own prefix on the shard that owns the hubs, the head of the halo
        on the others."""
        from .graph import HOT_FRACTION, L2_BYTES
        if not self.sorted_rows:
            return (0, 0)
        cache = self.__dict__.setdefault("_hot", {})
        if k not in cache:  # once per k: the search syncs the host
            H = int(min(self.n_global, HOT_FRACTION * L2_BYTES / (4 * max(k, 1))))
            if self.row0 < H:
                cache[k] = (0, min(H, self.row0 + self.n_own) - self.row0)
            else:
                halo = torch.as_tensor(self.plan.halo_cols)
                cache[k] = (self.n_own,
                            int(torch.searchsorted(halo, torch.tensor(H, device=halo.device))))
        return cache[k]

    def _plan_chunks(self):
        self.n_chunks, self.chunk_desc = _plan_chunks(
            self.n_own, self.nnz_local, self.indptr, self.long_threshold, self.chunk_len,
            self.device)

    # -- split CSR: own-column pass overlapping the halo exchange --------------
    @property
    def split_terms(self) -> bool:
        """Terms run as own-column pass + halo-column pass (halos exist)."""
        return self.plan.n_halo > 0

    @property
    def split(self):
        if self._split is None:
            parts = split_local_csr(self.indptr, self.indices, self.values, self.n_own)
            self._split = [SplitCSR(ipp, idx, v, self.device, self.long_threshold,
                                    self.chunk_len) for ipp, idx, v in parts]
        return self._split

    def partial_term(self, E, P, k, scaled_in=False, scaled_out=False):
        """Pass 0: P = L_own E[:n_own] (own-column entries, no epilogue)."""
        self.split[0].term(E, None, None, True, P, 0.0, 1.0, 0.0, 1.0, 0.0, 1.0, k,
                           self.row_scale, scaled_in, False, self.hot_range(k))

    def remote_term(self, E, x_own, out, P, alpha, beta, gamma, w0, lam_f, s_final, k,
                    scaled_in=False, scaled_out=False):
        """Pass 1: the term epilogue on L_halo E + P (= L E for the own rows)."""
        self.split[1].term(E, x_own, P, False, out, alpha, beta, gamma, w0, lam_f, s_final, k,
                           self.row_scale, scaled_in, scaled_out, self.hot_range(k))

    def segments(self, k):
        from .graph import segment_table
        key = min(k, 128)
        if key not in self._segments:
            self._segments[key] = segment_table(self.rowlen, key, self.sorted_rows,
                                                self.long_threshold if self.n_chunks else None)
        return self._segments[key]

    def local_term(self, E, x_own, out, alpha, beta, gamma, w0, lam_f, s_final, k,
                   scaled_in=False, scaled_out=False):
        if scaled_in or scaled_out or self.row_scale is not None:
            _shard_term_call(self, E, x_own, None, False, out, alpha, beta, gamma, w0, lam_f,
                             s_final, k, self.row_scale, scaled_in, scaled_out, self.hot_range(k))
            return
        lib = _lib.load()
        nseg, seg = self.segments(k)
        partials = (torch.empty(self.n_chunks * min(k, 128), dtype=torch.float32, device=self.device)
                    if self.n_chunks else None)
        tickets = (torch.zeros(self.n_chunks, dtype=torch.int32, device=self.device)
                   if self.n_chunks else None)
        rc = lib.sped_csr_poly_apply(
            self.n_own, k, _lib.ptr(self.indptr), _lib.ptr(self.indices), _lib.ptr(self.values),
            self.long_threshold, self.chunk_len, _lib.ptr(self.chunk_desc), self.n_chunks,
            _lib.ptr(partials), _lib.ptr(tickets), seg, nseg,
            self.n_own + self.plan.n_halo, None, _lib.ptr(x_own), _lib.ptr(E),
            None, None, _lib.ptr(out), 1, _lib.dbl_array([alpha]), _lib.dbl_array([beta]),
            _lib.dbl_array([gamma]), float(w0), float(lam_f), float(s_final),
            _lib.stream_ptr(self.device))
        _lib.check(rc, "sped_csr_poly_apply (shard)")

    # -- stochastic (edge-minibatch) term on the shard -------------------------
    def compact_batch(self, batch: torch.Tensor, terms: int = 1):
        """Global sampled edge ids (``terms`` equal slices, sample order) ->
        per term, the local indices of the samples with an endpoint in this
        shard, in sample order.  One host sync for the counts."""
        b = batch.to(torch.int64).view(terms, -1)
        ne = self._eid_sorted.numel()
        if ne == 0:
            return [torch.zeros(0, dtype=torch.int32, device=self.device) for _ in range(terms)]
        pos = torch.searchsorted(self._eid_sorted, b).clamp_max(ne - 1)
        hit = self._eid_sorted[pos] == b
        counts = hit.sum(1).cpu().tolist()
        loc = self._eid_order[pos[hit]].to(torch.int32)
        return list(torch.split(loc, counts))

    def local_batch_term(self, E, x_own, out, batch_t, B, alpha, beta, gamma, w0, lam_f,
                         s_final, k, local_batch: torch.Tensor | None = None):
        """One edge-minibatch term (sped_edge_batch_poly_apply_scaled) on the
        own rows over the term's global batch ``batch_t`` (B samples; or its
        precomputed compaction ``local_batch``), neighbour rows read from
        E = [own | halo], estimator scale m / B of the global batch."""
        lib = _lib.load()
        if local_batch is None:
            local_batch = self.compact_batch(batch_t)[0]
        bl = int(local_batch.numel())
        nbytes = int(lib.sped_edge_batch_workspace_bytes(self.n_own, max(bl, 1)))
        if self._bws is None or self._bws.numel() < nbytes:
            self._bws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        rc = lib.sped_edge_batch_poly_apply_scaled(
            self.n_own, k, int(self.edge_ids.numel()), _lib.ptr(self.indices),
            _lib.ptr(self.edge_w_l), _lib.ptr(self.epos_l), _lib.ptr(self.erow_l),
            _lib.ptr(local_batch) if bl else None, bl, float(self.m_global) / float(B),
            _lib.ptr(self._bws), self._bws.numel(), _lib.ptr(x_own), _lib.ptr(E), None, None,
            _lib.ptr(out), 1,
            _lib.dbl_array([alpha]), _lib.dbl_array([beta]), _lib.dbl_array([gamma]), float(w0),
            float(lam_f), float(s_final), _lib.stream_ptr(self.device))
        _lib.check(rc, "sped_edge_batch_poly_apply_scaled (shard)")

    @property
    def epos_local(self) -> torch.Tensor:
        """Per GLOBAL edge entry, its local CSR position (-1: not owned);
        O(m) -- for tests.  The product path uses the compact local arrays."""
        ep = torch.full((2 * self.m_global,), -1, dtype=torch.int32, device=self.device)
        if self.edge_ids.numel():
            ep.view(-1, 2)[self.edge_ids] = self.epos_l.view(-1, 2)
        return ep


def _all_gather_rows(x: torch.Tensor, offsets: np.ndarray, group) -> torch.Tensor:
    """Concatenate every rank's rows (rank order = row order); ranks hold
    offsets[r+1] - offsets[r] rows each (padded to the max for the
    collective)."""
    world = offsets.size - 1
    cdev = _comm_device(group)
    sizes = np.diff(offsets)
    mx = int(sizes.max()) if world else 0
    buf = torch.zeros((mx,) + tuple(x.shape[1:]), dtype=x.dtype, device=cdev)
    buf[: x.shape[0]] = x.to(cdev)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([parts[r][: int(sizes[r])] for r in range(world)])


class ShardedOperator:
    """Reversed polynomial operator over a ShardedLaplacian: same schedule
    as ``TransformedOperator`` with a halo exchange before every term."""

    def __init__(self, shard: ShardedLaplacian, transform, lambda_star: float, term_fn=None):
        from .transforms import term_schedule
        self.shard = shard
        self.transform = transform
        self.lambda_star = lambda_star
        self.schedule = term_schedule(transform, lambda_star)
        self.term_fn = term_fn or shard.local_term
        # own-column pass overlapping the exchange (product term kernels only)
        self.overlap = term_fn is None and bool(getattr(shard, "split_terms", False))
        self.allow_scaled = term_fn is None
        self._ex = {}
        self._bufs = {}
        self._pbuf = {}

    def _buffers(self, k):
        if k not in self._bufs:
            sh = self.shard
            rows = sh.n_own + sh.plan.n_halo
            self._bufs[k] = [torch.empty((rows, k), dtype=torch.float32, device=sh.device)
                             for _ in range(2)]
            self._ex[k] = HaloExchanger(sh.plan, k, sh.device, sh.group)
        return self._bufs[k], self._ex[k]

    def apply_local(self, x_own: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """p(L) applied to the distributed block whose local rows are x_own."""
        sh = self.shard
        k = int(x_own.shape[1])
        (Ea, Eb), ex = self._buffers(k)
        al, be, ga, w0, lf, s = self.schedule
        if out is None:
            out = torch.empty_like(x_own)
        if len(al) == 0:
            out.copy_(x_own * (lf + s * w0))
            return out
        Ea[: sh.n_own].copy_(x_own)
        cur, nxt = Ea, Eb
        P = None
        if self.overlap:
            if k not in self._pbuf:
                self._pbuf[k] = torch.empty((sh.n_own, k), dtype=torch.float32, device=sh.device)
            P = self._pbuf[k]
        scaled = (self.allow_scaled and len(al) >= 2
                  and getattr(sh, "scaled_terms", lambda k: False)(k))
        for t in range(len(al)):
            final = t == len(al) - 1
            dst = out if final else nxt[: sh.n_own]
            coeffs = (al[t], be[t], ga[t], w0 if t == 0 else 1.0, lf if final else 0.0,
                      s if final else 1.0)
            # scaled-normalized form: E carries u = D^-1/2 w after term 0
            sk = {"scaled_in": t > 0, "scaled_out": not final} if scaled else {}
            if P is not None:
                works = ex.start(cur)
                sh.partial_term(cur, P, k, **sk)       # overlaps the halo transfer
                ex.finish(works)
                sh.remote_term(cur, x_own, dst, P, *coeffs, k, **sk)
            else:
                ex.exchange(cur)
                self._term(t, cur, x_own, dst, *coeffs, k, **sk)
            cur, nxt = nxt, cur
        return out

    def _term(self, t, E, x_own, dst, al, be, ga, w0, lf, s, k, **kw):
        self.term_fn(E, x_own, dst, al, be, ga, w0, lf, s, k, **kw)


class ShardedStochasticOperator(ShardedOperator):
    """make_stochastic_oracle (solvers.py:150-180, per-term batches) over a
    ShardedLaplacian.  Every rank holds the same PCG64 stream (same seed), so
    the ranks draw identical global batches without communicating."""

    def __init__(self, shard: ShardedLaplacian, transform, lambda_star: float,
                 batch_size: int, seed: int, index_source: str = "device", term_fn=None):
        super().__init__(shard, transform, lambda_star)
        if index_source not in ("device", "host"):
            raise ValueError("index_source must be 'device' or 'host'")
        self.batch_size = int(batch_size)
        from .sampling import DeviceGenerator
        self.gen = DeviceGenerator(np.random.default_rng(seed), shard.device)
        self.index_source = index_source
        self.batch_fn = term_fn or shard.local_batch_term
        self._batch = None
        self.overlap = False  # edge-minibatch terms: one pass after the exchange
        self.allow_scaled = False  # the minibatch estimate reads unscaled w

    @property
    def rng(self) -> np.random.Generator:
        return self.gen.rng

    def draw(self, count: int) -> torch.Tensor:
        from .sampling import host_draw
        m = self.shard.m_global
        if self.index_source == "device":
            return self.gen.integers(m, count)
        return host_draw(self.gen.rng, m, count, self.shard.device)

    def apply_local(self, x_own: torch.Tensor, out: torch.Tensor | None = None,
                    batch: torch.Tensor | None = None) -> torch.Tensor:
        nt = len(self.schedule[0])
        self._batch = batch if batch is not None else (self.draw(nt * self.batch_size)
                                                       if nt > 0 else None)
        # this shard's samples of every term, compacted once per apply
        self._local = (self.shard.compact_batch(self._batch, nt)
                       if nt > 0 and hasattr(self.shard, "compact_batch") else None)
        return super().apply_local(x_own, out)

    def _term(self, t, E, x_own, dst, al, be, ga, w0, lf, s, k, **kw):
        B = self.batch_size
        bt = self._batch[t * B:(t + 1) * B]
        if self._local is not None:
            self.batch_fn(E, x_own, dst, bt, B, al, be, ga, w0, lf, s, k,
                          local_batch=self._local[t])
        else:
            self.batch_fn(E, x_own, dst, bt, B, al, be, ga, w0, lf, s, k)


class _Reducing:
    """Within the block every Gram the workspace forms is all-reduced."""

    def __init__(self, ws, group):
        self.ws, self.group = ws, group

    def __enter__(self):
        self.ws.reduce = lambda G: dist.all_reduce(G, op=dist.ReduceOp.SUM, group=self.group)

    def __exit__(self, *exc):
        self.ws.reduce = None


def sharded_mu_eg_step(op: ShardedOperator, V_own: torch.Tensor, eta: float, ws,
                       out: torch.Tensor, MV: torch.Tensor | None = None, group=None):
    """mu_eg_step (solvers.py:121-144) on row shards: local Gram, one
    all-reduce of the 3 k x k blocks, identical k x k algebra on every rank,
    local update."""
    MV = op.apply_local(V_own, out=MV)
    with _Reducing(ws, group):
        ws.mu_eg(V_own, MV, eta, out)
    return out


def sharded_oja_step(op: ShardedOperator, V_own: torch.Tensor, eta: float, ws,
                     out: torch.Tensor, MV: torch.Tensor | None = None, group=None):
    """oja_step (solvers.py:114-118, MGS as CholQR2) on row shards: the Gram
    of W = V + eta*MV and the Gram of the first CholQR pass are each one
    all-reduce; the triangular solves are identical on every rank."""
    MV = op.apply_local(V_own, out=MV)
    with _Reducing(ws, group):
        ws.oja(V_own, MV, eta, out)
    return out
