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

Stochastic mode: every rank draws the SAME global edge batch (same PCG64
seed), the histogram kernel drops the endpoints it does not own (local epos =
-1) and the row sweep writes only owned rows, gathering the other endpoint's
row from the halo-extended block -- the single-GPU arithmetic row for row.

The exchange/partition logic is device-agnostic (it also runs on CPU tensors
under gloo, which is how it is tested without GPUs); the local term on a GPU
is always ``sped_csr_poly_apply``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib

__all__ = ["partition_rows", "HaloPlan", "ShardedLaplacian", "ShardedOperator",
           "ShardedStochasticOperator", "sharded_mu_eg_step", "sharded_oja_step"]


def partition_rows(indptr: np.ndarray, parts: int) -> np.ndarray:
    """Node offsets (parts+1) splitting rows into contiguous ranges with
    about nnz/parts nonzeros each (each range non-empty when n >= parts)."""
    n = indptr.size - 1
    nnz = int(indptr[-1])
    targets = (np.arange(1, parts) * nnz) // parts
    cuts = np.searchsorted(indptr[1:], targets, side="left") + 1
    off = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    for i in range(1, parts + 1):  # strictly increasing when possible
        off[i] = max(off[i], min(off[i - 1] + 1, n))
    off[-1] = n
    return off


@dataclass
class HaloPlan:
    rank: int
    world: int
    offsets: np.ndarray          # parts+1 node offsets
    n_own: int
    halo_cols: np.ndarray        # global ids of halo rows, grouped by owner
    recv_counts: np.ndarray      # per owner
    send_rows: list              # per peer: local row ids this rank sends
    local_indices: np.ndarray    # local CSR columns remapped into E

    @property
    def n_halo(self) -> int:
        return int(self.halo_cols.size)

    @property
    def send_counts(self) -> np.ndarray:
        return np.array([s.size for s in self.send_rows], dtype=np.int64)


def _local_view(indices_global: np.ndarray, offsets: np.ndarray, rank: int, world: int):
    b, e = int(offsets[rank]), int(offsets[rank + 1])
    cols = indices_global.astype(np.int64)
    remote_mask = (cols < b) | (cols >= e)
    halo = np.unique(cols[remote_mask])                  # sorted => grouped by owner
    owners = np.searchsorted(offsets, halo, side="right") - 1
    recv_counts = np.bincount(owners, minlength=world).astype(np.int64)
    local = np.empty_like(cols)
    local[~remote_mask] = cols[~remote_mask] - b
    local[remote_mask] = (e - b) + np.searchsorted(halo, cols[remote_mask])
    return b, e, halo, recv_counts, local


def build_halo_plans_local(indptr: np.ndarray, indices: np.ndarray,
                           offsets: np.ndarray) -> list:
    """Every rank's HaloPlan computed in one process (no communication):
    the same result build_halo_plan agrees on collectively.  Used by
    single-device tests of the shard kernels and by planning tools."""
    world = offsets.size - 1
    views = []
    for r in range(world):
        p0, p1 = int(indptr[offsets[r]]), int(indptr[offsets[r + 1]])
        views.append(_local_view(indices[p0:p1], offsets, r, world))
    plans = []
    for r in range(world):
        b, e, halo, recv_counts, local = views[r]
        send_rows = []
        for q in range(world):
            if q == r:
                send_rows.append(np.zeros(0, dtype=np.int64))
                continue
            hq = views[q][2]
            oq = np.searchsorted(offsets, hq, side="right") - 1
            send_rows.append(hq[oq == r] - b)
        plans.append(HaloPlan(r, world, offsets, e - b, halo, recv_counts, send_rows, local))
    return plans


def _comm_device(group=None) -> torch.device:
    """Tensors for collectives must live where the backend expects them."""
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def build_halo_plan(indices_global: np.ndarray, offsets: np.ndarray, rank: int, world: int,
                    group=None) -> HaloPlan:
    """Remap a rank's CSR columns into [own | halo] and agree on the send
    lists with every peer (collective over ``group``)."""
    b, e, halo, recv_counts, local = _local_view(indices_global, offsets, rank, world)
    # exchange the request lists: counts first, then the ids (on the device
    # for NCCL groups, on the host for gloo)
    cdev = _comm_device(group)
    counts = torch.from_numpy(recv_counts.copy()).to(cdev)
    all_counts = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(all_counts, counts, group=group)
    send_counts = np.array([int(all_counts[q][rank]) for q in range(world)], dtype=np.int64)
    ops = []
    recv_bufs = {}
    starts = np.concatenate([[0], np.cumsum(recv_counts)])
    for q in range(world):
        if q == rank:
            continue
        if recv_counts[q]:
            req = torch.from_numpy(halo[starts[q]:starts[q + 1]].copy()).to(cdev)
            ops.append(dist.P2POp(dist.isend, req, q, group=group))
        if send_counts[q]:
            buf = torch.empty(int(send_counts[q]), dtype=torch.int64, device=cdev)
            recv_bufs[q] = buf
            ops.append(dist.P2POp(dist.irecv, buf, q, group=group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    send_rows = []
    for q in range(world):
        if q in recv_bufs:
            send_rows.append(recv_bufs[q].cpu().numpy() - b)
        else:
            send_rows.append(np.zeros(0, dtype=np.int64))
    return HaloPlan(rank, world, offsets, e - b, halo, recv_counts, send_rows, local)


class HaloExchanger:
    """Per-term halo fill of E = [own | halo] (grouped send/recv)."""

    def __init__(self, plan: HaloPlan, k: int, device, group=None):
        self.plan, self.k, self.device, self.group = plan, k, torch.device(device), group
        self.send_idx = torch.from_numpy(np.concatenate(plan.send_rows).astype(np.int32)
                                         if plan.send_rows else np.zeros(0, np.int32)).to(self.device)
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

    def __init__(self, indptr: np.ndarray, indices: np.ndarray, values: np.ndarray, device,
                 long_threshold: int, chunk_len: int):
        self.n = int(indptr.size - 1)
        self.nnz = int(indptr[-1])
        self.rowlen = np.diff(indptr)
        self.indptr = torch.from_numpy(indptr.astype(np.int32)).to(device)
        self.indices = torch.from_numpy(np.ascontiguousarray(indices, dtype=np.int32)).to(device)
        self.values = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float32)).to(device)
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

    def term(self, E, x_own, partial_in, raw_out, out, alpha, beta, gamma, w0, lam_f, s_final, k):
        lib = _lib.load()
        nseg, seg = self.segments(k)
        partials = (torch.empty(self.n_chunks * min(k, 128), dtype=torch.float32, device=E.device)
                    if self.n_chunks else None)
        tickets = (torch.zeros(self.n_chunks, dtype=torch.int32, device=E.device)
                   if self.n_chunks else None)
        rc = lib.sped_csr_term_split(
            self.n, k, _lib.ptr(self.indptr), _lib.ptr(self.indices), _lib.ptr(self.values),
            self.long_threshold, self.chunk_len, _lib.ptr(self.chunk_desc), self.n_chunks,
            _lib.ptr(partials), _lib.ptr(tickets), seg, nseg,
            _lib.ptr(x_own), _lib.ptr(E), _lib.ptr(partial_in), int(raw_out), _lib.ptr(out),
            float(alpha), float(beta), float(gamma), float(w0), float(lam_f), float(s_final),
            _lib.stream_ptr(E.device))
        _lib.check(rc, "sped_csr_term_split")


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


def split_local_csr(indptr: np.ndarray, local_indices: np.ndarray, values, n_own: int):
    """Split a shard's CSR (columns in E numbering) into own-column entries
    (col < n_own, diagonal included) and halo-column entries, keeping each
    row's entry order.  ``values`` None = implicit unit-weight combinatorial
    Laplacian (materialised: -1 off the diagonal, row length - 1 on it, the
    values the implicit kernel synthesises).  Returns two (indptr, indices,
    values) triples."""
    rowlen = np.diff(indptr)
    rows = np.repeat(np.arange(n_own, dtype=np.int64), rowlen)
    cols = np.asarray(local_indices, dtype=np.int64)
    if values is None:
        vals = np.full(cols.size, -1.0, dtype=np.float32)
        diag = cols == rows
        vals[diag] = (rowlen[rows[diag]] - 1).astype(np.float32)
    else:
        vals = np.asarray(values, dtype=np.float32)
    out = []
    for mask in (cols < n_own, cols >= n_own):
        ip = np.zeros(n_own + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows[mask], minlength=n_own), out=ip[1:])
        out.append((ip, cols[mask], vals[mask]))
    return out


class ShardedLaplacian:
    """This rank's rows of L on its GPU, plus the halo plan."""

    def __init__(self, full_laplacian, rank: int, world: int, group=None,
                 offsets: np.ndarray | None = None, plan: HaloPlan | None = None):
        lap = full_laplacian
        self.full = lap
        self.device = lap.device
        indptr_h = lap.indptr.cpu().numpy().astype(np.int64)
        self.offsets = partition_rows(indptr_h, world) if offsets is None else offsets
        b, e = int(self.offsets[rank]), int(self.offsets[rank + 1])
        p0, p1 = int(indptr_h[b]), int(indptr_h[e])
        if plan is None:
            cols = lap.indices[p0:p1].cpu().numpy()
            plan = build_halo_plan(cols, self.offsets, rank, world, group)
        self.plan = plan
        self.group = group
        self.rank, self.world = rank, world
        self.n_own = e - b
        self.row0 = b
        self.n_global = lap.n
        self.nnz_local = p1 - p0
        self.nnz_global = lap.nnz
        self.indptr = torch.from_numpy((indptr_h[b:e + 1] - p0).astype(np.int32)).to(self.device)
        self.indices = torch.from_numpy(self.plan.local_indices.astype(np.int32)).to(self.device)
        self.values = None if lap.values is None else lap.values[p0:p1].contiguous()
        self.implicit = lap.values is None
        self.long_threshold, self.chunk_len = lap.long_threshold, lap.chunk_len
        self.rowlen = np.diff(indptr_h[b:e + 1])
        self.sorted_rows = lap.reordered
        self.pos0, self.pos1 = p0, p1
        self._segments = {}
        self._epos = None
        self._erow = None
        self._bws = None
        self._split = None
        self._plan_chunks()

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
            ip = (self.rowlen.cumsum() if self.n_own else np.zeros(0, np.int64))
            indptr = np.concatenate([[0], ip]).astype(np.int64)
            vals = None if self.values is None else self.values.cpu().numpy()
            parts = split_local_csr(indptr, self.plan.local_indices, vals, self.n_own)
            self._split = [SplitCSR(ipp, idx, v, self.device, self.long_threshold,
                                    self.chunk_len) for ipp, idx, v in parts]
        return self._split

    def partial_term(self, E, P, k):
        """Pass 0: P = L_own E[:n_own] (own-column entries, no epilogue)."""
        self.split[0].term(E, None, None, True, P, 0.0, 1.0, 0.0, 1.0, 0.0, 1.0, k)

    def remote_term(self, E, x_own, out, P, alpha, beta, gamma, w0, lam_f, s_final, k):
        """Pass 1: the term epilogue on L_halo E + P (= L E for the own rows)."""
        self.split[1].term(E, x_own, P, False, out, alpha, beta, gamma, w0, lam_f, s_final, k)

    def segments(self, k):
        from .graph import segment_table
        key = min(k, 128)
        if key not in self._segments:
            self._segments[key] = segment_table(self.rowlen, key, self.sorted_rows,
                                                self.long_threshold if self.n_chunks else None)
        return self._segments[key]

    def local_term(self, E, x_own, out, alpha, beta, gamma, w0, lam_f, s_final, k):
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
    @property
    def epos_local(self) -> torch.Tensor:
        """Per edge, the local CSR positions of its two entries (-1 where the
        entry's row belongs to another shard)."""
        if self._epos is None:
            ep = self.full.epos.long()
            own = (ep >= self.pos0) & (ep < self.pos1)
            self._epos = torch.where(own, ep - self.pos0, torch.full_like(ep, -1)).to(torch.int32)
        return self._epos

    @property
    def erow_local(self) -> torch.Tensor:
        """Per edge entry, its local row (-1 where not owned)."""
        if self._erow is None:
            ep = self.epos_local.long()
            rows = torch.searchsorted(self.indptr.long(), ep.clamp_min(0), right=True) - 1
            self._erow = torch.where(ep >= 0, rows, torch.full_like(rows, -1)).to(torch.int32)
        return self._erow

    def local_batch_term(self, E, x_own, out, batch_t, B, alpha, beta, gamma, w0, lam_f,
                         s_final, k):
        """One edge-minibatch term (sped_edge_batch_poly_apply) on the own
        rows, neighbour rows read from E = [own | halo]."""
        lib = _lib.load()
        nbytes = int(lib.sped_edge_batch_workspace_bytes(self.n_own, int(B)))
        if self._bws is None or self._bws.numel() < nbytes:
            self._bws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        rc = lib.sped_edge_batch_poly_apply(
            self.n_own, k, self.full.graph.m, _lib.ptr(self.indices), _lib.ptr(self.full.edge_w),
            _lib.ptr(self.epos_local), _lib.ptr(self.erow_local), _lib.ptr(batch_t), int(B),
            _lib.ptr(self._bws), self._bws.numel(), _lib.ptr(x_own), _lib.ptr(E), None, None,
            _lib.ptr(out), 1,
            _lib.dbl_array([alpha]), _lib.dbl_array([beta]), _lib.dbl_array([gamma]), float(w0),
            float(lam_f), float(s_final), _lib.stream_ptr(self.device))
        _lib.check(rc, "sped_edge_batch_poly_apply (shard)")


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
        for t in range(len(al)):
            final = t == len(al) - 1
            dst = out if final else nxt[: sh.n_own]
            coeffs = (al[t], be[t], ga[t], w0 if t == 0 else 1.0, lf if final else 0.0,
                      s if final else 1.0)
            if P is not None:
                works = ex.start(cur)
                sh.partial_term(cur, P, k)       # overlaps the halo transfer
                ex.finish(works)
                sh.remote_term(cur, x_own, dst, P, *coeffs, k)
            else:
                ex.exchange(cur)
                self._term(t, cur, x_own, dst, *coeffs, k)
            cur, nxt = nxt, cur
        return out

    def _term(self, t, E, x_own, dst, al, be, ga, w0, lf, s, k):
        self.term_fn(E, x_own, dst, al, be, ga, w0, lf, s, k)


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

    @property
    def rng(self) -> np.random.Generator:
        return self.gen.rng

    def draw(self, count: int) -> torch.Tensor:
        from .sampling import host_draw
        m = self.shard.full.graph.m
        if self.index_source == "device":
            return self.gen.integers(m, count)
        return host_draw(self.gen.rng, m, count, self.shard.device)

    def apply_local(self, x_own: torch.Tensor, out: torch.Tensor | None = None,
                    batch: torch.Tensor | None = None) -> torch.Tensor:
        nt = len(self.schedule[0])
        self._batch = batch if batch is not None else (self.draw(nt * self.batch_size)
                                                       if nt > 0 else None)
        return super().apply_local(x_own, out)

    def _term(self, t, E, x_own, dst, al, be, ga, w0, lf, s, k):
        B = self.batch_size
        self.batch_fn(E, x_own, dst, self._batch[t * B:(t + 1) * B], B, al, be, ga, w0, lf, s, k)


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
