"""Row-sharded polynomial apply across 2 ranks (gloo, CPU): partitioning,
halo plans, the grouped send/recv halo exchange and the per-term schedule
must reproduce the single-process oracle.  The local term here is a scipy
SpMM on the CPU (test stand-in for the CUDA term kernel, which the GPU tests
cover); everything else is the product code."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class CpuShard:
    """Stand-in for ShardedLaplacian on the CPU: the product's halo plan and
    exchanger, with a scipy local term."""

    def __init__(self, csr, rank, world, offsets=None):
        from paper_2207_14589_b200.distributed import build_halo_plan, partition_rows
        import scipy.sparse as sps
        self.offsets = partition_rows(csr.indptr.astype(np.int64), world) if offsets is None else offsets
        b, e = int(self.offsets[rank]), int(self.offsets[rank + 1])
        p0, p1 = csr.indptr[b], csr.indptr[e]
        self.plan = build_halo_plan(csr.indices[p0:p1], self.offsets, rank, world)
        self.n_own = e - b
        self.row0 = b
        self.device = torch.device("cpu")
        self.group = None
        ncols = self.n_own + self.plan.n_halo
        self.local = sps.csr_matrix((csr.data[p0:p1], self.plan.local_indices,
                                     csr.indptr[b:e + 1] - p0), shape=(self.n_own, ncols))

    def term(self, E, x_own, out, al, be, ga, w0, lf, s, k):
        Ew = E.double().numpy()
        x = x_own.double().numpy()
        Lw = self.local @ Ew
        wnew = al * x + be * w0 * Lw + ga * w0 * Ew[: self.n_own]
        out.copy_(torch.from_numpy(lf * x + s * wnew))

    local_term = term

    # split-term protocol of ShardedLaplacian (overlapped exchange): the
    # product's split_local_csr, scipy passes standing in for the kernels
    @property
    def split_terms(self):
        return self.plan.n_halo > 0

    def _split(self):
        import scipy.sparse as sps
        from paper_2207_14589_b200.distributed import split_local_csr
        if not hasattr(self, "_parts"):
            ncols = self.n_own + self.plan.n_halo
            self._parts = [sps.csr_matrix((v, c, ip), shape=(self.n_own, ncols))
                           for ip, c, v in split_local_csr(self.local.indptr.astype(np.int64),
                                                           self.local.indices, self.local.data,
                                                           self.n_own)]
        return self._parts

    def partial_term(self, E, P, k):
        own = E[: self.n_own].double().numpy()  # the halo rows are still in flight
        A = self._split()[0]
        P.copy_(torch.from_numpy(A[:, : self.n_own] @ own))
        self.partial_calls = getattr(self, "partial_calls", 0) + 1

    def remote_term(self, E, x_own, out, P, al, be, ga, w0, lf, s, k):
        Ew = E.double().numpy()
        x = x_own.double().numpy()
        Lw = self._split()[1] @ Ew + P.double().numpy()
        wnew = al * x + be * w0 * Lw + ga * w0 * Ew[: self.n_own]
        out.copy_(torch.from_numpy(lf * x + s * wnew))


def _worker(rank, world, port, n, u, v, w, mode, kind, ell, k, result_q, split=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2207_14589_b200 as sp
        from paper_2207_14589_b200.distributed import ShardedOperator
        csr = O.laplacian_csr(n, u, v, w, mode)
        shard = CpuShard(csr, rank, world)
        lam = O.choose_lambda_star(kind, O.lambda_upper(n, u, v, w, mode))
        t = sp.SpectralTransform(kind, ell)
        op = ShardedOperator(shard, t, lam, term_fn=None if split else shard.term)
        assert op.overlap == split
        X = np.random.default_rng(0).standard_normal((n, k)).astype(np.float32)
        b, e = shard.row0, shard.row0 + shard.n_own
        y_own = op.apply_local(torch.from_numpy(X[b:e].copy()))
        # Gram all-reduce (C2): sum of local V^T V equals the global one
        G = torch.from_numpy(X[b:e].astype(np.float64).T @ X[b:e].astype(np.float64))
        dist.all_reduce(G)
        parts = [None] * world
        if split:
            assert shard.partial_calls == len(op.schedule[0])
        dist.all_gather_object(parts, (b, y_own.numpy(), G.numpy(), shard.plan.n_halo))
        if rank == 0:
            result_q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,graph,mode,kind,ell,split", [
    (2, "cfg4s", "normalized", "negexp-taylor", 6, False),
    (3, "cfg4s", "normalized", "negexp-taylor", 6, False),
    (2, "cfg5s", "unnormalized", "negexp-limit", 5, False),
    (3, "cfg3s", "unnormalized", "identity", None, False),
    (2, "cfg4s", "normalized", "negexp-taylor", 6, True),
    (3, "cfg5s", "unnormalized", "negexp-limit", 5, True),
])
def test_sharded_apply_matches_oracle(golden, world, graph, mode, kind, ell, split):
    """split=True: the overlapped schedule (exchange started, own-column
    pass, exchange finished, halo-column pass) of ShardedOperator."""
    n, u, v, w = golden.graph(graph)
    u, v, w = O.canonical_edges(n, u, v, w)
    k = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, u, v, w, mode, kind, ell, k, q,
                                               split))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    csr = O.laplacian_csr(n, u, v, w, mode)
    lam = O.choose_lambda_star(kind, O.lambda_upper(n, u, v, w, mode))
    X = np.random.default_rng(0).standard_normal((n, k)).astype(np.float32).astype(np.float64)
    ref = O.apply_transform(csr, kind, ell, 1e-6, lam, X)
    Y = np.zeros_like(ref)
    for b, y, G, nh in parts:
        Y[b:b + y.shape[0]] = y
        np.testing.assert_allclose(G, X.T @ X, rtol=1e-10)
        assert nh > 0  # a real halo exchange happened
    assert np.linalg.norm(Y - ref) / np.linalg.norm(ref) <= 1e-6


def test_partition_rows_balances_nnz():
    from paper_2207_14589_b200.distributed import partition_rows
    rng = np.random.default_rng(0)
    lens = rng.integers(1, 100, size=1000)
    lens[17] = 5000
    indptr = np.concatenate([[0], np.cumsum(lens)])
    for parts in (1, 2, 4, 8):
        off = partition_rows(indptr, parts)
        assert off[0] == 0 and off[-1] == 1000 and np.all(np.diff(off) > 0)
        loads = np.diff(indptr[off])
        assert loads.max() <= indptr[-1] / parts + 5000


def test_split_local_csr_partitions_entries():
    """Own-column + halo-column parts re-assemble the shard CSR; implicit
    unit-weight values are materialised as the kernel synthesises them."""
    from paper_2207_14589_b200.distributed import split_local_csr
    import scipy.sparse as sps
    indptr = np.array([0, 3, 5, 9], dtype=np.int64)
    cols = np.array([0, 2, 4, 1, 3, 0, 2, 5, 6], dtype=np.int64)   # n_own = 3, halo cols 3..6
    vals = np.arange(9, dtype=np.float32) + 1
    (ip0, c0, v0), (ip1, c1, v1) = split_local_csr(indptr, cols, vals, 3)
    A = sps.csr_matrix((vals, cols, indptr), shape=(3, 7)).toarray()
    B = (sps.csr_matrix((v0, c0, ip0), shape=(3, 7)) + sps.csr_matrix((v1, c1, ip1), shape=(3, 7)))
    np.testing.assert_array_equal(B.toarray(), A)
    assert np.all(c0 < 3) and np.all(c1 >= 3)
    (_, c0, v0), (_, c1, v1) = split_local_csr(indptr, cols, None, 3)
    np.testing.assert_array_equal(v0, [2, -1, 1, -1, 3])  # diag = row length - 1
    np.testing.assert_array_equal(v1, [-1, -1, -1, -1])


def _route_worker(rank, world, port, n, u, v, w, reorder, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2207_14589_b200.distributed import plan_shard_edges
        sl = np.arange(rank, u.size, world)  # a strided slice of the edge list per rank
        se = plan_shard_edges(n, torch.from_numpy(u[sl]), torch.from_numpy(v[sl]),
                              torch.from_numpy(w[sl]), torch.from_numpy(sl), rank, world,
                              reorder=reorder)
        parts = [None] * world
        dist.all_gather_object(parts, (rank, se.offsets, se.lo.numpy(), se.hi.numpy(),
                                       se.w.numpy(), se.eid.numpy(), se.m, se.unit_weight,
                                       None if se.perm is None else se.perm.numpy()))
        if rank == 0:
            result_q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,graph,reorder", [(2, "cfg4s", None), (3, "cfg4s", "degree"),
                                                 (3, "cfg5s", None), (2, "cfg3s", "degree")])
def test_plan_shard_edges_routes_incident_edges(golden, world, graph, reorder):
    """Edge routing without the whole graph on any rank: from strided edge
    slices, every rank ends up with exactly the edges incident to its rows
    (lexsorted in the agreed internal labels, original ids and weights
    kept), the nnz-balanced offsets of the whole graph, and -- with
    reorder -- the degree-descending relabelling of the single-GPU operator."""
    from paper_2207_14589_b200.distributed import partition_rows
    n, u, v, w = golden.graph(graph)
    u, v, w = O.canonical_edges(n, u, v, w)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_route_worker, args=(r, world, port, n, u, v, w, reorder, q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cnt = np.bincount(u, minlength=n) + np.bincount(v, minlength=n)
    rowlen = cnt + (cnt > 0)
    lo, hi = u.copy(), v.copy()
    if reorder == "degree":
        perm = np.argsort(-rowlen, kind="stable")
        iperm = np.empty(n, dtype=np.int64)
        iperm[perm] = np.arange(n)
        a, b = iperm[u], iperm[v]
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        rowlen = rowlen[perm]
    offsets = partition_rows(np.concatenate([[0], np.cumsum(rowlen)]), world)
    eid = np.arange(u.size)
    for r, off, plo, phi, pw, peid, m, unit, pperm in parts:
        np.testing.assert_array_equal(off, offsets)
        assert m == u.size and unit == bool(np.all(w == 1.0))
        if reorder == "degree":
            np.testing.assert_array_equal(pperm, perm)
        else:
            assert pperm is None
        b, e = offsets[r], offsets[r + 1]
        sel = ((lo >= b) & (lo < e)) | ((hi >= b) & (hi < e))
        order = np.lexsort((hi[sel], lo[sel]))
        np.testing.assert_array_equal(plo, lo[sel][order])
        np.testing.assert_array_equal(phi, hi[sel][order])
        np.testing.assert_array_equal(peid, eid[sel][order])
        np.testing.assert_array_equal(pw, w[sel][order])


def test_exchange_bytes_per_term_model():
    """Predicted halo bytes: deduplicated off-shard rows x 4k;
    hub-prefix replication moves the prefix rows out of the point-to-point
    halos into one all-gather."""
    from paper_2207_14589_b200.distributed import exchange_bytes_per_term, partition_rows
    # path 0-1-2-3-4-5 plus a hub 0 joined to everything
    n = 6
    edges = sorted({(i, i + 1) for i in range(5)} | {(0, j) for j in range(2, 6)})
    rows = [[] for _ in range(n)]
    for a, b in edges:
        rows[a].append(b)
        rows[b].append(a)
    indptr = np.zeros(n + 1, dtype=np.int64)
    cols = []
    for i in range(n):
        r = sorted(rows[i] + [i])
        cols += r
        indptr[i + 1] = indptr[i] + len(r)
    cols = np.array(cols, dtype=np.int64)
    off = np.array([0, 3, 6])
    d = exchange_bytes_per_term(indptr, cols, off, k=4)
    # rank 0 (rows 0-2) references 3, 4, 5; rank 1 (rows 3-5) references 0, 2
    assert [x["halo_rows"] for x in d["ranks"]] == [3, 2]
    assert d["max_bytes_per_rank"] == 3 * 16
    h = exchange_bytes_per_term(indptr, cols, off, k=4, replicate_rows=1)
    assert [x["p2p_rows"] for x in h["ranks"]] == [3, 1]
    assert [x["allgather_rows"] for x in h["ranks"]] == [0, 1]


def _plan_worker(rank, world, port, indptr, indices, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2207_14589_b200.distributed import build_halo_plan, partition_rows
        off = partition_rows(torch.from_numpy(indptr), world)
        p0, p1 = int(indptr[off[rank]]), int(indptr[off[rank + 1]])
        plan = build_halo_plan(torch.from_numpy(indices[p0:p1].copy()), off, rank, world)
        parts = [None] * world
        dist.all_gather_object(parts, (rank, off, plan.halo_cols.numpy(), plan.recv_counts,
                                       [s.numpy() for s in plan.send_rows],
                                       plan.local_indices.numpy()))
        if rank == 0:
            result_q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_build_halo_plan_torch_columns(golden, world):
    """The collective halo plan built from TORCH column tensors (the device
    path, here on CPU tensors under gloo) equals the one-process plans."""
    from paper_2207_14589_b200.distributed import build_halo_plans_local
    n, u, v, w = golden.graph("cfg4s")
    u, v, w = O.canonical_edges(n, u, v, w)
    csr = O.laplacian_csr(n, u, v, w, "normalized")
    indptr = csr.indptr.astype(np.int64)
    indices = csr.indices.astype(np.int64)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, world, port, indptr, indices, q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = build_halo_plans_local(indptr, indices, parts[0][1])
    for r, off, halo, rc, send, local in parts:
        np.testing.assert_array_equal(halo, ref[r].halo_cols)
        np.testing.assert_array_equal(rc, ref[r].recv_counts)
        np.testing.assert_array_equal(local, ref[r].local_indices)
        for q_ in range(world):
            np.testing.assert_array_equal(send[q_], ref[r].send_rows[q_])
