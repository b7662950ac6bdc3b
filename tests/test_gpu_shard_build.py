"""Row shards built WITHOUT the whole graph (replaces slicing a
LaplacianOperator built whole on every rank, ref graph.py:182-199):
``sped_laplacian_build_rows`` from each shard's incident edges must give
exactly rows [b, e) of the single-GPU CSR (indptr, global columns, fp32
values, degrees, edge positions), and shards made by
``ShardedLaplacian.from_shard_edges`` must reproduce the single-GPU exact and
stochastic applies.  One GPU, P shards in one process: the routing that
produces each shard's incident edges is ``plan_shard_edges`` (tested under
gloo, tests/test_distributed_gloo.py); here its outcome is formed directly."""

import ctypes as C

import numpy as np
import pytest
import torch

from conftest import rel_fro

pytestmark = pytest.mark.gpu


def _shard_edges(g, world, reorder):
    """Every rank's ShardEdges as plan_shard_edges would route them."""
    from paper_2207_14589_b200.distributed import ShardEdges, _degree_order, partition_rows
    u, v, w = g.device_edges("cuda")
    n, m = g.n, g.m
    eid = torch.arange(m, device="cuda")
    cnt = torch.bincount(u, minlength=n) + torch.bincount(v, minlength=n)
    rowlen = cnt + (cnt > 0).to(cnt.dtype)
    perm = None
    lo, hi = u, v
    if reorder:
        perm, iperm = _degree_order(rowlen)
        rowlen = rowlen[perm]
        a, b = iperm[u], iperm[v]
        lo, hi = torch.minimum(a, b), torch.maximum(a, b)
    indptr = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    torch.cumsum(rowlen, 0, out=indptr[1:])
    offsets = partition_rows(indptr, world)
    out = []
    for r in range(world):
        b, e = int(offsets[r]), int(offsets[r + 1])
        sel = ((lo >= b) & (lo < e)) | ((hi >= b) & (hi < e))
        order = torch.argsort(lo[sel] * n + hi[sel])
        out.append(ShardEdges(n, m, r, world, offsets, lo[sel][order], hi[sel][order],
                              w[sel][order], eid[sel][order], rowlen, perm,
                              g.is_unit_weight()))
    return out


def _graph(cfg, scale=0.02):
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200 import generators as G
    n, u, v, w = G.config_graph(cfg, device="cuda", scale=scale)
    return sp.Graph.from_canonical(n, u, v, w)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("cfg,mode", [(4, "normalized"), (5, "unnormalized"), (3, "unnormalized"),
                                      (5, "normalized")])
def test_row_build_equals_full_build_rows(cuda, cfg, mode, world):
    """sped_laplacian_build_rows == rows [b, e) of sped_laplacian_build, bit
    for bit (stored values, weighted diagonal fold, normalized scaling with
    the gathered degrees), in the relabelled order of power-law graphs."""
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200 import _lib
    g = _graph(cfg)
    L = sp.LaplacianOperator(g, mode, implicit=False)
    lib = _lib.load()
    ses = _shard_edges(g, world, L.reordered)
    if L.reordered:
        assert torch.equal(ses[0].perm.to(torch.int32), L.perm)
    deg_full = torch.from_numpy(L.degrees).cuda()
    if L.reordered:
        deg_full = deg_full[L.perm.long()]
    indptr_full = L.indptr.long()
    seen = torch.zeros(2 * g.m, dtype=torch.int32, device="cuda")
    for se in ses:
        b, e = se.row_range
        nr, ml = e - b, int(se.lo.numel())
        indptr = torch.empty(nr + 1, dtype=torch.int32, device="cuda")
        cap = max(2 * ml + nr, 1)
        indices = torch.empty(cap, dtype=torch.int32, device="cuda")
        vals = torch.empty(cap, dtype=torch.float32, device="cuda")
        deg = torch.empty(max(nr, 1), dtype=torch.float64, device="cuda")
        epos = torch.empty(max(2 * ml, 1), dtype=torch.int32, device="cuda")
        nnz = C.c_int64(0)
        rc = lib.sped_laplacian_build_rows(g.n, b, e, ml, _lib.ptr(se.lo), _lib.ptr(se.hi),
                                           _lib.ptr(se.w), _lib.ptr(deg_full),
                                           1 if mode == "normalized" else 0, 1,
                                           _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(vals),
                                           _lib.ptr(deg), _lib.ptr(epos), C.byref(nnz),
                                           _lib.stream_ptr(cuda))
        _lib.check(rc)
        p0, p1 = int(indptr_full[b]), int(indptr_full[e])
        assert int(nnz.value) == p1 - p0
        assert torch.equal(indptr.long(), indptr_full[b:e + 1] - p0)
        assert torch.equal(indices[: p1 - p0], L.indices[p0:p1])
        assert torch.equal(vals[: p1 - p0], L.values[p0:p1])          # bit-exact fp32
        assert torch.equal(deg[:nr], deg_full[b:e])                    # bincount order
        # each input edge's entries: the same CSR positions as the full
        # build's epos (re-keyed by original edge id), -1 off the shard
        ep = epos[: 2 * ml].view(-1, 2).long()
        full = L.epos[: 2 * g.m].view(-1, 2).long()[se.eid]
        own = (full >= p0) & (full < p1)
        assert torch.equal(ep, torch.where(own, full - p0, torch.full_like(full, -1)))
        seen.view(-1, 2)[se.eid] += own.to(torch.int32)
    assert bool((seen == 1).all())  # every entry built by exactly one shard


def _halo_fill(E, shards, plans, cur, world):
    for r in range(world):
        roff = np.concatenate([[0], np.cumsum(plans[r].recv_counts)])
        for q in range(world):
            if q == r or plans[r].recv_counts[q] == 0:
                continue
            rows = torch.as_tensor(plans[q].send_rows[r]).cuda()
            dst = E[r][cur][shards[r].n_own + roff[q]: shards[r].n_own + roff[q + 1]]
            dst.copy_(E[q][cur][rows])


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("cfg,kind,ell", [(4, "negexp-taylor", 12), (5, "negexp-limit", 9),
                                          (3, "negexp-taylor", 16), (2, "negexp-limit", 17)])
def test_shards_from_edges_apply(cuda, world, cfg, kind, ell):
    """Shards built from their incident edges run the overlapped split
    schedule (own-column pass while the halo is NaN, halo-column pass after)
    and reproduce the single-GPU apply.  Normalized unit-weight graphs
    (configs 2, 4) run the single-GPU scaled form: terms after the first
    exchange and gather u = D^-1/2 w without values (sped_csr_term_shard)."""
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200 import generators as G
    from paper_2207_14589_b200.distributed import ShardedLaplacian, build_halo_plans_local
    spec = G.CONFIGS[cfg]
    g = _graph(cfg)
    op = sp.make_reversed_operator(g, sp.SpectralTransform(kind, ell), spec["mode"])
    L = op.laplacian
    k = spec["k"]
    X = torch.randn((g.n, k), device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
    ref = op.apply_internal(X)
    ses = _shard_edges(g, world, L.reordered)
    offsets = ses[0].offsets
    plans = build_halo_plans_local(L.indptr.long(), L.indices[: L.nnz], offsets)
    deg = torch.from_numpy(L.degrees).cuda()
    if L.reordered:
        deg = deg[L.perm.long()]
    shards = [ShardedLaplacian.from_shard_edges(se, spec["mode"], col_degrees=deg, plan=plans[r],
                                                long_threshold=L.long_threshold,
                                                chunk_len=L.chunk_len)
              for r, se in enumerate(ses)]
    assert sum(s.nnz_local for s in shards) == L.nnz
    al, be, ga, w0, lf, s = op.schedule
    E = [[torch.empty((sh.n_own + sh.plan.n_halo, k), device="cuda") for _ in range(2)]
         for sh in shards]
    xs = [X[int(offsets[r]):int(offsets[r + 1])].contiguous() for r in range(world)]
    outs = [torch.empty_like(xs[r]) for r in range(world)]
    P = [torch.empty_like(xs[r]) for r in range(world)]
    for r in range(world):
        E[r][0][: shards[r].n_own].copy_(xs[r])
    scaled = shards[0].scaled_terms(k)
    assert scaled == (spec["mode"] == "normalized" and g.is_unit_weight())
    cur = 0
    for tt in range(len(al)):
        final = tt == len(al) - 1
        sk = {"scaled_in": tt > 0, "scaled_out": not final} if scaled else {}
        coeffs = (al[tt], be[tt], ga[tt], w0 if tt == 0 else 1.0, lf if final else 0.0,
                  s if final else 1.0)
        if world == 1:  # no halo: one unsplit pass
            shards[0].local_term(E[0][cur], xs[0], outs[0] if final else E[0][1 - cur], *coeffs,
                                 k, **sk)
            cur = 1 - cur
            continue
        for r in range(world):
            E[r][cur][shards[r].n_own:].fill_(float("nan"))
            shards[r].partial_term(E[r][cur], P[r], k, **sk)
        _halo_fill(E, shards, plans, cur, world)
        for r in range(world):
            sh = shards[r]
            dst = outs[r] if final else E[r][1 - cur][: sh.n_own]
            sh.remote_term(E[r][cur], xs[r], dst, P[r], *coeffs, k, **sk)
        cur = 1 - cur
    got = torch.cat(outs)
    assert torch.isfinite(got).all()
    assert rel_fro(got.cpu().numpy(), ref.cpu().numpy()) <= 1e-5


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("cfg", [3, 5, 4])
def test_shards_from_edges_stochastic(cuda, world, cfg):
    """Compacted edge-minibatch terms on shards built from their edges: each
    shard sorts only its own samples' records (O(B/P)), with the global
    estimator scale m/B, and the assembled block equals the single-GPU
    stochastic apply on the same batch."""
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200 import generators as G
    from paper_2207_14589_b200.distributed import ShardedLaplacian, build_halo_plans_local
    spec = G.CONFIGS[cfg]
    g = _graph(cfg)
    op = sp.make_reversed_operator(g, sp.SpectralTransform("negexp-limit", 9), spec["mode"])
    L = op.laplacian
    B = 5000
    orc = sp.make_stochastic_oracle(op, B, seed=13, estimator="edge-batch")
    k = min(spec["k"], 64)
    X = torch.randn((g.n, k), device="cuda", generator=torch.Generator(device="cuda").manual_seed(4))
    al, be, ga, w0, lf, s = op.schedule
    batch = orc.draw(len(al) * B)
    ref = orc.apply_internal(X, batch=batch)
    ses = _shard_edges(g, world, L.reordered)
    offsets = ses[0].offsets
    plans = build_halo_plans_local(L.indptr.long(), L.indices[: L.nnz], offsets)
    deg = torch.from_numpy(L.degrees).cuda()
    if L.reordered:
        deg = deg[L.perm.long()]
    shards = [ShardedLaplacian.from_shard_edges(se, spec["mode"], col_degrees=deg, plan=plans[r])
              for r, se in enumerate(ses)]
    local = [sh.compact_batch(batch, len(al)) for sh in shards]
    # every sampled entry lands in exactly one shard's records
    for tt in range(len(al)):
        tot = sum(int((sh.epos_l.view(-1, 2)[loc[tt].long()] >= 0).sum())
                  for sh, loc in zip(shards, local))
        assert tot == 2 * B
        assert max(int(loc[tt].numel()) for loc in local) < B  # O(B/P) per shard
    E = [[torch.empty((sh.n_own + sh.plan.n_halo, k), device="cuda") for _ in range(2)]
         for sh in shards]
    xs = [X[int(offsets[r]):int(offsets[r + 1])].contiguous() for r in range(world)]
    outs = [torch.empty_like(xs[r]) for r in range(world)]
    for r in range(world):
        E[r][0][: shards[r].n_own].copy_(xs[r])
    cur = 0
    for tt in range(len(al)):
        _halo_fill(E, shards, plans, cur, world)
        final = tt == len(al) - 1
        for r in range(world):
            sh = shards[r]
            dst = outs[r] if final else E[r][1 - cur][: sh.n_own]
            sh.local_batch_term(E[r][cur], xs[r], dst, batch[tt * B:(tt + 1) * B], B, al[tt],
                                be[tt], ga[tt], w0 if tt == 0 else 1.0, lf if final else 0.0,
                                s if final else 1.0, k, local_batch=local[r][tt])
        cur = 1 - cur
    got = torch.cat(outs)
    assert rel_fro(got.cpu().numpy(), ref.cpu().numpy()) <= 1e-6


def test_shard_with_no_sampled_endpoint(cuda):
    """B_local = 0 (sped_edge_batch_poly_apply_scaled): the term is its
    epilogue alone -- the estimate of every own row is 0."""
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200.distributed import ShardedLaplacian
    g = sp.Graph.from_edges(4, [(0, 1), (2, 3)])
    L = sp.LaplacianOperator(g, "unnormalized")
    sh = ShardedLaplacian(L, 0, 1)
    x = torch.randn((4, 8), device="cuda")
    out = torch.empty_like(x)
    sh.local_batch_term(x, x, out, None, 10, 0.5, 1.0, 0.25, 1.0, 0.0, 1.0, 8,
                        local_batch=torch.zeros(0, dtype=torch.int32, device="cuda"))
    torch.testing.assert_close(out, 0.5 * x + 0.25 * x, rtol=1e-6, atol=0)


def test_shard_build_zero_degree_normalized_raises(cuda):
    """An isolated node makes the normalized Laplacian undefined: the shard
    build raises the reference's ValueError (graph.py:187-188) on every
    shard, from the gathered degree vector, not only on the owner."""
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200.distributed import ShardedLaplacian
    g = sp.Graph.from_edges(6, [(0, 1), (1, 2), (3, 4)])   # node 5 isolated
    ses = _shard_edges(g, 2, False)
    deg = torch.zeros(6, dtype=torch.float64, device="cuda")
    deg[:5] = torch.tensor([1, 2, 1, 1, 1], dtype=torch.float64)
    for se in ses:
        with pytest.raises(ValueError, match="degrees"):
            ShardedLaplacian.from_shard_edges(se, "normalized", col_degrees=deg,
                                              plan=None if se.world == 1 else _plan_for(g, se))


def _plan_for(g, se):
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200.distributed import build_halo_plans_local
    L = sp.LaplacianOperator(g, "unnormalized", implicit=False)
    return build_halo_plans_local(L.indptr.long(), L.indices[: L.nnz], se.offsets)[se.rank]
