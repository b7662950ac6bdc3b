"""Row-sharded apply on ONE GPU: every shard's fused term kernel runs on its
[own | halo] block with halos filled by in-process copies that follow the
shards' HaloPlans (the NCCL send/recv of a real run), and the assembled
result must equal the single-operator apply.  (The collective plan
agreement and the send/recv exchange itself are tested under gloo on CPU.)"""

import numpy as np
import pytest
import torch

from conftest import rel_fro

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("cfg,kind,ell", [(4, "negexp-taylor", 12), (5, "negexp-limit", 9),
                                          (3, "identity", None), (1, "negexp-limit", 9)])
def test_sharded_terms_match_single_gpu(cuda, world, cfg, kind, ell, split):
    """split=True: the own-column pass runs BEFORE the halo rows arrive (the
    halo region holds NaN then), the halo-column pass after, as in the
    overlapped NCCL path (sped_csr_term_split)."""
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200 import generators as G
    from paper_2207_14589_b200.distributed import (ShardedLaplacian, build_halo_plans_local,
                                                   partition_rows)
    spec = G.CONFIGS[cfg]
    n, u, v, w = G.config_graph(cfg, device="cuda", scale=0.02 if cfg > 2 else 1.0)
    g = sp.Graph.from_canonical(n, u, v, w)
    L = sp.LaplacianOperator(g, spec["mode"])
    t = sp.SpectralTransform(kind, ell)
    lam = 0.0 if kind != "identity" else 2.0
    op = sp.TransformedOperator(L, t, lam, 2.0)
    k = spec["k"]
    X = torch.randn((n, k), device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
    ref = op.apply_internal(X)
    indptr = L.indptr.cpu().numpy().astype(np.int64)
    indices = L.indices[: L.nnz].cpu().numpy()
    offsets = partition_rows(indptr, world)
    plans = build_halo_plans_local(indptr, indices, offsets)
    shards = [ShardedLaplacian(L, r, world, offsets=offsets, plan=plans[r]) for r in range(world)]
    assert sum(p.n_halo for p in plans) > 0
    al, be, ga, w0, lf, s = op.schedule
    E = [[torch.empty((sh.n_own + sh.plan.n_halo, k), device="cuda") for _ in range(2)]
         for sh in shards]
    xs = [X[int(offsets[r]):int(offsets[r + 1])].contiguous() for r in range(world)]
    outs = [torch.empty_like(xs[r]) for r in range(world)]
    for r in range(world):
        E[r][0][: shards[r].n_own].copy_(xs[r])
    P = [torch.empty_like(xs[r]) for r in range(world)]
    cur = 0
    for tt in range(len(al)):
        final = tt == len(al) - 1
        if split:
            for r in range(world):
                E[r][cur][shards[r].n_own:].fill_(float("nan"))
                shards[r].partial_term(E[r][cur], P[r], k)
        # halo fill: rank r receives from owner q the rows q's send list names
        for r in range(world):
            roff = np.concatenate([[0], np.cumsum(plans[r].recv_counts)])
            for q in range(world):
                if q == r or plans[r].recv_counts[q] == 0:
                    continue
                rows = torch.from_numpy(plans[q].send_rows[r]).cuda()
                dst = E[r][cur][shards[r].n_own + roff[q]: shards[r].n_own + roff[q + 1]]
                dst.copy_(E[q][cur][rows])
        for r in range(world):
            sh = shards[r]
            dst = outs[r] if final else E[r][1 - cur][: sh.n_own]
            coeffs = (al[tt], be[tt], ga[tt], w0 if tt == 0 else 1.0, lf if final else 0.0,
                      s if final else 1.0)
            if split:
                sh.remote_term(E[r][cur], xs[r], dst, P[r], *coeffs, k)
            else:
                sh.local_term(E[r][cur], xs[r], dst, *coeffs, k)
        cur = 1 - cur
    got = torch.cat(outs)
    assert torch.isfinite(got).all()
    assert rel_fro(got.cpu().numpy(), ref.cpu().numpy()) <= 1e-5


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("cfg", [3, 5])
def test_sharded_stochastic_terms_match_single_gpu(cuda, world, cfg):
    """Edge-minibatch terms on row shards: every shard replays the same
    global batch, keeps only the endpoints it owns (local epos = -1 for the
    others) and gathers the other endpoint from its halo; the assembled block
    equals the single-GPU stochastic apply on the same batch."""
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200 import generators as G
    from paper_2207_14589_b200.distributed import (ShardedLaplacian, build_halo_plans_local,
                                                   partition_rows)
    spec = G.CONFIGS[cfg]
    n, u, v, w = G.config_graph(cfg, device="cuda", scale=0.02)
    g = sp.Graph.from_canonical(n, u, v, w)
    op = sp.make_reversed_operator(g, sp.SpectralTransform("negexp-limit", 9), spec["mode"])
    L = op.laplacian
    B = 5000
    orc = sp.make_stochastic_oracle(op, B, seed=11, estimator="edge-batch")
    k = spec["k"]
    X = torch.randn((n, k), device="cuda", generator=torch.Generator(device="cuda").manual_seed(2))
    al, be, ga, w0, lf, s = op.schedule
    batch = orc.draw(len(al) * B)
    ref = orc.apply_internal(X, batch=batch)
    indptr = L.indptr.cpu().numpy().astype(np.int64)
    indices = L.indices[: L.nnz].cpu().numpy()
    offsets = partition_rows(indptr, world)
    plans = build_halo_plans_local(indptr, indices, offsets)
    shards = [ShardedLaplacian(L, r, world, offsets=offsets, plan=plans[r]) for r in range(world)]
    # every edge entry is owned by exactly one shard
    owned = sum((sh.epos_local >= 0).long() for sh in shards)
    assert bool((owned == 1).all())
    E = [[torch.empty((sh.n_own + sh.plan.n_halo, k), device="cuda") for _ in range(2)]
         for sh in shards]
    xs = [X[int(offsets[r]):int(offsets[r + 1])].contiguous() for r in range(world)]
    outs = [torch.empty_like(xs[r]) for r in range(world)]
    for r in range(world):
        E[r][0][: shards[r].n_own].copy_(xs[r])
    cur = 0
    for tt in range(len(al)):
        for r in range(world):
            roff = np.concatenate([[0], np.cumsum(plans[r].recv_counts)])
            for q in range(world):
                if q == r or plans[r].recv_counts[q] == 0:
                    continue
                rows = torch.from_numpy(plans[q].send_rows[r]).cuda()
                dst = E[r][cur][shards[r].n_own + roff[q]: shards[r].n_own + roff[q + 1]]
                dst.copy_(E[q][cur][rows])
        final = tt == len(al) - 1
        for r in range(world):
            sh = shards[r]
            dst = outs[r] if final else E[r][1 - cur][: sh.n_own]
            sh.local_batch_term(E[r][cur], xs[r], dst, batch[tt * B:(tt + 1) * B], B, al[tt],
                                be[tt], ga[tt], w0 if tt == 0 else 1.0, lf if final else 0.0,
                                s if final else 1.0, k)
        cur = 1 - cur
    got = torch.cat(outs)
    assert rel_fro(got.cpu().numpy(), ref.cpu().numpy()) <= 1e-6


def test_sharded_solver_steps_single_rank(cuda):
    """sharded_mu_eg_step / sharded_oja_step / the sharded stochastic
    operator through a real (one-rank NCCL) process group equal the
    single-GPU steps: the collective path end to end."""
    import socket
    import torch.distributed as dist
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200 import generators as G
    from paper_2207_14589_b200.distributed import (ShardedLaplacian, ShardedOperator,
                                                   ShardedStochasticOperator, sharded_mu_eg_step,
                                                   sharded_oja_step)
    from paper_2207_14589_b200.solvers import StepWorkspace
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        n, u, v, w = G.config_graph(3, device="cuda", scale=0.02)
        g = sp.Graph.from_canonical(n, u, v, w)
        t = sp.SpectralTransform("negexp-limit", 9)
        op = sp.make_reversed_operator(g, t, "unnormalized")
        k = 64
        V = sp.init_state(n, k, 3).V
        Vi = op.laplacian.to_internal(V)
        shard = ShardedLaplacian(op.laplacian, 0, 1)
        sop = ShardedOperator(shard, t, op.lambda_star)
        ws1, ws2 = StepWorkspace(n, k, "cuda"), StepWorkspace(n, k, "cuda")
        for name, sstep, body in (("mu-eg", sharded_mu_eg_step, "mu_eg"),
                                  ("oja", sharded_oja_step, "oja")):
            out_s = torch.empty_like(Vi)
            sstep(sop, Vi, 0.1, ws1, out_s)
            out_r = torch.empty_like(Vi)
            getattr(ws2, body)(Vi, op.apply_internal(Vi), 0.1, out_r)
            assert rel_fro(out_s.cpu().numpy(), out_r.cpu().numpy()) <= 1e-6, name
            assert ws1.reduce is None
        sto = ShardedStochasticOperator(shard, t, op.lambda_star, 4000, seed=5)
        orc = sp.make_stochastic_oracle(op, 4000, seed=5, estimator="edge-batch")
        y_s = sto.apply_local(Vi)
        y_r = orc.apply_internal(Vi)  # same seed: the same batches
        assert rel_fro(y_s.cpu().numpy(), y_r.cpu().numpy()) <= 1e-6
    finally:
        dist.destroy_process_group()
