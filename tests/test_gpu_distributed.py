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


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("cfg,kind,ell", [(4, "negexp-taylor", 12), (5, "negexp-limit", 9),
                                          (3, "identity", None)])
def test_sharded_terms_match_single_gpu(cuda, world, cfg, kind, ell):
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200 import generators as G
    from paper_2207_14589_b200.distributed import (ShardedLaplacian, build_halo_plans_local,
                                                   partition_rows)
    spec = G.CONFIGS[cfg]
    n, u, v, w = G.config_graph(cfg, device="cuda", scale=0.02)
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
    cur = 0
    for tt in range(len(al)):
        # halo fill: rank r receives from owner q the rows q's send list names
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
            sh.local_term(E[r][cur], xs[r], dst, al[tt], be[tt], ga[tt], w0 if tt == 0 else 1.0,
                          lf if final else 0.0, s if final else 1.0, k)
        cur = 1 - cur
    got = torch.cat(outs)
    assert rel_fro(got.cpu().numpy(), ref.cpu().numpy()) <= 1e-5
