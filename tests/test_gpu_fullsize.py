"""Parity at the BASELINE sizes the perf claims are quoted on.

* configs 3 / 4 / 5, exact mode: the bench's own schedule (the operator
  ``bench.py`` builds -- degree relabelling, 4096/1024 hub chunks, the
  scaled-normalized (VM 2) terms and the persisting-L2 hub window at config 4)
  against the fp64 oracle (scipy CSR, threaded row blocks) at full n, plus
  the device CSR bit for bit against the oracle's, and one whole mu-EG step;
* configs 3s / 5s, stochastic mode: the edge-minibatch apply on identical
  (bit-exact, device-drawn) batches against the restated oracle;
* config 2 run to convergence and a stochastic run_solver on an SBM:
  angle / Ritz values / k-means labels against eigsh and the CPU port.

Reference lines: transforms.py:229-262 (apply), graph.py:182-199 (CSR),
solvers.py:121-144 (mu_eg_step), solvers.py:150-178 (minibatches),
metrics.py:57-79,143-176, tests/test_acceptance.py:169-183,289-302.
"""

import os

import numpy as np
import pytest
import torch

import oracle as O
from conftest import rel_fro

pytestmark = pytest.mark.gpu

PV_TOL = 1e-5   # north_star: p(L)V within 1e-5 relative Frobenius (fp32)
THREADS = max(1, min(32, len(os.sched_getaffinity(0))))


def _sp():
    import paper_2207_14589_b200 as sp
    return sp


def _bench_operator(cfg):
    """The operator exactly as bench.py builds it (device generator ->
    Graph.from_canonical -> make_reversed_operator)."""
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    spec = G.CONFIGS[cfg]
    n, u, v, w = G.config_graph(cfg, device="cuda")
    g = sp.Graph.from_canonical(n, u, v, w, validate=False)
    t = sp.SpectralTransform("negexp-taylor", spec["ell"])
    op = sp.make_reversed_operator(g, t, spec["mode"], device="cuda")
    return spec, g, op


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_fullsize_exact_apply_and_step(cuda, cfg):
    """The headline schedules at full size: CSR bit-exact, p(L)V <= 1e-5,
    one mu-EG step (tcgen05 Gram + update) <= 1e-5, against fp64."""
    sp = _sp()
    from paper_2207_14589_b200.solvers import StepWorkspace
    spec, g, op = _bench_operator(cfg)
    lap = op.laplacian
    n, k, ell, mode = g.n, spec["k"], spec["ell"], spec["mode"]
    if cfg == 4:
        # the plan the headline number runs
        assert lap.reordered and lap.n_chunks > 0 and lap.row_scale is not None
        assert (lap.long_threshold, lap.chunk_len) == (4096, 1024)
        assert 0 < lap.hot_rows(k) < n
    # CSR, bit for bit (original order), against the oracle's
    csr = O.laplacian_csr(n, g.u, g.v, g.w, mode)
    indptr, indices, data = lap.csr_host()
    np.testing.assert_array_equal(indptr, csr.indptr)
    np.testing.assert_array_equal(indices, csr.indices)
    np.testing.assert_array_equal(data, csr.data.astype(np.float32))
    del indptr, indices, data
    # V as bench.py draws it, in the solver's internal order
    gen = torch.Generator(device="cuda").manual_seed(1234)
    V = torch.randn((n, k), device="cuda", generator=gen)
    V /= torch.linalg.norm(V, dim=0)
    Vi = lap.to_internal(V)
    MVi = torch.empty_like(Vi)
    op.apply_internal(Vi, out=MVi)           # the bench's call
    ws = StepWorkspace(n, k, Vi.device)
    Vn = torch.empty_like(Vi)
    ws.mu_eg(Vi, MVi, 0.1, Vn)               # the bench's step body
    MV = lap.from_internal(MVi).cpu().numpy()
    Vnew = lap.from_internal(Vn).cpu().numpy()
    Vh = V.cpu().numpy().astype(np.float64)
    ref = O.apply_transform(csr, "negexp-taylor", ell, 1e-6, op.lambda_star, Vh, threads=THREADS)
    err = rel_fro(MV, ref)
    assert err <= PV_TOL, err
    Vref = O.mu_eg_step(Vh, ref, 0.1)
    err_step = rel_fro(Vnew, Vref)
    assert err_step <= PV_TOL, err_step
    assert not ws.take_flag()
    print(f"cfg{cfg}: p(L)V rel err {err:.2e}, mu-EG step rel err {err_step:.2e}")


@pytest.mark.parametrize("cfg", [3, 5])
def test_fullsize_stochastic_apply(cuda, cfg):
    """Configs 3s / 5s (B = 1e6 / 4e6 per term, k = 64 / 128): the bench's
    edge-minibatch kernels on identical device-drawn batches (bit-exact
    against numpy's PCG64) vs the restated oracle; 3 terms bound the CPU
    time.  Deterministic: the same batch gives bit-identical output."""
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    spec = G.CONFIGS[cfg]
    n, u, v, w = G.config_graph(cfg, device="cuda")
    g = sp.Graph.from_canonical(n, u, v, w, validate=False)
    k, B = spec["k"], spec["batch"]
    t = sp.SpectralTransform("negexp-limit", 3)
    op = sp.make_reversed_operator(g, t, spec["mode"], device="cuda")
    orc = sp.make_stochastic_oracle(op, B, seed=7, estimator="edge-batch")
    X = torch.randn((n, k), device="cuda", generator=torch.Generator("cuda").manual_seed(cfg))
    batch = orc.draw(op.n_terms * B)
    Y = orc.apply_internal(X, batch=batch)
    Y2 = orc.apply_internal(X, batch=batch)
    assert torch.equal(Y, Y2)
    bh = batch.cpu().numpy().astype(np.int64)
    np.testing.assert_array_equal(bh, np.random.default_rng(7).integers(0, g.m, size=bh.size))
    batches = [bh[i * B:(i + 1) * B] for i in range(op.n_terms)]
    ref = O.edge_batch_poly_apply(g.u, g.v, g.w, "negexp-limit", 3, 1e-6, op.lambda_star,
                                  batches, X.cpu().numpy().astype(np.float64), threads=THREADS)
    err = rel_fro(Y.cpu().numpy(), ref)
    assert err <= PV_TOL, err
    print(f"cfg{cfg}s: rel err {err:.2e}")


def _room_truth(g, k):
    import scipy.sparse.linalg as sla
    csr = O.laplacian_csr(g.n, g.u, g.v, g.w, "normalized")
    vals, vecs = sla.eigsh(csr, k=k + 4, sigma=-1e-2, which="LM")
    order = np.argsort(vals)[:k]
    return csr, vals[order], vecs[:, order]


def test_config2_run_to_convergence(cuda):
    """Config 2 (4-room grid, normalized, k = 16), mu-EG with
    negexp-limit(17) at eta = 1.0 for 4,500 steps (bench time_to_angle):
    max principal angle <= 1e-3 to the true bottom-16 eigenvectors and to
    the CPU port's converged block, Ritz values within 1e-4 (relative, the
    zero eigenvalue absolute), identical k-means room labels."""
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    n, u, v, w = G.config_graph(2)
    g = sp.Graph(n, u.numpy(), v.numpy(), w.numpy())
    k, steps, eta = 16, 4500, 1.0
    t = sp.SpectralTransform("negexp-limit", 17)
    cfg = sp.SolverConfig(solver="mu-eg", k=k, eta=eta, steps=steps, eval_every=steps, seed=0)
    run = sp.run_solver(g, t, cfg, mode="normalized", record_timing=False)
    V = run.V.cpu().numpy().astype(np.float64)
    csr, lam, U = _room_truth(g, k)
    ang = sp.principal_angles(V, U)
    assert ang <= 1e-3, ang
    # the CPU port from the same seeded initial block
    init_seed, _, _ = O.solver_seeds(0)
    lam_star = O.choose_lambda_star("negexp-limit", 2.0)
    Vc = O.init_state(n, k, init_seed)
    for _ in range(steps):
        Vc = O.mu_eg_step(Vc, O.apply_transform(csr, "negexp-limit", 17, 1e-6, lam_star, Vc), eta)
    assert O.principal_angles(Vc, U) <= 1e-3
    ang_cpu = sp.principal_angles(V, Vc)
    assert ang_cpu <= 1e-3, ang_cpu
    ritz = O.ritz_values(csr, V)
    assert abs(ritz[0] - lam[0]) <= 1e-4 * abs(lam[1])
    np.testing.assert_allclose(ritz[1:], lam[1:], rtol=1e-4)
    labels = sp.kmeans_cluster(V[:, :4], 4, seed=0)
    labels_cpu = O.kmeans_cluster(Vc[:, :4], 4, seed=0)
    assert sp.match_labels(labels, labels_cpu) == 1.0
    print(f"cfg2: angle {ang:.2e} (truth) {ang_cpu:.2e} (CPU port), ritz max rel "
          f"{np.max(np.abs(ritz[1:] - lam[1:]) / lam[1:]):.2e}")


def test_stochastic_run_solver_sbm(cuda):
    """Stochastic mode end to end: run_solver(batch_size > 0) with the
    per-term edge-minibatch oracle (the north-star path) on the config-1 SBM
    (10 blocks x 100), mu-EG, negexp-limit(13), eta = 0.1, B = 16 m edges per
    term, 1,500 steps: max principal angle to the true bottom-10
    eigenvectors <= 1e-2 (measured 5.4e-3; the exact run reaches 1e-3), the
    k-means labels identical to the exact run's, seed-deterministic.
    (tools/probe_stochastic_solver.py: the walk oracle, the reference's
    default for polynomial kinds, diverges at these settings -- its
    per-column estimates have too much variance for negexp-limit(13) -- so
    it is pinned call by call against the reference's goldens instead,
    tests/test_gpu_walks.py.)"""
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    n, u, v, w = G.sbm_dense(10, 100, 0.1, 0.002, seed=3)
    g = sp.Graph(n, u.numpy(), v.numpy(), w.numpy())
    t = sp.SpectralTransform("negexp-limit", 13)
    cfg = sp.SolverConfig(solver="mu-eg", k=10, eta=0.1, steps=1500, eval_every=500,
                          batch_size=16 * g.m, seed=2)
    run = sp.run_solver(g, t, cfg, record_timing=False, estimator="edge-batch")
    run2 = sp.run_solver(g, t, cfg, record_timing=False, estimator="edge-batch")
    assert torch.equal(run.V, run2.V)
    exact = sp.run_solver(g, t, sp.SolverConfig(solver="mu-eg", k=10, eta=0.1, steps=1500,
                                                eval_every=500, seed=2), record_timing=False)
    gt = sp.graph_ground_truth(g)
    U = gt.bottom(10)
    V = run.V.cpu().numpy().astype(np.float64)
    Ve = exact.V.cpu().numpy().astype(np.float64)
    ang, ang_exact = sp.principal_angles(V, U), sp.principal_angles(Ve, U)
    labels = sp.kmeans_cluster(V, 10, seed=5)
    labels_exact = sp.kmeans_cluster(Ve, 10, seed=5)
    print(f"stochastic run: angle {ang:.3e} (exact run {ang_exact:.3e})")
    assert ang_exact <= 1e-3
    assert ang <= 1e-2, ang
    assert sp.match_labels(labels, labels_exact) == 1.0
    # the subspace-error trajectory is recorded at the eval steps, decreasing
    errs = [r.subspace_error for r in run.records]
    assert len(errs) == 4 and errs[-1] < errs[0]
