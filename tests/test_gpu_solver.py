"""Device solver steps, stochastic oracle and end-to-end runs vs the
reference goldens / oracle (run on a B200)."""

import numpy as np
import pytest
import torch

import oracle as O
from conftest import rel_fro

pytestmark = pytest.mark.gpu


def _sp():
    import paper_2207_14589_b200 as sp
    return sp


def _graph(golden, name):
    sp = _sp()
    n, u, v, w = golden.graph(name)
    return sp.Graph(n, u, v, w)


# --- solver steps --------------------------------------------------------------------

def test_init_state_vs_reference(cuda, golden):
    sp = _sp()
    for key in golden.keys("init/"):
        _, n, k, seed = key.split("/")
        V = sp.init_state(int(n), int(k), int(seed)).V
        assert V.is_cuda
        np.testing.assert_allclose(V.cpu().numpy(), golden[key], atol=2e-5, err_msg=key)


def test_steps_vs_reference(cuda, golden):
    sp = _sp()
    for key in golden.keys("step/"):
        if not key.endswith("/V0"):
            continue
        base = key[: -len("/V0")]
        _, name, mode, kind, ell, k = base.split("/")
        ell = None if ell == "None" else int(ell)
        op = sp.make_reversed_operator(_graph(golden, name), sp.SpectralTransform(kind, ell), mode)
        V0 = golden[key]
        for eta in (0.05, 0.5):
            for rule, fn in (("mueg", sp.mu_eg_step), ("oja", sp.oja_step)):
                ref = golden[f"{base}/{rule}/{eta}"]
                # numpy state in -> numpy out (reference-facing)
                out = fn(sp.EigenState(V0.copy()), op, eta)
                assert isinstance(out.V, np.ndarray) and out.step == 1
                assert rel_fro(out.V, ref) <= 1e-5, (base, rule, eta)
                # device state in -> device state out
                outd = fn(sp.EigenState(torch.as_tensor(V0, dtype=torch.float32, device="cuda")),
                          op, eta)
                assert outd.V.is_cuda
                assert rel_fro(outd.V.cpu().numpy(), ref) <= 1e-5, (base, rule, eta)


def test_mu_eg_reference_behaviours(cuda):
    sp = _sp()
    st = sp.init_state(5, 2, seed=9)
    nxt = sp.mu_eg_step(st, lambda V: 2 * V, eta=0.0)
    np.testing.assert_allclose(nxt.V.cpu().numpy(), st.V.cpu().numpy(), atol=1e-6)
    st = sp.init_state(10, 3, seed=2)
    nxt = sp.oja_step(st, lambda V: V, eta=0.7)
    np.testing.assert_allclose(nxt.V.cpu().numpy(), st.V.cpu().numpy(), atol=1e-5)
    # unit-norm columns every step
    g = sp.Graph.from_edges(6, [(0, 1), (0, 2), (1, 2), (3, 4), (3, 5), (4, 5), (2, 3)])
    op = sp.make_reversed_operator(g, sp.SpectralTransform("identity"))
    st = sp.init_state(6, 3, seed=20)
    for _ in range(25):
        st = sp.mu_eg_step(st, op, eta=0.05)
        np.testing.assert_allclose(torch.linalg.norm(st.V, dim=0).cpu().numpy(), 1.0, atol=1e-5)


def test_mu_eg_known_top_two(cuda):
    sp = _sp()
    rng = np.random.default_rng(7)
    q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    M = torch.as_tensor((q * np.array([3.0, 2.0, 1.0])) @ q.T, dtype=torch.float32, device="cuda")
    st = sp.init_state(3, 2, seed=8)
    for _ in range(2000):
        st = sp.mu_eg_step(st, lambda V: M @ V, eta=0.1)
    V = st.V.cpu().numpy()
    for i in range(2):
        assert abs(abs(V[:, i] @ q[:, i]) - 1) < 0.01


# --- stochastic oracle ---------------------------------------------------------------

def test_device_pcg64_bit_exact(cuda, golden):
    from paper_2207_14589_b200.sampling import pcg64_draw
    for case in sorted({k.rsplit("/", 1)[0] for k in golden.keys("pcg/")}):
        _, m, seed = case.split("/")
        rng = np.random.default_rng()
        rng.bit_generator.state = golden.state(case + "/state0")
        i = 0
        while f"{case}/draw{i}" in golden:
            ref = golden[f"{case}/draw{i}"]
            got = pcg64_draw(rng, int(m), ref.size, "cuda").cpu().numpy()
            np.testing.assert_array_equal(got, ref, err_msg=case)
            assert rng.bit_generator.state == golden.state(f"{case}/state{i + 1}"), case
            i += 1


@pytest.mark.parametrize("m,count", [(10_000_000, 16_000_000), (31_600_000, 4_000_000),
                                     (2**31 - 1, 1_000_000), (5, 100_000)])
def test_device_pcg64_large_streams(cuda, m, count):
    from paper_2207_14589_b200.sampling import pcg64_draw
    rng = np.random.default_rng(123)
    mirror = np.random.default_rng(123)
    for _ in range(2):
        got = pcg64_draw(rng, m, count, "cuda").cpu().numpy()
        ref = mirror.integers(0, m, size=count)
        np.testing.assert_array_equal(got, ref)
        assert rng.bit_generator.state == mirror.bit_generator.state


def test_device_generator_stream_and_state(cuda):
    """DeviceGenerator (state resident on the device, no host sync per draw):
    successive draws equal numpy's integers(0, m, count) stream, the host
    Generator re-synchronised from the device words equals numpy's state,
    and host/device hand-over in both directions keeps one stream."""
    from paper_2207_14589_b200.sampling import DeviceGenerator
    for m, sizes in ((5, [7, 1, 300]), (80_296_541, [1_000_001, 3, 17_000_000]),
                     (2**31 - 1, [999, 1000])):
        gen = DeviceGenerator(np.random.default_rng(11), "cuda")
        mirror = np.random.default_rng(11)
        for c in sizes:
            got = gen.integers(m, c).cpu().numpy()
            np.testing.assert_array_equal(got, mirror.integers(0, m, size=c))
        assert gen.rng.bit_generator.state == mirror.bit_generator.state
        # the host takes over, then the device again
        np.testing.assert_array_equal(gen.rng.integers(0, m, size=5), mirror.integers(0, m, size=5))
        np.testing.assert_array_equal(gen.integers(m, 9).cpu().numpy(),
                                      mirror.integers(0, m, size=9))
        assert gen.rng.bit_generator.state == mirror.bit_generator.state


def test_stochastic_run_solver_cuda_graph_equals_eager(cuda, golden):
    """Stochastic mu-EG / Oja steps replayed as CUDA graphs (device draws from
    the resident PCG64 state inside the graph) are bit-identical to the eager
    steps, and the oracle's stream ends where numpy's does."""
    sp = _sp()
    g = _graph(golden, "cfg1")
    t = sp.SpectralTransform("negexp-limit", 13)
    for solver in ("mu-eg", "oja"):
        cfg = sp.SolverConfig(solver=solver, k=10, eta=0.1, steps=30, eval_every=10, seed=4,
                              batch_size=3 * g.m)
        a = sp.run_solver(g, t, cfg, record_timing=False, estimator="edge-batch",
                          use_cuda_graphs=True)
        b = sp.run_solver(g, t, cfg, record_timing=False, estimator="edge-batch",
                          use_cuda_graphs=False)
        assert torch.equal(a.V, b.V), solver
        assert [r.subspace_error for r in a.records] == [r.subspace_error for r in b.records]


@pytest.mark.parametrize("source", ["device", "host"])
def test_identity_stochastic_oracle_vs_reference(cuda, golden, source):
    sp = _sp()
    for case in sorted({k.rsplit("/", 1)[0] for k in golden.keys("sto/")}):
        _, name, B, seed = case.split("/")
        g = _graph(golden, name)
        op = sp.make_reversed_operator(g, sp.SpectralTransform("identity"))
        oracle = sp.make_stochastic_oracle(op, int(B), int(seed), index_source=source)
        x = golden[case + "/x"]
        for call in range(3):
            y = oracle(x)
            np.testing.assert_array_equal(oracle.last_batch.cpu().numpy(),
                                          golden[f"{case}/batch{call}"])
            assert rel_fro(y, golden[f"{case}/y{call}"]) <= 1e-5, (case, call)


def test_stochastic_single_edge_is_exact(cuda):
    sp = _sp()
    g = sp.Graph.from_edges(2, [(0, 1)])
    op = sp.make_reversed_operator(g, sp.SpectralTransform("identity"))
    oracle = sp.make_stochastic_oracle(op, 3, seed=1)
    v = np.array([0.4, -1.2])
    np.testing.assert_allclose(oracle(v), op.apply(v), atol=1e-6)
    assert sp.make_stochastic_oracle(op, 0, seed=0) == op.apply
    op2 = sp.make_reversed_operator(g, sp.SpectralTransform("negexp"))
    with pytest.raises(ValueError, match="polynomial"):
        sp.make_stochastic_oracle(op2, 4, seed=0)


@pytest.mark.parametrize("kind,ell,k", [("negexp-limit", 9, 4), ("negexp-taylor", 6, 16),
                                        ("log-taylor", 5, 64), ("negexp-limit", 3, 128),
                                        ("negexp-limit", 5, 10)])
def test_edge_batch_poly_vs_restated_oracle(cuda, kind, ell, k):
    """Per-term minibatch composition: same batches -> oracle (fp64)."""
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    n, u, v, w = G.lp_sbm(2000, 10, 24.0, 0.1, 5, 0.8)
    g = sp.Graph(n, u.numpy(), v.numpy(), w.numpy())
    eps = 0.5 if kind == "log-taylor" else 1e-6
    op = sp.make_reversed_operator(g, sp.SpectralTransform(kind, ell, eps))
    oracle = sp.make_stochastic_oracle(op, 5000, seed=3, estimator="edge-batch")
    x = np.random.default_rng(k).standard_normal((n, k)).astype(np.float32).astype(np.float64)
    y = oracle(x)
    B = 5000
    batch = oracle.last_batch.cpu().numpy().astype(np.int64)
    batches = [batch[t * B:(t + 1) * B] for t in range(op.n_terms)]
    ref = O.edge_batch_poly_apply(g.u, g.v, g.w, kind, ell, eps, op.lambda_star, batches, x)
    rng = np.random.default_rng(3)
    np.testing.assert_array_equal(np.concatenate(O.draw_batches(rng, g.m, B, op.n_terms)), batch)
    assert rel_fro(y, ref) <= 1e-5
    # deterministic: the same batch gives bit-identical output
    xd = torch.as_tensor(x, dtype=torch.float32, device="cuda")
    bd = oracle.last_batch
    assert torch.equal(oracle.apply_device(xd, batch=bd), oracle.apply_device(xd, batch=bd))


@pytest.mark.parametrize("B", [31, 33, 700, 4000])
def test_edge_batch_hub_runs_vs_restated_oracle(cuda, B):
    """Rows whose record run spans several 32-record chunks of the sweep
    (a star's hub) next to short runs (a path)."""
    sp = _sp()
    hub = [(0, j) for j in range(1, 301)]
    tail = [(300 + j, 301 + j) for j in range(40)]
    wts = np.linspace(0.5, 2.0, len(hub) + len(tail))
    g = sp.Graph.from_edges(341, [(a, b, c) for (a, b), c in zip(hub + tail, wts)])
    op = sp.make_reversed_operator(g, sp.SpectralTransform("negexp-limit", 5))
    oracle = sp.make_stochastic_oracle(op, B, seed=11, estimator="edge-batch")
    x = np.random.default_rng(B).standard_normal((g.n, 8)).astype(np.float32).astype(np.float64)
    y = oracle(x)
    batch = oracle.last_batch.cpu().numpy().astype(np.int64)
    batches = [batch[t * B:(t + 1) * B] for t in range(op.n_terms)]
    ref = O.edge_batch_poly_apply(g.u, g.v, g.w, "negexp-limit", 5, 1e-6, op.lambda_star,
                                  batches, x)
    assert rel_fro(y, ref) <= 1e-5
    xd = torch.as_tensor(x, dtype=torch.float32, device="cuda")
    bd = oracle.last_batch
    assert torch.equal(oracle.apply_device(xd, batch=bd), oracle.apply_device(xd, batch=bd))


@pytest.mark.parametrize("k", [16, 200])
def test_edge_batch_all_terms_sort_equals_per_term(cuda, k):
    """The all-terms (grouped) sort and the per-term overlapped sorts -- the
    path a workspace of sped_edge_batch_workspace_bytes(n, B) takes -- give
    bit-identical output."""
    sp = _sp()
    from paper_2207_14589_b200 import _lib
    from paper_2207_14589_b200 import generators as G
    n, u, v, w = G.lp_sbm(3000, 12, 20.0, 0.1, 7, 0.8)
    g = sp.Graph(n, u.numpy(), v.numpy(), w.numpy())
    op = sp.make_reversed_operator(g, sp.SpectralTransform("negexp-limit", 9))
    orc = sp.make_stochastic_oracle(op, 4000, seed=5, estimator="edge-batch")
    x = torch.randn((n, k), device="cuda", generator=torch.Generator("cuda").manual_seed(k))
    y_all = orc.apply_internal(x).clone()
    batch = orc.last_batch
    per = int(_lib.load().sped_edge_batch_workspace_bytes(op.laplacian.n, 4000))
    assert per < orc.ws_bytes
    full = orc.ws_bytes
    try:
        orc.ws_bytes = per
        y_per = orc.apply_internal(x, batch=batch)
    finally:
        orc.ws_bytes = full
    assert torch.equal(y_all, y_per)


def test_edge_batch_unbiased_on_device(cuda):
    sp = _sp()
    g = sp.Graph.from_edges(3, [(0, 1), (1, 2)])
    op = sp.make_reversed_operator(g, sp.SpectralTransform("negexp-limit", 3))
    oracle = sp.make_stochastic_oracle(op, 2, seed=3, estimator="edge-batch")
    v = torch.tensor([0.2, -0.5, 0.9], device="cuda")
    exact = op.apply(v).cpu().numpy()
    draws = np.stack([oracle(v).cpu().numpy() for _ in range(4000)])
    se = draws.std(axis=0, ddof=1) / np.sqrt(draws.shape[0])
    assert np.all(np.abs(draws.mean(axis=0) - exact) <= 3.5 * se + 1e-6)


# --- end to end ------------------------------------------------------------------------

def test_run_solver_small_graphs(cuda, golden):
    sp = _sp()
    k3 = _graph(golden, "k3")
    cfg = sp.SolverConfig(k=2, steps=0, seed=0)
    run = sp.run_solver(k3, sp.SpectralTransform("identity"), cfg)
    assert len(run.records) == 1 and run.records[0].step == 0
    cfg = sp.SolverConfig(k=2, steps=120, eval_every=30, seed=5)
    a = sp.run_to_csv(sp.run_solver(k3, sp.SpectralTransform("identity"), cfg, record_timing=False))
    b = sp.run_to_csv(sp.run_solver(k3, sp.SpectralTransform("identity"), cfg, record_timing=False))
    assert a == b
    cfg = sp.SolverConfig(k=2, steps=50, eval_every=10, seed=5, batch_size=2)
    a = sp.run_to_csv(sp.run_solver(k3, sp.SpectralTransform("identity"), cfg, record_timing=False))
    b = sp.run_to_csv(sp.run_solver(k3, sp.SpectralTransform("identity"), cfg, record_timing=False))
    assert a == b
    with pytest.raises(ValueError):
        sp.run_solver(k3, sp.SpectralTransform("identity"), sp.SolverConfig(k=4, steps=1))


def test_run_solver_cfg1_matches_reference(cuda, golden):
    """Config 1 (SBM 10x100), mu-EG, negexp-limit(13), 1500 steps: the
    device run reaches the reference's subspace (max principal angle
    <= 1e-3 between the two final blocks' spans and the truth), Ritz values
    within 1e-4 relative, and k-means labels identical to the reference's."""
    sp = _sp()
    g = _graph(golden, "cfg1")
    cfg = sp.SolverConfig(solver="mu-eg", k=10, eta=0.1, steps=1500, eval_every=50, seed=5)
    run = sp.run_solver(g, sp.SpectralTransform("negexp-limit", 13), cfg, record_timing=False)
    V = run.V.cpu().numpy().astype(np.float64)
    Vref = golden["run/cfg1/mu-eg/V"]
    gt = sp.graph_ground_truth(g)
    U = gt.bottom(10)
    assert sp.principal_angles(V, U) <= 1e-3
    assert sp.principal_angles(V, Vref) <= 1e-3
    L = sp.build_laplacian(g)
    ritz = sp.ritz_values(L, V)
    np.testing.assert_allclose(ritz[1:], gt.eigenvalues[1:10], rtol=1e-4)
    assert abs(ritz[0]) <= 1e-4
    labels = sp.kmeans_cluster(V, 10, seed=5)
    assert sp.match_labels(labels, golden["run/cfg1/mu-eg/labels"]) == 1.0
    # the planted blocks themselves are recovered as well as by the reference
    ref_acc = sp.match_labels(golden["run/cfg1/mu-eg/labels"], np.arange(1000) // 100)
    assert sp.match_labels(labels, np.arange(1000) // 100) >= ref_acc


def test_run_solver_cuda_graph_equals_eager(cuda, golden):
    sp = _sp()
    g = _graph(golden, "cfg1")
    t = sp.SpectralTransform("negexp-limit", 13)
    cfg = sp.SolverConfig(solver="mu-eg", k=10, eta=0.1, steps=40, eval_every=20, seed=1)
    a = sp.run_solver(g, t, cfg, record_timing=False, use_cuda_graphs=True,
                      use_persistent_kernel=False)
    b = sp.run_solver(g, t, cfg, record_timing=False, use_cuda_graphs=False)
    assert torch.equal(a.V, b.V)
    # the grid-resident kernel (K7, the default here): same to fp32 rounding,
    # and bit-reproducible run to run
    d = sp.run_solver(g, t, cfg, record_timing=False)
    e = sp.run_solver(g, t, cfg, record_timing=False, use_persistent_kernel=True)
    assert rel_fro(d.V.cpu().numpy(), b.V.cpu().numpy()) <= 1e-5
    assert torch.equal(d.V, e.V)
    cfg = sp.SolverConfig(solver="oja", k=10, eta=0.1, steps=40, eval_every=20, seed=1)
    a = sp.run_solver(g, t, cfg, record_timing=False, use_cuda_graphs=True,
                      use_persistent_kernel=False)
    b = sp.run_solver(g, t, cfg, record_timing=False, use_cuda_graphs=False)
    assert torch.equal(a.V, b.V)
    # the grid-resident Oja (K7, CholQR2 in-kernel; the default here)
    d = sp.run_solver(g, t, cfg, record_timing=False)
    e = sp.run_solver(g, t, cfg, record_timing=False, use_persistent_kernel=True)
    assert rel_fro(d.V.cpu().numpy(), b.V.cpu().numpy()) <= 1e-5
    assert torch.equal(d.V, e.V)


def test_reference_solver_accepts_device_operator(cuda, golden):
    """The drop-in seam: the device operator satisfies the duck type the
    reference's run_solver/oja_step consume (numpy in, numpy out)."""
    sp = _sp()
    g = _graph(golden, "two_triangles_bridge")
    op = sp.make_reversed_operator(g, sp.SpectralTransform("identity"))
    V = O.init_state(6, 2, 3)
    for _ in range(200):
        V = O.oja_step(V, op.apply(V), 0.5)
    gt = sp.graph_ground_truth(g)
    assert sp.subspace_error(V, gt, 2) <= 1e-3


def test_run_solver_relabelled_operator(cuda):
    """run_solver keeps its state in the operator's internal order; the
    result (original order) matches the unrelabelled run."""
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    n, u, v, w = G.chung_lu(6000, device="cuda")
    g = sp.Graph.from_canonical(n, u, v, w)
    t = sp.SpectralTransform("negexp-limit", 7)
    runs = []
    for reorder in (None, "degree"):
        L = sp.LaplacianOperator(g, "normalized", reorder=reorder)
        op = sp.TransformedOperator(L, t, 0.0, 2.0)
        cfg = sp.SolverConfig(solver="mu-eg", k=8, eta=0.5, steps=30, eval_every=10, seed=2)
        runs.append(sp.run_solver(g, t, cfg, mode="normalized", operator=op,
                                  record_timing=False).V.cpu().numpy())
    assert rel_fro(runs[1], runs[0]) <= 1e-4


@pytest.mark.parametrize("k", [10, 16, 32, 64, 128])
@pytest.mark.parametrize("n", [8191, 20000, 100003])
def test_gram_kernels_vs_fp64(cuda, k, n):
    """sped_gram (tcgen05 3xTF32 path for k in {32,64,128}, SIMT otherwise)
    against an fp64 reference: S = V^T V, C = V^T M, Q = M^T M.  Bar: 1e-5 of
    the largest entry (fp32-class; the tensor core's truncating fp32
    accumulation is bounded by draining NACC accumulators every SPLIT rows)."""
    from paper_2207_14589_b200.solvers import StepWorkspace
    gen = torch.Generator(device="cuda").manual_seed(k * 7 + n)
    V = torch.randn((n, k), device="cuda", generator=gen) / n ** 0.5
    M = 3.0 * torch.randn((n, k), device="cuda", generator=gen) / n ** 0.5 + 0.5 * V
    ws = StepWorkspace(n, k, torch.device("cuda"))
    ws.gram(V, M)
    G = ws.G.cpu().numpy()
    Vh, Mh = V.double().cpu().numpy(), M.double().cpu().numpy()
    for blk, ref in ((0, Vh.T @ Vh), (1, Vh.T @ Mh), (2, Mh.T @ Mh)):
        got = G[blk * k * k:(blk + 1) * k * k].reshape(k, k)
        scale = np.abs(ref).max()
        assert np.abs(got - ref).max() <= 1e-5 * scale, (blk, np.abs(got - ref).max() / scale)
    ws.gram(V)
    S = ws.G.cpu().numpy()[: k * k].reshape(k, k)
    assert np.abs(S - Vh.T @ Vh).max() <= 1e-5 * np.abs(Vh.T @ Vh).max()
    # sped_gram_mueg (the mu-EG Gram): S, C and diag(Q); at k = 128 the Q
    # block's MMAs are skipped and its off-diagonal comes back 0
    ws.gram(V, M, diag_q=True)
    G = ws.G.cpu().numpy()
    for blk, ref in ((0, Vh.T @ Vh), (1, Vh.T @ Mh)):
        got = G[blk * k * k:(blk + 1) * k * k].reshape(k, k)
        assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max(), blk
    Q = G[2 * k * k:].reshape(k, k)
    qref = (Mh * Mh).sum(0)
    assert np.abs(np.diag(Q) - qref).max() <= 1e-5 * qref.max()
    if k == 128:
        assert not np.any(Q - np.diag(np.diag(Q)))
        assert np.abs(np.diag(Q) - qref).max() <= 1e-12 * qref.max()  # fp64 sums of squares


@pytest.mark.parametrize("k", [10, 16, 32, 64, 128])
def test_block_update_vs_fp64(cuda, k):
    from paper_2207_14589_b200.solvers import StepWorkspace
    n = 50001
    gen = torch.Generator(device="cuda").manual_seed(k)
    P = torch.randn((n, k), device="cuda", generator=gen)
    M = torch.randn((n, k), device="cuda", generator=gen)
    A = torch.triu(torch.randn((k, k), device="cuda", generator=gen))
    B = torch.randn((k, k), device="cuda", generator=gen)
    sc = torch.rand(k, device="cuda", generator=gen) + 0.5
    ws = StepWorkspace(n, k, torch.device("cuda"))
    out = torch.empty_like(P)
    Pd, Md, Ad, Bd, sd = (t.double() for t in (P, M, A, B, sc))
    # k = 128 runs on tcgen05 in 3xTF32 (no lo*lo term, fp32 accumulation in
    # TMEM): ~7e-7 relative on random data; the SIMT kernels are ~1e-7
    tol = 3e-6 if k == 128 else 1e-6
    for upper, Bm, eta in ((True, None, 0.3), (False, None, 0.7), (False, B, 0.0)):
        ws.update(P, A.contiguous(), M, Bm, eta, sc, out, upper=upper)
        ref = (Pd @ Ad + (Md @ Bd if Bm is not None else eta * Md)) * sd
        assert rel_fro(out.cpu().numpy(), ref.cpu().numpy()) <= tol, (upper, Bm is not None)
    # no M, no scale (the CholQR2 / orthonormalisation form)
    ws.update(P, A.contiguous(), None, None, 0.0, None, out)
    assert rel_fro(out.cpu().numpy(), (Pd @ Ad).cpu().numpy()) <= tol


def test_block_update_k32_unaligned_coefficients(cuda):
    """The packed-FMA k = 32 update reads A / scale as float2; pointers that
    are only 4-B aligned take the lane-per-column kernel -- same result, and
    the packed kernel's output is bit-identical to it (same per-element sums
    in the same order)."""
    from paper_2207_14589_b200.solvers import StepWorkspace
    n, k = 20011, 32
    gen = torch.Generator(device="cuda").manual_seed(5)
    P = torch.randn((n, k), device="cuda", generator=gen)
    M = torch.randn((n, k), device="cuda", generator=gen)
    A = torch.triu(torch.randn((k, k), device="cuda", generator=gen)).contiguous()
    sc = torch.rand(k, device="cuda", generator=gen) + 0.5
    ws = StepWorkspace(n, k, torch.device("cuda"))
    out = torch.empty_like(P)
    ws.update(P, A, M, None, 0.3, sc, out, upper=True)
    buf = torch.empty(k * k + 1, device="cuda")
    A_odd = buf[1:]                       # 4-B aligned view of the same coefficients
    A_odd.copy_(A.flatten())
    assert A_odd.data_ptr() % 8 == 4
    out2 = torch.empty_like(P)
    ws.update(P, A_odd, M, None, 0.3, sc, out2, upper=True)
    assert torch.equal(out, out2)
    ref = (P.double() @ A.double() + 0.3 * M.double()) * sc.double()
    assert rel_fro(out.cpu().numpy(), ref.cpu().numpy()) <= 1e-6


@pytest.mark.parametrize("name,mode,kind,ell,k", [("cfg1", "unnormalized", "negexp-limit", 13, 10),
                                                  ("er0", "unnormalized", "negexp-limit", 9, 3),
                                                  ("er1", "normalized", "negexp-taylor", 8, 4)])
def test_persistent_solver_vs_reference(cuda, golden, name, mode, kind, ell, k):
    """sped_persistent_mueg (K7): one whole mu-EG step in one cooperative
    launch == the reference's mu_eg_step (goldens) to 1e-5."""
    sp = _sp()
    from paper_2207_14589_b200.solvers import _PersistentStepper, persistent_solver_eligible
    op = sp.make_reversed_operator(_graph(golden, name), sp.SpectralTransform(kind, ell), mode)
    base = f"step/{name}/{mode}/{kind}/{ell}/{k}"
    V0 = torch.as_tensor(golden[base + "/V0"], dtype=torch.float32, device="cuda")
    assert persistent_solver_eligible(op, k, "mu-eg")
    for eta in (0.05, 0.5):
        st = _PersistentStepper(op, eta, op.laplacian.to_internal(V0))
        st.advance(1)
        V1 = op.laplacian.from_internal(st.V).cpu().numpy()
        assert rel_fro(V1, golden[f"{base}/mueg/{eta}"]) <= 1e-5, eta
        assert not st.ws.take_flag()


@pytest.mark.parametrize("graph,mode,kind,ell,eta,k", [
    ("cfg2", "normalized", "negexp-limit", 17, 1.0, 16),
    ("sbm20k", "normalized", "negexp-taylor", 12, 0.1, 32),
    ("sbm20k", "unnormalized", "negexp-limit", 9, 0.3, 7),
    ("sbm20k", "normalized", "negexp-limit", 151, 0.5, 8)])  # > 64 terms in the parameters
def test_persistent_solver_multi_cta(cuda, graph, mode, kind, ell, eta, k):
    """K7 on graphs spread over every SM (config 2's 10^4-node grid; a 2x10^4
    node SBM with stored normalized values / implicit unit weights, odd k):
    25 steps equal the CUDA-graph multi-kernel path and the oracle's fp64
    steps to 1e-4 (fp32 rounding of two summation orders, compounded over 25
    steps; the single-step contract of 1e-5 is checked against the goldens
    above)."""
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    from paper_2207_14589_b200.solvers import (_GraphStepper, _PersistentStepper,
                                               persistent_solver_eligible)
    if graph == "cfg2":
        n, u, v, w = G.config_graph(2)
    else:
        n, u, v, w = G.sbm_sparse(20000, 100, 20.0, 0.9)
    g = sp.Graph(n, u.numpy(), v.numpy(), w.numpy())
    op = sp.make_reversed_operator(g, sp.SpectralTransform(kind, ell), mode)
    assert persistent_solver_eligible(op, k, "mu-eg")
    V0 = sp.init_state(n, k, 11).V
    Vi = op.laplacian.to_internal(V0)
    p = _PersistentStepper(op, eta, Vi)
    q = _GraphStepper(op, "mu-eg", eta, Vi)
    p.advance(25)
    q.advance(25)
    Vp = op.laplacian.from_internal(p.V).cpu().numpy()
    Vq = op.laplacian.from_internal(q.V).cpu().numpy()
    assert rel_fro(Vp, Vq) <= 1e-4
    csr = O.laplacian_csr(n, g.u, g.v, g.w, mode)
    lam = O.choose_lambda_star(kind, O.lambda_upper(n, g.u, g.v, g.w, mode))
    Vo = V0.cpu().numpy().astype(np.float64)
    for _ in range(25):
        Vo = O.mu_eg_step(Vo, O.apply_transform(csr, kind, ell, 1e-6, lam, Vo), eta)
    assert rel_fro(Vp, Vo) <= 1e-4
    p2 = _PersistentStepper(op, eta, Vi)
    p2.advance(25)
    assert torch.equal(p.V, p2.V)
    # split over launches: the tagged term blocks carry stale words of the
    # previous launch, which the per-launch tag base must never match
    p3 = _PersistentStepper(op, eta, Vi)
    for m in (1, 1, 10, 13):
        p3.advance(m)
    assert torch.equal(p.V, p3.V)
    assert not p3.ws.take_flag()


@pytest.mark.parametrize("n,d,c,spread", [(3000, 8, 6, 0.3), (20000, 16, 12, 1.0)])
def test_kmeans_labels_vs_oracle_and_deterministic(cuda, n, d, c, spread):
    """kmeans_cluster (device assignment, fixed-point centroid sums) gives the
    oracle's labels (metrics.py:143-176 restated; index work, bit-exact) on
    blobs of increasing overlap, and identical labels run to run at a size
    where fp64 atomics would reorder their sums."""
    sp = _sp()
    rng = np.random.default_rng(n + c)
    centers = rng.standard_normal((c, d)) * 3.0
    X = (centers[rng.integers(0, c, n)] + spread * rng.standard_normal((n, d))).astype(np.float32)
    got = sp.kmeans_cluster(X, c, seed=3)
    ref = O.kmeans_cluster(X.astype(np.float64), c, seed=3)
    assert np.array_equal(got, ref)
    Xd = torch.as_tensor(X, device="cuda")
    big = torch.cat([Xd] * 10)  # 2e5 rows
    a = sp.kmeans_cluster(big, c, seed=1)
    b = sp.kmeans_cluster(big, c, seed=1)
    assert np.array_equal(a, b)


def test_power_law_graph_capture_with_l2_window(cuda):
    """A degree-relabelled power-law graph whose SpMM sets the persisting-L2
    window over the hub prefix: whole steps captured as CUDA graphs equal
    the eager steps bit for bit, and the apply equals the oracle."""
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    from paper_2207_14589_b200.solvers import _GraphStepper
    n, u, v, w = G.chung_lu(600_000, cap=20000.0, device="cuda")
    g = sp.Graph.from_canonical(n, u, v, w)
    op = sp.make_reversed_operator(g, sp.SpectralTransform("negexp-taylor", 6), "normalized")
    lap = op.laplacian
    assert lap.reordered and 0 < lap.hot_rows(32) < n  # the window is in play
    V = torch.randn((n, 32), device="cuda", generator=torch.Generator(device="cuda").manual_seed(2))
    V /= torch.linalg.norm(V, dim=0)
    a = _GraphStepper(op, "mu-eg", 0.1, V)
    a.advance(3)
    from paper_2207_14589_b200.solvers import StepWorkspace
    ws = StepWorkspace(n, 32, "cuda")
    X = V.clone()
    Y, MV = torch.empty_like(X), torch.empty_like(X)
    for _ in range(3):
        op.apply_internal(X, out=MV)
        ws.mu_eg(X, MV, 0.1, Y)
        X, Y = Y, X
    assert torch.equal(a.V, X)
    csr = O.laplacian_csr(n, g.u, g.v, g.w, "normalized")
    x = np.random.default_rng(1).standard_normal((n, 8)).astype(np.float32)
    got = op.apply(torch.as_tensor(x, device="cuda")).cpu().numpy()
    ref = O.apply_transform(csr, "negexp-taylor", 6, 1e-6, op.lambda_star, x.astype(np.float64))
    assert rel_fro(got, ref) <= 1e-5


@pytest.mark.parametrize("n", [1, 127, 128, 129, 1000])
def test_k128_tensor_core_kernels_small_n(cuda, n):
    """The k = 128 tcgen05 update and the mu-EG Gram at tile-edge sizes
    (one partial tile, exactly one tile, one row over) against fp64."""
    from paper_2207_14589_b200.solvers import StepWorkspace
    k = 128
    gen = torch.Generator(device="cuda").manual_seed(n)
    P = torch.randn((n, k), device="cuda", generator=gen)
    M = torch.randn((n, k), device="cuda", generator=gen)
    A = torch.triu(torch.randn((k, k), device="cuda", generator=gen)).contiguous()
    sc = torch.rand(k, device="cuda", generator=gen) + 0.5
    ws = StepWorkspace(n, k, torch.device("cuda"))
    out = torch.empty_like(P)
    ws.update(P, A, M, None, 0.3, sc, out, upper=True)
    ref = ((P.double() @ A.double() + 0.3 * M.double()) * sc.double()).cpu().numpy()
    assert rel_fro(out.cpu().numpy(), ref) <= 3e-6
    ws.gram(P, M, diag_q=True)
    G = ws.G.cpu().numpy()
    Ph, Mh = P.double().cpu().numpy(), M.double().cpu().numpy()
    S, C = G[: k * k].reshape(k, k), G[k * k: 2 * k * k].reshape(k, k)
    assert np.abs(S - Ph.T @ Ph).max() <= 1e-5 * np.abs(Ph.T @ Ph).max()
    assert np.abs(C - Ph.T @ Mh).max() <= 1e-5 * np.abs(Ph.T @ Mh).max()
    Q = G[2 * k * k:].reshape(k, k)
    np.testing.assert_allclose(np.diag(Q), (Mh * Mh).sum(0), rtol=1e-12)


@pytest.mark.parametrize("k,kind,ell", [(1, "negexp-limit", 1), (3, "negexp-taylor", 2),
                                        (5, "identity", None)])
def test_persistent_solver_tiny(cuda, golden, k, kind, ell):
    """K7 at the small end (k = 1, one-term and identity transforms, a
    6-node graph): whole steps equal the oracle's fp64 steps."""
    sp = _sp()
    from paper_2207_14589_b200.solvers import _PersistentStepper, persistent_solver_eligible
    g = _graph(golden, "two_triangles_bridge")
    op = sp.make_reversed_operator(g, sp.SpectralTransform(kind, ell))
    assert persistent_solver_eligible(op, k, "mu-eg")
    V0 = O.init_state(g.n, k, 4)
    st = _PersistentStepper(op, 0.2, op.laplacian.to_internal(
        torch.as_tensor(V0, dtype=torch.float32, device="cuda")))
    st.advance(5)
    csr = O.laplacian_csr(g.n, g.u, g.v, g.w)
    V = V0.copy()
    for _ in range(5):
        V = O.mu_eg_step(V, O.apply_transform(csr, kind, ell, 1e-6, op.lambda_star, V), 0.2)
    got = op.laplacian.from_internal(st.V).cpu().numpy()
    assert rel_fro(got, V) <= 1e-4
    assert not st.ws.take_flag()



@pytest.mark.parametrize("graph,mode,kind,ell,eta,k", [
    ("cfg1", "unnormalized", "negexp-limit", 13, 0.1, 10),
    ("cfg2", "normalized", "negexp-limit", 17, 1.0, 16),
    ("sbm20k", "normalized", "negexp-taylor", 12, 0.5, 32)])
def test_persistent_oja_vs_oracle(cuda, golden, graph, mode, kind, ell, eta, k):
    """K7 Oja (sped_persistent_oja: CholQR2 inside the grid-resident launch)
    over 20 steps against the oracle's fp64 oja_step (MGS, solvers.py:114-118)
    and the multi-kernel path; bit-reproducible run to run."""
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    from paper_2207_14589_b200.solvers import (_GraphStepper, _PersistentStepper,
                                               persistent_solver_eligible)
    if graph == "cfg1":
        g = _graph(golden, "cfg1")
    else:
        n, u, v, w = G.config_graph(2) if graph == "cfg2" else G.sbm_sparse(20000, 100, 20.0, 0.9)
        g = sp.Graph(n, u.numpy(), v.numpy(), w.numpy())
    op = sp.make_reversed_operator(g, sp.SpectralTransform(kind, ell), mode)
    assert persistent_solver_eligible(op, k, "oja")
    V0 = sp.init_state(g.n, k, 5).V
    Vi = op.laplacian.to_internal(V0)
    p = _PersistentStepper(op, eta, Vi, "oja")
    q = _GraphStepper(op, "oja", eta, Vi)
    p.advance(20)
    q.advance(20)
    Vp = op.laplacian.from_internal(p.V).cpu().numpy()
    assert rel_fro(Vp, op.laplacian.from_internal(q.V).cpu().numpy()) <= 1e-4
    csr = O.laplacian_csr(g.n, g.u, g.v, g.w, mode)
    lam = O.choose_lambda_star(kind, O.lambda_upper(g.n, g.u, g.v, g.w, mode))
    Vo = V0.cpu().numpy().astype(np.float64)
    for _ in range(20):
        Vo = O.oja_step(Vo, O.apply_transform(csr, kind, ell, 1e-6, lam, Vo), eta)
    assert rel_fro(Vp, Vo) <= 1e-4
    np.testing.assert_allclose(np.linalg.norm(Vp, axis=0), 1.0, atol=1e-5)
    p2 = _PersistentStepper(op, eta, Vi, "oja")
    for m in (7, 13):
        p2.advance(m)
    assert torch.equal(p.V, p2.V)
    assert not p.ws.take_flag()
