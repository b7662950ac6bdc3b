"""CUDA path vs the reference goldens and the CPU oracle (run on a B200).

Tolerances (BASELINE north_star): graph construction and sampled indices
bit-exact; p(L)V within 1e-5 relative Frobenius in fp32.
"""

import numpy as np
import pytest
import torch

import oracle as O
from conftest import rel_fro

pytestmark = pytest.mark.gpu

PV_TOL = 1e-5


def _sp():
    import paper_2207_14589_b200 as sp
    return sp


def _graph(golden, name):
    sp = _sp()
    n, u, v, w = golden.graph(name)
    return sp.Graph(n, u, v, w)


# --- graph construction (bit-exact) -----------------------------------------------

@pytest.mark.parametrize("mode", ["unnormalized", "normalized"])
def test_csr_bit_exact_vs_reference(cuda, golden, mode):
    sp = _sp()
    checked = 0
    for name in golden.graph_names():
        key = f"csr/{name}/{mode}"
        g = _graph(golden, name)
        if f"{key}/error" in golden:
            with pytest.raises(ValueError, match="degrees"):
                sp.build_laplacian(g, mode)
            continue
        if f"{key}/indptr" not in golden:
            continue
        for implicit in (False, True):
            if implicit and not (mode == "unnormalized" and g.is_unit_weight()):
                continue
            L = sp.LaplacianOperator(g, mode, implicit=implicit)
            indptr, indices, data = L.csr_host()
            np.testing.assert_array_equal(indptr, golden[f"{key}/indptr"], err_msg=name)
            np.testing.assert_array_equal(indices, golden[f"{key}/indices"], err_msg=name)
            ref32 = golden[f"{key}/data"].astype(np.float32)
            assert np.array_equal(data.view(np.uint32), ref32.view(np.uint32)), (name, mode)
            np.testing.assert_array_equal(L.degrees, golden[f"csr/{name}/{mode}/degrees"])
        checked += 1
    assert checked >= 10


def test_csr_bit_exact_config_scale(cuda):
    """Config-5-shaped weighted graph (n=2e5) and config-4-shaped normalized
    Chung-Lu (n=2e5): device CSR == fp32(scipy CSR) bit for bit."""
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    for (n, u, v, w), mode in [(G.lp_sbm(200_000, 20, 24.0, 0.1, 5, 0.8, device="cuda"), "unnormalized"),
                               (G.chung_lu(200_000, device="cuda"), "normalized"),
                               (G.sbm_sparse(200_000, 20, 20.0, 0.9, device="cuda"), "normalized")]:
        g = sp.Graph.from_canonical(n, u, v, w)
        L = sp.LaplacianOperator(g, mode, implicit=False)
        indptr, indices, data = L.csr_host()
        ref = O.laplacian_csr(n, g.u, g.v, g.w, mode)
        np.testing.assert_array_equal(indptr, ref.indptr)
        np.testing.assert_array_equal(indices, ref.indices)
        mism = np.flatnonzero(data.view(np.uint32) != ref.data.astype(np.float32).view(np.uint32))
        assert mism.size == 0, (mode, mism[:10])
        np.testing.assert_array_equal(L.degrees, O.degrees(n, g.u, g.v, g.w))


# --- polynomial apply ----------------------------------------------------------------

def test_apply_vs_reference_goldens(cuda, golden):
    sp = _sp()
    cases = sorted({k.rsplit("/", 1)[0] for k in golden.keys("apply/")})
    worst = 0.0
    ops = {}
    for case in cases:
        _, name, mode, kind, ell, eps, k = case.split("/")
        ell = None if ell == "None" else int(ell)
        key = (name, mode, kind, ell, eps)
        if key not in ops:
            import warnings
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", RuntimeWarning)
                ops[key] = sp.make_reversed_operator(_graph(golden, name),
                                                     sp.SpectralTransform(kind, ell, float(eps)), mode)
        op = ops[key]
        assert op.lambda_star == float(golden[case + "/lambda_star"])
        x = golden[case + "/x"]
        y = op.apply(x.astype(np.float64))          # numpy in -> numpy out (drop-in)
        assert isinstance(y, np.ndarray) and y.dtype == np.float64 and y.shape == x.shape
        err = rel_fro(y, golden[case + "/y"])
        worst = max(worst, err)
        assert err <= PV_TOL, (case, err)
        # device tensors in -> device tensors out
        yd = op.apply(torch.as_tensor(x, dtype=torch.float32, device="cuda"))
        assert yd.is_cuda and yd.dtype == torch.float32
        assert rel_fro(yd.cpu().numpy(), golden[case + "/y"]) <= PV_TOL
    print("worst rel Frobenius vs reference:", worst)


@pytest.mark.parametrize("k", [1, 3, 4, 8, 10, 16, 32, 64, 128, 130, 256])
def test_apply_all_widths_vs_oracle(cuda, k):
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    n, u, v, w = G.lp_sbm(3000, 10, 24.0, 0.1, 5, 0.8)
    g = sp.Graph(n, u.numpy(), v.numpy(), w.numpy())
    csr = O.laplacian_csr(n, g.u, g.v, g.w)
    rng = np.random.default_rng(k)
    x = rng.standard_normal((n, k)).astype(np.float32)
    for kind, ell in (("negexp-limit", 9), ("negexp-taylor", 6), ("identity", None)):
        op = sp.make_reversed_operator(g, sp.SpectralTransform(kind, ell))
        ref = O.apply_transform(csr, kind, ell, 1e-6, op.lambda_star, x.astype(np.float64))
        y = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        assert rel_fro(y, ref) <= PV_TOL, (k, kind)


@pytest.mark.parametrize("k", [16, 32, 64, 128])
def test_long_row_chunk_path(cuda, k):
    """Power-law graph with hubs, tiny long-row threshold: every hub row is
    split into chunks folded by the last-arriving warp (deterministic)."""
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    n, u, v, w = G.chung_lu(20000, device="cuda")
    g = sp.Graph.from_canonical(n, u, v, w)
    L = sp.LaplacianOperator(g, "normalized", long_threshold=64, chunk_len=48)
    assert L.n_long_rows > 10 and L.n_chunks > L.n_long_rows
    csr = O.laplacian_csr(n, g.u, g.v, g.w, "normalized")
    x = np.random.default_rng(0).standard_normal((n, k)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    y1 = L.matvec(xd)
    y2 = L.matvec(xd)
    assert torch.equal(y1, y2)  # deterministic
    assert rel_fro(y1.cpu().numpy(), csr @ x.astype(np.float64)) <= PV_TOL
    t = sp.SpectralTransform("negexp-limit", 13)
    op = sp.TransformedOperator(L, t, 0.0, 2.0)
    ref = O.apply_transform(csr, "negexp-limit", 13, 1e-6, 0.0, x.astype(np.float64))
    assert rel_fro(op.apply(xd).cpu().numpy(), ref) <= PV_TOL


def test_matvec_reference_cases(cuda, golden):
    sp = _sp()
    L = sp.build_laplacian(sp.Graph.from_edges(2, [(0, 1)]))
    np.testing.assert_allclose(L.matvec(np.array([1.0, -1.0])), [2, -2])
    L = sp.build_laplacian(_graph(golden, "two_triangles_bridge"))
    np.testing.assert_allclose(L.matvec(np.ones(6)), 0, atol=1e-6)
    with pytest.raises(ValueError, match="dimension"):
        L.matvec(np.ones(5))
    g = sp.Graph.from_edges(3, [])
    np.testing.assert_allclose(sp.build_laplacian(g).matvec(np.ones(3)), 0)
    op = sp.make_reversed_operator(_graph(golden, "k3"), sp.SpectralTransform("identity"))
    with pytest.raises(ValueError, match="dimension"):
        op.apply(np.ones(4))
    op0 = sp.make_reversed_operator(_graph(golden, "k3"), sp.SpectralTransform("negexp-taylor", 0))
    v = np.random.default_rng(1).standard_normal(3)
    np.testing.assert_allclose(op0.apply(v), op0.lambda_star * v + v, atol=1e-6)


def test_exact_kinds_dense_oracle(cuda, golden):
    sp = _sp()
    g = _graph(golden, "k3")
    op = sp.make_reversed_operator(g, sp.SpectralTransform("negexp-limit", 251))
    dense = sp.exact_transform_dense(sp.SpectralTransform("negexp"), sp.dense_laplacian(g))
    v = np.random.default_rng(0).standard_normal(3)
    want = -dense @ v
    assert np.linalg.norm(op.apply(v) - want) / np.linalg.norm(want) <= 1e-2
    lap = sp.build_laplacian(g)
    op2 = sp.TransformedOperator(lap, sp.SpectralTransform("negexp"), 0.0, 4.0, None)
    with pytest.raises(ValueError, match="dense"):
        op2.apply(np.ones(3))


# --- full BASELINE sizes: size-independent properties ------------------------------------

@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_full_size_properties(cuda, cfg):
    """At BASELINE sizes (n = 1e6 / 1e7 / 2e6): exact-row parity on a random
    row sample (oracle SpMM restricted to the sampled rows, fp64), linearity
    of p(L), symmetry <y, Lx> = <Ly, x>, L 1 = 0 (combinatorial), and
    run-to-run determinism."""
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    spec = G.CONFIGS[cfg]
    n, u, v, w = G.config_graph(cfg, device="cuda")
    g = sp.Graph.from_canonical(n, u, v, w)
    mode, k, ell = spec["mode"], spec["k"], spec["ell"]
    L = sp.LaplacianOperator(g, mode)
    gen = torch.Generator(device="cuda").manual_seed(cfg)
    X = torch.randn((n, k), device="cuda", generator=gen)
    Y = torch.randn((n, k), device="cuda", generator=gen)
    LX = L.matvec(X)
    # row-sample parity against the oracle (fp64 on host)
    indptr, indices, data = L.csr_host()
    rows = np.sort(np.random.default_rng(cfg).choice(n, 2000, replace=False))
    Xh = X.cpu().numpy().astype(np.float64)
    ref_rows = np.stack([data[indptr[r]:indptr[r + 1]].astype(np.float64)
                         @ Xh[indices[indptr[r]:indptr[r + 1]]] for r in rows])
    assert rel_fro(LX[rows].cpu().numpy(), ref_rows) <= PV_TOL
    # symmetry
    a = float((Y.double() * LX.double()).sum())
    b = float((L.matvec(Y).double() * X.double()).sum())
    assert abs(a - b) <= 1e-4 * max(abs(a), 1.0)
    if mode == "unnormalized":
        ones = torch.ones((n, k), device="cuda")
        assert float(L.matvec(ones).abs().max()) <= 1e-3
    # linearity of the full polynomial
    t = sp.SpectralTransform("negexp-limit", ell + 1)
    op = sp.TransformedOperator(L, t, 0.0, 2.0)
    pX, pY = op.apply(X), op.apply(Y)
    pZ = op.apply(2.0 * X - 0.5 * Y)
    assert rel_fro(pZ.cpu().numpy(), (2.0 * pX - 0.5 * pY).cpu().numpy()) <= 1e-5
    assert torch.equal(op.apply(X), pX)


# --- degree-ordered (relabelled) operators ---------------------------------------------

@pytest.mark.parametrize("k", [4, 16, 32, 64, 128, 10])
def test_relabelled_operator_matches_oracle(cuda, k):
    """The degree-descending relabelling is internal: matvec/apply in the
    original order equal the oracle's, with hubs chunked and segments active."""
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    n, u, v, w = G.chung_lu(30000, device="cuda")
    g = sp.Graph.from_canonical(n, u, v, w)
    L = sp.LaplacianOperator(g, "normalized", reorder="degree", long_threshold=256, chunk_len=128)
    assert L.reordered and L.n_chunks > 0
    nseg, _ = L.segments(k)
    assert nseg >= 1
    csr = O.laplacian_csr(n, g.u, g.v, g.w, "normalized")
    x = np.random.default_rng(k).standard_normal((n, k)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    assert rel_fro(L.matvec(xd).cpu().numpy(), csr @ x.astype(np.float64)) <= PV_TOL
    # internal order round trip
    assert torch.equal(L.from_internal(L.to_internal(xd)), xd)
    t = sp.SpectralTransform("negexp-taylor", 12)
    op = sp.TransformedOperator(L, t, 0.0, 2.0)
    ref = O.apply_transform(csr, "negexp-taylor", 12, 1e-6, 0.0, x.astype(np.float64))
    assert rel_fro(op.apply(xd).cpu().numpy(), ref) <= PV_TOL
    yi = op.apply_internal(L.to_internal(xd))
    assert rel_fro(L.from_internal(yi).cpu().numpy(), ref) <= PV_TOL


def test_relabelled_csr_host_is_original_order(cuda, golden):
    sp = _sp()
    g = _graph(golden, "cfg4s")
    L = sp.LaplacianOperator(g, "normalized", reorder="degree")
    indptr, indices, data = L.csr_host()
    np.testing.assert_array_equal(indptr, golden["csr/cfg4s/normalized/indptr"])
    np.testing.assert_array_equal(indices, golden["csr/cfg4s/normalized/indices"])
    assert np.array_equal(data, golden["csr/cfg4s/normalized/data"].astype(np.float32))


def test_relabelled_stochastic_oracle_matches_unrelabelled(cuda):
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    n, u, v, w = G.chung_lu(20000, device="cuda")
    g = sp.Graph.from_canonical(n, u, v, w)
    t = sp.SpectralTransform("negexp-limit", 5)
    x = torch.randn((n, 16), device="cuda")
    outs = []
    for reorder in (None, "degree"):
        L = sp.LaplacianOperator(g, "normalized", reorder=reorder)
        op = sp.TransformedOperator(L, t, 0.0, 2.0)
        oracle = sp.make_stochastic_oracle(op, 20000, seed=9, estimator="edge-batch")
        outs.append(oracle(x).cpu().numpy())
    assert rel_fro(outs[1], outs[0]) <= PV_TOL


@pytest.mark.parametrize("k", [4, 32, 64, 128, 10])
def test_scaled_normalized_path(cuda, k, monkeypatch):
    """Unit-weight normalized Laplacians run terms after the first on
    u = D^-1/2 w without the values stream (row_scale set): every kind
    matches the oracle, and the stored-values path (SPED_SCALED_NORM=0) to
    fp32 rounding.  k = 10 (generic kernel) silently keeps stored values."""
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    n, u, v, w = G.chung_lu(30000, device="cuda")
    g = sp.Graph.from_canonical(n, u, v, w)
    L = sp.LaplacianOperator(g, "normalized", long_threshold=256, chunk_len=128)
    assert L.row_scale is not None and L.reordered and L.n_chunks > 0
    monkeypatch.setenv("SPED_SCALED_NORM", "0")
    L0 = sp.LaplacianOperator(g, "normalized", long_threshold=256, chunk_len=128)
    assert L0.row_scale is None
    csr = O.laplacian_csr(n, g.u, g.v, g.w, "normalized")
    x = np.random.default_rng(k).standard_normal((n, k)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    for kind, ell in (("negexp-taylor", 12), ("negexp-limit", 9), ("log-taylor", 7),
                      ("identity", None)):
        t = sp.SpectralTransform(kind, ell, 0.5 if kind == "log-taylor" else 1e-6)
        ref = O.apply_transform(csr, kind, ell, t.epsilon, 0.0, x.astype(np.float64))
        y = sp.TransformedOperator(L, t, 0.0, 2.0).apply(xd)
        y0 = sp.TransformedOperator(L0, t, 0.0, 2.0).apply(xd)
        assert rel_fro(y.cpu().numpy(), ref) <= PV_TOL, kind
        assert rel_fro(y.cpu().numpy(), y0.cpu().numpy()) <= 2e-6, kind
    # weighted graphs keep the stored values
    wg = sp.Graph(n, g.u, g.v, np.full(g.m, 2.0))
    assert sp.LaplacianOperator(wg, "normalized").row_scale is None


def test_device_canonicalisation_matches_host(cuda):
    """Graph(n, u, v, w) canonicalises on the device (sped_canonicalize_edges)
    and returns the reference's canonical edge list (the oracle restatement of
    graph.py:64-88) bit for bit -- orientation, lexsort, dropped zero weights
    -- for host arrays, CUDA tensors and device=, and raises the same
    ValueErrors in the same order of precedence."""
    import torch
    import paper_2207_14589_b200 as sp
    rng = np.random.default_rng(7)
    for n, m in ((1, 0), (5, 4), (1000, 20000), (300_000, 2_000_000)):
        a = rng.integers(0, n, m)
        b = rng.integers(0, n, m)
        keep = a != b
        a, b = a[keep], b[keep]
        key = np.unique(np.minimum(a, b) * n + np.maximum(a, b))
        lo, hi = key // n, key % n
        perm = rng.permutation(lo.size)
        flip = rng.random(lo.size) < 0.5
        u = np.where(flip, hi, lo)[perm]
        v = np.where(flip, lo, hi)[perm]
        w = rng.uniform(0.0, 2.0, lo.size)
        w[rng.random(lo.size) < 0.05] = 0.0  # dropped, as in the reference
        ru, rv, rw = O.canonical_edges(n, u, v, w)
        for g in (sp.Graph(n, u, v, w), sp.Graph(n, u, v, w, device="cuda"),
                  sp.Graph(n, torch.as_tensor(u, device="cuda"), torch.as_tensor(v, device="cuda"),
                           torch.as_tensor(w, device="cuda"))):
            assert g.m == ru.size
            assert np.array_equal(g.u, ru) and np.array_equal(g.v, rv) and np.array_equal(g.w, rw)
            assert g.u.dtype == np.int64
    cases = [  # (u, v, w, message) -- precedence as in the reference
        ([0, 1], [1, 2], [1.0, -1.0], "nonnegative"),
        ([0, 2, 1], [0, 9, 2], [1.0, 1.0, -0.5], "nonnegative"),
        ([0, 2], [0, 9], [1.0, 1.0], "self-loops"),
        ([0, 2], [1, 9], [1.0, 1.0], "out of range"),
        ([0, 1, 2], [1, 0, 3], [1.0, 2.0, 1.0], "duplicate"),
        ([3, 3], [3, 3], [0.0, 0.0], None),  # zero-weight self loops are dropped first
    ]
    for u, v, w, msg in cases:
        if msg is None:
            assert O.canonical_edges(5, u, v, w)[0].size == 0
        else:
            with pytest.raises(ValueError, match=msg):
                O.canonical_edges(5, u, v, w)
        for kw in ({}, {"device": "cuda"}):
            if msg is None:
                assert sp.Graph(5, u, v, w, **kw).m == 0
            else:
                with pytest.raises(ValueError, match=msg):
                    sp.Graph(5, u, v, w, **kw)


def test_operator_shared_across_threads(cuda):
    """The reference's operators are immutable and safe to share across
    threads (transforms.py:207-208): two host threads applying one
    relabelled operator (hub chunks in play) on their own streams get the
    single-thread result bit for bit."""
    import threading
    import torch
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200 import generators as G
    n, u, v, w = G.chung_lu(200_000, cap=20000.0, device="cuda")
    g = sp.Graph.from_canonical(n, u, v, w)
    L = sp.LaplacianOperator(g, "normalized", long_threshold=256, chunk_len=128)
    assert L.n_chunks > 0
    op = sp.TransformedOperator(L, sp.SpectralTransform("negexp-limit", 9), 0.0, 2.0)
    xs = [torch.randn((n, 32), device="cuda", generator=torch.Generator(device="cuda").manual_seed(s))
          for s in (1, 2)]
    ref = [op.apply_internal(x) for x in xs]
    torch.cuda.synchronize()
    got = [None, None]

    def work(i):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(20):
                y = op.apply_internal(xs[i])
            s.synchronize()
            got[i] = y
    ts = [threading.Thread(target=work, args=(i,)) for i in (0, 1)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i in (0, 1):
        assert torch.equal(got[i], ref[i])


def test_mu_eg_step_concurrent_threads(cuda):
    """The reference's step functions are pure: two host threads running
    mu_eg_step on the SAME (default) stream with their own states get the
    single-thread results bit for bit -- each thread has its own step
    workspace (Gram, coefficients, collapse flag)."""
    import threading
    import torch
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200 import generators as G
    n, u, v, w = G.lp_sbm(20000, 20, 24.0, 0.1, 5, 0.8, device="cuda")
    g = sp.Graph.from_canonical(n, u, v, w)
    op = sp.make_reversed_operator(g, sp.SpectralTransform("negexp-limit", 5), device="cuda")
    V0 = [sp.init_state(n, 32, s).V for s in (1, 2)]

    def run(V):
        st = sp.EigenState(V)
        for _ in range(10):
            st = sp.mu_eg_step(st, op, 0.1)
        return st.V

    ref = [run(V) for V in V0]
    torch.cuda.synchronize()
    got = [None, None]

    def work(i):
        got[i] = run(V0[i])
        torch.cuda.synchronize()
    ts = [threading.Thread(target=work, args=(i,)) for i in (0, 1)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for i in (0, 1):
        assert torch.equal(got[i], ref[i])


def test_bench_sped_arm_contract(cuda):
    """`bench.py` (default arm, scaled-down graph) prints one JSON line with
    the driver's keys plus roofline / cpu_baseline / e2e / gpu_launches /
    clocks, and W >= 3 warm-up steps."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--scale", "0.02", "--steps", "3",
                        "--warmup", "3", "--no-extra"],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 3
    rf = d["roofline"]
    assert rf["bound"] in ("hbm", "tensor") and 0 < rf["frac"] < 1.5 and rf["peak"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and d["cpu_baseline"]["cores"] >= 1
    assert "workload" in d["config"]


def test_debug_checks_detect_bad_column(cuda):
    """The debug-check build (SPED_LIB=... built with -DSPED_DEBUG_CHECKS=1)
    flags a gather outside the input block (bit 1) instead of reading
    silently; the release build compiles the checks away."""
    from paper_2207_14589_b200 import _lib
    lib = _lib.load()
    if int(lib.sped_debug_checks()) != 1:
        pytest.skip("release build (checks compiled out)")
    lib.sped_debug_take()
    n, k = 4, 8
    indptr = torch.tensor([0, 1, 2, 3, 4], dtype=torch.int32, device="cuda")
    indices = torch.tensor([0, 1, 2, n], dtype=torch.int32, device="cuda")  # row 3 -> col n
    values = torch.ones(4, dtype=torch.float32, device="cuda")
    x = torch.zeros((2 * n, k), device="cuda")   # room behind row n: the bad read stays in bounds
    out = torch.empty((n, k), device="cuda")
    rc = lib.sped_csr_poly_apply(n, k, _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(values),
                                 1 << 30, 1, None, 0, None, None, None, 0, 0, None,
                                 _lib.ptr(x), None, None, None, _lib.ptr(out), 1,
                                 _lib.dbl_array([0.0]), _lib.dbl_array([1.0]),
                                 _lib.dbl_array([0.0]), 1.0, 0.0, 1.0, _lib.stream_ptr(cuda))
    _lib.check(rc)
    assert int(lib.sped_debug_take()) & 1


def test_large_nk_int64_offsets(cuda):
    """n * k >= 2^31 (n = 1.7e7, k = 128: 2.2e9 floats per block): every row
    offset and gather address is 64-bit (the round-1 int32 overflow of
    ADVICE/VERDICT).  A power-law graph so hub chunks, warp rows and short
    rows all run; exact rows against the oracle on a sample that includes
    the last rows, whose offsets exceed 2^31."""
    sp = _sp()
    from paper_2207_14589_b200 import generators as G
    n, k = 17_000_000, 128
    assert n * k >= 2 ** 31
    nn, u, v, w = G.chung_lu(n, 2.1, 2.0, 4.0, 1e4, device="cuda")
    g = sp.Graph.from_canonical(nn, u, v, w)
    L = sp.LaplacianOperator(g, "unnormalized", implicit=False)
    del u, v, w
    assert L.reordered and L.n_chunks > 0
    X = torch.empty((nn, k), device="cuda").uniform_(-1, 1)
    Y = L.poly_apply_internal(X, [0.0], [1.0], [0.0], 1.0, 0.0, 1.0)
    indptr = L.indptr.cpu().numpy().astype(np.int64)
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([rng.choice(nn, 400, replace=False),
                                     np.arange(nn - 50, nn), np.arange(0, 20)]))
    got = Y[torch.as_tensor(rows, device="cuda")].double().cpu().numpy()
    ref = []
    for r in rows:
        p0, p1 = int(indptr[r]), int(indptr[r + 1])
        cols = L.indices[p0:p1].long()
        vals = L.values[p0:p1].double()
        ref.append((vals[:, None] * X[cols].double()).sum(0).cpu().numpy())
    assert rel_fro(got, np.stack(ref)) <= PV_TOL
