"""Pin the CPU oracle restatement (oracle/) to the reference's own outputs.

The golden vectors were produced by running the reference ``specgap`` package
(tests/golden/make_golden.py).  Every check here is CPU-only.
"""

import numpy as np
import pytest

import oracle as O
from conftest import rel_fro


def _graph(golden, name):
    n, u, v, w = golden.graph(name)
    return n, *O.canonical_edges(n, u, v, w)


def test_canonical_edges_match_reference(golden):
    for name in golden.graph_names():
        n, u, v, w = golden.graph(name)
        # shuffle + flip orientation; the restated canonicalisation must
        # recover the reference's order exactly
        rng = np.random.default_rng(len(name))
        p = rng.permutation(u.size)
        flip = rng.random(u.size) < 0.5
        uu = np.where(flip, v, u)[p]
        vv = np.where(flip, u, v)[p]
        lo, hi, ww = O.canonical_edges(n, uu, vv, w[p])
        np.testing.assert_array_equal(lo, u)
        np.testing.assert_array_equal(hi, v)
        np.testing.assert_array_equal(ww, w)


def test_degrees_bit_exact(golden):
    for name in golden.graph_names():
        n, u, v, w = _graph(golden, name)
        np.testing.assert_array_equal(O.degrees(n, u, v, w), golden[f"g/{name}/degrees"])


@pytest.mark.parametrize("mode", ["unnormalized", "normalized"])
def test_csr_bit_exact(golden, mode):
    checked = 0
    for name in golden.graph_names():
        key = f"csr/{name}/{mode}"
        n, u, v, w = _graph(golden, name)
        if f"{key}/error" in golden:
            with pytest.raises(ValueError, match="degrees"):
                O.laplacian_csr(n, u, v, w, mode)
            continue
        if f"{key}/indptr" not in golden:
            continue
        c = O.laplacian_csr(n, u, v, w, mode)
        np.testing.assert_array_equal(c.indptr, golden[f"{key}/indptr"])
        np.testing.assert_array_equal(c.indices, golden[f"{key}/indices"])
        ref = golden[f"{key}/data"]
        np.testing.assert_array_equal(c.data.astype(ref.dtype), ref)
        checked += 1
    assert checked >= 10


def test_apply_matches_reference(golden):
    keys = golden.keys("apply/")
    cases = sorted({k.rsplit("/", 1)[0] for k in keys})
    assert len(cases) > 50
    for case in cases:
        _, name, mode, kind, ell, eps, k = case.split("/")
        ell = None if ell == "None" else int(ell)
        eps = float(eps)
        n, u, v, w = _graph(golden, name)
        csr = O.laplacian_csr(n, u, v, w, mode)
        lam = O.choose_lambda_star(kind, O.lambda_upper(n, u, v, w, mode), eps)
        assert lam == pytest.approx(float(golden[case + "/lambda_star"]), rel=0, abs=0)
        x = golden[case + "/x"].astype(np.float64)
        y = O.apply_transform(csr, kind, ell, eps, lam, x)
        ref = golden[case + "/y"]
        tol = 1e-12 if ref.dtype == np.float64 else 2e-7
        assert rel_fro(y, ref) <= tol, case


def test_term_schedule_reproduces_apply(golden):
    """The (alpha, beta, gamma) schedule the CUDA kernels run is the same
    recurrence as transforms.py:241-262 (checked in fp64 with scipy)."""
    for case in sorted({k.rsplit("/", 1)[0] for k in golden.keys("apply/")}):
        _, name, mode, kind, ell, eps, k = case.split("/")
        ell = None if ell == "None" else int(ell)
        eps = float(eps)
        n, u, v, w = _graph(golden, name)
        csr = O.laplacian_csr(n, u, v, w, mode)
        lam = float(golden[case + "/lambda_star"])
        x = golden[case + "/x"].astype(np.float64)
        al, be, ga, w0, lf, s = O.term_schedule(kind, ell, eps, lam)
        cur = w0 * x
        for t in range(len(al)):
            cur = al[t] * x + be[t] * (csr @ cur) + ga[t] * cur
        y = lf * x + s * cur
        ref = golden[case + "/y"]
        tol = 1e-10 if ref.dtype == np.float64 else 2e-7
        assert rel_fro(y, ref) <= tol, case


def test_solver_steps_match_reference(golden):
    for key in golden.keys("step/"):
        if not key.endswith("/V0"):
            continue
        base = key[: -len("/V0")]
        _, name, mode, kind, ell, k = base.split("/")
        ell = None if ell == "None" else int(ell)
        n, u, v, w = _graph(golden, name)
        csr = O.laplacian_csr(n, u, v, w, mode)
        lam = O.choose_lambda_star(kind, O.lambda_upper(n, u, v, w, mode))
        V0 = golden[key]
        MV = O.apply_transform(csr, kind, ell, 1e-6, lam, V0)
        for eta in (0.05, 0.5):
            np.testing.assert_allclose(O.mu_eg_step(V0, MV, eta), golden[f"{base}/mueg/{eta}"],
                                       rtol=0, atol=1e-12)
            np.testing.assert_allclose(O.oja_step(V0, MV, eta), golden[f"{base}/oja/{eta}"],
                                       rtol=0, atol=1e-12)


def test_init_state_matches_reference(golden):
    for key in golden.keys("init/"):
        _, n, k, seed = key.split("/")
        np.testing.assert_array_equal(O.init_state(int(n), int(k), int(seed)), golden[key])


def test_identity_minibatch_oracle_bit_exact(golden):
    cases = sorted({k.rsplit("/", 1)[0] for k in golden.keys("sto/")})
    for case in cases:
        _, name, B, seed = case.split("/")
        n, u, v, w = _graph(golden, name)
        lam = O.choose_lambda_star("identity", O.lambda_upper(n, u, v, w))
        rng = np.random.default_rng(int(seed))
        x = golden[case + "/x"]
        for call in range(3):
            batch = rng.integers(0, u.size, size=int(B))
            np.testing.assert_array_equal(batch, golden[f"{case}/batch{call}"])
            y = O.identity_minibatch_apply(u, v, w, lam, batch, x)
            np.testing.assert_array_equal(y, golden[f"{case}/y{call}"])


def test_edge_batch_poly_identity_reduces_to_reference(golden):
    case = "sto/two_triangles_bridge/4/2"
    n, u, v, w = _graph(golden, "two_triangles_bridge")
    lam = O.choose_lambda_star("identity", O.lambda_upper(n, u, v, w))
    rng = np.random.default_rng(2)
    x = golden[case + "/x"]
    batches = O.draw_batches(rng, u.size, 4, 1)
    y = O.edge_batch_poly_apply(u, v, w, "identity", None, 1e-6, lam, batches, x)
    np.testing.assert_array_equal(y, golden[case + "/y0"])


def test_edge_batch_poly_unbiased():
    """Restated per-term composition is unbiased (Monte Carlo, 3.5 s.e.),
    modelled on tests/test_solvers.py:155-162 of the reference."""
    n = 6
    u, v, w = O.canonical_edges(n, np.array([0, 0, 1, 3, 3, 4, 2]),
                                np.array([1, 2, 2, 4, 5, 5, 3]),
                                np.array([1.0, 2.0, 0.5, 1.0, 1.5, 1.0, 0.7]))
    csr = O.laplacian_csr(n, u, v, w)
    x = np.array([0.3, -0.7, 1.1, 0.2, -0.4, 0.9])
    for kind, ell in (("negexp-limit", 3), ("negexp-taylor", 2), ("log-taylor", 2)):
        eps = 0.5 if kind == "log-taylor" else 1e-6
        exact = O.apply_transform(csr, kind, ell, eps, 0.0, x)
        rng = np.random.default_rng(5)
        draws = np.array([O.edge_batch_poly_apply(u, v, w, kind, ell, eps, 0.0,
                                                  O.draw_batches(rng, u.size, 3, ell), x)
                          for _ in range(20000)])
        se = draws.std(axis=0, ddof=1) / np.sqrt(draws.shape[0])
        assert np.all(np.abs(draws.mean(axis=0) - exact) <= 3.5 * se + 1e-12), kind


def test_pcg64_restatement_bit_exact(golden):
    cases = sorted({k.rsplit("/", 1)[0] for k in golden.keys("pcg/")})
    assert cases
    for case in cases:
        _, m, seed = case.split("/")
        st = golden.state(case + "/state0")
        i = 0
        while f"{case}/draw{i}" in golden:
            ref = golden[f"{case}/draw{i}"]
            vals, st, _ = O.pcg64_integers(st, int(m), ref.size)
            np.testing.assert_array_equal(vals, ref)
            assert st["state"] == golden.state(f"{case}/state{i + 1}")["state"]
            assert st["has_uint32"] == golden.state(f"{case}/state{i + 1}")["has_uint32"]
            i += 1


def test_kmeans_matches_reference(golden):
    np.testing.assert_array_equal(O.kmeans_cluster(golden["kmeans/X"], 3, seed=1),
                                  golden["kmeans/labels"])


def test_oracle_versions_recorded():
    v = O.versions()
    assert "numpy" in v and "scipy" in v


@pytest.mark.parametrize("mode", ["unnormalized", "normalized"])
def test_row_sample_csr_equals_full_rows(golden, mode):
    """The bench's bounded CPU sample builds rows [r0, r1) only; they equal
    the corresponding rows of the full restated CSR."""
    for name in ("cfg4s", "cfg5s", "er_dense_w"):
        n, u, v, w = _graph(golden, name)
        full = O.laplacian_csr(n, u, v, w, mode)
        for r0, r1 in ((0, n // 3), (n // 3, n)):
            part = O.laplacian_csr_rows(n, u, v, w, mode, r0, r1)
            ref = full[r0:r1]
            np.testing.assert_array_equal(part.indptr, ref.indptr)
            np.testing.assert_array_equal(part.indices, ref.indices)
            np.testing.assert_array_equal(part.data.astype(np.float32), ref.data.astype(np.float32))


# --- walk-based estimator (walks.py) --------------------------------------------------

def test_walk_estimator_oracle_vs_reference(golden):
    """The restated walk sampler reproduces the reference's walks (chunk-0
    edge sequences and log-probabilities bit for bit) and its importance /
    rejection estimates."""
    for key in golden.keys("walk/"):
        if not key.endswith("/y"):
            continue
        base = key[:-2]
        name, seed = base.split("/")[1], int(base.split("/")[2])
        n, u, v, w = golden.graph(name)
        coeffs = golden[base + "/coeffs"]
        W = int(golden[base + "/walks"])
        x = golden[base + "/x"]
        inc = O.incidence_lists(n, u, v)
        ell = coeffs.size - 1
        rng = np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, 0))))
        E, lp = O.walk_sample_chunk(inc, u.size, ell, min(8192, W), rng)
        assert np.array_equal(E[:256], golden[base + "/E0"]), base
        assert np.array_equal(lp[:256], golden[base + "/logp0"]), base
        y = O.walk_estimate(n, u, v, w, coeffs, x, W, seed, inc=inc)
        np.testing.assert_allclose(y, golden[key], rtol=1e-12, atol=1e-12)
        e = np.zeros_like(coeffs)
        e[-1] = 1.0
        yr = O.walk_estimate(n, u, v, w, e, x, W, seed, mode="rejection", inc=inc)
        np.testing.assert_allclose(yr, golden[base + "/rejection"], rtol=1e-12, atol=1e-12)


def test_walk_oracle_composition_vs_reference(golden):
    """make_stochastic_oracle's walk oracle (solvers.py:183-200): per-column
    call seeds from SeedSequence((seed, counter)), counter carried across
    calls."""
    for key in golden.keys("walkorc/"):
        if not key.endswith("/y0"):
            continue
        base = key[:-3]
        _, name, kind, ell, B, seed = base.split("/")
        n, u, v, w = golden.graph(name)
        coeffs = O.polynomial_coefficients(kind, int(ell))
        lam = float(golden[base + "/lambda_star"])
        X = golden[base + "/x"]
        y0, c = O.walk_oracle_apply(n, u, v, w, coeffs, lam, X, int(B), int(seed), 0)
        y1, _ = O.walk_oracle_apply(n, u, v, w, coeffs, lam, X, int(B), int(seed), c)
        np.testing.assert_allclose(y0, golden[base + "/y0"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(y1, golden[base + "/y1"], rtol=1e-12, atol=1e-12)
