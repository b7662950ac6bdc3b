"""Walk-based polynomial estimator (csrc/walks.cu) vs the reference's
estimates (goldens) and the oracle restatement: the device replays numpy's
Philox draws, so the walks are the reference's and the fp64 estimates agree
to rounding."""

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

TOL = dict(rtol=1e-10, atol=1e-12)


def _graph(golden, name):
    import paper_2207_14589_b200 as sp
    n, u, v, w = golden.graph(name)
    return sp.Graph(n, u, v, w)


def test_walk_estimates_vs_reference(cuda, golden):
    import paper_2207_14589_b200 as sp
    checked = 0
    for key in golden.keys("walk/"):
        if not key.endswith("/y"):
            continue
        base = key[:-2]
        name, seed = base.split("/")[1], int(base.split("/")[2])
        g = _graph(golden, name)
        coeffs = golden[base + "/coeffs"]
        W = int(golden[base + "/walks"])
        x = golden[base + "/x"]
        ell = coeffs.size - 1
        y = sp.estimate_polynomial_matvec(g, coeffs, x, sp.SamplerConfig(ell, W, 1, "importance", seed))
        np.testing.assert_allclose(y, golden[key], **TOL, err_msg=base)
        yr = sp.estimate_power_matvec(g, ell, x, sp.SamplerConfig(ell, W, 4, "rejection", seed))
        np.testing.assert_allclose(yr, golden[base + "/rejection"], **TOL, err_msg=base)
        # device in, device out; deterministic
        xd = torch.as_tensor(x, device="cuda")
        cfg = sp.SamplerConfig(ell, W, 1, "importance", seed)
        y1 = sp.estimate_polynomial_matvec(g, coeffs, xd, cfg)
        y2 = sp.estimate_polynomial_matvec(g, coeffs, xd, cfg)
        assert y1.is_cuda and torch.equal(y1, y2)
        checked += 1
    assert checked >= 5


def test_walk_oracle_vs_reference(cuda, golden):
    """make_stochastic_oracle(..., estimator='walk') reproduces the
    reference's walk oracle call by call (per-column seeds, counter state)."""
    import paper_2207_14589_b200 as sp
    for key in golden.keys("walkorc/"):
        if not key.endswith("/y0"):
            continue
        base = key[:-3]
        _, name, kind, ell, B, seed = base.split("/")
        g = _graph(golden, name)
        op = sp.make_reversed_operator(g, sp.SpectralTransform(kind, int(ell)))
        assert abs(op.lambda_star - float(golden[base + "/lambda_star"])) <= 1e-12
        orc = sp.make_stochastic_oracle(op, int(B), seed=int(seed), estimator="walk")
        X = golden[base + "/x"]
        np.testing.assert_allclose(orc(X), golden[base + "/y0"], **TOL)
        np.testing.assert_allclose(orc(X), golden[base + "/y1"], **TOL)
        # the reference's own signature: sampler=SamplerConfig(...)
        cfg = sp.SamplerConfig(int(ell), int(B))
        orc2 = sp.make_stochastic_oracle(op, int(B), seed=int(seed), sampler=cfg)
        np.testing.assert_allclose(orc2(X), golden[base + "/y0"], **TOL)
        # and the reference's default call (no sampler, no estimator) is the
        # walk oracle too, as in solvers.py:181-202
        orc3 = sp.make_stochastic_oracle(op, int(B), seed=int(seed))
        np.testing.assert_allclose(orc3(X), golden[base + "/y0"], **TOL)
        np.testing.assert_allclose(orc3(X), golden[base + "/y1"], **TOL)


@pytest.mark.parametrize("graph", ["sbm1k", "chunglu"])
def test_walk_estimates_vs_oracle_larger(cuda, graph):
    """Larger graphs (SBM 10x100; a power-law graph whose hub incidence lists
    exercise the two-list selection) against the CPU restatement."""
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200 import generators as G
    if graph == "sbm1k":
        n, u, v, w = G.config_graph(1)
    else:
        n, u, v, w = G.chung_lu(3000)
    g = sp.Graph(n, u.numpy(), v.numpy(), w.numpy())
    coeffs = np.array([0.3, -0.2, 0.05, -0.01])
    x = np.random.default_rng(1).standard_normal(n)
    W = 20000
    y = sp.estimate_polynomial_matvec(g, coeffs, x, sp.SamplerConfig(3, W, 1, "importance", 17))
    ref = O.walk_estimate(n, g.u, g.v, g.w, coeffs, x, W, 17)
    np.testing.assert_allclose(y, ref, **TOL)


# --- device mirrors of the reference's walk-estimator tests
# (specgap tests/test_walks.py:157-252) --------------------------------------

def _small(name):
    import paper_2207_14589_b200 as sp
    edges = {"path2": (2, [(0, 1)]), "path3": (3, [(0, 1), (1, 2)]),
             "star4": (4, [(0, 1), (0, 2), (0, 3)]),
             "bridge": (6, [(0, 1), (0, 2), (1, 2), (3, 4), (3, 5), (4, 5), (2, 3)])}[name]
    return sp.Graph.from_edges(*edges)


def test_walk_power_estimate_exact_on_single_edge(cuda):
    import paper_2207_14589_b200 as sp
    cfg = sp.SamplerConfig(ell=2, walks_per_estimate=1, seed=0)
    np.testing.assert_allclose(sp.estimate_power_matvec(_small("path2"), 2,
                                                        np.array([1.0, -1.0]), cfg), [4.0, -4.0])


def test_walk_power_estimate_unbiased(cuda):
    import paper_2207_14589_b200 as sp
    g = _small("path3")
    v = np.array([0.5, -1.0, 2.0])
    exact = np.linalg.matrix_power(sp.dense_laplacian(g), 2) @ v
    means = np.array([sp.estimate_power_matvec(g, 2, v, sp.SamplerConfig(2, 4000, seed=100 + b))
                      for b in range(30)])
    se = means.std(axis=0, ddof=1) / np.sqrt(30)
    assert np.all(np.abs(means.mean(axis=0) - exact) <= 3 * se)


def test_walk_rejection_errors_and_validation(cuda):
    import paper_2207_14589_b200 as sp
    with pytest.raises(RuntimeError, match="importance"):
        sp.estimate_power_matvec(_small("star4"), 8, np.ones(4),
                                 sp.SamplerConfig(8, 4, mode="rejection", seed=12))
    cfg = sp.SamplerConfig(2, 10, seed=0)
    with pytest.raises(ValueError):
        sp.estimate_power_matvec(_small("path3"), 0, np.ones(3), cfg)
    with pytest.raises(ValueError):
        sp.estimate_power_matvec(_small("path3"), 2, np.ones(4), cfg)
    with pytest.raises(ValueError, match="importance"):
        sp.estimate_polynomial_matvec(_small("path3"), [0.0, 0.0, 1.0], np.ones(3),
                                      sp.SamplerConfig(2, 10, mode="rejection", seed=0))


def test_walk_reproducibility_and_walker_count(cuda):
    import paper_2207_14589_b200 as sp
    g = _small("bridge")
    v = np.random.default_rng(10).standard_normal(6)
    a = sp.estimate_power_matvec(g, 3, v, sp.SamplerConfig(3, 30000, n_walkers=1, seed=13))
    b = sp.estimate_power_matvec(g, 3, v, sp.SamplerConfig(3, 30000, n_walkers=5, seed=13))
    np.testing.assert_array_equal(a, b)
    c = sp.estimate_power_matvec(g, 3, v, sp.SamplerConfig(3, 30000, n_walkers=1, seed=13))
    np.testing.assert_array_equal(a, c)


def test_walk_polynomial_exact_cases(cuda):
    import paper_2207_14589_b200 as sp
    p3 = _small("path3")
    v = np.array([3.0, 1.0, -2.0])
    out = sp.estimate_polynomial_matvec(p3, [1.0, 0.0, 0.0, 0.0], v, sp.SamplerConfig(3, 10, seed=0))
    np.testing.assert_array_equal(out, v)
    p2 = _small("path2")
    t = sp.SpectralTransform("negexp-limit", 3)
    coeffs = sp.polynomial_coefficients(t)
    v2 = np.array([0.7, -0.2])
    est = sp.estimate_polynomial_matvec(p2, coeffs, v2, sp.SamplerConfig(3, 1, seed=5))
    dense = sp.exact_transform_dense(t, sp.dense_laplacian(p2))
    np.testing.assert_allclose(est, dense @ v2, atol=1e-12)
