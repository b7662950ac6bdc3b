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
