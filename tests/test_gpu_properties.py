"""Property tests on random graphs (hypothesis, seeded numpy draws), modelled
on the reference's own (tests/test_graph.py:105-127, tests/test_solvers.py
:95-137): device CSR bit-exact vs the oracle's fp32 CSR, matvec / p(L)V vs
the fp64 oracle, Laplacian null vectors, and solver-step identities."""

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle as O
from conftest import rel_fro

pytestmark = pytest.mark.gpu

# derandomize: the same examples on every run and every box (a GPU-box run
# must not depend on a fresh random draw)
SETTINGS = settings(max_examples=40, deadline=None, derandomize=True, database=None,
                    suppress_health_check=[HealthCheck.function_scoped_fixture])


def _recurrence_bound(csr, kind, ell, epsilon, lam_star, x):
    """Norm of the same recurrence run on absolute values: what an fp32
    evaluation's rounding errors are proportional to.  When the true result
    is much smaller (cancellation between terms, e.g. log-taylor outside its
    radius of convergence or an edgeless graph), 1e-5 of the RESULT is below
    fp32 resolution and the error is judged against this instead."""
    al, be, ga, w0, lf, s = O.term_schedule(kind, ell, epsilon, lam_star)
    A = abs(csr)
    ax = np.abs(x)
    w = abs(w0) * ax
    for a_, b_, g_ in zip(al, be, ga):
        w = abs(a_) * ax + abs(b_) * (A @ w) + abs(g_) * w
    return float(np.linalg.norm(abs(lf) * ax + abs(s) * w))


def _random_graph(seed, n, p, weighted):
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, k=1)  # the reference rejects self loops
    keep = rng.random(iu.size) < p
    u, v = iu[keep], ju[keep]
    w = rng.uniform(0.1, 2.0, u.size) if weighted else np.ones(u.size)
    # fp32-representable weights, as SURVEY 8d prescribes for the parity inputs
    return n, u.astype(np.int64), v.astype(np.int64), w.astype(np.float32).astype(np.float64)


graphs = st.tuples(st.integers(0, 2**31 - 1), st.integers(2, 70), st.floats(0.03, 0.6),
                   st.booleans())


@SETTINGS
@given(gspec=graphs, mode=st.sampled_from(["unnormalized", "normalized"]),
       k=st.sampled_from([1, 3, 4, 8, 32]))
def test_random_graph_csr_and_matvec(cuda, gspec, mode, k):
    import paper_2207_14589_b200 as sp
    n, u, v, w = _random_graph(*gspec)
    g = sp.Graph(n, u, v, w)
    deg = np.bincount(g.u, g.w, n) + np.bincount(g.v, g.w, n)
    if mode == "normalized" and np.any(deg == 0):
        with pytest.raises(ValueError):
            sp.LaplacianOperator(g, mode)
        return
    L = sp.LaplacianOperator(g, mode)
    ref = O.laplacian_csr(n, g.u, g.v, g.w, mode)
    indptr, indices, data = L.csr_host()
    assert np.array_equal(indptr, ref.indptr) and np.array_equal(indices, ref.indices)
    assert np.array_equal(data, ref.data.astype(np.float32))
    x = np.random.default_rng(gspec[0] + 1).standard_normal((n, k))
    y = L.matvec(x)
    assert y.dtype == np.float64 and y.shape == (n, k)
    assert rel_fro(y, ref @ x) <= 1e-5
    # null vector: L 1 = 0 (combinatorial), L D^1/2 1 = 0 (normalized)
    z = np.ones(n) if mode == "unnormalized" else np.sqrt(deg)
    assert np.abs(L.matvec(z)).max() <= 1e-5 * max(1.0, np.abs(z).max() * deg.max())


@SETTINGS
@given(gspec=graphs, kind=st.sampled_from(["negexp-limit", "negexp-taylor", "log-taylor",
                                            "identity"]),
       ell=st.integers(1, 9), k=st.sampled_from([2, 4, 16]))
def test_random_graph_poly_apply(cuda, gspec, kind, ell, k):
    import paper_2207_14589_b200 as sp
    n, u, v, w = _random_graph(*gspec)
    if kind == "negexp-limit" and ell % 2 == 0:
        ell += 1
    g = sp.Graph(n, u, v, w)
    t = sp.SpectralTransform(kind, None if kind == "identity" else ell,
                             0.5 if kind == "log-taylor" else 1e-6)
    op = sp.make_reversed_operator(g, t)
    csr = O.laplacian_csr(n, g.u, g.v, g.w)
    x = np.random.default_rng(gspec[0] + 2).standard_normal((n, k))
    ref = O.apply_transform(csr, kind, t.ell, t.epsilon, op.lambda_star, x)
    y = op.apply(x)
    # north-star tolerance: 1e-5 relative Frobenius; under cancellation, 16
    # fp32 ulps of the absolute-value recurrence (the evaluation's own scale)
    err = float(np.linalg.norm(y - ref))
    bound = _recurrence_bound(csr, kind, t.ell, t.epsilon, op.lambda_star, x)
    assert err <= max(1e-5 * float(np.linalg.norm(ref)), 16 * 2.0 ** -24 * bound), \
        (err, float(np.linalg.norm(ref)), bound)


@SETTINGS
@given(gspec=graphs, k=st.integers(1, 5))
def test_mu_eg_zero_step_keeps_normalized_state(cuda, gspec, k):
    """eta = 0: mu-EG returns the column-normalized input (solvers.py:121-144),
    and the k = 1 case works (reference tests/test_solvers.py:118-137)."""
    import paper_2207_14589_b200 as sp
    n, u, v, w = _random_graph(*gspec)
    k = min(k, n)
    g = sp.Graph(n, u, v, w)
    op = sp.make_reversed_operator(g, sp.SpectralTransform("negexp-limit", 5))
    V0 = O.init_state(n, k, gspec[0] % 1000)
    st0 = sp.EigenState(V0, 0)
    st1 = sp.mu_eg_step(st0, op, 0.0)
    ref = O.mu_eg_step(V0, O.apply_transform(O.laplacian_csr(n, g.u, g.v, g.w), "negexp-limit", 5,
                                             1e-6, op.lambda_star, V0), 0.0)
    assert rel_fro(np.asarray(st1.V), ref) <= 1e-5
    assert rel_fro(np.asarray(st1.V), V0) <= 1e-5


def test_oja_fixed_point_on_true_eigenvectors(cuda, golden):
    """The top-k eigenvectors of the reversed operator are an Oja fixed point
    (reference tests/test_solvers.py:30-50): the span does not move."""
    import paper_2207_14589_b200 as sp
    n, u, v, w = golden.graph("cfg1")
    g = sp.Graph(n, u, v, w)
    gt = sp.graph_ground_truth(g)
    U = gt.bottom(6)
    op = sp.make_reversed_operator(g, sp.SpectralTransform("negexp-limit", 13))
    st1 = sp.oja_step(sp.EigenState(U, 0), op, 0.3)
    assert sp.principal_angles(np.asarray(st1.V), U) <= 1e-3
