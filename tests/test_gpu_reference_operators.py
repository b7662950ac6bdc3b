"""Device mirrors of the reference's operator tests that are on the hot path
(specgap tests/test_graph.py:59-127, tests/test_transforms.py:133-200):
matvec semantics and errors, quadratic form, empty graph, reversal."""

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


def _sp():
    import paper_2207_14589_b200 as sp
    return sp


def _k3(sp):
    return sp.Graph(3, [0, 0, 1], [1, 2, 2], [1.0, 1.0, 1.0])


def _dense(g, mode="unnormalized"):
    return O.laplacian_csr(g.n, g.u, g.v, g.w, mode).toarray()


def test_matvec_block_input_and_vector(cuda):
    """test_graph.py:70-84"""
    sp = _sp()
    g = _k3(sp)
    L = sp.build_laplacian(g)
    V = np.random.default_rng(1).standard_normal((3, 4))
    np.testing.assert_allclose(L.matvec(V), _dense(g) @ V, rtol=1e-6, atol=1e-6)
    x = np.array([1.0, -1.0, 0.5])
    y = L.matvec(x)
    assert y.shape == (3,)
    np.testing.assert_allclose(y, _dense(g) @ x, rtol=1e-6, atol=1e-6)


def test_matvec_dimension_mismatch(cuda):
    """test_graph.py:76-78, test_transforms.py:170-173"""
    sp = _sp()
    g = _k3(sp)
    with pytest.raises(ValueError, match="dimension"):
        sp.build_laplacian(g).matvec(np.ones(4))
    op = sp.make_reversed_operator(g, sp.SpectralTransform("identity"))
    with pytest.raises(ValueError, match="dimension"):
        op.apply(np.ones(4))


def test_empty_graph_zero_operator(cuda):
    """test_graph.py:87-89, 99-104"""
    sp = _sp()
    g = sp.Graph.from_edges(3, [])
    np.testing.assert_allclose(sp.build_laplacian(g).matvec(np.ones(3)), 0)
    with pytest.raises(ValueError, match="degree"):
        sp.build_laplacian(g, "normalized")


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_quadratic_form_matches_edge_sum(cuda, seed):
    """test_graph.py:107-117: x^T L x = sum_e w_e (x_u - x_v)^2"""
    sp = _sp()
    rng = np.random.default_rng(seed)
    n = int(rng.integers(5, 60))
    iu, ju = np.triu_indices(n, k=1)
    keep = rng.random(iu.size) < 0.3
    u, v = iu[keep], ju[keep]
    w = rng.uniform(0.1, 2.0, u.size).astype(np.float32).astype(np.float64)
    g = sp.Graph(n, u, v, w)
    x = rng.standard_normal(n)
    q = float(x @ sp.build_laplacian(g).matvec(x))
    ref = float(np.sum(w * (x[u] - x[v]) ** 2))
    assert abs(q - ref) <= 1e-5 * max(1.0, abs(ref))


def test_exact_kind_without_dense_oracle(cuda):
    """test_transforms.py:176-180"""
    sp = _sp()
    lap = sp.build_laplacian(_k3(sp))
    op = sp.TransformedOperator(lap, sp.SpectralTransform("negexp"), 0.0, 4.0, None)
    with pytest.raises(ValueError, match="dense"):
        op.apply(np.ones(3))


def test_log_taylor_divergence_warning(cuda):
    """test_transforms.py:183-186"""
    sp = _sp()
    with pytest.warns(RuntimeWarning, match="diverges"):
        sp.make_reversed_operator(_k3(sp), sp.SpectralTransform("log-taylor", 11))


def test_reversed_top_k_is_bottom_k(cuda):
    """test_transforms.py:189-200 (polynomial kinds on the device): the top-k
    eigenvectors of lambda* I - f(L) span the bottom-k of L."""
    sp = _sp()
    rng = np.random.default_rng(21)
    for _ in range(4):
        n = int(rng.integers(6, 30))
        iu, ju = np.triu_indices(n, k=1)
        keep = rng.random(iu.size) < 0.5
        u, v = iu[keep], ju[keep]
        if u.size == 0:
            continue
        w = rng.uniform(0.1, 2.0, u.size).astype(np.float32).astype(np.float64)
        g = sp.Graph(n, u, v, w)
        gt = sp.graph_ground_truth(g)
        for t in (sp.SpectralTransform("identity"), sp.SpectralTransform("negexp-limit", 41)):
            op = sp.make_reversed_operator(g, t)
            M = op.apply(np.eye(n))
            M = 0.5 * (M + M.T)
            vals, vecs = np.linalg.eigh(M)
            top = vecs[:, ::-1][:, :2]
            gaps = np.diff(gt.eigenvalues[:3])
            if np.all(gaps > 1e-3):  # well-defined bottom-2 subspace
                assert sp.subspace_error(top, gt, k=2) <= 1e-4, t.kind


def test_kmeans_reference_cases(cuda):
    """specgap tests/test_metrics.py:127-152 on the device k-means (incl. the
    degenerate identical-points case, where empty clusters are re-seeded at
    the farthest point exactly as metrics.py:161-165)."""
    sp = _sp()
    rng = np.random.default_rng(0)
    X = np.vstack([rng.normal(0, 0.1, (40, 2)), rng.normal(5, 0.1, (40, 2))])
    truth = np.repeat([0, 1], 40)
    assert sp.cluster_accuracy(sp.kmeans_cluster(X, 2, seed=1), truth) == 1.0
    X0 = np.zeros((10, 2))
    truth0 = np.array([0] * 7 + [1] * 3)
    labels0 = sp.kmeans_cluster(X0, 2, seed=1)
    assert sp.cluster_accuracy(labels0, truth0) == pytest.approx(0.7)
    np.testing.assert_array_equal(labels0, O.kmeans_cluster(X0, 2, seed=1))
    assert sp.cluster_accuracy(np.array([2, 2, 0, 0, 1, 1]), np.array([0, 0, 1, 1, 2, 2])) == 1.0
