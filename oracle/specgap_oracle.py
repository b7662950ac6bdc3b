"""numpy/scipy restatement of the reference SPED hot path (TEST INFRASTRUCTURE).

Every function cites the reference lines it restates; paths are relative to
``/root/reference/pkg/src/specgap/``.  Arithmetic is fp64 exactly as in the
reference; the sparse product is scipy's ``csr @ dense`` (the reference's own
L0 dependency, ``graph.py:211``).  Nothing here is imported by the product
package ``paper_2207_14589_b200``.

Third-party boundary: the SpMM arithmetic lives in scipy's
``csr_matvecs`` and the minibatch RNG in numpy's PCG64; both are used here
as-is (versions recorded by ``versions()``).
"""

from __future__ import annotations

import math
import warnings

import numpy as np
import scipy.sparse as sp

__all__ = [
    "walk_chunk_key",
    "incidence_lists",
    "walk_sample_chunk",
    "walk_estimate",
    "walk_oracle_apply",
    "versions",
    "canonical_edges",
    "degrees",
    "degree_counts",
    "laplacian_csr",
    "laplacian_csr_rows",
    "lambda_upper",
    "check_transform",
    "choose_lambda_star",
    "polynomial_coefficients",
    "scalar_map",
    "apply_transform",
    "term_schedule",
    "identity_minibatch_apply",
    "sampled_laplacian_apply",
    "edge_batch_poly_apply",
    "draw_batches",
    "orthonormalize",
    "init_state",
    "solver_seeds",
    "mu_eg_step",
    "oja_step",
    "subspace_error",
    "dense_ground_truth",
    "principal_angles",
    "ritz_values",
    "kmeans_cluster",
    "pcg64_integers",
    "threaded_csr_matmul",
]

_NORM_TOL = 1e-12  # solvers.py:42


def versions() -> dict:
    import scipy
    return {"numpy": np.__version__, "scipy": scipy.__version__}


# ---------------------------------------------------------------- graph (L1)

def canonical_edges(n: int, u, v, w):
    """Canonical edge list; restates ``Graph.__post_init__`` (graph.py:64-88)."""
    if n < 0:
        raise ValueError("node count must be nonnegative")
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    w = np.asarray(w, dtype=np.float64)
    if not (u.shape == v.shape == w.shape):
        raise ValueError("edge arrays must have identical length")
    if np.any(w < 0):
        raise ValueError("edge weights must be nonnegative")
    keep = w > 0
    u, v, w = u[keep], v[keep], w[keep]
    if u.size:
        if np.any(u == v):
            raise ValueError("self-loops are not allowed")
        if np.any((u < 0) | (u >= n) | (v < 0) | (v >= n)):
            raise ValueError("edge endpoint out of range")
    lo = np.minimum(u, v)
    hi = np.maximum(u, v)
    order = np.lexsort((hi, lo))
    lo, hi, w = lo[order], hi[order], w[order]
    pair = lo * n + hi
    if pair.size and np.any(np.diff(pair) == 0):
        raise ValueError("duplicate edge for an unordered node pair")
    return lo, hi, w


def degrees(n, u, v, w):
    """Weighted degree; graph.py:118-122."""
    d = np.bincount(u, weights=w, minlength=n)
    d += np.bincount(v, weights=w, minlength=n)
    return d


def degree_counts(n, u, v):
    """Unweighted degree; graph.py:124-128."""
    d = np.bincount(u, minlength=n)
    d += np.bincount(v, minlength=n)
    return d


def laplacian_csr(n, u, v, w, mode="unnormalized") -> sp.csr_matrix:
    """CSR Laplacian; restates ``LaplacianOperator.__post_init__`` (graph.py:182-199).

    Returned with sorted column indices (canonical form), fp64 data, int32
    indices/indptr as scipy produces them.
    """
    if mode not in ("unnormalized", "normalized"):
        raise ValueError(f"unknown Laplacian mode: {mode!r}")
    deg = degrees(n, u, v, w)
    if mode == "normalized" and n and np.any(deg == 0):
        raise ValueError("normalized Laplacian requires all degrees > 0")
    rows = np.concatenate([u, v, u, v])
    cols = np.concatenate([v, u, u, v])
    vals = np.concatenate([-w, -w, w, w])
    lap = sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr()
    if mode == "normalized":
        with np.errstate(divide="ignore"):
            dinv = 1.0 / np.sqrt(deg)
        dinv[~np.isfinite(dinv)] = 0.0
        scale = sp.diags(dinv)
        lap = scale @ lap @ scale
    lap = sp.csr_matrix(lap)
    lap.sort_indices()
    return lap


def laplacian_csr_rows(n, u, v, w, mode, r0, r1) -> sp.csr_matrix:
    """Rows [r0, r1) of ``laplacian_csr`` (same construction, restricted to
    the sampled rows): the bounded CPU-baseline sample of a BASELINE-size
    graph.  Canonical edges in, (r1-r0) x n CSR out."""
    deg = degrees(n, u, v, w)
    if mode == "normalized" and n and np.any(deg == 0):
        raise ValueError("normalized Laplacian requires all degrees > 0")
    su = (u >= r0) & (u < r1)
    sv = (v >= r0) & (v < r1)
    rows = np.concatenate([u[su], v[sv], u[su], v[sv]]) - r0
    cols = np.concatenate([v[su], u[sv], u[su], v[sv]])
    vals = np.concatenate([-w[su], -w[sv], w[su], w[sv]])
    lap = sp.coo_matrix((vals, (rows, cols)), shape=(r1 - r0, n)).tocsr()
    if mode == "normalized":
        dinv = 1.0 / np.sqrt(deg)
        lap = sp.diags(dinv[r0:r1]) @ lap @ sp.diags(dinv)
    lap = sp.csr_matrix(lap)
    lap.sort_indices()
    return lap


def lambda_upper(n, u, v, w, mode="unnormalized") -> float:
    """Spectral upper bound; transforms.py:280-284 with graph.py:351-362."""
    if mode == "normalized":
        return 2.0
    if n == 0 or u.size == 0:
        return 0.0
    return 2.0 * float(degrees(n, u, v, w).max())


# ----------------------------------------------------------- transforms (L2)

_POLY = {"identity", "log-taylor", "negexp-taylor", "negexp-limit"}
_KINDS = ("identity", "log", "log-taylor", "negexp", "negexp-taylor", "negexp-limit")


def check_transform(kind, ell=None, epsilon=1e-6):
    """SpectralTransform validation; transforms.py:74-85."""
    if kind not in _KINDS:
        raise ValueError(f"unknown transform kind {kind!r}")
    if kind in ("log-taylor", "negexp-taylor", "negexp-limit"):
        min_ell = 0 if kind == "negexp-taylor" else 1
        if ell is None or ell < min_ell:
            raise ValueError(f"{kind} requires a series degree >= {min_ell}")
        if kind == "negexp-limit" and ell % 2 == 0:
            raise ValueError("negexp-limit requires an odd series degree")
    if kind in ("log", "log-taylor") and epsilon <= 0:
        raise ValueError("log transforms require epsilon > 0")


def choose_lambda_star(kind, lam_upper, epsilon=1e-6) -> float:
    """transforms.py:180-192."""
    if kind == "identity":
        return 1.01 * lam_upper
    if kind in ("log", "log-taylor"):
        top = math.log(lam_upper + epsilon)
        return top + 0.01 * abs(top)
    return 0.0


def polynomial_coefficients(kind, ell=None, epsilon=1e-6) -> np.ndarray:
    """Monomial coefficients; transforms.py:152-177."""
    from numpy.polynomial import polynomial as P
    if kind == "identity":
        return np.array([0.0, 1.0])
    if kind == "negexp-taylor":
        return np.array([-((-1.0) ** i) / math.factorial(i) for i in range(ell + 1)])
    if kind == "negexp-limit":
        return -P.polypow(np.array([1.0, -1.0 / ell]), ell)
    if kind == "log-taylor":
        shift = np.array([epsilon - 1.0, 1.0])
        out = np.zeros(ell + 1)
        power = np.array([1.0])
        for i in range(1, ell + 1):
            power = P.polymul(power, shift)
            out[: power.size] += ((1.0 if i % 2 == 1 else -1.0) / i) * power
        return out
    raise ValueError(f"{kind} has no polynomial expansion")


def scalar_map(kind, lam, ell=None, epsilon=1e-6):
    """transforms.py:120-149."""
    lam = np.asarray(lam, dtype=np.float64)
    if kind == "identity":
        return lam.copy()
    if kind == "log":
        return np.log(lam + epsilon)
    if kind == "log-taylor":
        y = lam + epsilon - 1.0
        out = np.zeros_like(y)
        term = np.ones_like(y)
        for i in range(1, ell + 1):
            term = term * y
            out += (1.0 if i % 2 == 1 else -1.0) * term / i
        return out
    if kind == "negexp":
        return -np.exp(-lam)
    if kind == "negexp-taylor":
        out = np.zeros_like(lam)
        term = np.ones_like(lam)
        out -= term
        for i in range(1, ell + 1):
            term = term * (-lam) / i
            out -= term
        return out
    if kind == "negexp-limit":
        return -((1.0 - lam / ell) ** ell)
    raise AssertionError(kind)


def apply_transform(csr, kind, ell, epsilon, lam_star, x, threads=1):
    """Reversed polynomial apply; restates ``TransformedOperator.apply``
    (transforms.py:229-262) with ``L.matvec = csr @ w`` (graph.py:211).
    ``threads > 1`` splits each ``csr @ w`` into row blocks on a thread pool
    (``threaded_csr_matmul``: the same scipy kernel per row, so the same
    fp64 result) for the full-size parity tests."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape[0] != csr.shape[0]:
        raise ValueError("dimension mismatch in transformed matvec")

    def L(w):
        return csr @ w if threads <= 1 else threaded_csr_matmul(csr, w, threads)

    if kind == "identity":                                  # :241-242
        return lam_star * x - L(x)
    if kind == "negexp-limit":                              # :243-248
        w = x.copy()
        inv = 1.0 / ell
        for _ in range(ell):
            w -= inv * L(w)
        return lam_star * x + w
    if kind == "negexp-taylor":                             # :249-254
        c = [-((-1.0) ** i) / math.factorial(i) for i in range(ell + 1)]
        w = c[-1] * x
        for i in range(ell - 1, -1, -1):
            w = c[i] * x + L(w)
        return lam_star * x - w
    if kind == "log-taylor":                                # :255-262
        shift = epsilon - 1.0
        c = [0.0] + [(1.0 if i % 2 == 1 else -1.0) / i for i in range(1, ell + 1)]
        w = c[-1] * x
        for i in range(ell - 1, -1, -1):
            w = c[i] * x + L(w) + shift * w
        return lam_star * x - w
    raise ValueError(f"{kind} is not a polynomial transform")


def term_schedule(kind, ell, epsilon, lam_star):
    """The (alpha, beta, gamma) per-term form of transforms.py:241-262
    (SURVEY §8a a8), plus the final ``out = lam_f*x + s*w``.  Returns
    ``(alpha, beta, gamma, w0_scale, lam_f, s)``; term t computes
    ``w <- alpha_t x + beta_t L w + gamma_t w`` starting from ``w = w0_scale*x``.
    Used by the restated stochastic composition below."""
    if kind == "identity":
        return [0.0], [1.0], [0.0], 1.0, lam_star, -1.0
    if kind == "negexp-limit":
        return [0.0] * ell, [-1.0 / ell] * ell, [1.0] * ell, 1.0, lam_star, 1.0
    if kind == "negexp-taylor":
        c = [-((-1.0) ** i) / math.factorial(i) for i in range(ell + 1)]
        return ([c[i] for i in range(ell - 1, -1, -1)], [1.0] * ell, [0.0] * ell,
                c[ell], lam_star, -1.0)
    if kind == "log-taylor":
        c = [0.0] + [(1.0 if i % 2 == 1 else -1.0) / i for i in range(1, ell + 1)]
        return ([c[i] for i in range(ell - 1, -1, -1)], [1.0] * ell,
                [epsilon - 1.0] * ell, c[ell], lam_star, -1.0)
    raise ValueError(kind)


# ------------------------------------------------- stochastic oracle (L3/L2)

def draw_batches(rng: np.random.Generator, m: int, batch: int, count: int):
    """``count`` successive ``rng.integers(0, m, size=batch)`` draws
    (solvers.py:171), one per polynomial term."""
    return [rng.integers(0, m, size=batch) for _ in range(count)]


def sampled_laplacian_apply(u, v, w, batch, x, threads=1):
    """Unscaled sampled-edge Laplacian product ``est`` of solvers.py:172-176:
    ``diff = (x[u_b]-x[v_b])*w_b; est[u_b] += diff; est[v_b] -= diff``.

    ``threads > 1`` (full-size tests): the same sum written as the sampled
    Laplacian ``sum_b w_b (e_u - e_v)(e_u - e_v)^T`` in scipy CSR (duplicate
    samples summed) times ``x`` on a thread pool -- equal to the ``np.add.at``
    form up to fp64 summation order."""
    x = np.asarray(x, dtype=np.float64)
    if threads > 1:
        ub, vb = u[batch], v[batch]
        wb = np.asarray(w, dtype=np.float64)[batch]
        n = x.shape[0]
        S = sp.coo_matrix((np.concatenate([wb, -wb, -wb, wb]),
                           (np.concatenate([ub, ub, vb, vb]), np.concatenate([ub, vb, ub, vb]))),
                          shape=(n, n)).tocsr()
        return threaded_csr_matmul(S, x, threads)
    diff = (x[u[batch]] - x[v[batch]]) * (w[batch] if x.ndim == 1 else w[batch][:, None])
    est = np.zeros_like(x)
    np.add.at(est, u[batch], diff)
    np.subtract.at(est, v[batch], diff)
    return est


def identity_minibatch_apply(u, v, w, lam_star, batch, x):
    """The identity edge-minibatch oracle body; solvers.py:169-178."""
    m = u.size
    est = sampled_laplacian_apply(u, v, w, batch, x)
    est *= m / batch.size
    return lam_star * np.asarray(x, dtype=np.float64) - est


def edge_batch_poly_apply(u, v, w, kind, ell, epsilon, lam_star, batches, x, threads=1):
    """RESTATED (no reference implementation): the reversed
    polynomial recurrence of transforms.py:241-262 with term t's ``L w``
    replaced by the unbiased minibatch estimate of solvers.py:171-177 drawn
    from ``batches[t]`` (term order = application order).  Identity kind with
    one batch reduces exactly to ``identity_minibatch_apply``."""
    x = np.asarray(x, dtype=np.float64)
    m = u.size
    al, be, ga, w0, lam_f, s = term_schedule(kind, ell, epsilon, lam_star)
    if len(batches) != len(al):
        raise ValueError("need one batch per polynomial term")
    if kind == "identity":
        return identity_minibatch_apply(u, v, w, lam_star, batches[0], x)
    cur = w0 * x
    for t in range(len(al)):
        est = sampled_laplacian_apply(u, v, w, batches[t], cur, threads) * (m / batches[t].size)
        cur = al[t] * x + be[t] * est + ga[t] * cur
    return lam_f * x + s * cur


# ------------------------------------------------------------ solvers (L3)

def orthonormalize(V, rng=None):
    """Thin QR by MGS; solvers.py:84-102."""
    V = V.copy()
    n, k = V.shape
    for j in range(k):
        for i in range(j):
            V[:, j] -= (V[:, i] @ V[:, j]) * V[:, i]
        norm = np.linalg.norm(V[:, j])
        if norm < _NORM_TOL:
            warnings.warn(f"rank collapse in column {j}; re-randomizing", RuntimeWarning)
            if rng is None:
                rng = np.random.default_rng(0)
            V[:, j] = rng.standard_normal(n)
            for i in range(j):
                V[:, j] -= (V[:, i] @ V[:, j]) * V[:, i]
            norm = np.linalg.norm(V[:, j])
        V[:, j] /= norm
    return V


def init_state(n, k, seed):
    """solvers.py:105-111."""
    if k > n:
        raise ValueError("cannot ask for more eigenvectors than dimensions")
    rng = np.random.default_rng(seed)
    return orthonormalize(rng.standard_normal((n, k)), rng)


def solver_seeds(seed):
    """(init, aux, oracle) seeds; solvers.py:245-246."""
    ss = np.random.SeedSequence(seed)
    return tuple(int(x) for x in ss.generate_state(3))


def mu_eg_step(V, MV, eta, rng=None):
    """solvers.py:121-144 with ``MV = oracle(V)`` precomputed."""
    C = V.T @ MV
    G = MV - V @ np.triu(C, 1)
    d = np.einsum("nk,nk->k", V, G)
    W = V + eta * (G - V * d)
    norms = np.linalg.norm(W, axis=0)
    bad = norms < _NORM_TOL
    if np.any(bad):
        if rng is None:
            rng = np.random.default_rng(0)
        W[:, bad] = rng.standard_normal((W.shape[0], int(bad.sum())))
        norms = np.linalg.norm(W, axis=0)
    return W / norms


def oja_step(V, MV, eta, rng=None):
    """solvers.py:114-118."""
    return orthonormalize(V + eta * MV, rng)


# ------------------------------------------------------------- metrics

def dense_ground_truth(csr):
    """Dense eigendecomposition (metrics.py:39-54), desk scale only."""
    vals, vecs = np.linalg.eigh(csr.toarray())
    return vals, vecs


def subspace_error(V, U):
    """``1 - tr(U*^T P U*)/k``; metrics.py:57-79 (U = bottom-k truth)."""
    V = np.atleast_2d(np.asarray(V, dtype=np.float64))
    k = U.shape[1]
    gram = V.T @ V
    B = U.T @ V
    sol = np.linalg.solve(gram, B.T)
    trace = float(np.einsum("ij,ji->", B, sol))
    return float(np.clip(1.0 - trace / k, 0.0, 1.0))


def principal_angles(V, U):
    """RESTATED: largest principal angle via scipy."""
    import scipy.linalg as sla
    return float(np.max(sla.subspace_angles(np.asarray(V, np.float64), U)))


def ritz_values(csr, V):
    """RESTATED: ``eigvalsh(Q^T L Q)`` with Q = orth(V)."""
    Q, _ = np.linalg.qr(np.asarray(V, np.float64))
    return np.linalg.eigvalsh(Q.T @ (csr @ Q))


def kmeans_cluster(X, k, seed=0, max_iter=100):
    """Farthest-point Lloyd's; metrics.py:143-176."""
    if k < 2:
        raise ValueError("k must be at least 2")
    X = np.atleast_2d(np.asarray(X, dtype=np.float64))
    npts = X.shape[0]
    rng = np.random.default_rng(seed)
    centers = np.empty((k, X.shape[1]))
    centers[0] = X[rng.integers(npts)]
    dist = np.linalg.norm(X - centers[0], axis=1)
    for j in range(1, k):
        centers[j] = X[int(np.argmax(dist))]
        dist = np.minimum(dist, np.linalg.norm(X - centers[j], axis=1))
    labels = np.zeros(npts, dtype=np.int64)
    for _ in range(max_iter):
        d2 = ((X[:, None, :] - centers[None, :, :]) ** 2).sum(axis=2)
        new_labels = np.argmin(d2, axis=1)
        for j in range(k):
            members = X[new_labels == j]
            if members.shape[0] == 0:
                nearest = d2[np.arange(npts), new_labels]
                centers[j] = X[int(np.argmax(nearest))]
            else:
                centers[j] = members.mean(axis=0)
        if np.array_equal(new_labels, labels):
            break
        labels = new_labels
    return labels


# ------------------------------------------------ PCG64 + Lemire (restated)

_PCG_MULT = (2549297995355413924 << 64) | 4865540595714422341
_M128 = (1 << 128) - 1


def pcg64_integers(state: dict, m: int, size: int):
    """Pure-Python restatement of numpy ``Generator(PCG64).integers(0, m, size)``
    for ``1 <= m < 2**32`` (numpy ``random_bounded_uint64_fill`` ->
    ``buffered_bounded_lemire_uint32`` -> ``pcg64_next32``).  ``state`` is
    ``bit_generator.state``; returns ``(values, new_state, draws32)`` where
    ``draws32`` counts the 32-bit draws consumed.  Small sizes only
    (pure Python); it pins the GPU K4 kernel's algorithm."""
    st = state["state"]["state"]
    inc = state["state"]["inc"]
    has = state["has_uint32"]
    uint = state["uinteger"]
    out = np.empty(size, dtype=np.int64)
    ndraw = 0

    def next32():
        nonlocal st, has, uint, ndraw
        ndraw += 1
        if has:
            has = 0
            return uint
        st = (st * _PCG_MULT + inc) & _M128
        hi, lo = st >> 64, st & ((1 << 64) - 1)
        rot = hi >> 58
        x = hi ^ lo
        r = ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)
        has = 1
        uint = r >> 32
        return r & 0xFFFFFFFF

    rng = m - 1
    if rng == 0:
        out[:] = 0
    else:
        rng_excl = rng + 1
        for i in range(size):
            mm = next32() * rng_excl
            left = mm & 0xFFFFFFFF
            if left < rng_excl:
                thresh = ((1 << 32) - rng_excl) % rng_excl
                while left < thresh:
                    mm = next32() * rng_excl
                    left = mm & 0xFFFFFFFF
            out[i] = mm >> 32
    new = {"bit_generator": "PCG64", "state": {"state": st, "inc": inc},
           "has_uint32": has, "uinteger": uint}
    return out, new, ndraw


# ---------------------------------------------- threaded CPU baseline helper

def threaded_csr_matmul(csr, x, threads):
    """``csr @ x`` split into ``threads`` row blocks on a thread pool.
    scipy's csr_matvecs releases the GIL, so this is the reference's own
    kernel on all host cores (used only by bench.py's CPU baseline)."""
    from concurrent.futures import ThreadPoolExecutor
    n = csr.shape[0]
    if threads <= 1:
        return csr @ x
    bounds = np.linspace(0, n, threads + 1).astype(np.int64)
    out = np.empty((n,) + x.shape[1:], dtype=np.result_type(csr.dtype, x.dtype))

    def work(i):
        a, b = bounds[i], bounds[i + 1]
        out[a:b] = csr[a:b] @ x

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, range(threads)))
    return out


# ---------------------------------------------------------------------------
# walk-based polynomial estimator (walks.py), restated.  numpy's Philox is the
# reference's own RNG (walks.py:196-198); the incidence lists are built
# directly from the canonical (lexsorted) edge list.

_WALK_CHUNK = 8192  # walks.py:45


def walk_chunk_key(seed: int, chunk: int) -> np.ndarray:
    """Philox key of chunk ``chunk`` (walks.py:196-198: Philox(SeedSequence((seed, chunk))),
    counter 0): the two uint64 words SeedSequence hands the bit generator."""
    return np.random.SeedSequence((seed, chunk)).generate_state(2, np.uint64)


def incidence_lists(n, u, v):
    """Edge incidence graph (graph.py:326-342): for edge e the sorted union of
    the edge ids at its two endpoints (e itself included once).  Returns
    (indptr, indices, deg_inc)."""
    m = u.size
    at = [[] for _ in range(n)]
    for e in range(m):
        at[int(u[e])].append(e)
        at[int(v[e])].append(e)
    indptr = [0]
    indices = []
    for e in range(m):
        inc = np.unique(np.asarray(at[int(u[e])] + at[int(v[e])], dtype=np.int64))
        indices.extend(inc.tolist())
        indptr.append(len(indices))
    indptr = np.asarray(indptr, dtype=np.int64)
    return indptr, np.asarray(indices, dtype=np.int64), np.diff(indptr)


def walk_sample_chunk(inc, m, ell, count, rng):
    """walks.py:175-193: uniform first edge, uniform incident successor."""
    indptr, indices, deg_inc = inc
    E = np.empty((count, ell), dtype=np.int64)
    E[:, 0] = (rng.random(count) * m).astype(np.int64)
    log_p = np.full(count, -math.log(m))
    for j in range(ell - 1):
        cur = E[:, j]
        deg = deg_inc[cur]
        pick = (rng.random(count) * deg).astype(np.int64)
        E[:, j + 1] = indices[indptr[cur] + pick]
        log_p -= np.log(deg)
    return E, log_p


def _alpha(u, v, e1, e2):
    """Incidence inner product (walks.py:83-103)."""
    return ((u[e1] == u[e2]).astype(np.int64) + (v[e1] == v[e2])
            - (u[e1] == v[e2]) - (v[e1] == u[e2]))


def walk_estimate(n, u, v, w, coeffs, x, walks, seed, mode="importance", inc=None):
    """estimate_polynomial_matvec / estimate_power_matvec (walks.py:225-341):
    sum over chunks (reduced in chunk order) of each walk's prefix
    contributions coeffs[i] * chain / p, accumulated at the first edge's
    endpoints; importance mode returns coeffs[0] x + total / N, rejection
    mode (single power coeffs = e_ell) total / (N p_min)."""
    coeffs = np.asarray(coeffs, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    m = u.size
    ell = coeffs.size - 1
    if inc is None:
        inc = incidence_lists(n, u, v)
    deg_star = int(np.max(np.bincount(u, minlength=n) + np.bincount(v, minlength=n)))
    lpmin = -ell * math.log(2 * deg_star - 1) - math.log(m)
    n_chunks = -(-walks // _WALK_CHUNK)
    total = np.zeros(n)
    n_acc = 0
    for c in range(n_chunks):
        size = min(_WALK_CHUNK, walks - c * _WALK_CHUNK)
        rng = np.random.Generator(np.random.Philox(np.random.SeedSequence((seed, c))))
        E, log_p_full = walk_sample_chunk(inc, m, ell, size, rng)
        logmag = np.cumsum(np.log(w[E]), axis=1)
        sign = np.ones((size, ell))
        if ell > 1:
            a = _alpha(u, v, E[:, :-1].ravel(), E[:, 1:].ravel()).reshape(size, ell - 1)
            sign[:, 1:] = np.cumprod(np.sign(a), axis=1)
            logmag[:, 1:] += np.cumsum(np.log(np.abs(a)), axis=1)
        acc = np.zeros(n)

        def accumulate(Es, coefs, which):
            e_last = Es[:, which - 1]
            contrib = coefs * (x[u[e_last]] - x[v[e_last]])
            acc[:] += np.bincount(u[Es[:, 0]], weights=contrib, minlength=n)
            acc[:] -= np.bincount(v[Es[:, 0]], weights=contrib, minlength=n)

        if mode == "importance":
            deg_logs = np.zeros((size, ell))
            if ell > 1:
                deg_logs[:, 1:] = np.cumsum(np.log(inc[2][E[:, :-1]]), axis=1)
            for i in range(1, ell + 1):
                if coeffs[i] == 0.0:
                    continue
                lp = -math.log(m) - deg_logs[:, i - 1]
                accumulate(E, coeffs[i] * sign[:, i - 1] * np.exp(logmag[:, i - 1] - lp), i)
        else:
            keep = rng.random(size) < np.exp(lpmin - log_p_full)
            n_acc += int(keep.sum())
            if keep.any():
                accumulate(E[keep], coeffs[ell] * sign[keep, ell - 1]
                           * np.exp(logmag[keep, ell - 1]), ell)
        total += acc
    if mode == "importance":
        return coeffs[0] * x + total / walks
    if n_acc == 0:
        raise RuntimeError("no walk survived rejection")
    return total / (walks * math.exp(lpmin))


def walk_oracle_apply(n, u, v, w, coeffs, lam_star, x, walks, seed, call0):
    """make_stochastic_oracle's walk oracle (solvers.py:183-200): one estimate
    per column, column j of call c seeded with
    SeedSequence((seed, counter)).generate_state(1)[0]; returns
    (lam_star x - f(L) x, next counter)."""
    x = np.asarray(x, dtype=np.float64)
    cols = x[:, None] if x.ndim == 1 else x
    out = np.empty_like(cols)
    inc = incidence_lists(n, u, v)
    counter = call0
    for j in range(cols.shape[1]):
        call_seed = int(np.random.SeedSequence((seed, counter)).generate_state(1)[0])
        counter += 1
        fx = walk_estimate(n, u, v, w, coeffs, cols[:, j], walks, call_seed, inc=inc)
        out[:, j] = lam_star * cols[:, j] - fx
    return (out[:, 0] if x.ndim == 1 else out), counter
