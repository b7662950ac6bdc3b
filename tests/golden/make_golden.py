"""Generate golden vectors by running the REFERENCE ``specgap`` package.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/golden.npz`` (+ ``golden_meta.json``).  Every array is
produced by the reference's own public API on edge lists stored alongside, so
the fixtures pin the oracle restatement (``oracle/``) and the CUDA path to the
reference itself.  Graph inputs are the reference's conftest fixtures, seeded
Erdos-Renyi graphs (the reference's ``random_graph`` recipe) and small
BASELINE-shaped graphs from ``paper_2207_14589_b200.generators``.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

import specgap as sg  # noqa: E402  (reference, read-only)
from specgap import transforms as tf  # noqa: E402


def random_graph(rng, n, p=0.5, weighted=False, require_connected=False):
    """The reference conftest helper (pkg/tests/conftest.py:34-46)."""
    while True:
        iu, iv = np.triu_indices(n, k=1)
        keep = rng.random(iu.size) < p
        if not keep.any():
            continue
        w = rng.uniform(0.2, 2.0, int(keep.sum())) if weighted else np.ones(int(keep.sum()))
        g = sg.Graph(n, iu[keep], iv[keep], w)
        if not require_connected or g.is_connected():
            return g


def graphs():
    out = {
        "path2": sg.Graph.from_edges(2, [(0, 1)]),
        "path3": sg.Graph.from_edges(3, [(0, 1), (1, 2)]),
        "k3": sg.Graph.from_edges(3, [(0, 1), (0, 2), (1, 2)]),
        "star4": sg.Graph.from_edges(4, [(0, 1), (0, 2), (0, 3)]),
        "two_triangles_bridge": sg.Graph.from_edges(
            6, [(0, 1), (0, 2), (1, 2), (3, 4), (3, 5), (4, 5), (2, 3)]),
        "isolated": sg.Graph.from_edges(5, [(0, 1), (1, 3)]),
    }
    rng = np.random.default_rng(2024)
    for i in range(6):
        g = random_graph(rng, int(rng.integers(5, 50)), p=0.3, weighted=(i % 2 == 0),
                         require_connected=True)
        out[f"er{i}"] = g
    # fp64 weights with many incident edges per node (diagonal fold order)
    rng = np.random.default_rng(7)
    g = random_graph(rng, 60, p=0.5, weighted=True, require_connected=True)
    out["er_dense_w"] = g
    import torch  # noqa: F401  (generators use torch on the CPU)
    from paper_2207_14589_b200 import generators as G
    for name, (n, u, v, w) in {
        "cfg1": G.config_graph(1),
        "cfg3s": G.sbm_sparse(2000, 20, 20.0, 0.9),
        "cfg4s": G.chung_lu(1500, 2.1, 2.0, 16.0, 1e5),
        "cfg5s": G.lp_sbm(1200, 12, 24.0, 0.1, 5, 0.8),
    }.items():
        out[name] = sg.Graph(n, u.numpy(), v.numpy(), w.numpy())
    return out


def main():
    data = {}
    meta = {"numpy": np.__version__, "reference": str(sg.__version__), "cases": {}}
    import scipy
    meta["scipy"] = scipy.__version__
    G = graphs()
    for name, g in G.items():
        data[f"g/{name}/n"] = np.array(g.n)
        data[f"g/{name}/u"] = g.u.astype(np.int32)
        data[f"g/{name}/v"] = g.v.astype(np.int32)
        data[f"g/{name}/w"] = g.w
        data[f"g/{name}/degrees"] = g.degrees()
        for mode in ("unnormalized", "normalized"):
            if name in ("cfg1", "cfg3s", "cfg5s") and mode == "normalized":
                continue
            try:
                L = sg.build_laplacian(g, mode)
            except ValueError as e:
                data[f"csr/{name}/{mode}/error"] = np.array(str(e))
                continue
            c = L._csr.copy()
            c.sort_indices()
            data[f"csr/{name}/{mode}/indptr"] = c.indptr.astype(np.int32)
            data[f"csr/{name}/{mode}/indices"] = c.indices.astype(np.int32)
            # large cases keep fp32(data): exactly what the device CSR must equal
            data[f"csr/{name}/{mode}/data"] = c.data if g.n < 100 else c.data.astype(np.float32)
            data[f"csr/{name}/{mode}/degrees"] = L.degrees
    # ---- polynomial applies ------------------------------------------------
    kinds = [("identity", None, 1e-6), ("negexp-limit", 9, 1e-6), ("negexp-limit", 3, 1e-6),
             ("negexp-taylor", 8, 1e-6), ("negexp-taylor", 0, 1e-6), ("log-taylor", 9, 0.5),
             ("negexp-limit", 17, 1e-6), ("negexp-taylor", 16, 1e-6)]
    apply_graphs = ["path2", "k3", "star4", "two_triangles_bridge", "er0", "er1", "er2",
                    "er_dense_w", "cfg1", "cfg3s", "cfg4s", "cfg5s"]
    import warnings
    for gi, name in enumerate(apply_graphs):
        g = G[name]
        for mode in ("unnormalized", "normalized"):
            if name in ("cfg1", "cfg3s", "cfg5s") and mode == "normalized":
                continue
            if name == "cfg4s" and mode == "unnormalized":
                continue
            for ki, (kind, ell, eps) in enumerate(kinds):
                big = name in ("cfg1", "cfg3s", "cfg4s", "cfg5s")
                if ell is not None and ell >= 16 and not big:
                    continue
                if big and (kind, ell) not in (("identity", None), ("negexp-limit", 9),
                                               ("negexp-taylor", 16), ("log-taylor", 9)):
                    continue
                t = sg.SpectralTransform(kind, ell, eps)
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore", RuntimeWarning)
                    op = sg.make_reversed_operator(g, t, mode)
                for k in ((1, 3) if g.n < 100 else (4,)):
                    rng = np.random.default_rng(1000 * gi + 10 * ki + k)
                    x = rng.standard_normal((g.n, k)).astype(np.float32).astype(np.float64)
                    if k == 1:
                        x = x[:, 0]
                    y = op.apply(x)
                    key = f"apply/{name}/{mode}/{kind}/{ell}/{eps}/{k}"
                    small = g.n < 100
                    data[key + "/x"] = x if small else x.astype(np.float32)
                    data[key + "/y"] = y if small else y.astype(np.float32)
                    data[key + "/lambda_star"] = np.array(op.lambda_star)
    # ---- solver steps ------------------------------------------------------
    for name, mode, kind, ell, k in [("two_triangles_bridge", "unnormalized", "identity", None, 3),
                                     ("er0", "unnormalized", "negexp-limit", 9, 3),
                                     ("er1", "normalized", "negexp-taylor", 8, 4),
                                     ("cfg1", "unnormalized", "negexp-limit", 13, 10)]:
        g = G[name]
        op = sg.make_reversed_operator(g, sg.SpectralTransform(kind, ell), mode)
        st = sg.init_state(g.n, k, seed=11)
        key = f"step/{name}/{mode}/{kind}/{ell}/{k}"
        data[key + "/V0"] = st.V
        for eta in (0.05, 0.5):
            data[key + f"/mueg/{eta}"] = sg.mu_eg_step(st, op.apply, eta).V
            data[key + f"/oja/{eta}"] = sg.oja_step(st, op.apply, eta).V
    for n, k, seed in [(3, 3, 0), (50, 4, 9), (100, 8, 1), (1000, 10, 123)]:
        data[f"init/{n}/{k}/{seed}"] = sg.init_state(n, k, seed).V
    # ---- identity edge-minibatch oracle ------------------------------------
    for name, B, seed in [("path2", 3, 1), ("k3", 2, 5), ("two_triangles_bridge", 4, 2),
                          ("er2", 50, 3), ("cfg1", 1000, 4)]:
        g = G[name]
        op = sg.make_reversed_operator(g, tf.identity())
        oracle = sg.make_stochastic_oracle(op, B, seed=seed)
        rng = np.random.default_rng(seed)
        x = np.random.default_rng(99).standard_normal((g.n, 3)).astype(np.float32).astype(np.float64)
        key = f"sto/{name}/{B}/{seed}"
        data[key + "/x"] = x
        for call in range(3):
            data[key + f"/batch{call}"] = rng.integers(0, g.m, size=B)
            data[key + f"/y{call}"] = oracle(x)
    # ---- PCG64 index streams -------------------------------------------------
    for m, seed, sizes in [(3, 1, (5, 7)), (1000, 2, (1001, 3)), (9_990_000, 3, (4096, 17)),
                           (2**31 - 1, 4, (333, 64)), (1, 5, (10,)), (7, 6, (1, 1, 1))]:
        rng = np.random.default_rng(seed)
        key = f"pcg/{m}/{seed}"
        data[key + "/state0"] = np.array(json.dumps(rng.bit_generator.state))
        for i, s in enumerate(sizes):
            data[key + f"/draw{i}"] = rng.integers(0, m, size=s)
            data[key + f"/state{i + 1}"] = np.array(json.dumps(rng.bit_generator.state))
    # ---- run_solver trajectories -------------------------------------------
    for name, solver, eta, kind, ell in [("k3", "oja", 0.1, "identity", None),
                                         ("two_triangles_bridge", "mu-eg", 0.05, "identity", None),
                                         ("cfg1", "mu-eg", 0.1, "negexp-limit", 13)]:
        g = G[name]
        k = 2 if g.n < 10 else 10
        steps = 200 if g.n < 10 else 1500
        cfg = sg.SolverConfig(solver=solver, k=k, eta=eta, steps=steps, eval_every=50, seed=5)
        run = sg.run_solver(g, sg.SpectralTransform(kind, ell), cfg, record_timing=False)
        key = f"run/{name}/{solver}"
        data[key + "/csv"] = np.array(sg.run_to_csv(run))
        data[key + "/V"] = run.V
        gt = sg.graph_ground_truth(g)
        data[key + "/gt_vals"] = gt.eigenvalues[: k + 1]
        if name == "cfg1":
            data[key + "/labels"] = sg.kmeans_cluster(run.V, 10, seed=5)
            data[key + "/gt_labels"] = sg.kmeans_cluster(gt.bottom(10), 10, seed=5)
    # ---- walk-based polynomial estimator (walks.py) --------------------------
    from specgap import walks as wk
    for name, coeffs, W, seed in [("path3", [0.5, -1.0, 0.25], 3000, 1),
                                  ("k3", [0.0, 0.0, 1.0], 5000, 2),
                                  ("two_triangles_bridge", [1.0, -0.5, 0.1, -0.02], 20000, 3),
                                  ("er0", [0.2, -0.3, 0.05, 0.0, 0.01], 30000, 4),
                                  ("er1", [1.0, -0.7, 0.2], 20000, 5)]:
        g = G[name]
        ell = len(coeffs) - 1
        x = np.random.default_rng(seed).standard_normal(g.n)
        key = f"walk/{name}/{seed}"
        data[key + "/coeffs"] = np.asarray(coeffs)
        data[key + "/walks"] = np.array(W)
        data[key + "/x"] = x
        data[key + "/y"] = wk.estimate_polynomial_matvec(
            g, coeffs, x, wk.SamplerConfig(ell, W, 1, "importance", seed))
        E, lp = wk._sample_chunk(wk.edge_incidence_graph(g), ell, min(8192, W),
                                 wk._chunk_generator(seed, 0))
        data[key + "/E0"] = E[:256]
        data[key + "/logp0"] = lp[:256]
        if ell >= 1:
            data[key + "/rejection"] = wk.estimate_power_matvec(
                g, ell, x, wk.SamplerConfig(ell, W, 1, "rejection", seed))
    for name, kind, ell, B, seed in [("two_triangles_bridge", "negexp-limit", 3, 4000, 7),
                                     ("er2", "negexp-taylor", 4, 3000, 8)]:
        g = G[name]
        op = sg.make_reversed_operator(g, sg.SpectralTransform(kind, ell))
        orc = sg.make_stochastic_oracle(op, B, seed=seed)
        X = np.random.default_rng(seed).standard_normal((g.n, 2))
        key = f"walkorc/{name}/{kind}/{ell}/{B}/{seed}"
        data[key + "/x"] = X
        data[key + "/lambda_star"] = np.array(op.lambda_star)
        data[key + "/y0"] = orc(X)
        data[key + "/y1"] = orc(X)
    # ---- k-means -------------------------------------------------------------
    rng = np.random.default_rng(0)
    X = np.concatenate([rng.normal(0, 0.1, (40, 3)), rng.normal(3, 0.1, (50, 3)),
                        rng.normal(-3, 0.1, (30, 3))]).astype(np.float32).astype(np.float64)
    data["kmeans/X"] = X
    data["kmeans/labels"] = sg.kmeans_cluster(X, 3, seed=1)
    np.savez_compressed(HERE / "golden.npz", **data)
    (HERE / "golden_meta.json").write_text(json.dumps(meta, indent=1))
    print(f"wrote {len(data)} arrays to {HERE / 'golden.npz'}")


if __name__ == "__main__":
    main()
