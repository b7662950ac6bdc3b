"""Sweep stochastic run_solver settings on the config-1 SBM (angle to the
truth, planted-block recovery, wall time) to choose the end-to-end test."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2207_14589_b200 as sp  # noqa: E402
from paper_2207_14589_b200 import generators as G  # noqa: E402

n, u, v, w = G.sbm_dense(10, 100, 0.1, 0.002, seed=3)
g = sp.Graph(n, u.numpy(), v.numpy(), w.numpy())
gt = sp.graph_ground_truth(g)
U = gt.bottom(10)
print("m", g.m, "lam_max", gt.eigenvalues[-1], flush=True)
for est, ell, B, eta, sched, steps in [
        ("edge-batch", 13, 4, 0.1, "constant", 1500),
        ("edge-batch", 13, 4, 0.1, "invsqrt", 1500),
        ("edge-batch", 13, 16, 0.1, "constant", 1500),
        ("edge-batch", 13, 16, 0.05, "constant", 3000),
        ("edge-batch", 13, 1, 0.1, "constant", 1500),
        ("walk", 13, 1000, 0.1, "constant", 300),
        ("walk", 13, 4000, 0.1, "constant", 300),
        ("walk", 13, 4000, 0.1, "invsqrt", 600)]:
    bs = B * g.m if est == "edge-batch" else B
    cfg = sp.SolverConfig(solver="mu-eg", k=10, eta=eta, steps=steps, eval_every=steps,
                          batch_size=bs, seed=2, eta_schedule=sched)
    t0 = time.perf_counter()
    run = sp.run_solver(g, sp.SpectralTransform("negexp-limit", ell), cfg, record_timing=False,
                        estimator=est)
    V = run.V.cpu().numpy().astype(np.float64)
    dt = time.perf_counter() - t0
    ang = sp.principal_angles(V, U)
    acc = sp.match_labels(sp.kmeans_cluster(V, 10, seed=5), np.arange(n) // 100)
    print(f"{est:10s} ell={ell} B={bs} eta={eta} {sched:8s} steps={steps}: angle {ang:.3e} "
          f"acc {acc:.3f} {dt:.1f}s", flush=True)
