"""The reference's acceptance criterion 6 (tests/test_acceptance.py:196-220,
arXiv 2207.14589's central claim) on the device: on a 1000-node graph of 5
cliques joined by 25 random edges, negexp-limit(251) reaches the eigenvector
streak k = 5 at least 3x sooner than the identity transform (Oja, eta 3).

    python tools/criterion6.py
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

import paper_2207_14589_b200 as sp  # noqa: E402


def clique_clusters(n=1000, c=5, bridges=25, seed=0):
    size = n // c
    us, vs = [], []
    for b in range(c):
        iu, ju = np.triu_indices(size, k=1)
        us.append(iu + b * size)
        vs.append(ju + b * size)
    rng = np.random.default_rng(seed)
    have = set()
    while len(have) < bridges:
        a, b = rng.integers(0, n, 2)
        if a // size != b // size:
            have.add((min(a, b), max(a, b)))
    br = np.array(sorted(have))
    u = np.concatenate(us + [br[:, 0]])
    v = np.concatenate(vs + [br[:, 1]])
    return sp.Graph(n, u, v, np.ones(u.size))


def steps_to_streak(g, gt, t, solver, k, eta, steps, eval_every):
    cfg = sp.SolverConfig(solver=solver, k=k, eta=eta, steps=steps, eval_every=eval_every,
                          seed=11)
    t0 = time.perf_counter()
    run = sp.run_solver(g, t, cfg, ground_truth=gt, stop_on_targets=True, record_timing=False)
    return run.steps_to_streak, time.perf_counter() - t0


def main():
    g = clique_clusters()
    gt = sp.graph_ground_truth(g)
    s_id, t_id = steps_to_streak(g, gt, sp.SpectralTransform("identity"), "oja", 5, 3.0,
                                 120_000, 500)
    s_251, t_251 = steps_to_streak(g, gt, sp.SpectralTransform("negexp-limit", 251), "oja", 5,
                                   3.0, 20_000, 25)
    print(json.dumps({"graph": "5 cliques x 200 + 25 bridges", "k": 5, "solver": "oja",
                      "eta": 3.0, "identity_steps_to_streak": s_id, "identity_s": t_id,
                      "negexp_limit_251_steps_to_streak": s_251, "negexp_limit_251_s": t_251,
                      "step_ratio": (s_id / s_251) if (s_id and s_251) else None}), flush=True)


if __name__ == "__main__":
    main()
