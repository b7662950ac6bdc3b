"""Per-step time of the small-graph solver paths (configs 1-2): CUDA-graph
multi-kernel steps vs the grid-resident K7 kernel.

    python tools/bench_small.py [--steps 2000]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2207_14589_b200 as sp  # noqa: E402
from paper_2207_14589_b200 import generators as G  # noqa: E402
from paper_2207_14589_b200.solvers import _GraphStepper, _PersistentStepper  # noqa: E402

CASES = [(1, "negexp-limit", 13, 0.1), (2, "negexp-limit", 17, 1.0)]


def per_step_us(stepper, steps):
    stepper.advance(10)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    stepper.advance(steps)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2000)
    args = ap.parse_args()
    for cfg, kind, ell, eta in CASES:
        spec = G.CONFIGS[cfg]
        n, u, v, w = G.config_graph(cfg)
        g = sp.Graph(n, u.numpy(), v.numpy(), w.numpy())
        op = sp.make_reversed_operator(g, sp.SpectralTransform(kind, ell), spec["mode"])
        k = spec["k"]
        Vi = op.laplacian.to_internal(sp.init_state(n, k, 1).V)
        row = {"config": spec["name"], "n": n, "nnz": op.laplacian.nnz, "k": k,
               "terms": op.n_terms, "steps": args.steps}
        row["cuda_graph_us_per_step"] = per_step_us(_GraphStepper(op, "mu-eg", eta, Vi), args.steps)
        t0 = time.perf_counter()
        row["persistent_us_per_step"] = per_step_us(_PersistentStepper(op, eta, Vi), args.steps)
        row["oja_cuda_graph_us_per_step"] = per_step_us(_GraphStepper(op, "oja", eta, Vi), args.steps)
        row["oja_persistent_us_per_step"] = per_step_us(_PersistentStepper(op, eta, Vi, "oja"),
                                                        args.steps)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
