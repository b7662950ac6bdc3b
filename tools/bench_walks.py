"""Walk estimator throughput (walk steps / s) on a BASELINE-shaped graph,
beside the CPU restatement (numpy, one core) on a small sample.

    python tools/bench_walks.py [--config 3] [--walks 1000000] [--ell 16]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2207_14589_b200 as sp  # noqa: E402
from paper_2207_14589_b200 import generators as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--walks", type=int, default=1_000_000)
    ap.add_argument("--ell", type=int, default=16)
    ap.add_argument("--k", type=int, default=1)
    a = ap.parse_args()
    n, u, v, w = G.config_graph(a.config)
    g = sp.Graph(n, u.numpy(), v.numpy(), w.numpy())
    coeffs = np.full(a.ell + 1, 0.1)
    X = torch.randn((n, a.k), dtype=torch.float64, device="cuda")
    from paper_2207_14589_b200.walks import _estimate
    _estimate(g, coeffs, X, list(range(a.k)), a.walks, "importance", "cuda")
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    _estimate(g, coeffs, X, list(range(a.k)), a.walks, "importance", "cuda")
    e.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = s.elapsed_time(e)
    steps = a.walks * a.k * a.ell
    row = {"config": G.CONFIGS[a.config]["name"], "n": n, "m": g.m, "walks": a.walks, "k": a.k,
           "ell": a.ell, "ms_device": ms, "ms_wall_incl_host_keys": wall * 1e3,
           "walk_steps_per_s": steps / (ms / 1e3)}
    print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
