"""Graph construction (SURVEY 8a rows a1 + a3) at a BASELINE size: the
reference's host path (numpy lexsort canonicalisation, graph.py:64-88) vs
the device path (sped_canonicalize_edges incl. the H2D copy of the host edge
arrays, then the device CSR build sped_laplacian_build).  The input is the
config's edge list shuffled and randomly re-oriented (non-canonical).

    python tools/bench_graph.py [--config 4]
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
    ap.add_argument("--config", type=int, default=4)
    a = ap.parse_args()
    spec = G.CONFIGS[a.config]
    n, u, v, w = G.config_graph(a.config, device="cuda")
    rng = np.random.default_rng(0)
    u, v, w = u.cpu().numpy(), v.cpu().numpy(), w.cpu().numpy()
    perm = rng.permutation(u.size)
    flip = rng.random(u.size) < 0.5
    uh, vh, wh = np.where(flip, v, u)[perm], np.where(flip, u, v)[perm], w[perm]
    # warm-up (library load, allocator) on a small graph
    sp.Graph(100, np.arange(10), np.arange(1, 11), np.ones(10), device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gd = sp.Graph(n, uh, vh, wh, device="cuda")
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t0
    t0 = time.perf_counter()
    L = sp.LaplacianOperator(gd, spec["mode"], reorder=None)
    torch.cuda.synchronize()
    t_csr = time.perf_counter() - t0
    import os
    os.environ["SPED_GRAPH_HOST"] = "1"  # the reference's numpy path
    t0 = time.perf_counter()
    gh = sp.Graph(n, uh, vh, wh)
    t_host = time.perf_counter() - t0
    del os.environ["SPED_GRAPH_HOST"]
    same = (np.array_equal(gh.u, gd.u) and np.array_equal(gh.v, gd.v)
            and np.array_equal(gh.w, gd.w))
    print(json.dumps({"config": spec["name"], "n": n, "m": int(gh.m),
                      "graph_host_s": t_host, "graph_device_s_incl_h2d": t_dev,
                      "laplacian_csr_device_s": t_csr, "nnz": int(L.nnz),
                      "identical": bool(same), "speedup": t_host / t_dev}), flush=True)


if __name__ == "__main__":
    main()
