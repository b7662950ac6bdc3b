"""Config-4 SpMM per-term time vs the long-row plan: rows longer than
long_threshold are cut into chunk_len-nonzero chunks (hub-chunk kernel), the
rest of the rows above 64 nonzeros take the warp-per-row kernel.

    python tools/sweep_chunking.py
"""
import itertools
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2207_14589_b200 as sp  # noqa: E402
from paper_2207_14589_b200 import generators as G  # noqa: E402


def main():
    spec = G.CONFIGS[4]
    dev = torch.device("cuda")
    n, u, v, w = G.config_graph(4, device=dev)
    g = sp.Graph.from_canonical(n, u, v, w, validate=False)
    t = sp.SpectralTransform("negexp-taylor", spec["ell"])
    X = torch.randn((n, spec["k"]), device=dev)
    out = torch.empty_like(X)
    import os
    plan = os.environ.get("PLAN", "1024:512,2048:512,4096:512,2048:1024,4096:1024,8192:1024,"
                                  "8192:2048,1024:512")
    for thr, cl in [tuple(int(x) for x in p.split(":")) for p in plan.split(",")]:
        L = sp.LaplacianOperator(g, spec["mode"], long_threshold=thr, chunk_len=cl)
        op = sp.TransformedOperator(L, t, 0.0, 2.0)
        for _ in range(2):
            op.apply_internal(X, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            op.apply_internal(X, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(json.dumps({"long_threshold": thr, "chunk_len": cl, "n_chunks": L.n_chunks,
                          "ms_per_term": ms / op.n_terms}), flush=True)
        del L, op


if __name__ == "__main__":
    main()
