"""Per-term SpMM timing sweep on one BASELINE config (tuning aid).

    python tools/sweep_spmm.py --config 4 --hot 0.2 0.35 0.5 0.7 --reorder auto none
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2207_14589_b200 as sp  # noqa: E402
from paper_2207_14589_b200 import generators as G, graph as GR  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--hot", type=float, nargs="*", default=[GR.HOT_FRACTION])
    ap.add_argument("--reorder", nargs="*", default=["auto"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--kind", default="negexp-taylor")
    ap.add_argument("--k", type=int, nargs="*", default=None, help="block widths (default: the config's k)")
    a = ap.parse_args()
    spec = G.CONFIGS[a.config]
    dev = torch.device("cuda")
    n, u, v, w = G.config_graph(a.config, device=dev)
    g = sp.Graph.from_canonical(n, u, v, w, validate=False)
    k, ell = spec["k"], spec["ell"]
    t = sp.SpectralTransform(a.kind, ell if a.kind != "negexp-limit" else ell + 1)
    for ro in a.reorder:
      L = sp.LaplacianOperator(g, spec["mode"], reorder=None if ro == "none" else ro)
      op = sp.TransformedOperator(L, t, 0.0, 2.0)
      for k in (a.k or [spec["k"]]):
        X = torch.randn((n, k), device=dev)
        out = torch.empty_like(X)
        for hot in a.hot:
            GR.HOT_FRACTION = hot
            for _ in range(2):
                op.apply_internal(X, out=out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                op.apply_internal(X, out=out)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            print(json.dumps({"config": a.config, "k": k, "reorder": ro, "reordered": L.reordered,
                              "hot_fraction": hot, "hot_rows": L.hot_rows(k), "terms": op.n_terms,
                              "ms_per_apply": ms, "ms_per_term": ms / op.n_terms,
                              "segments": [list(L.segments(k)[1])[:3 * L.segments(k)[0]]]}),
                  flush=True)
        del X, out
      del L, op


if __name__ == "__main__":
    main()
