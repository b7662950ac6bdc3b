"""Config-4 SpMM per-term time vs the row-length segment table (rows sorted
by descending length; each segment picks the nonzero-parallel lane groups
per row, `sub`).  Segments are (min_len_exclusive, sub) from long to short;
rows above the long-row threshold are chunked as usual.

    python tools/sweep_segments.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2207_14589_b200 as sp  # noqa: E402
from paper_2207_14589_b200 import _lib, generators as G  # noqa: E402

VARIANTS = {
    "current": [(64, 4), (0, 1)],
    "w8_512_h4": [(512, 8), (64, 4), (0, 1)],
    "w8_64": [(64, 8), (0, 1)],
    "w8_256_h2_32": [(256, 8), (32, 2), (0, 1)],
    "h4_128_h2_16": [(128, 4), (16, 2), (0, 1)],
    "h4_32": [(32, 4), (0, 1)],
    "h4_128_h1": [(128, 4), (0, 1)],
}


def table(rowlen, thr, spec):
    L = rowlen
    r_long = int(np.searchsorted(-L, -thr, side="left"))
    seg, start = [], r_long
    for lo, sub in spec:
        end = max(int(np.searchsorted(-L, -lo, side="left")), start) if lo > 0 else L.size
        if end > start:
            seg.append((start, end, sub))
        start = end
    return len(seg), _lib.i64_array([x for t in seg for x in t])


def main():
    spec = G.CONFIGS[4]
    dev = torch.device("cuda")
    n, u, v, w = G.config_graph(4, device=dev)
    g = sp.Graph.from_canonical(n, u, v, w, validate=False)
    L = sp.LaplacianOperator(g, spec["mode"])
    op = sp.TransformedOperator(L, sp.SpectralTransform("negexp-taylor", spec["ell"]), 0.0, 2.0)
    X = torch.randn((n, spec["k"]), device=dev)
    out = torch.empty_like(X)
    for rnd in range(2):
        for name, vspec in VARIANTS.items():
            L._segments[32] = table(L.rowlen, L.long_threshold, vspec)
            for _ in range(2):
                op.apply_internal(X, out=out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                op.apply_internal(X, out=out)
            e1.record()
            torch.cuda.synchronize()
            print(json.dumps({"variant": name, "ms_per_term": e0.elapsed_time(e1) / 5 / op.n_terms}),
                  flush=True)


if __name__ == "__main__":
    main()
