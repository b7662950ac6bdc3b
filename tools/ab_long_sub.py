"""Same-process interleaved A/B of the lane slices per long row (config 4):
patches the operator's segment table between timings.

    python tools/ab_long_sub.py [--rounds 5]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2207_14589_b200 as sp  # noqa: E402
from paper_2207_14589_b200 import _lib, generators as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    spec = bench.cfg_spec(4)
    k = spec["k"]
    n, u, v, w = G.config_graph(4, device=dev)
    g = sp.Graph.from_canonical(n, u, v, w, validate=False)
    op = sp.make_reversed_operator(g, bench.transform_for(spec), spec["mode"], device=dev)
    lap = op.laplacian
    nseg, seg = lap.segments(k)
    base = [int(seg[i]) for i in range(3 * nseg)]
    x = torch.randn((n, k), device=dev)
    y = torch.empty_like(x)
    nt = len(op.schedule[0])
    out = {}
    for r in range(a.rounds):
        for sub in (4, 2, 8):
            tab = list(base)
            tab[2] = sub  # the long-row segment comes first
            lap._segments[min(k, 128)] = (nseg, _lib.i64_array(tab))
            for _ in range(2):
                op.apply_internal(x, out=y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                op.apply_internal(x, out=y)
            e1.record()
            torch.cuda.synchronize()
            out.setdefault(sub, []).append(round(e0.elapsed_time(e1) / a.reps / nt, 4))
    print(json.dumps({"segment_table": base, "ms_per_term_by_sub": out}))


if __name__ == "__main__":
    main()
