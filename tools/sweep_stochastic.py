"""Stochastic (per-term edge-minibatch) apply timing on a BASELINE config:
device PCG64 draw of ell*B edge ids + the per-term batch kernels.

    python tools/sweep_stochastic.py --config 3
"""
import argparse
import hashlib
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2207_14589_b200 as sp  # noqa: E402
from paper_2207_14589_b200 import generators as G  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    spec = G.CONFIGS[a.config]
    dev = torch.device("cuda")
    n, u, v, w = G.config_graph(a.config, device=dev)
    g = sp.Graph.from_canonical(n, u, v, w, validate=False)
    k, ell, B = spec["k"], spec["ell"], spec["batch"]
    t = sp.SpectralTransform("negexp-limit", ell + 1)
    op = sp.make_reversed_operator(g, t, spec["mode"], device=dev)
    orc = sp.make_stochastic_oracle(op, B, seed=7, estimator="edge-batch")
    torch.manual_seed(0)
    X = torch.randn((n, k), device=dev)
    nt = op.n_terms
    for _ in range(2):
        orc.apply_internal(X)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    draw_ms = apply_ms = 0.0
    for _ in range(a.reps):
        ev[0].record()
        batch = orc.draw(nt * B)
        ev[1].record()
        Y = orc.apply_internal(X, batch=batch)
        ev[2].record()
        torch.cuda.synchronize()
        draw_ms += ev[0].elapsed_time(ev[1])
        apply_ms += ev[1].elapsed_time(ev[2])
    draw_ms /= a.reps
    apply_ms /= a.reps
    print(json.dumps({"config": a.config, "n": n, "nnz": op.laplacian.nnz, "k": k, "terms": nt,
                      "batch": B, "draw_ms_per_apply": draw_ms, "apply_ms": apply_ms,
                      "ms_per_term": apply_ms / nt,
                      "sampled_edges_k_per_s": nt * B * k / (apply_ms / 1e3),
                      # bit pattern of the last apply (A/B builds must agree)
                      "out_hash": hashlib.sha1(Y.cpu().numpy().tobytes()).hexdigest()[:16]}),
          flush=True)


if __name__ == "__main__":
    main()
