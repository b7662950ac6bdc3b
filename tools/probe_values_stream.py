"""What does the CSR values stream cost on config 4?  Times one polynomial
term over the same Chung-Lu graph with stored values (normalized) and with
implicit values (unnormalized, unit weights: -1 / row_len-1 synthesised in
the kernel).  Same sparsity, same gathers; only the 4 B/nnz values stream
and the epilogue constants differ."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2207_14589_b200 as sp  # noqa: E402
from paper_2207_14589_b200 import generators as G  # noqa: E402

n, u, v, w = G.config_graph(4, device="cuda")
g = sp.Graph.from_canonical(n, u, v, w)
k = 32
x = torch.randn(n, k, device="cuda")
for mode in ("normalized", "unnormalized"):
    L = sp.LaplacianOperator(g, mode, device="cuda")
    xi = L.to_internal(x)
    al, be, ga = [1.0] * 12, [1.0] * 12, [0.0] * 12
    for _ in range(2):
        L.poly_apply_internal(xi, al, be, ga, 1.0, 0.0, 1.0)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        L.poly_apply_internal(xi, al, be, ga, 1.0, 0.0, 1.0)
    e.record()
    torch.cuda.synchronize()
    print(json.dumps({"mode": mode, "implicit_values": L.values is None, "nnz": L.nnz,
                      "ms_per_term": s.elapsed_time(e) / 5 / 12}), flush=True)
    del L
    torch.cuda.empty_cache()
