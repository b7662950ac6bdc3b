"""SURVEY 8a rows a10 (init_state: Gaussian block + orthonormalisation) and
a14 (k-means on the embedding) at config-3 size (n = 10^6, k = 64; k-means
with 100 clusters), device paths timed on the GPU box.

    python tools/bench_rows_a10_a14.py
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2207_14589_b200 as sp  # noqa: E402


def main():
    n, k = 1_000_000, 64
    sp.init_state(1000, 8, 0)  # warm-up (library, cuBLAS-free path, allocator)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = sp.init_state(n, k, 7)
    V = st.V
    torch.cuda.synchronize() if isinstance(V, torch.Tensor) else None
    t_init = time.perf_counter() - t0
    Vd = torch.as_tensor(V, device="cuda", dtype=torch.float32) if not isinstance(V, torch.Tensor) \
        else V.to("cuda", torch.float32)
    G = (Vd.double().T @ Vd.double()).cpu().numpy()
    orth_err = float(np.abs(G - np.eye(k)).max())
    # k-means: 100 clusters on a 64-dim embedding with planted structure
    rng = np.random.default_rng(0)
    centers = rng.standard_normal((100, k)).astype(np.float32)
    lab = rng.integers(0, 100, n)
    X = torch.as_tensor(centers[lab] + 0.3 * rng.standard_normal((n, k)).astype(np.float32),
                        device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    labels = sp.kmeans_cluster(X, 100, seed=0, max_iter=20)
    t_km = time.perf_counter() - t0
    acc = sp.match_labels(labels, lab)
    print(json.dumps({"n": n, "k": k, "init_state_s": t_init, "init_orthonormality_err": orth_err,
                      "kmeans_clusters": 100, "kmeans_max_iter": 20, "kmeans_s": t_km,
                      "kmeans_match_vs_planted": acc,
                      "reference_note": "SURVEY 8a: init_state 99 s (MGS, n=1e6 k=64); "
                                        "kmeans (n,c,d) broadcast needs 51 GB"}), flush=True)


if __name__ == "__main__":
    main()
