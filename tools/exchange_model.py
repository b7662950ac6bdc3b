"""Predicted halo exchange bytes per polynomial term for the row-sharded
configs at P = 2/4/8: contiguous nnz-balanced row partitions of
the operator's internal order, deduplicated halo rows x 4k bytes per rank,
and (power-law config 4) hub-prefix replication of the top H rows.

    python tools/exchange_model.py > profiles/r02_exchange_model.jsonl
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2207_14589_b200 as sp  # noqa: E402
from paper_2207_14589_b200 import generators as G  # noqa: E402
from paper_2207_14589_b200.distributed import exchange_bytes_per_term, partition_rows  # noqa: E402


def main():
    dev = torch.device("cuda")
    for cfg in (3, 4, 5):
        spec = G.CONFIGS[cfg]
        n, u, v, w = G.config_graph(cfg, device=dev)
        g = sp.Graph.from_canonical(n, u, v, w, validate=False)
        L = sp.LaplacianOperator(g, spec["mode"])
        k = spec["k"]
        ip = L.indptr.long()
        idx = L.indices[: L.nnz]
        term_s = None
        for P in (2, 4, 8):
            off = partition_rows(ip, P)
            reps = [0] + ([400_000, 1_000_000] if L.reordered else [])
            for H in reps:
                d = exchange_bytes_per_term(ip, idx, off, k, replicate_rows=H)
                own_nnz = [int(ip[int(off[r + 1])] - ip[int(off[r])]) for r in range(P)]
                rec = {"config": cfg, "P": P, "k": k, "n": n, "nnz": L.nnz,
                       "reordered": L.reordered, "replicate_rows": H,
                       "max_halo_rows": max(x["halo_rows"] for x in d["ranks"]),
                       "max_bytes_per_rank": d["max_bytes_per_rank"],
                       "max_own_nnz": max(own_nnz),
                       "halo_over_own_rows": max(x["halo_rows"] / max(x["own_rows"], 1)
                                                 for x in d["ranks"]),
                       "ms_at_900GBps": d["max_bytes_per_rank"] / 900e9 * 1e3}
                print(json.dumps(rec), flush=True)
        del L, g


if __name__ == "__main__":
    main()
