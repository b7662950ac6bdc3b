"""Time the solver-step block kernels at BASELINE sizes on random data:
tcgen05 Gram (sped_gram with M) and the mu-EG update (sped_block_update,
upper-triangular A), for (n, k) in {(1e7, 32), (1e6, 64), (2e6, 128)}.
Checks the Gram against an fp64 torch reference (relative to the largest
entry) so a tuning variant cannot silently break it.

    python tools/bench_gram.py [--reps 20] [--only 32]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2207_14589_b200.solvers import StepWorkspace  # noqa: E402

CASES = [(10_000_000, 32), (1_000_000, 64), (2_000_000, 128)]


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", type=int, default=0)
    args = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    for n, k in CASES:
        if args.only and k != args.only:
            continue
        V = torch.randn(n, k, device="cuda", generator=g) / n ** 0.5
        M = torch.randn(n, k, device="cuda", generator=g) / n ** 0.5
        ws = StepWorkspace(n, k, "cuda")
        gram_ms = timed(lambda: ws.gram(V, M), args.reps)
        Z = torch.cat([V, M], 1).double()
        ref = Z.T @ Z
        G = ws.G.double()
        S, C, Q = G[: k * k].view(k, k), G[k * k: 2 * k * k].view(k, k), G[2 * k * k:].view(k, k)
        err = max((S - ref[:k, :k]).abs().max().item(), (C - ref[:k, k:]).abs().max().item(),
                  (Q.diagonal() - ref[k:, k:].diagonal()).abs().max().item()) / ref.abs().max().item()
        gram_mueg_ms = timed(lambda: ws.gram(V, M, diag_q=True), args.reps)
        G = ws.G.double()
        S, C, Q = G[: k * k].view(k, k), G[k * k: 2 * k * k].view(k, k), G[2 * k * k:].view(k, k)
        err_mueg = max((S - ref[:k, :k]).abs().max().item(), (C - ref[:k, k:]).abs().max().item(),
                       (Q.diagonal() - ref[k:, k:].diagonal()).abs().max().item()) / ref.abs().max().item()
        del Z, ref
        A = torch.triu(torch.randn(k, k, device="cuda", generator=g))
        sc = torch.rand(k, device="cuda", generator=g) + 0.5
        out = torch.empty_like(V)
        upd_ms = timed(lambda: ws.update(V, A, M, None, 0.1, sc, out, upper=True), args.reps)
        ref_u = ((V.double() @ A.double() + 0.1 * M.double()) * sc.double())
        upd_err = ((out.double() - ref_u).norm() / ref_u.norm()).item()
        del ref_u
        gb = 8 * n * k / 1e9
        print(json.dumps({"n": n, "k": k, "gram_ms": gram_ms, "gram_GBps": gb / gram_ms * 1e3,
                          "gram_rel_err": err, "gram_mueg_ms": gram_mueg_ms, "gram_mueg_rel_err": err_mueg, "update_ms": upd_ms, "update_rel_err": upd_err,
                          "update_GBps": 1.5 * gb / upd_ms * 1e3}), flush=True)
        del V, M, out, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
