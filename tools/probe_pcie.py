"""Pinned host <-> device copy rate for the e2e step's block (n x k fp32):
one cudaMemcpyAsync against the block split over 2 / 4 streams.

    python tools/probe_pcie.py [--mb 1280]
"""
import argparse
import json
import time

import torch


def rate(fn, nbytes, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t0) / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=1280)
    a = ap.parse_args()
    n = a.mb * 1000 * 1000 // 4
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h.normal_()
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
    out = {"bytes": n * 4}
    for parts in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(parts)]
        cuts = [n * i // parts for i in range(parts + 1)]

        def h2d():
            for s, lo, hi in zip(streams, cuts[:-1], cuts[1:]):
                with torch.cuda.stream(s):
                    d[lo:hi].copy_(h[lo:hi], non_blocking=True)

        def d2h():
            for s, lo, hi in zip(streams, cuts[:-1], cuts[1:]):
                with torch.cuda.stream(s):
                    h2[lo:hi].copy_(d[lo:hi], non_blocking=True)

        def both():
            h2d()
            d2h()

        out[f"h2d_GBps_{parts}"] = rate(h2d, n * 4)
        out[f"d2h_GBps_{parts}"] = rate(d2h, n * 4)
        out[f"duplex_GBps_{parts}"] = rate(both, 2 * n * 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
