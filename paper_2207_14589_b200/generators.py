"""Seeded synthetic graph families for the BASELINE configurations.

The reference ships none of these (SURVEY §0 finding 5: "general stochastic
block model sampling" is a non-goal); they exist so the bench
and the parity tests have config-shaped inputs.  Each generator returns a
canonical edge list ``(n, u, v, w)`` — ``u < v``, lexsorted, unique, no
self-loops — built with torch so that the 10^7-node families are generated on
the device in seconds (``device="cuda"``) and the small parity cases on the
host (``device="cpu"``).  The same edge arrays are fed to the CPU oracle and to
the CUDA path, so generator RNG streams never enter a parity comparison.

Config map (BASELINE.json ``configs``):
  1 ``sbm_dense(10, 100, 0.1, 0.002)``             combinatorial, unweighted
  2 ``grid_rooms(100)``                            normalized, unweighted
  3 ``sbm_sparse(10**6, 100, 20.0, 0.9)``          combinatorial, unweighted
  4 ``chung_lu(10**7, 2.1, 2.0, 16.0, 1e5)``       normalized, unweighted
  5 ``lp_sbm(2*10**6, 200, 24.0, 0.1, 5, 0.8)``    combinatorial, weighted
"""

from __future__ import annotations

import math

import torch

__all__ = [
    "canonicalize_pairs",
    "sbm_dense",
    "sbm_sparse",
    "grid_rooms",
    "chung_lu",
    "lp_sbm",
    "config_graph",
    "CONFIGS",
]


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def canonicalize_pairs(n: int, a: torch.Tensor, b: torch.Tensor,
                       w: torch.Tensor | None = None):
    """Drop self-loops, orient ``u < v``, sort lexicographically, drop
    duplicate pairs (first weight wins).  Returns int64 ``u, v`` and float64
    ``w`` on the input device."""
    a = a.to(torch.int64)
    b = b.to(torch.int64)
    keep = a != b
    a, b = a[keep], b[keep]
    if w is not None:
        w = w[keep]
    lo = torch.minimum(a, b)
    hi = torch.maximum(a, b)
    key = lo * n + hi
    if w is None:
        key = torch.unique(key, sorted=True)
        wout = torch.ones(key.numel(), dtype=torch.float64, device=key.device)
    else:
        key, order = torch.sort(key, stable=True)
        w = w[order]
        first = torch.ones_like(key, dtype=torch.bool)
        first[1:] = key[1:] != key[:-1]
        key = key[first]
        wout = w[first].to(torch.float64)
    return key // n, key % n, wout


def sbm_dense(blocks: int, size: int, p_in: float, p_out: float, seed: int = 1,
              device="cpu"):
    """Config 1: Bernoulli over all pairs (desk scale only)."""
    n = blocks * size
    g = _gen(seed, device)
    iu = torch.triu_indices(n, n, offset=1, device=device)
    same = (iu[0] // size) == (iu[1] // size)
    p = torch.where(same, torch.tensor(p_in, device=device),
                    torch.tensor(p_out, device=device))
    keep = torch.rand(iu.shape[1], generator=g, device=device) < p
    u, v = iu[0][keep], iu[1][keep]
    return n, u, v, torch.ones(u.numel(), dtype=torch.float64, device=device)


def sbm_sparse(n: int, blocks: int, mean_degree: float, intra_frac: float,
               seed: int = 3, device="cpu"):
    """Config 3: ``n*mean_degree/2`` edge draws, ``intra_frac`` of them inside
    a uniformly chosen block; duplicates and self-loops removed."""
    g = _gen(seed, device)
    size = n // blocks
    m = int(round(n * mean_degree / 2))
    m_in = int(round(m * intra_frac))
    m_out = m - m_in
    blk = torch.randint(0, blocks, (m_in,), generator=g, device=device)
    a_in = blk * size + torch.randint(0, size, (m_in,), generator=g, device=device)
    b_in = blk * size + torch.randint(0, size, (m_in,), generator=g, device=device)
    a_out = torch.randint(0, n, (m_out,), generator=g, device=device)
    ba = a_out // size
    shift = torch.randint(1, blocks, (m_out,), generator=g, device=device)
    bb = (ba + shift) % blocks
    b_out = bb * size + torch.randint(0, size, (m_out,), generator=g, device=device)
    u, v, w = canonicalize_pairs(n, torch.cat([a_in, a_out]), torch.cat([b_in, b_out]))
    return n, u, v, w


def grid_rooms(side: int = 100, device="cpu"):
    """Config 2: ``side x side`` 4-neighbour grid split into 4 rooms by two
    full-length walls (a vertical and a horizontal cut through the middle,
    realised as removed edges).  Each wall keeps one 1-cell doorway per
    half-wall so the rooms stay connected (SURVEY §8d note (iii))."""
    n = side * side
    mid = side // 2
    r = torch.arange(side, device=device)
    rr, cc = torch.meshgrid(r, r, indexing="ij")
    node = rr * side + cc
    # horizontal neighbours (r, c)-(r, c+1)
    hu = node[:, :-1].reshape(-1)
    hv = node[:, 1:].reshape(-1)
    hrow = rr[:, :-1].reshape(-1)
    hcol = cc[:, :-1].reshape(-1)
    # vertical wall between columns mid-1 and mid, doors at rows mid//2 and mid+mid//2
    hcut = (hcol == mid - 1) & (hrow != mid // 2) & (hrow != mid + mid // 2)
    # vertical neighbours (r, c)-(r+1, c)
    vu = node[:-1, :].reshape(-1)
    vv = node[1:, :].reshape(-1)
    vrow = rr[:-1, :].reshape(-1)
    vcol = cc[:-1, :].reshape(-1)
    vcut = (vrow == mid - 1) & (vcol != mid // 2) & (vcol != mid + mid // 2)
    a = torch.cat([hu[~hcut], vu[~vcut]])
    b = torch.cat([hv[~hcut], vv[~vcut]])
    u, v, w = canonicalize_pairs(n, a, b)
    return n, u, v, w


def chung_lu(n: int, exponent: float = 2.1, d_min: float = 2.0,
             mean_degree: float = 16.0, cap: float = 1e5, seed: int = 4,
             device="cpu"):
    """Config 4: Chung-Lu graph with Pareto expected degrees (density exponent
    ``exponent``, minimum ``d_min``, capped at ``cap``, rescaled to
    ``mean_degree``).  ``n*mean_degree/2`` endpoint pairs are drawn
    proportionally to the expected degrees; self-loops and duplicates are
    dropped.  Every node left isolated gets one edge to a uniformly random
    node, so the normalized Laplacian is defined (SURVEY §8d note (iv)).
    Node labels are a random permutation (no locality by construction)."""
    g = _gen(seed, device)
    shape = exponent - 1.0
    uu = torch.rand(n, generator=g, device=device, dtype=torch.float64)
    wts = d_min * torch.pow(1.0 - uu, -1.0 / shape)
    wts = torch.clamp(wts, max=cap)
    wts = wts * (mean_degree / wts.mean())
    m = int(round(n * mean_degree / 2))
    cdf = torch.cumsum(wts, 0)
    cdf = cdf / cdf[-1]
    perm = torch.randperm(n, generator=g, device=device)
    a = torch.empty(0, dtype=torch.int64, device=device)
    b = torch.empty(0, dtype=torch.int64, device=device)
    # hubs collide often, so top the unique edge count up to m in rounds and
    # drop a uniform random excess at the end (keeps the degree law)
    for _ in range(6):
        need = m - a.numel()
        if need <= 0:
            break
        draw = int(need * 1.25) + 16
        ends = torch.searchsorted(cdf, torch.rand(2 * draw, generator=g, device=device,
                                                  dtype=torch.float64)).clamp_(max=n - 1)
        ends = perm[ends]
        u_, v_, _ = canonicalize_pairs(n, torch.cat([a, ends[:draw]]),
                                       torch.cat([b, ends[draw:]]))
        a, b = u_, v_
    if a.numel() > m:
        sel = torch.randperm(a.numel(), generator=g, device=device)[:m]
        sel, _ = torch.sort(sel)
        a, b = a[sel], b[sel]
    deg = torch.zeros(n, dtype=torch.int64, device=device)
    deg.scatter_add_(0, a, torch.ones_like(a))
    deg.scatter_add_(0, b, torch.ones_like(b))
    iso = torch.nonzero(deg == 0).flatten()
    if iso.numel():
        other = torch.randint(0, n - 1, (iso.numel(),), generator=g, device=device)
        other = other + (other >= iso).to(other.dtype)
        a = torch.cat([a, iso])
        b = torch.cat([b, other])
    u, v, w = canonicalize_pairs(n, a, b)
    return n, u, v, w


def lp_sbm(n: int, blocks: int, mean_degree: float, drop_frac: float,
           candidates: int, cand_intra: float, seed: int = 5, device="cpu"):
    """Config 5: "link-prediction-filled" SBM.  Start from an SBM with
    ``mean_degree`` (90% intra-block), drop ``drop_frac`` of its edges
    uniformly, then add ``candidates`` candidate edges per node
    (``cand_intra`` intra-block), every edge weighted U(0,1) and rounded to
    fp32 so both paths consume identical weights (SURVEY §8d "Weights")."""
    g = _gen(seed, device)
    _, u0, v0, _ = sbm_sparse(n, blocks, mean_degree, 0.9, seed=seed + 1000, device=device)
    keep = torch.rand(u0.numel(), generator=g, device=device) >= drop_frac
    u0, v0 = u0[keep], v0[keep]
    size = n // blocks
    src = torch.arange(n, device=device).repeat_interleave(candidates)
    intra = torch.rand(src.numel(), generator=g, device=device) < cand_intra
    blk = src // size
    other_blk = (blk + torch.randint(1, blocks, (src.numel(),), generator=g, device=device)) % blocks
    tb = torch.where(intra, blk, other_blk)
    dst = tb * size + torch.randint(0, size, (src.numel(),), generator=g, device=device)
    a = torch.cat([u0, src])
    b = torch.cat([v0, dst])
    w = torch.rand(a.numel(), generator=g, device=device, dtype=torch.float32)
    w = torch.where(w == 0, torch.full_like(w, 0.5), w).to(torch.float64)
    u, v, ww = canonicalize_pairs(n, a, b, w)
    return n, u, v, ww


CONFIGS = {
    1: dict(name="cfg1-sbm1k", mode="unnormalized", k=10, ell=8,
            gen=lambda device="cpu", scale=1.0: sbm_dense(10, 100, 0.1, 0.002, device=device)),
    2: dict(name="cfg2-grid4rooms", mode="normalized", k=16, ell=16,
            gen=lambda device="cpu", scale=1.0: grid_rooms(100, device=device)),
    3: dict(name="cfg3-sbm1M", mode="unnormalized", k=64, ell=16, batch=1_000_000,
            gen=lambda device="cpu", scale=1.0: sbm_sparse(
                int(10**6 * scale) // 100 * 100, 100, 20.0, 0.9, device=device)),
    4: dict(name="cfg4-chunglu10M", mode="normalized", k=32, ell=12,
            gen=lambda device="cpu", scale=1.0: chung_lu(
                int(10**7 * scale), 2.1, 2.0, 16.0, 1e5, device=device)),
    5: dict(name="cfg5-lpsbm2M", mode="unnormalized", k=128, ell=20, batch=4_000_000,
            gen=lambda device="cpu", scale=1.0: lp_sbm(
                int(2 * 10**6 * scale) // 200 * 200, 200, 24.0, 0.1, 5, 0.8, device=device)),
}


def config_graph(cfg: int, device="cpu", scale: float = 1.0):
    """Edge arrays for BASELINE config ``cfg`` (1-based), optionally scaled
    down in node count for parity tests (``scale < 1``)."""
    return CONFIGS[cfg]["gen"](device=device, scale=scale)


def _expected_edges(n, mean_degree):  # pragma: no cover - documentation helper
    return int(math.ceil(n * mean_degree / 2))
