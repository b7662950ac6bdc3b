"""Walk-based polynomial estimator on the device (walks.py).

Mirrors the reference's ``SamplerConfig`` / ``estimate_power_matvec`` /
``estimate_polynomial_matvec`` (walks.py:63-341) and the walk oracle of
``make_stochastic_oracle`` (solvers.py:183-200).  The walks are the
reference's own, bit for bit: the Philox keys come from
``SeedSequence((seed, chunk))`` on the host exactly as walks.py:196-198
derives them, and the kernel (csrc/walks.cu) replays numpy's draw order;
values are fp64 and agree to fp64 rounding.  ``n_walkers`` only affects the
reference's thread count, never its result, and is accepted and ignored.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .arrays import is_device_array
from .graph import Graph, degree_bounds

__all__ = ["SamplerConfig", "estimate_power_matvec", "estimate_polynomial_matvec",
           "WalkOracle", "WALK_CHUNK"]

WALK_CHUNK = 8192  # walks.py:45


@dataclass(frozen=True)
class SamplerConfig:
    """walks.py:63-80."""

    ell: int
    walks_per_estimate: int
    n_walkers: int = 1
    mode: str = "importance"
    seed: int = 0

    def __post_init__(self):
        if self.ell < 1:
            raise ValueError("walk length must be at least 1")
        if self.walks_per_estimate < 1:
            raise ValueError("need at least one walk per estimate")
        if self.mode not in ("importance", "rejection"):
            raise ValueError(f"unknown sampler mode {self.mode!r}")
        if self.n_walkers < 1:
            raise ValueError("n_walkers must be positive")
        if self.seed < 0:
            raise ValueError("seed must be a nonnegative integer")


def chunk_keys(seed: int, walks: int) -> np.ndarray:
    """Philox keys of the estimate's chunks (walks.py:196-198), uint64[n_chunks, 2]."""
    n_chunks = -(-walks // WALK_CHUNK)
    return np.stack([np.random.SeedSequence((seed, c)).generate_state(2, np.uint64)
                     for c in range(n_chunks)])


class _WalkIndex:
    """Device incidence index of a graph: the u-runs of the lexsorted edge
    list and the v-runs of a stable sort by v (csrc/walks.cu)."""

    def __init__(self, g: Graph, device):
        lib = _lib.load()
        self.device = torch.device(device)
        self.g = g
        self.u, self.v, self.w = g.device_edges(self.device)
        n, m = g.n, g.m
        self.up_start = torch.empty(n + 1, dtype=torch.int32, device=self.device)
        self.lo_start = torch.empty(n + 1, dtype=torch.int32, device=self.device)
        self.sorted_e = torch.empty(max(m, 1), dtype=torch.int32, device=self.device)
        nbytes = int(lib.sped_walk_index_workspace_bytes(n, m))
        ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        rc = lib.sped_walk_index_build(n, m, _lib.ptr(self.u), _lib.ptr(self.v),
                                       _lib.ptr(self.up_start), _lib.ptr(self.lo_start),
                                       _lib.ptr(self.sorted_e), _lib.ptr(ws), nbytes,
                                       _lib.stream_ptr(self.device))
        _lib.check(rc, "sped_walk_index_build")
        self.deg_star_inc = degree_bounds(g).deg_star_inc


_INDEX_CACHE: dict = {}


def _index(g: Graph, device) -> _WalkIndex:
    key = (id(g), str(torch.device(device)))
    hit = _INDEX_CACHE.get(key)
    if hit is None or hit.g is not g:
        if g.m == 0:
            raise ValueError("edge incidence graph undefined for an edgeless graph")
        hit = _WalkIndex(g, device)
        _INDEX_CACHE[key] = hit
    return hit


def _estimate(g: Graph, coeffs: np.ndarray, X: torch.Tensor, seeds, walks: int, mode: str,
              device) -> torch.Tensor:
    """Device estimate for the columns of X (n x k fp64, CUDA), column j with
    seed seeds[j]; returns n x k fp64."""
    lib = _lib.load()
    idx = _index(g, device)
    n, k = int(X.shape[0]), int(X.shape[1])
    ell = coeffs.size - 1
    keys = np.concatenate([chunk_keys(int(s), walks) for s in seeds])
    keys_d = torch.from_numpy(keys.astype(np.uint64).view(np.int64)).to(idx.device)
    out = torch.empty_like(X)
    nbytes = int(lib.sped_walk_workspace_bytes(n, k, walks))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=idx.device)
    rc = lib.sped_walk_poly_estimate(n, g.m, k, _lib.ptr(idx.u), _lib.ptr(idx.v), _lib.ptr(idx.w),
                                     _lib.ptr(idx.up_start), _lib.ptr(idx.lo_start),
                                     _lib.ptr(idx.sorted_e), ell, _lib.dbl_array(coeffs),
                                     0 if mode == "importance" else 1, idx.deg_star_inc, walks,
                                     _lib.ptr(keys_d), _lib.ptr(X), _lib.ptr(out), _lib.ptr(ws),
                                     nbytes, _lib.stream_ptr(idx.device))
    _lib.check(rc, "sped_walk_poly_estimate")
    return out


def _as_fp64_block(v, n, device):
    if is_device_array(v):
        t = v.to(device=device, dtype=torch.float64)
        back = "device"
    else:
        t = torch.as_tensor(np.asarray(v, dtype=np.float64), device=device)
        back = "host"
    if t.shape[0] != n:
        raise ValueError("vector length must match the node count")
    return t, back


def estimate_polynomial_matvec(g: Graph, coeffs, v, cfg: SamplerConfig, device=None):
    """walks.py:311-341: ``sum_i coeffs[i] L^i v`` from one walk per sample,
    every prefix reused."""
    coeffs = np.asarray(coeffs, dtype=np.float64)
    if coeffs.ndim != 1 or coeffs.size < 1:
        raise ValueError("coeffs must be a nonempty 1-D sequence")
    dev = _lib.require_cuda(device)
    vt, back = _as_fp64_block(v, g.n, dev)
    if vt.dim() != 1:
        raise ValueError("vector length must match the node count")
    if cfg.mode == "rejection":
        raise ValueError("rejection mode estimates single powers only; "
                         "polynomials use importance weighting")
    out = coeffs[0] * vt
    if coeffs.size == 1 or not np.any(coeffs[1:]):
        return out.cpu().numpy() if back == "host" else out
    y = _estimate(g, coeffs, vt[:, None].contiguous(), [cfg.seed], cfg.walks_per_estimate,
                  "importance", dev)[:, 0]
    return y.cpu().numpy() if back == "host" else y


def estimate_power_matvec(g: Graph, ell: int, v, cfg: SamplerConfig, device=None):
    """walks.py:276-308: Monte Carlo ``L^ell v`` (importance or rejection)."""
    if ell < 1:
        raise ValueError("power must be at least 1")
    dev = _lib.require_cuda(device)
    vt, back = _as_fp64_block(v, g.n, dev)
    if vt.dim() != 1:
        raise ValueError("vector length must match the node count")
    coeffs = np.zeros(ell + 1)
    coeffs[ell] = 1.0
    y = _estimate(g, coeffs, vt[:, None].contiguous(), [cfg.seed], cfg.walks_per_estimate,
                  cfg.mode, dev)[:, 0]
    if cfg.mode == "rejection" and not bool(torch.any(y != 0)) and bool(torch.any(vt != 0)):
        raise RuntimeError("no walk survived rejection; increase "
                           "walks_per_estimate or use importance mode")
    return y.cpu().numpy() if back == "host" else y


class WalkOracle:
    """The walk oracle of make_stochastic_oracle (solvers.py:183-200): every
    column of every call is one importance estimate of f(L)x_j with
    ``walks`` walks, seeded SeedSequence((seed, counter)).generate_state(1)[0]
    with the counter running over columns and calls; returns
    ``lambda* x - f(L) x``."""

    def __init__(self, op, walks: int, seed: int):
        from .transforms import polynomial_coefficients
        self.op = op
        self.walks = int(walks)
        self.seed = int(seed)
        self.counter = 0
        self.coeffs = np.asarray(polynomial_coefficients(op.transform), dtype=np.float64)
        self.device = op.laplacian.device

    @property
    def n(self) -> int:
        return self.op.n

    def _seeds(self, k):
        s = [int(np.random.SeedSequence((self.seed, self.counter + j)).generate_state(1)[0])
             for j in range(k)]
        self.counter += k
        return s

    def apply_device(self, X: torch.Tensor) -> torch.Tensor:
        Xd = X.to(torch.float64)
        cols = Xd[:, None] if Xd.dim() == 1 else Xd
        lam = float(self.op.lambda_star)
        g = self.op.laplacian.graph
        if self.coeffs.size == 1 or not np.any(self.coeffs[1:]):
            self._seeds(cols.shape[1])
            fx = self.coeffs[0] * cols
        else:
            fx = _estimate(g, self.coeffs, cols.contiguous(), self._seeds(cols.shape[1]),
                           self.walks, "importance", self.device)
        out = lam * cols - fx
        out = out[:, 0] if Xd.dim() == 1 else out
        return out.to(X.dtype)

    def apply_internal(self, X: torch.Tensor) -> torch.Tensor:
        """The solver's internal (relabelled) row order in and out; the walks
        run on the reference's node ids."""
        lap = self.op.laplacian
        if not lap.reordered:
            return self.apply_device(X)
        return lap.to_internal(self.apply_device(lap.from_internal(X)))

    def __call__(self, x):
        if is_device_array(x):
            return self.apply_device(x)
        xd = torch.as_tensor(np.asarray(x, dtype=np.float64), device=self.device)
        if xd.shape[0] != self.n:
            raise ValueError("dimension mismatch in transformed matvec")
        return self.apply_device(xd).cpu().numpy()
