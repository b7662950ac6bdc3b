"""Graphs and the device Laplacian operator.

Mirrors the reference ``specgap.graph`` surface used by the hot path
(``/root/reference/pkg/src/specgap/graph.py``):

* :class:`Graph` — canonical edge list with the same validation and error
  messages as ``Graph.__post_init__`` (graph.py:64-88).  Host input is
  canonicalised with numpy exactly as the reference does; generator output
  that is already canonical and lives on the GPU can enter through
  :meth:`Graph.from_canonical` without a host round trip.
* :class:`LaplacianOperator` — the CSR of ``L = D - A`` or
  ``D^-1/2 L D^-1/2`` built ON THE DEVICE by ``sped_laplacian_build``
  (bit-identical to fp32 of scipy's CSR, graph.py:182-199) and applied by the
  fused SpMM kernel (``matvec``, graph.py:205-211).
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Iterable, NamedTuple, Sequence

import numpy as np
import torch

from . import _lib
from .arrays import as_device_block, from_device_block

__all__ = [
    "Graph",
    "LaplacianOperator",
    "DegreeBounds",
    "build_laplacian",
    "laplacian_matvec",
    "dense_laplacian",
    "degree_bounds",
]

_DENSE_MAX_NODES = 5000
LONG_ROW_THRESHOLD = 1024   # floor of the adaptive long-row threshold
CHUNK_LEN = 512


def long_row_plan(nnz: int, sms: int = 148) -> tuple[int, int]:
    """(long_threshold, chunk_len) for the hub-chunk kernel: rows longer than
    the threshold are cut into chunks; shorter rows go to one warp.  The
    threshold follows the per-warp share of the nonzeros (a row no longer
    than ~1/4 of it cannot form a tail), clamped to [1024, 4096]; chunks are
    a quarter of it (>= 512).  Config 4 (1.7e8 nnz): 4096 / 1024, 3.18 ->
    ~3.10 ms/term against 1024 / 512 (tools/sweep_chunking.py)."""
    thr = max(LONG_ROW_THRESHOLD, min(4096, nnz // (sms * 256)))
    return thr, max(CHUNK_LEN, thr // 4)


class Graph:
    """Undirected weighted graph stored as a canonical edge list (u < v,
    lexsorted, unique, w > 0).  Same contract as ``specgap.Graph``."""

    def __init__(self, n: int, u, v, w, *, device=None, _canonical: bool = False):
        """Edges are canonicalised on the GPU (``device``, the CUDA tensors'
        device, or the current one): ``sped_canonicalize_edges`` produces the
        reference's canonical list (graph.py:64-88) bit for bit and raises
        the same ValueErrors.  There is no host path: without CUDA this
        raises (no CPU fallback)."""
        if n < 0:
            raise ValueError("node count must be nonnegative")
        self.n = int(n)
        self._dev = {}
        if _canonical:
            self._u, self._v, self._w = u, v, w
            return
        self._canonicalize_on_device(u, v, w, device)

    def _canonicalize_on_device(self, u, v, w, device):
        import ctypes as C
        if device is None:
            device = next((a.device for a in (u, v, w) if isinstance(a, torch.Tensor) and a.is_cuda),
                          None)
        dev = _lib.require_cuda(device)
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())

        def put(a, dt):
            if isinstance(a, torch.Tensor):
                return a.to(device=dev, dtype=dt).contiguous()
            return torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dt).contiguous()
        u, v, w = put(u, torch.int64), put(v, torch.int64), put(w, torch.float64)
        if not (u.shape == v.shape == w.shape) or u.dim() != 1:
            raise ValueError("edge arrays must have identical length")
        m = int(u.numel())
        u2, v2, w2 = torch.empty_like(u), torch.empty_like(v), torch.empty_like(w)
        mk, st = C.c_int64(0), C.c_int32(0)
        lib = _lib.load()
        rc = lib.sped_canonicalize_edges(self.n, m, _lib.ptr(u), _lib.ptr(v), _lib.ptr(w),
                                         _lib.ptr(u2), _lib.ptr(v2), _lib.ptr(w2), C.byref(mk),
                                         C.byref(st), _lib.stream_ptr(dev))
        _lib.check(rc, "sped_canonicalize_edges")
        st = int(st.value)
        if st & 1:
            raise ValueError("edge weights must be nonnegative")
        if st & 2:
            raise ValueError("self-loops are not allowed")
        if st & 4:
            raise ValueError("edge endpoint out of range")
        if st & 8:
            raise ValueError("duplicate edge for an unordered node pair")
        k = int(mk.value)
        self._u, self._v, self._w = u2[:k], v2[:k], w2[:k]
        self._dev[torch.device(dev)] = (self._u, self._v, self._w)

    # -- construction ------------------------------------------------------
    @classmethod
    def from_edges(cls, n: int, edges: Iterable[Sequence]) -> "Graph":
        us, vs, ws = [], [], []
        for e in edges:
            if len(e) == 2:
                a, b = e
                c = 1.0
            else:
                a, b, c = e
            us.append(a)
            vs.append(b)
            ws.append(c)
        return cls(n, np.array(us, dtype=np.int64), np.array(vs, dtype=np.int64),
                   np.array(ws, dtype=np.float64))

    @classmethod
    def from_canonical(cls, n: int, u, v, w, validate: bool = True) -> "Graph":
        """Wrap an edge list that is already canonical (u < v, strictly
        increasing ``u*n+v``, w > 0) — e.g. generator output on the GPU —
        without the host lexsort.  ``validate`` checks the invariants with
        device-side reductions and raises the reference's errors."""
        if isinstance(u, torch.Tensor):
            u = u.to(torch.int64)
            v = v.to(torch.int64)
            w = w.to(torch.float64)
            if validate and u.numel():
                if bool((w <= 0).any()):
                    raise ValueError("edge weights must be positive in canonical form")
                if bool((u >= v).any()) or bool((u < 0).any()) or bool((v >= n).any()):
                    raise ValueError("canonical edges need 0 <= u < v < n")
                key = u * n + v
                if key.numel() > 1 and bool((key[1:] <= key[:-1]).any()):
                    raise ValueError("canonical edges must be lexsorted without duplicates")
            g = cls(n, u, v, w, _canonical=True)
            if u.is_cuda:
                g._dev[u.device] = (u, v, w)
            return g
        g = cls(n, u, v, w)
        return g

    # -- host views (API parity with specgap.Graph) --------------------------
    def _host(self, a):
        return a.cpu().numpy() if isinstance(a, torch.Tensor) else a

    @property
    def u(self) -> np.ndarray:
        self._u = self._host(self._u)
        return self._u

    @property
    def v(self) -> np.ndarray:
        self._v = self._host(self._v)
        return self._v

    @property
    def w(self) -> np.ndarray:
        self._w = self._host(self._w)
        return self._w

    @property
    def m(self) -> int:
        return int(self._u.shape[0])

    @property
    def num_edges(self) -> int:
        return self.m

    def is_unit_weight(self) -> bool:
        w = self._w
        if isinstance(w, torch.Tensor):
            return bool((w == 1.0).all()) if w.numel() else True
        return bool(np.all(w == 1.0))

    def degrees(self) -> np.ndarray:
        """Weighted degree (graph.py:118-122)."""
        d = np.bincount(self.u, weights=self.w, minlength=self.n)
        d += np.bincount(self.v, weights=self.w, minlength=self.n)
        return d

    def degree_counts(self) -> np.ndarray:
        d = np.bincount(self.u, minlength=self.n)
        d += np.bincount(self.v, minlength=self.n)
        return d

    def neighbors(self, i: int) -> np.ndarray:
        return np.sort(np.concatenate([self.v[self.u == i], self.u[self.v == i]]))

    def has_edge(self, i: int, j: int) -> bool:
        return j in self.neighbors(i)

    def device_edges(self, device):
        """(u int64, v int64, w float64) on ``device`` (cached)."""
        device = torch.device(device)
        hit = self._dev.get(device)
        if hit is None:
            def dev(a, dt):
                if isinstance(a, torch.Tensor):
                    return a.to(device=device, dtype=dt)
                return torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dt)
            hit = (dev(self._u, torch.int64), dev(self._v, torch.int64), dev(self._w, torch.float64))
            self._dev[device] = hit
        return hit

    def __repr__(self) -> str:
        return f"Graph(n={self.n}, m={self.m})"


class DegreeBounds(NamedTuple):
    deg_star: int
    deg_star_inc: int
    lambda_upper: float


def degree_bounds(g: Graph) -> DegreeBounds:
    """graph.py:351-362."""
    if g.n == 0 or g.m == 0:
        return DegreeBounds(0, 0, 0.0)
    deg_star = int(g.degree_counts().max())
    return DegreeBounds(deg_star, 2 * deg_star - 1, 2.0 * float(g.degrees().max()))


L2_BYTES = 126 * 1024 * 1024
HOT_FRACTION = 0.3          # share of L2 held by the hub-prefix persisting window
SKEW_REORDER = 16.0         # max degree / mean degree above which rows are degree-ordered


def segment_table(rowlen: np.ndarray, k: int, sorted_desc: bool, long_threshold):
    """Row ranges of similar length sharing a lanes-per-row choice for the
    SpMM (``sped_csr_poly_apply`` ``segments``).  Rows sorted by descending
    length (degree-ordered graphs) get: long rows (> 64 nonzeros) one warp per
    row, the rest (k/4) lanes per row; chunked rows (> long_threshold) are
    skipped (their own kernel).  Unsorted graphs get one range sized from the
    mean row length.  Returns ``(n_segments, int64 ctypes array)``."""
    n = int(rowlen.size)
    lpr = max(1, min(32, k // 4))
    smax = max(1, 32 // lpr)
    if n == 0:
        seg = []
    elif sorted_desc:
        L = rowlen
        thr = long_threshold if long_threshold is not None else np.iinfo(np.int64).max
        r_long = int(np.searchsorted(-L, -thr, side="left"))    # rows with len > thr
        r_64 = max(int(np.searchsorted(-L, -64, side="left")), r_long)
        seg = []
        if r_64 > r_long:
            # long rows: several lane slices per row.  At k = 32 two slices
            # (8 lanes per row, four rows per warp) beat four: config 4
            # 2.457 -> 2.424 ms/term (profiles/r02_ab_long_sub_cfg4.log)
            seg.append((r_long, r_64, max(1, smax // 2) if k <= 32 else smax))
        if n > r_64:
            seg.append((r_64, n, 1))              # medium/short rows: LPR lanes per row
    else:
        mean = float(rowlen.sum()) / n
        sub = int(os.environ.get("SPED_SUB", "0")) or (smax if mean >= 64 else 1)
        seg = [(0, n, min(sub, smax))]
    flat = [x for t in seg for x in t]
    return len(seg), _lib.i64_array(flat)


class LaplacianOperator:
    """Device CSR Laplacian; ``mode`` in {"unnormalized", "normalized"}.

    Attributes mirror the reference (``graph``, ``mode``, ``degrees`` — host
    fp64, bit-identical to ``Graph.degrees()``) plus the device arrays
    ``indptr``, ``indices``, ``values`` (None for implicit unit-weight
    combinatorial Laplacians), ``epos`` and the long-row plan.

    ``reorder``: ``"auto"`` relabels power-law graphs (max degree >
    SKEW_REORDER x mean) by descending degree, ``"degree"`` always, ``None``
    never.  With a relabelling the device arrays describe ``P L P^T``
    (internal order; ``perm[i]`` = original id of internal row i).  The
    reference-facing ``matvec`` still takes and returns blocks in the
    original order; solver internals work in the internal order
    (``to_internal`` / ``from_internal``).
    """

    def __init__(self, graph: Graph, mode: str = "unnormalized", device=None,
                 long_threshold: int | None = None, chunk_len: int | None = None,
                 implicit: bool | None = None, reorder: str | None = "auto"):
        if mode not in ("unnormalized", "normalized"):
            raise ValueError(f"unknown Laplacian mode: {mode!r}")
        if reorder not in ("auto", "degree", None):
            raise ValueError(f"unknown reorder {reorder!r}")
        dev = _lib.require_cuda(device)
        self.graph = graph
        self.mode = mode
        self.device = dev
        n, m = graph.n, graph.m
        if implicit is None:
            implicit = (mode == "unnormalized") and graph.is_unit_weight()
        self.implicit = bool(implicit)
        u, v, w = graph.device_edges(dev)
        indptr, indices, vals, deg, epos, nnz = self._build(n, m, u, v, w)
        self.degrees = deg[:n].cpu().numpy()
        self.perm = self.iperm = None
        rowlen = np.diff(indptr.cpu().numpy().astype(np.int64))
        mean = float(rowlen.mean()) if n else 0.0
        skewed = n > 0 and mean > 0 and rowlen.max() > SKEW_REORDER * mean
        if reorder == "degree" or (reorder == "auto" and skewed and n >= 4096):
            indptr, indices, vals, epos = self._relabel(n, m, u, v, w, indptr)
        self.indptr, self.nnz = indptr, nnz
        self.indices = indices[: max(nnz, 1)]
        self.values = None if vals is None else vals[: max(nnz, 1)]
        # unit-weight normalized Laplacian without self loops: the SpMM runs
        # terms after the first on u = D^-1/2 w without reading values
        # (row_scale = d^-1/2 in internal order; SPED_SCALED_NORM=0 disables)
        self.row_scale = None
        if (mode == "normalized" and self.values is not None and n > 0
                and os.environ.get("SPED_SCALED_NORM", "1") != "0" and graph.is_unit_weight()
                and not bool((u == v).any())):
            rs = torch.rsqrt(deg[:n].double()).float()
            self.row_scale = rs[self.perm_rows.long()] if self.perm is not None else rs
        self.epos = epos
        self.edge_w = None if graph.is_unit_weight() else w.to(torch.float32)
        self.rowlen = np.diff(self.indptr.cpu().numpy().astype(np.int64))
        self.max_row_nnz = int(self.rowlen.max()) if n else 0
        thr, cl = long_row_plan(self.nnz)
        self.long_threshold = int(long_threshold if long_threshold is not None else thr)
        self.chunk_len = int(chunk_len if chunk_len is not None else cl)
        self._plan()
        self._segments = {}

    # -- construction --------------------------------------------------------
    def _build(self, n, m, u, v, w):
        lib = _lib.load()
        dev = self.device
        cap = 2 * m + n
        indptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
        indices = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
        vals = None if self.implicit else torch.empty(max(cap, 1), dtype=torch.float32, device=dev)
        deg = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        epos = torch.empty(max(2 * m, 1), dtype=torch.int32, device=dev)
        nnz = C.c_int64(0)
        with torch.cuda.device(dev):
            rc = lib.sped_laplacian_build(n, m, _lib.ptr(u), _lib.ptr(v), _lib.ptr(w),
                                          1 if self.mode == "normalized" else 0,
                                          0 if self.implicit else 1,
                                          _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(vals),
                                          _lib.ptr(deg), _lib.ptr(epos), C.byref(nnz),
                                          _lib.stream_ptr(dev))
        _lib.check(rc, "sped_laplacian_build")
        return indptr, indices, vals, deg, epos, int(nnz.value)

    def _relabel(self, n, m, u, v, w, indptr):
        """Degree-descending relabelling: rebuild the CSR of P L P^T and
        re-key epos by ORIGINAL edge id (the stochastic path samples original
        edge ids)."""
        lib = _lib.load()
        dev = self.device
        stream = _lib.stream_ptr(dev)
        perm = torch.empty(n, dtype=torch.int32, device=dev)
        iperm = torch.empty(n, dtype=torch.int32, device=dev)
        _lib.check(lib.sped_degree_order(n, _lib.ptr(indptr), _lib.ptr(perm), _lib.ptr(iperm),
                                         stream), "sped_degree_order")
        u2 = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
        v2 = torch.empty_like(u2)
        w2 = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
        emap = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
        _lib.check(lib.sped_relabel_edges(n, m, _lib.ptr(u), _lib.ptr(v), _lib.ptr(w),
                                          _lib.ptr(iperm), _lib.ptr(u2), _lib.ptr(v2), _lib.ptr(w2),
                                          _lib.ptr(emap), stream), "sped_relabel_edges")
        indptr2, indices2, vals2, _, epos_new, nnz2 = self._build(n, m, u2[:m], v2[:m], w2[:m])
        epos = torch.empty_like(epos_new)
        if m:
            e = emap[:m].long()
            epos.view(-1, 2)[e] = epos_new[: 2 * m].view(-1, 2)
        self.perm, self.iperm = perm, iperm
        self.perm_rows = perm  # gather index: internal row i <- original row perm[i]
        return indptr2, indices2, vals2, epos

    def _plan(self):
        lib = _lib.load()
        n = self.n
        maxc = int(lib.sped_spmm_plan_max_chunks(n, self.nnz, self.long_threshold, self.chunk_len))
        desc = torch.empty(max(4 * maxc, 4), dtype=torch.int32, device=self.device)
        nch, nlong = C.c_int64(0), C.c_int64(0)
        with torch.cuda.device(self.device):
            rc = lib.sped_spmm_plan(n, _lib.ptr(self.indptr), self.long_threshold, self.chunk_len,
                                    _lib.ptr(desc), maxc, C.byref(nch), C.byref(nlong),
                                    _lib.stream_ptr(self.device))
        _lib.check(rc, "sped_spmm_plan")
        self.n_chunks = int(nch.value)
        self.n_long_rows = int(nlong.value)
        self.chunk_desc = desc[: max(4 * self.n_chunks, 4)].clone() if self.n_chunks else None


    @property
    def reordered(self) -> bool:
        return self.perm is not None

    def segments(self, k: int):
        """Row-range table ``[(begin, end, sub), ...]`` for width k (cached)."""
        key = min(k, 128)
        if key not in self._segments:
            self._segments[key] = segment_table(self.rowlen, key, self.reordered,
                                                self.long_threshold if self.n_chunks else None)
        return self._segments[key]

    def hot_rows(self, k: int) -> int:
        if not self.reordered:
            return self.n
        return int(min(self.n, HOT_FRACTION * L2_BYTES / (4 * max(k, 1))))

    # -- ordering ----------------------------------------------------------------
    def to_internal(self, xd: torch.Tensor) -> torch.Tensor:
        """Original-order block -> internal (relabelled) order."""
        if self.perm is None:
            return xd
        return self._gather(xd, self.perm)

    def from_internal(self, yd: torch.Tensor) -> torch.Tensor:
        if self.perm is None:
            return yd
        return self._gather(yd, self.iperm)

    def _gather(self, src: torch.Tensor, rows: torch.Tensor) -> torch.Tensor:
        lib = _lib.load()
        k = 1 if src.dim() == 1 else int(src.shape[1])
        out = torch.empty_like(src)
        rc = lib.sped_gather_rows(self.n, k, _lib.ptr(rows), _lib.ptr(src.contiguous()),
                                  _lib.ptr(out), _lib.stream_ptr(self.device))
        _lib.check(rc, "sped_gather_rows")
        return out

    # -- reference surface ---------------------------------------------------
    @property
    def n(self) -> int:
        return self.graph.n

    def matvec(self, x):
        """``L @ x`` for a vector of length n or an (n, k) block (numpy in ->
        numpy float64 out, torch CUDA in -> torch fp32 out)."""
        shape0 = x.shape[0] if hasattr(x, "shape") and len(x.shape) else None
        if shape0 != self.n:
            raise ValueError(f"dimension mismatch: operator is {self.n}, "
                             f"input has leading dimension {shape0}")
        return self.poly_apply(x, [0.0], [1.0], [0.0], 1.0, 0.0, 1.0)

    __call__ = matvec

    # -- device entry points ---------------------------------------------------
    def poly_apply(self, x, alpha, beta, gamma, w0, lam_f, s_final, out=None):
        """Run a (alpha, beta, gamma) term schedule (see ``sped.h``)."""
        xd, back = as_device_block(x, self.device)
        yd = self.poly_apply_device(xd, alpha, beta, gamma, w0, lam_f, s_final, out=out)
        return from_device_block(yd, back)

    def poly_apply_device(self, xd: torch.Tensor, alpha, beta, gamma, w0, lam_f, s_final,
                          out: torch.Tensor | None = None) -> torch.Tensor:
        """Original-order block in, original-order block out."""
        if self.perm is None:
            return self.poly_apply_internal(xd, alpha, beta, gamma, w0, lam_f, s_final, out=out)
        y = self.poly_apply_internal(self.to_internal(xd), alpha, beta, gamma, w0, lam_f, s_final)
        y = self.from_internal(y)
        if out is not None:
            out.copy_(y)
            return out
        return y

    def poly_apply_internal(self, xd: torch.Tensor, alpha, beta, gamma, w0, lam_f, s_final,
                            out: torch.Tensor | None = None) -> torch.Tensor:
        lib = _lib.load()
        n = self.n
        k = 1 if xd.dim() == 1 else int(xd.shape[1])
        nt = len(alpha)
        if out is None:
            out = torch.empty_like(xd)
        wa = torch.empty_like(xd) if nt >= 2 else None
        wb = torch.empty_like(xd) if nt >= 3 else None
        # per-call chunk scratch (partial rows and arrival tickets), so one
        # operator can be applied from several threads / streams at once
        partials = (torch.empty(self.n_chunks * min(k, 128), dtype=torch.float32, device=self.device)
                    if self.n_chunks else None)
        tickets = (torch.zeros(self.n_chunks, dtype=torch.int32, device=self.device)
                   if self.n_chunks else None)
        nseg, seg = self.segments(k)
        with torch.cuda.device(self.device):
            rc = lib.sped_csr_poly_apply(
                n, k, _lib.ptr(self.indptr), _lib.ptr(self.indices), _lib.ptr(self.values),
                self.long_threshold, self.chunk_len, _lib.ptr(self.chunk_desc), self.n_chunks,
                _lib.ptr(partials), _lib.ptr(tickets), seg, nseg, self.hot_rows(k),
                _lib.ptr(self.row_scale), _lib.ptr(xd), None, _lib.ptr(wa), _lib.ptr(wb),
                _lib.ptr(out), nt,
                _lib.dbl_array(alpha), _lib.dbl_array(beta), _lib.dbl_array(gamma), float(w0),
                float(lam_f), float(s_final), _lib.stream_ptr(self.device))
        _lib.check(rc, "sped_csr_poly_apply")
        return out

    def csr_host(self, original_order: bool = True):
        """(indptr, indices, data) as numpy (data fp32; implicit values are
        materialised).  For a relabelled operator the ORIGINAL-order CSR is
        rebuilt on the device (the exact sped_laplacian_build output)."""
        if original_order and self.perm is not None:
            u, v, w = self.graph.device_edges(self.device)
            indptr, indices, vals, _, _, nnz = self._build(self.n, self.graph.m, u, v, w)
            return self._host_arrays(indptr, indices[:nnz], None if vals is None else vals[:nnz])
        return self._host_arrays(self.indptr, self.indices[: self.nnz],
                                 None if self.values is None else self.values[: self.nnz])

    def _host_arrays(self, indptr_d, indices_d, vals_d):
        indptr = indptr_d.cpu().numpy()
        indices = indices_d.cpu().numpy()
        if vals_d is not None:
            data = vals_d.cpu().numpy()
        else:
            rows = np.repeat(np.arange(self.n), np.diff(indptr))
            rl = np.diff(indptr)[rows]
            data = np.where(indices == rows, rl - 1, -1).astype(np.float32)
        return indptr, indices, data


def build_laplacian(g: Graph, mode: str = "unnormalized", device=None) -> LaplacianOperator:
    return LaplacianOperator(g, mode, device=device)


def laplacian_matvec(op: LaplacianOperator, x):
    return op.matvec(x)


def dense_laplacian(g: Graph, mode: str = "unnormalized", device=None) -> np.ndarray:
    """Dense Laplacian (desk scale only, graph.py:224-229): densified from the
    device CSR (fp32 values, returned as float64)."""
    if g.n > _DENSE_MAX_NODES:
        raise ValueError(f"dense Laplacian refused for n={g.n} (limit {_DENSE_MAX_NODES})")
    op = build_laplacian(g, mode, device=device)
    indptr, indices, data = op.csr_host()
    out = np.zeros((g.n, g.n))
    rows = np.repeat(np.arange(g.n), np.diff(indptr))
    out[rows, indices] = data
    return out
