"""Seeded edge minibatches and the stochastic (edge-minibatch) oracle.

The reference draws ``rng.integers(0, m, size=B)`` from a numpy PCG64
generator created once per oracle (solvers.py:167,171).  Here the same
indices are produced either

* on the device by ``sped_pcg64_integers_device`` (bit-exact numpy PCG64 +
  Lemire, the default) with the generator state kept in device memory and
  advanced there (no host synchronisation, CUDA-graph capturable); the host
  ``Generator`` is re-synchronised from it lazily (``DeviceGenerator``), or
* on the host by the numpy generator itself (``index_source="host"``),
  uploaded through pinned memory.

Both are bit-identical to the reference stream; a whole apply's ``ell`` term
batches are one draw of ``ell*B`` values (numpy's buffered uint32 carries
across calls, so consecutive calls concatenate).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .arrays import as_device_block, from_device_block

__all__ = ["pcg64_draw", "host_draw", "EdgeBatchOracle", "pcg64_advance_state",
           "DeviceGenerator"]

_MULT = (2549297995355413924 << 64) | 4865540595714422341
_M128 = (1 << 128) - 1
_M64 = (1 << 64) - 1


def _advance(state: int, inc: int, delta: int) -> int:
    acc_mult, acc_plus = 1, 0
    cur_mult, cur_plus = _MULT, inc
    while delta > 0:
        if delta & 1:
            acc_mult = (acc_mult * cur_mult) & _M128
            acc_plus = (acc_plus * cur_mult + cur_plus) & _M128
        cur_plus = ((cur_mult + 1) * cur_plus) & _M128
        cur_mult = (cur_mult * cur_mult) & _M128
        delta >>= 1
    return (acc_mult * state + acc_plus) & _M128


def _output(state: int) -> int:
    hi, lo = state >> 64, state & _M64
    rot = hi >> 58
    x = hi ^ lo
    return ((x >> rot) | (x << ((64 - rot) & 63))) & _M64


def pcg64_advance_state(st: dict, draws32: int) -> dict:
    """numpy PCG64 state after ``draws32`` calls of next_uint32."""
    if draws32 <= 0:
        return st
    s = st["state"]["state"]
    inc = st["state"]["inc"]
    has = st["has_uint32"]
    uint = st["uinteger"]
    r = draws32 - (1 if has else 0)
    if r <= 0:
        has = 0
    else:
        steps = (r + 1) // 2
        s = _advance(s, inc, steps)
        has = r % 2
        uint = _output(s) >> 32
    return {"bit_generator": "PCG64", "state": {"state": s, "inc": inc},
            "has_uint32": int(has), "uinteger": int(uint)}


def pcg64_draw(rng: np.random.Generator, m: int, count: int, device) -> torch.Tensor:
    """``rng.integers(0, m, size=count)`` generated on the device (int32),
    advancing ``rng`` exactly as numpy would."""
    if m <= 0:
        raise ValueError("high <= 0")
    if m > np.iinfo(np.int32).max:
        raise ValueError("edge count exceeds int32 indices")
    st = rng.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise ValueError("device draws need a PCG64 generator")
    lib = _lib.load()
    out = torch.empty(max(count, 1), dtype=torch.int32, device=device)
    nbytes = int(lib.sped_pcg64_workspace_bytes(count))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
    s = st["state"]["state"]
    inc = st["state"]["inc"]
    draws = C.c_int64(0)
    rc = lib.sped_pcg64_integers(s >> 64, s & _M64, inc >> 64, inc & _M64,
                                 int(st["has_uint32"]), int(st["uinteger"]), int(m), int(count),
                                 _lib.ptr(out), C.byref(draws), _lib.ptr(ws), nbytes,
                                 _lib.stream_ptr(device))
    _lib.check(rc, "sped_pcg64_integers")
    rng.bit_generator.state = pcg64_advance_state(st, int(draws.value))
    return out[:count]


def _state_words(st: dict) -> np.ndarray:
    s, inc = st["state"]["state"], st["state"]["inc"]
    return np.array([s >> 64, s & _M64, inc >> 64, inc & _M64, int(st["has_uint32"]),
                     int(st["uinteger"])], dtype=np.uint64)


def _words_state(w: np.ndarray) -> dict:
    w = [int(x) for x in np.asarray(w, dtype=np.uint64)]
    return {"bit_generator": "PCG64", "state": {"state": (w[0] << 64) | w[1],
                                                "inc": (w[2] << 64) | w[3]},
            "has_uint32": int(w[4]), "uinteger": int(w[5])}


class DeviceGenerator:
    """A numpy ``Generator(PCG64)`` whose state lives on the device between
    draws.  ``integers(m, count)`` runs ``sped_pcg64_integers_device``: the
    same values and the same state evolution as ``rng.integers(0, m, count)``
    (solvers.py:171), with no host round trip.  ``rng`` returns the host
    Generator re-synchronised from the device words (one small D2H copy);
    touching it hands authority back to the host until the next draw."""

    def __init__(self, rng: np.random.Generator, device):
        if rng.bit_generator.state.get("bit_generator") != "PCG64":
            raise ValueError("device draws need a PCG64 generator")
        self._rng = rng
        self.device = torch.device(device)
        self._words = torch.empty(6, dtype=torch.int64, device=self.device)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._ws = torch.empty(0, dtype=torch.uint8, device=self.device)
        self._where = "host"  # which copy of the state is current

    @property
    def rng(self) -> np.random.Generator:
        if self._where == "device":
            self._rng.bit_generator.state = _words_state(self._words.cpu().numpy().view(np.uint64))
            self.check()
        self._where = "host"
        return self._rng

    def to_device(self):
        """Make the device words the current state (upload if the host copy
        is current)."""
        if self._where == "host":
            w = _state_words(self._rng.bit_generator.state).view(np.int64)
            self._words.copy_(torch.from_numpy(w))
            self._where = "device"

    def snapshot(self) -> torch.Tensor:
        self.to_device()
        return self._words.clone()

    def restore(self, words: torch.Tensor):
        self._words.copy_(words)
        self._where = "device"

    def check(self):
        if int(self.status.item()) & 1:
            raise RuntimeError("pcg64: candidate pool exhausted")

    def integers(self, m: int, count: int) -> torch.Tensor:
        if m <= 0:
            raise ValueError("high <= 0")
        if m > np.iinfo(np.int32).max:
            raise ValueError("edge count exceeds int32 indices")
        self.to_device()
        lib = _lib.load()
        out = torch.empty(max(count, 1), dtype=torch.int32, device=self.device)
        nbytes = int(lib.sped_pcg64_workspace_bytes(count))
        if self._ws.numel() < nbytes:
            self._ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            rc = lib.sped_pcg64_integers_device(_lib.ptr(self._words), int(m), int(count),
                                                _lib.ptr(out), _lib.ptr(self.status),
                                                _lib.ptr(self._ws), self._ws.numel(),
                                                _lib.stream_ptr(self.device))
        _lib.check(rc, "sped_pcg64_integers_device")
        return out[:count]


def host_draw(rng: np.random.Generator, m: int, count: int, device) -> torch.Tensor:
    """The reference's own host draw, uploaded through pinned memory."""
    idx = rng.integers(0, m, size=count)
    pinned = torch.empty(count, dtype=torch.int32, pin_memory=True)
    np.copyto(pinned.numpy(), idx, casting="unsafe")
    return pinned.to(device, non_blocking=True)


class EdgeBatchOracle:
    """Stochastic reversed operator (solvers.py:150-180, restated per term).

    Each call draws ``n_terms * batch_size`` edge ids from the oracle's PCG64
    stream and runs ``sped_edge_batch_poly_apply``.  Stateful (owns the
    stream), like the reference's closure."""

    def __init__(self, op, batch_size: int, seed: int, index_source: str = "device"):
        if index_source not in ("device", "host"):
            raise ValueError("index_source must be 'device' or 'host'")
        self.op = op
        self.batch_size = int(batch_size)
        self.index_source = index_source
        lap = op.laplacian
        self.device = lap.device
        self.gen = DeviceGenerator(np.random.default_rng(seed), self.device)
        self.m = lap.graph.m
        lib = _lib.load()
        # room for every term's records (one sort per apply, not per term)
        self.ws_bytes = int(lib.sped_edge_batch_workspace_bytes_terms(
            lap.n, self.batch_size, max(int(op.n_terms), 1)))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        self.last_batch = None

    @property
    def n(self) -> int:
        return self.op.n

    @property
    def rng(self) -> np.random.Generator:
        """The oracle's numpy stream (solvers.py:167), current as of the last
        draw (re-synchronised from the device on access)."""
        return self.gen.rng

    def draw(self, count: int) -> torch.Tensor:
        if self.index_source == "device":
            return self.gen.integers(self.m, count)
        return host_draw(self.gen.rng, self.m, count, self.device)

    @property
    def graph_capturable(self) -> bool:
        """Whole applies can be captured in a CUDA graph: device-resident
        draws, and one stream (all terms sorted at once, or a single term)."""
        if self.index_source != "device":
            return False
        per_term = int(_lib.load().sped_edge_batch_workspace_bytes(self.op.laplacian.n,
                                                                   self.batch_size))
        return self.op.n_terms <= 1 or self.ws_bytes > per_term

    def apply_device(self, xd: torch.Tensor, batch: torch.Tensor | None = None,
                     out: torch.Tensor | None = None) -> torch.Tensor:
        """Original-order CUDA block in/out."""
        lap = self.op.laplacian
        if not lap.reordered:
            return self.apply_internal(xd, batch, out)
        y = lap.from_internal(self.apply_internal(lap.to_internal(xd), batch))
        if out is not None:
            out.copy_(y)
            return out
        return y

    def apply_internal(self, xd: torch.Tensor, batch: torch.Tensor | None = None,
                       out: torch.Tensor | None = None) -> torch.Tensor:
        lib = _lib.load()
        lap = self.op.laplacian
        al, be, ga, w0, lf, s = self.op.schedule
        nt = len(al)
        B = self.batch_size
        if batch is None:
            batch = self.draw(nt * B) if nt > 0 else torch.empty(1, dtype=torch.int32,
                                                                  device=self.device)
        self.last_batch = batch
        k = 1 if xd.dim() == 1 else int(xd.shape[1])
        if out is None:
            out = torch.empty_like(xd)
        wa = torch.empty_like(xd) if nt >= 2 else None
        wb = torch.empty_like(xd) if nt >= 3 else None
        rc = lib.sped_edge_batch_poly_apply(
            self.n, k, self.m, _lib.ptr(lap.indices), _lib.ptr(lap.edge_w), _lib.ptr(lap.epos),
            None, _lib.ptr(batch), B, _lib.ptr(self.ws), self.ws_bytes, _lib.ptr(xd), None,
            _lib.ptr(wa), _lib.ptr(wb), _lib.ptr(out), nt, _lib.dbl_array(al),
            _lib.dbl_array(be), _lib.dbl_array(ga), float(w0), float(lf), float(s),
            _lib.stream_ptr(self.device))
        _lib.check(rc, "sped_edge_batch_poly_apply")
        return out

    def __call__(self, x):
        shape0 = x.shape[0] if hasattr(x, "shape") and len(x.shape) else None
        if shape0 != self.n:
            raise ValueError("dimension mismatch in transformed matvec")
        xd, back = as_device_block(x, self.device)
        return from_device_block(self.apply_device(xd), back)
