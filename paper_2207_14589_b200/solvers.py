"""Streaming top-k eigensolvers on the device.

Mirrors ``specgap.solvers`` (/root/reference/pkg/src/specgap/solvers.py):
``EigenState``, ``SolverConfig``, ``init_state``, ``oja_step``,
``mu_eg_step``, ``make_stochastic_oracle``, ``run_solver``, ``run_to_csv``.

A step never leaves the GPU: oracle (fused polynomial SpMM, or the
edge-minibatch kernel) -> Gram of [V | MV] (``sped_gram``) -> k x k algebra
in fp64 on the device (``sped_mueg_coeffs`` / ``sped_oja_coeffs``) -> one
fused update pass (``sped_block_update``).  ``run_solver`` replays whole
steps as CUDA graphs between metric evaluations (exact oracle, constant eta).
Public step functions accept numpy or CUDA states; numpy in -> numpy out.
"""

from __future__ import annotations

import ctypes
import math
import threading
import time
import warnings
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .arrays import as_device_block, from_device_block
from .graph import Graph
from .metrics import GroundTruth, eigenvector_streak, graph_ground_truth, subspace_error
from .sampling import EdgeBatchOracle
from .transforms import SpectralTransform, TransformedOperator, make_reversed_operator

__all__ = [
    "EigenState",
    "SolverConfig",
    "MetricRow",
    "SolverRun",
    "StepWorkspace",
    "init_state",
    "orthonormalize",
    "oja_step",
    "mu_eg_step",
    "make_stochastic_oracle",
    "run_solver",
    "run_to_csv",
]

_NORM_TOL = 1e-12


@dataclass
class EigenState:
    """Candidate eigenvector block plus a step counter (solvers.py:46-58).
    ``V`` is a CUDA fp32 tensor (device solver) or a numpy array."""

    V: object
    step: int = 0

    @property
    def n(self) -> int:
        return int(self.V.shape[0])

    @property
    def k(self) -> int:
        return int(self.V.shape[1])

    def numpy(self) -> np.ndarray:
        V = self.V
        return V.detach().cpu().numpy().astype(np.float64) if isinstance(V, torch.Tensor) else V


@dataclass(frozen=True)
class SolverConfig:
    """solvers.py:61-81."""

    solver: str = "oja"
    k: int = 2
    eta: float = 0.1
    steps: int = 1000
    batch_size: int = 0
    seed: int = 0
    eval_every: int = 100
    eta_schedule: str = "constant"
    streak_epsilon: float = 0.01

    def __post_init__(self):
        if self.solver not in ("oja", "mu-eg"):
            raise ValueError(f"unknown solver {self.solver!r}")
        if self.eta <= 0:
            raise ValueError("step size must be positive")
        if self.steps < 0 or self.eval_every < 1 or self.k < 1:
            raise ValueError("invalid solver configuration")
        if self.eta_schedule not in ("constant", "invsqrt"):
            raise ValueError(f"unknown eta schedule {self.eta_schedule!r}")


class StepWorkspace:
    """Static device buffers for one (n, k) solver step (graph-capturable)."""

    def __init__(self, n: int, k: int, device):
        lib = _lib.load()
        self.n, self.k, self.device = n, k, device
        self.G = torch.empty(3 * k * k, dtype=torch.float64, device=device)
        self.gram_bytes = int(lib.sped_gram_workspace_bytes(n, k))
        self.gram_ws = torch.empty(self.gram_bytes, dtype=torch.uint8, device=device)
        self.A = torch.empty(k * k, dtype=torch.float32, device=device)
        self.B = torch.empty(k * k, dtype=torch.float32, device=device)
        self.scale = torch.empty(k, dtype=torch.float32, device=device)
        self.flag = torch.zeros(1, dtype=torch.int32, device=device)
        self.tmp = torch.empty((n, k), dtype=torch.float32, device=device)
        # row shards: called on G after every Gram (the all-reduce, C2)
        self.reduce = None

    def gram(self, V, M=None, diag_q=False):
        """G = {S, C, Q}; diag_q: Q's diagonal only (mu-EG, sped_gram_mueg)."""
        lib = _lib.load()
        fn = lib.sped_gram_mueg if (diag_q and M is not None) else lib.sped_gram
        with torch.cuda.device(self.device):
            rc = fn(self.n, self.k, _lib.ptr(V), _lib.ptr(M), _lib.ptr(self.G),
                    _lib.ptr(self.gram_ws), self.gram_bytes, _lib.stream_ptr(self.device))
        _lib.check(rc, "sped_gram")
        if self.reduce is not None:
            self.reduce(self.G)

    def update(self, P, A, M, B, eta, scale, out, upper=False):
        lib = _lib.load()
        with torch.cuda.device(self.device):
            rc = lib.sped_block_update(self.n, self.k, _lib.ptr(P), _lib.ptr(A), _lib.ptr(M),
                                       _lib.ptr(B), float(eta), _lib.ptr(scale), int(upper),
                                       _lib.ptr(out), _lib.stream_ptr(self.device))
        _lib.check(rc, "sped_block_update")

    def oja_coeffs(self, eta, with_m, T):
        lib = _lib.load()
        with torch.cuda.device(self.device):
            rc = lib.sped_oja_coeffs(self.k, _lib.ptr(self.G), float(eta), int(with_m),
                                     _lib.ptr(T), _lib.ptr(self.flag),
                                     _lib.stream_ptr(self.device))
        _lib.check(rc, "sped_oja_coeffs")

    # -- step bodies (device, stream-ordered, no host sync) -------------------
    def mu_eg(self, V, MV, eta, out):
        """solvers.py:121-144 in Gram form."""
        lib = _lib.load()
        self.gram(V, MV, diag_q=True)
        with torch.cuda.device(self.device):
            rc = lib.sped_mueg_coeffs(self.k, _lib.ptr(self.G), float(eta), _lib.ptr(self.A),
                                      _lib.ptr(self.scale), _lib.ptr(self.flag),
                                      _lib.stream_ptr(self.device))
        _lib.check(rc, "sped_mueg_coeffs")
        self.update(V, self.A, MV, None, eta, self.scale, out, upper=True)

    def oja(self, V, MV, eta, out):
        """oja_step (solvers.py:114-118) with MGS replaced by CholQR2."""
        lib = _lib.load()
        self.gram(V, MV)
        self.oja_coeffs(eta, 1, self.A)
        with torch.cuda.device(self.device):
            rc = lib.sped_axpby(self.k * self.k, float(eta), _lib.ptr(self.A), 0.0, None,
                                _lib.ptr(self.B), _lib.stream_ptr(self.device))
        _lib.check(rc, "sped_axpby")
        self.update(V, self.A, MV, self.B, 0.0, None, self.tmp)
        self.gram(self.tmp)
        self.oja_coeffs(0.0, 0, self.A)
        self.update(self.tmp, self.A, None, None, 0.0, None, out)

    def cholqr2(self, V, out):
        """_orthonormalize (solvers.py:84-102) as CholQR2 (same Q as MGS)."""
        self.gram(V)
        self.oja_coeffs(0.0, 0, self.A)
        self.update(V, self.A, None, None, 0.0, None, self.tmp)
        self.gram(self.tmp)
        self.oja_coeffs(0.0, 0, self.A)
        self.update(self.tmp, self.A, None, None, 0.0, None, out)

    def take_flag(self) -> bool:
        fv = int(self.flag.item())
        if fv & 2:
            raise RuntimeError("sped_persistent_mueg: a tagged term wait timed out")
        if fv & 4:
            raise RuntimeError("sped_persistent_mueg: tagged-term protocol violated "
                               "(a row was overwritten before it was read)")
        f = bool(fv)
        if f:
            self.flag.zero_()
        return f


_WS_LOCAL = threading.local()
_WS_MAX = 4  # workspaces kept per thread (each pins an n x k fp32 block)


def _workspace(n, k, device) -> StepWorkspace:
    """The calling thread's workspace for (n, k, device, current stream).
    Per thread, so concurrent step calls never share the Gram / coefficient
    / flag buffers (the reference's step functions are pure); a small LRU
    bounds the device memory the cache pins."""
    cache = getattr(_WS_LOCAL, "cache", None)
    if cache is None:
        cache = _WS_LOCAL.cache = OrderedDict()
    key = (n, k, str(device), torch.cuda.current_stream(device).cuda_stream)
    ws = cache.get(key)
    if ws is None:
        ws = StepWorkspace(n, k, device)
        cache[key] = ws
        while len(cache) > _WS_MAX:
            cache.popitem(last=False)
    else:
        cache.move_to_end(key)
    return ws


def _device_of(oracle, default=None):
    for obj in (getattr(oracle, "__self__", None), oracle):
        for attr in ("device",):
            d = getattr(obj, attr, None)
            if d is not None:
                return torch.device(d)
        lap = getattr(obj, "laplacian", None)
        if lap is not None and getattr(lap, "device", None) is not None:
            return lap.device
    return _lib.require_cuda(default)


def orthonormalize(V, rng=None, device=None):
    """Column-orthonormalise (same Q as MGS).  Collapsed columns are
    re-randomised as in solvers.py:91-100."""
    dev = _lib.require_cuda(device)
    Vd, back = as_device_block(V, dev)
    Vd = Vd.contiguous()
    n, k = Vd.shape
    ws = _workspace(n, k, dev)
    out = torch.empty_like(Vd)
    ws.cholqr2(Vd, out)
    if ws.take_flag():
        warnings.warn("rank collapse in orthonormalization; re-randomizing", RuntimeWarning)
        out = _mgs_repair(Vd, rng)
    return from_device_block(out, back)


def _mgs_repair(Vd, rng):
    """Rare path: column-sequential Gram-Schmidt with re-randomisation,
    following solvers.py:84-102 (device torch ops, fp64)."""
    V = Vd.double().clone()
    n, k = V.shape
    for j in range(k):
        for i in range(j):
            V[:, j] -= (V[:, i] @ V[:, j]) * V[:, i]
        nrm = torch.linalg.norm(V[:, j])
        if float(nrm) < _NORM_TOL:
            if rng is None:
                rng = np.random.default_rng(0)
            V[:, j] = torch.from_numpy(rng.standard_normal(n)).to(V.device)
            for i in range(j):
                V[:, j] -= (V[:, i] @ V[:, j]) * V[:, i]
            nrm = torch.linalg.norm(V[:, j])
        V[:, j] /= nrm
    return V.float()


def init_state(n: int, k: int, seed: int, device=None) -> EigenState:
    """Seeded Gaussian block (the reference's exact numpy stream,
    solvers.py:105-111), orthonormalised on the device.  V is a CUDA tensor."""
    if k > n:
        raise ValueError("cannot ask for more eigenvectors than dimensions")
    dev = _lib.require_cuda(device)
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((n, k))
    Vd = orthonormalize(torch.from_numpy(G.astype(np.float32)).to(dev), rng, device=dev)
    return EigenState(Vd, 0)


def _device_oracle(oracle):
    """The device-side apply of our operators (also when the reference-style
    bound method ``op.apply`` is passed), else None."""
    if isinstance(oracle, _InternalOracle):
        return oracle.apply_device
    obj = getattr(oracle, "__self__", oracle)
    if isinstance(obj, TransformedOperator) and obj.transform.is_polynomial:
        return obj.apply_device
    if isinstance(obj, EdgeBatchOracle):
        return obj.apply_device
    from .walks import WalkOracle
    if isinstance(obj, WalkOracle):
        return obj.apply_device
    return None


def _oracle_block(oracle, V, Vd, dev):
    """MV on the device.  Our operators run directly on the device copy of V
    (one H2D per step for host states); foreign callables get V as passed."""
    fn = _device_oracle(oracle)
    if fn is not None:
        return fn(Vd)
    MVd, _ = as_device_block(oracle(V), dev)
    return MVd


def mu_eg_step(state: EigenState, oracle, eta: float, rng=None) -> EigenState:
    """One parallel EigenGame update (solvers.py:121-144)."""
    dev = _device_of(oracle)
    Vd, back = as_device_block(state.V, dev)
    MVd = _oracle_block(oracle, state.V, Vd, dev)
    n, k = Vd.shape
    ws = _workspace(n, k, dev)
    out = torch.empty_like(Vd)
    ws.mu_eg(Vd, MVd, eta, out)
    if ws.take_flag():
        out = _mueg_repair(Vd, MVd, ws, eta, rng)
    return EigenState(from_device_block(out, back), state.step + 1)


def _mueg_repair(Vd, MVd, ws, eta, rng):
    warnings.warn("rank collapse in mu-eg update; re-randomizing", RuntimeWarning)
    W = torch.empty_like(Vd)
    ws.update(Vd, ws.A, MVd, None, eta, None, W)
    W = W.double()
    norms = torch.linalg.norm(W, dim=0)
    bad = (norms < _NORM_TOL).cpu().numpy()
    if rng is None:
        rng = np.random.default_rng(0)
    W[:, torch.from_numpy(bad).to(W.device)] = torch.from_numpy(
        rng.standard_normal((W.shape[0], int(bad.sum())))).to(W.device)
    return (W / torch.linalg.norm(W, dim=0)).float()


def oja_step(state: EigenState, oracle, eta: float, rng=None) -> EigenState:
    """One Oja update ``V <- orthonormalize(V + eta M V)`` (solvers.py:114-118)."""
    dev = _device_of(oracle)
    Vd, back = as_device_block(state.V, dev)
    MVd = _oracle_block(oracle, state.V, Vd, dev)
    n, k = Vd.shape
    ws = _workspace(n, k, dev)
    out = torch.empty_like(Vd)
    ws.oja(Vd, MVd, eta, out)
    if ws.take_flag():
        warnings.warn("rank collapse in oja update; re-randomizing", RuntimeWarning)
        out = _mgs_repair(Vd + eta * MVd, rng)
    return EigenState(from_device_block(out, back), state.step + 1)


_STEP_RULES = {"oja": oja_step, "mu-eg": mu_eg_step}


def make_stochastic_oracle(op: TransformedOperator, batch_size: int, seed: int,
                           sampler=None, index_source: str = "device",
                           estimator: str | None = None):
    """Unbiased stochastic estimate of the reversed transformed matvec
    (solvers.py:150-202).  Batch size 0 returns ``op.apply``.

    * Default (``estimator=None``): the reference's own estimators.  Identity
      kind: ``batch_size`` seeded edge minibatches from ONE numpy PCG64
      stream (solvers.py:164-178, bit-identical indices); other polynomial
      kinds: the reference's walk oracle (solvers.py:183-200), one importance
      estimate per column with the reference's per-call seeds and
      bit-identical walks (``walks.WalkOracle``; ``sampler=`` as in the
      reference).
    * ``estimator="edge-batch"`` (the north-star device path, opt-in for
      non-identity kinds): per-term seeded edge minibatches of ``batch_size``
      edges drawn from ONE PCG64 stream seeded with ``seed`` -- the restated
      per-term composition of SURVEY 8c(1).
    * ``estimator="walk"``: the walk oracle explicitly."""
    if batch_size == 0:
        return op.apply
    if batch_size < 0:
        raise ValueError("batch size must be nonnegative")
    if estimator not in (None, "edge-batch", "walk"):
        raise ValueError(f"unknown estimator {estimator!r}")
    if not op.transform.is_polynomial:
        raise ValueError("stochastic sampling needs a polynomial transform")
    if op.transform.kind != "identity" and (estimator == "walk" or
                                            (estimator is None)):
        from .walks import WalkOracle
        walks = sampler.walks_per_estimate if sampler is not None else batch_size
        return WalkOracle(op, walks, seed)
    return EdgeBatchOracle(op, batch_size, seed, index_source=index_source)


@dataclass
class MetricRow:
    step: int
    subspace_error: float
    streak: int
    elapsed_ns: int


@dataclass
class SolverRun:
    records: list
    state: EigenState
    config: SolverConfig
    ground_truth: GroundTruth | None
    steps_to_streak: int | None = None
    steps_to_subspace: int | None = None

    @property
    def V(self):
        return self.state.V


class _GraphStepper:
    """Whole solver steps captured as CUDA graphs (ping-pong buffers).
    ``op`` is the exact operator or an edge-minibatch oracle whose draws run
    on the device (each replay draws the next batches from the device-resident
    PCG64 state, so replays continue the reference's stream)."""

    def __init__(self, op, solver: str, eta: float, V0: torch.Tensor):
        self.dev = V0.device
        n, k = V0.shape
        self.bufs = [V0.clone(), torch.empty_like(V0)]
        self.MV = torch.empty_like(V0)
        self.ws = StepWorkspace(n, k, self.dev)
        self.op, self.solver, self.eta = op, solver, eta
        self.cur = 0
        self.graphs = [None, None]
        gen = getattr(op, "gen", None)
        if gen is not None:  # the warm-up must not consume the oracle's stream
            saved = gen.snapshot()
        s = torch.cuda.Stream(self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            for i in (0, 1):  # warm-up (allocations, attributes)
                self._body(self.bufs[i], self.bufs[1 - i])
        torch.cuda.current_stream(self.dev).wait_stream(s)
        torch.cuda.synchronize(self.dev)
        if gen is not None:
            gen.restore(saved)
        self.bufs[0].copy_(V0)
        for i in (0, 1):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._body(self.bufs[i], self.bufs[1 - i])
            self.graphs[i] = g

    def _body(self, V, out):
        self.op.apply_internal(V, out=self.MV)
        if self.solver == "mu-eg":
            self.ws.mu_eg(V, self.MV, self.eta, out)
        else:
            self.ws.oja(V, self.MV, self.eta, out)

    def step(self):
        self.graphs[self.cur].replay()
        self.cur ^= 1

    def advance(self, m: int):
        for _ in range(m):
            self.step()

    @property
    def V(self):
        return self.bufs[self.cur]


PERSISTENT_MAX_NK = 1 << 22


def persistent_solver_eligible(op, k: int, solver: str) -> bool:
    """Graphs small enough that a solver step is launch bound run whole steps
    inside one grid-resident launch (sped_persistent_mueg / _oja, K7):
    polynomial transforms, k <= 32, n*k <= 4M, no row longer than 512
    nonzeros (one thread per output entry walks its row, so a hub row would
    serialise the term)."""
    if not (solver in ("mu-eg", "oja") and isinstance(op, TransformedOperator)
            and op.transform.is_polynomial and k <= 32 and op.n * k <= PERSISTENT_MAX_NK
            and op.n_terms <= 256):
        return False
    return op.laplacian.max_row_nnz <= 512


class _PersistentStepper:
    """Many whole mu-EG (or Oja) steps per cooperative launch (K7)."""

    def __init__(self, op: TransformedOperator, eta: float, V0: torch.Tensor,
                 solver: str = "mu-eg"):
        if solver not in ("mu-eg", "oja"):
            raise ValueError(f"persistent solver: unknown solver {solver!r}")
        self.op, self.eta, self.solver = op, eta, solver
        self.V_ = V0.clone().contiguous()
        k = int(V0.shape[1])
        self.ws = StepWorkspace(op.n, k, V0.device)
        lib = _lib.load()
        nbytes = ctypes.c_int64(0)
        _lib.check(lib.sped_persistent_workspace_bytes(op.n, k, ctypes.byref(nbytes)),
                   "sped_persistent_workspace_bytes")
        # zeroed once: the tagged term blocks start at tag 0, the tag base too
        self.scratch = torch.zeros(int(nbytes.value), dtype=torch.uint8, device=V0.device)
        al, be, ga, w0, lf, s = op.schedule
        self._coef = (len(al), _lib.dbl_array(al), _lib.dbl_array(be), _lib.dbl_array(ga),
                      float(w0), float(lf), float(s))

    def advance(self, m: int):
        if m <= 0:
            return
        lib = _lib.load()
        lap = self.op.laplacian
        nt, al, be, ga, w0, lf, s = self._coef
        fn = lib.sped_persistent_oja if self.solver == "oja" else lib.sped_persistent_mueg
        rc = fn(lap.n, int(self.V_.shape[1]), int(lap.nnz), _lib.ptr(lap.indptr),
                _lib.ptr(lap.indices), _lib.ptr(lap.values), nt, al, be, ga, w0, lf, s,
                float(self.eta), int(m), _lib.ptr(self.V_), _lib.ptr(self.ws.flag),
                _lib.ptr(self.scratch), self.scratch.numel(), _lib.stream_ptr(self.V_.device))
        _lib.check(rc, "sped_persistent_" + self.solver.replace("-", ""))

    def step(self):
        self.advance(1)

    @property
    def V(self):
        return self.V_

    @property
    def bufs(self):
        return [self.V_]

    cur = 0


def run_solver(g: Graph, transform: SpectralTransform, config: SolverConfig,
               mode: str = "unnormalized", ground_truth: GroundTruth | None = None,
               operator: TransformedOperator | None = None,
               streak_target: int | None = None, subspace_target: float | None = None,
               stop_on_targets: bool = False, record_timing: bool = True,
               device=None, use_cuda_graphs: bool = True,
               index_source: str = "device",
               use_persistent_kernel: bool | None = None,
               estimator: str | None = None) -> SolverRun:
    """Run a solver on the reversed transformed Laplacian (solvers.py:227-292),
    entirely on the device.  Metrics are evaluated on the host every
    ``eval_every`` steps against the original Laplacian's bottom-k truth
    (dense, n <= 5000, as in the reference).  Deterministic polynomial
    mu-EG runs on small graphs use the grid-resident kernel K7
    (``use_persistent_kernel=None`` = when eligible), other graphable runs
    replay whole steps as CUDA graphs.  ``estimator`` selects the stochastic
    oracle for ``batch_size > 0`` (``make_stochastic_oracle``: None = the
    reference's; "edge-batch" = per-term edge minibatches)."""
    if config.k > g.n:
        raise ValueError("k exceeds the node count")
    dev = _lib.require_cuda(device)
    op = operator if operator is not None else make_reversed_operator(g, transform, mode, device=dev)
    ss = np.random.SeedSequence(config.seed)
    init_seed, aux_seed, oracle_seed = (int(x) for x in ss.generate_state(3))
    rng = np.random.default_rng(aux_seed)
    stochastic = config.batch_size > 0
    oracle = make_stochastic_oracle(op, config.batch_size, oracle_seed,
                                    index_source=index_source,
                                    estimator=estimator) if stochastic else op
    if ground_truth is None and g.n <= 5000:
        ground_truth = graph_ground_truth(g, mode)
    state = init_state(g.n, config.k, init_seed, device=dev)
    target_streak = config.k if streak_target is None else streak_target

    records: list[MetricRow] = []
    run = SolverRun(records, state, config, ground_truth)
    t0 = time.perf_counter_ns()

    def evaluate(V, step):
        elapsed = time.perf_counter_ns() - t0 if record_timing else 0
        if ground_truth is None:
            records.append(MetricRow(step, float("nan"), 0, elapsed))
            return
        Vh = V.detach().cpu().numpy().astype(np.float64)
        err = subspace_error(Vh, ground_truth, config.k)
        stk = eigenvector_streak(Vh, ground_truth, config.streak_epsilon)
        records.append(MetricRow(step, err, stk, elapsed))
        if run.steps_to_streak is None and stk >= target_streak:
            run.steps_to_streak = step
        if subspace_target is not None and run.steps_to_subspace is None and err <= subspace_target:
            run.steps_to_subspace = step

    def targets_met():
        if run.steps_to_streak is None:
            return False
        if subspace_target is not None and run.steps_to_subspace is None:
            return False
        return True

    evaluate(state.V, 0)
    graphable = (use_cuda_graphs and config.eta_schedule == "constant"
                 and isinstance(op, TransformedOperator) and op.transform.is_polynomial
                 and config.steps > 0
                 and (not stochastic or (isinstance(oracle, EdgeBatchOracle)
                                         and oracle.graph_capturable)))
    lap = op.laplacian if isinstance(op, TransformedOperator) else None
    internal = lap is not None and lap.reordered
    # the solver state lives in the operator's internal (relabelled) order
    V = lap.to_internal(state.V) if internal else state.V
    out_order = (lambda X: lap.from_internal(X)) if internal else (lambda X: X)
    steps_done = 0
    if graphable:
        persistent = not stochastic and (persistent_solver_eligible(op, config.k, config.solver)
                                         if use_persistent_kernel is None
                                         else use_persistent_kernel)
        if persistent:
            stepper = _PersistentStepper(op, config.eta, V, config.solver)
        else:
            stepper = _GraphStepper(oracle if stochastic else op, config.solver, config.eta, V)
        t = 0
        while t < config.steps:
            m = min(config.eval_every - t % config.eval_every, config.steps - t)
            stepper.advance(m)
            t += m
            steps_done = t
            if t % config.eval_every == 0 or t == config.steps:
                if stepper.ws.take_flag():
                    # rare: redo with the eager path's repair semantics
                    warnings.warn("rank collapse detected; re-randomizing", RuntimeWarning)
                    stepper.bufs[stepper.cur].copy_(orthonormalize(stepper.V, rng, device=dev))
                evaluate(out_order(stepper.V), t)
                if stop_on_targets and targets_met():
                    break
        V = stepper.V.clone()
    else:
        step_fn = _STEP_RULES[config.solver]
        ioracle = _InternalOracle(oracle) if internal else oracle
        st = EigenState(V, 0)
        for t in range(1, config.steps + 1):
            eta = config.eta if config.eta_schedule == "constant" else config.eta / math.sqrt(t)
            st = step_fn(st, ioracle, eta, rng)
            steps_done = t
            if t % config.eval_every == 0 or t == config.steps:
                evaluate(out_order(st.V), t)
                if stop_on_targets and targets_met():
                    break
        V = st.V
    run.state = EigenState(out_order(V), steps_done)
    return run


class _InternalOracle:
    """Adapter: the solver's internal-order state through an operator's
    internal-order device apply."""

    def __init__(self, oracle):
        self.obj = getattr(oracle, "__self__", oracle)
        self.device = self.obj.device

    def apply_device(self, Vd):
        return self.obj.apply_internal(Vd)

    __call__ = apply_device


def run_to_csv(run: SolverRun) -> str:
    """solvers.py:295-300."""
    lines = ["step,subspace_error,streak,elapsed_ns"]
    for row in run.records:
        lines.append(f"{row.step},{row.subspace_error!r},{row.streak},{row.elapsed_ns}")
    return "\n".join(lines) + "\n"
