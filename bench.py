#!/usr/bin/env python
"""SPED hot-path benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl sped|reference]

Workload (default, ``--config 4``): BASELINE configs[3] — Chung-Lu power-law
graph, n = 10^7, Pareto(2.1) expected degrees (mean 16), normalized Laplacian
fp32, k = 32, polynomial degree 12 (negexp-taylor, the literal degree).  One
STEP = one mu-EigenGame solver step: MV = p(L)V (12 fused SpMM terms), Gram of
[V | MV], k x k algebra, fused update.  ``value`` = 12*nnz*k per step / step
time (p(L)V nnz*k/s, whole job).  Inputs (V: 1.28 GB, CSR: 1.4 GB) are far
larger than the 126 MB L2, so no flush is needed between steps.

N > 1 (torchrun): rows are sharded across ranks (strong scaling: the same
graph), halo rows exchanged per term over NCCL, one Gram all-reduce per step.

``--impl reference`` times the reference's CPU algorithm (the oracle port:
scipy csr_matvecs + numpy, fp64) on all host cores: whole mu-EG steps on the
same graph (at most 3 timed steps; the line reports the steps it ran).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "p(L)V nnz*k/s (mu-EG step incl. Gram+update)"
UNIT = "nnz*k/s"
REF_MAX_STEPS = 3  # reference arm: whole host steps are ~10 s at config 4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", choices=["sped", "reference"], default="sped")
    ap.add_argument("--scale", type=float, default=1.0, help="node-count scale (debug only)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--no-extra", action="store_true", help="skip the stochastic (config 3s) line")
    return ap.parse_args()


def cfg_spec(c):
    from paper_2207_14589_b200 import generators as G
    spec = dict(G.CONFIGS[c])
    spec["index"] = c
    return spec


def transform_for(spec):
    import paper_2207_14589_b200 as sp
    return sp.SpectralTransform("negexp-taylor", spec["ell"])


def workload_config(spec, cfg_index, n, m, nnz, world, eta):
    """The ``config`` dict both arms print (identical keys and values)."""
    return {"workload": f"{spec['name']} (BASELINE configs[{cfg_index - 1}])",
            "n": n, "m": m, "nnz": nnz, "k": spec["k"], "mode": spec["mode"],
            "transform": f"negexp-taylor({spec['ell']})", "terms": spec["ell"],
            "solver": "mu-eg", "eta": eta,
            "parallelism": f"row-shard x{world}" if world > 1 else "single GPU",
            "l2": "inputs (V 4nk B, CSR) larger than the 126 MB L2; no flush"}


def cpu_mueg_steps(n, u, v, w, mode, k, ell, eta, steps, warmup, threads, csr=None):
    """Whole reference mu-EG steps on the host: ``MV = apply_transform(V)``
    (transforms.py:229-262, negexp-taylor(ell): ell Horner terms of scipy
    ``csr @ w`` in fp64, row blocks on ``threads`` threads) then
    ``mu_eg_step`` (solvers.py:121-144, numpy/BLAS).  Returns (seconds per
    step, steps timed, csr)."""
    import oracle as O
    if csr is None:
        csr = O.laplacian_csr(n, u, v, w, mode)
    lam = O.choose_lambda_star("negexp-taylor", O.lambda_upper(n, u, v, w, mode)
                               if mode != "normalized" else 2.0)
    rng = np.random.default_rng(1234)
    V = rng.standard_normal((n, k))
    V /= np.linalg.norm(V, axis=0)
    for _ in range(warmup):
        V = O.mu_eg_step(V, O.apply_transform(csr, "negexp-taylor", ell, 1e-6, lam, V,
                                              threads=threads), eta)
    t0 = time.perf_counter()
    for _ in range(steps):
        V = O.mu_eg_step(V, O.apply_transform(csr, "negexp-taylor", ell, 1e-6, lam, V,
                                              threads=threads), eta)
    dt = (time.perf_counter() - t0) / max(steps, 1)
    return dt, steps, csr


def bytes_per_term(n, nnz, k, stored_values, x_term, final_x):
    """Algorithmic (compulsory) HBM bytes of one fused term:
    indptr + indices (+ values) + read w + write w' (+ read x)."""
    b = 4 * (n + 1) + (4 + (4 if stored_values else 0)) * nnz + 4 * n * k * 2
    if x_term or final_x:
        b += 4 * n * k
    return b


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_traffic(workload):
    """DRAM bytes per term of the SpMM launches from the latest committed
    ncu capture (profiles/r02_traffic.json, else r01), or None."""
    p = ROOT / "profiles" / "r02_traffic.json"
    if not p.exists():
        p = ROOT / "profiles" / "r01_traffic.json"
    if not p.exists():
        return None, None
    d = json.loads(p.read_text()).get(workload)
    if not d:
        return None, None
    return float(d["dram_bytes_per_term"]), d["source"]


class DramMeter:
    """In-run DRAM traffic: bench_support/libdram_meter.so runs the CUPTI
    Range Profiler over one user range (single pass, no kernel replay) and
    returns dram__bytes_read.sum + dram__bytes_write.sum of everything the
    region launched -- the bytes the SpMM applies moved while they ran, on
    the bench's own process and clocks.  ``ok`` is False (with ``err``) when
    the library or the profiler is unavailable; nothing is guessed then."""

    def __init__(self, device_index=0):
        import ctypes as C
        self.ok, self.err = False, None
        path = ROOT / "bench_support" / "libdram_meter.so"
        try:
            lib = C.CDLL(str(path))
            lib.dm_error.restype = C.c_char_p
            lib.dm_end.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double)]
            if lib.dm_init(int(device_index)) != 0:
                self.err = lib.dm_error().decode()
                return
            self.lib, self.C = lib, C
            self.ok = True
        except OSError as exc:
            self.err = repr(exc)

    def bytes(self, fn):
        import torch
        C = self.C
        torch.cuda.synchronize()
        if self.lib.dm_begin() != 0:
            raise RuntimeError(self.lib.dm_error().decode())
        fn()
        torch.cuda.synchronize()
        rd, wr = C.c_double(0), C.c_double(0)
        if self.lib.dm_end(C.byref(rd), C.byref(wr)) != 0:
            raise RuntimeError(self.lib.dm_error().decode())
        return rd.value, wr.value


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


L2_BYTES = 126 * 1024 * 1024


def l2_capacity_bound(rowlen, k, algorithmic_bytes):
    """What a perfect static cache of the whole L2 would leave: gathers of row
    j happen (len_j - 1) times per term (once per neighbour); with the N =
    L2 / 4k most-gathered rows resident, the others cost one 4k-byte DRAM
    access each.  ``max_frac`` = algorithmic / (algorithmic + miss bytes): the
    roofline fraction a kernel running at 100 % of DRAM peak would report."""
    deg = np.sort(np.asarray(rowlen, dtype=np.int64) - 1)[::-1]
    deg = np.maximum(deg, 0)
    total = int(deg.sum())
    if total == 0:
        return None
    rows = int(min(deg.size, L2_BYTES // (4 * k)))
    hit = float(deg[:rows].sum()) / total
    miss_bytes = (1.0 - hit) * total * 4 * k
    return {"l2_bytes": L2_BYTES, "rows_resident": rows, "gathers_per_term": total,
            "hit_share": hit, "miss_bytes_per_term": miss_bytes,
            "min_traffic_per_term": algorithmic_bytes + miss_bytes,
            "max_frac": algorithmic_bytes / (algorithmic_bytes + miss_bytes)}


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def max_angle(V, Qu):
    """Largest principal angle between span(V) and span(Qu) (Qu orthonormal),
    numpy or torch (fp64): sin^2 = lambda_max(G^-1 P), G = V^T V,
    P = V^T (I - Qu Qu^T) V -- the same angle as scipy's subspace_angles
    (the oracle's), with the fixed truth factored once instead of per call."""
    if isinstance(V, np.ndarray):
        V = V.astype(np.float64)
        B = Qu.T @ V
        G = V.T @ V
        P = G - B.T @ B
        L = np.linalg.cholesky(G)
        Li = np.linalg.inv(L)
        lam = np.linalg.eigvalsh(Li @ P @ Li.T).max()
        return float(np.arcsin(min(1.0, max(lam, 0.0) ** 0.5)))
    # device block: the two k x k products on the GPU, the k x k rest on the host
    V = V.double()
    B = (Qu.T @ V).cpu().numpy()
    G = (V.T @ V).cpu().numpy()
    P = G - B.T @ B
    Li = np.linalg.inv(np.linalg.cholesky(G))
    lam = np.linalg.eigvalsh(Li @ P @ Li.T).max()
    return float(np.arcsin(min(1.0, max(lam, 0.0) ** 0.5)))


def time_to_angle(cfg=1, target=1e-3, eval_every=50, max_steps=20000, cpu=True,
                  kind="negexp-limit", ell=13, eta=0.1, cpu_sample_steps=None):
    """Time to max principal angle <= target between span(V) and the true
    bottom-k eigenvectors (BASELINE metric, part 3), GPU solver vs the CPU
    reference algorithm (oracle port), same graph / transform / seeds.
    Config 1: SBM 10x100, mu-EG, eta = 0.1, negexp-limit(13) (the smallest
    odd degree covering the spectrum, SURVEY 8d note (ii))."""
    import torch
    import oracle as O
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200 import generators as G
    from paper_2207_14589_b200.solvers import (_GraphStepper, _PersistentStepper,
                                               persistent_solver_eligible)
    spec = G.CONFIGS[cfg]
    k = spec["k"]
    n, u, v, w = G.config_graph(cfg)
    g = sp.Graph(n, u.numpy(), v.numpy(), w.numpy())
    if n <= 5000:
        U = sp.graph_ground_truth(g, spec["mode"]).bottom(k)
    else:  # sparse shift-invert ground truth (fp64, host) beyond the dense limit
        import scipy.sparse.linalg as sla
        vals, vecs = sla.eigsh(O.laplacian_csr(n, g.u, g.v, g.w, spec["mode"]),
                               k=k + 4, sigma=-1e-2, which="LM")
        U = vecs[:, np.argsort(vals)[:k]]
    init_seed, _, _ = O.solver_seeds(0)
    op = sp.make_reversed_operator(g, sp.SpectralTransform(kind, ell), spec["mode"])
    V0 = sp.init_state(n, k, init_seed).V
    Vi = op.laplacian.to_internal(V0)
    Qu = np.linalg.qr(U)[0]
    # the truth in the solver's internal row order, on the device (fp64)
    Qu_d = torch.as_tensor(Qu, dtype=torch.float64, device=Vi.device)
    if op.laplacian.perm is not None:
        Qu_d = Qu_d[op.laplacian.perm.long()].contiguous()
    Vchk = O.init_state(n, k, init_seed)
    assert abs(max_angle(Vchk, Qu) - O.principal_angles(Vchk, U)) < 1e-9
    max_angle(Vi, Qu_d)  # cuBLAS fp64 handle set up outside the timed loops

    def run_gpu(stepper):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for t in range(eval_every, max_steps + 1, eval_every):
            stepper.advance(eval_every)
            if max_angle(stepper.V, Qu_d) <= target:  # evaluated on the device
                return t, time.perf_counter() - t0
        return None, time.perf_counter() - t0

    # the multi-kernel CUDA-graph path, and the grid-resident K7 kernel (the
    # default for graphs this small) -- same steps, same result to fp32 rounding
    graph_steps, graph_s = run_gpu(_GraphStepper(op, "mu-eg", eta, Vi))
    gpu_path, gpu_steps, gpu_s = "CUDA-graph steps", graph_steps, graph_s
    out = {"config": spec["name"], "transform": f"{kind}({ell})", "eta": eta, "k": k,
           "target_angle": target, "eval_every": eval_every,
           "gpu_steps_cuda_graph": graph_steps, "gpu_s_cuda_graph": graph_s}
    if persistent_solver_eligible(op, k, "mu-eg"):
        p_steps, p_s = run_gpu(_PersistentStepper(op, eta, Vi))
        out.update(gpu_steps_persistent=p_steps, gpu_s_persistent=p_s)
        if p_steps is not None:
            gpu_path, gpu_steps, gpu_s = ("grid-resident K7 kernel (sped_persistent_mueg)",
                                          p_steps, p_s)
    out.update(gpu_path=gpu_path, gpu_steps=gpu_steps, gpu_s=gpu_s)
    # per-step latency of the same stepper without evaluations (SURVEY 8d:
    # configs 1-2 report latency, not a roofline fraction)
    stp = (_PersistentStepper(op, eta, Vi) if gpu_path.startswith("grid")
           else _GraphStepper(op, "mu-eg", eta, Vi))
    stp.advance(20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    stp.advance(500)
    e1.record()
    torch.cuda.synchronize()
    out["gpu_us_per_step"] = e0.elapsed_time(e1) * 1e3 / 500
    if cpu:
        csr = O.laplacian_csr(n, g.u, g.v, g.w, spec["mode"])
        lam = O.choose_lambda_star(kind, O.lambda_upper(n, g.u, g.v, g.w, spec["mode"]))
        V = O.init_state(n, k, init_seed)
        t0 = time.perf_counter()
        cpu_steps = None
        limit = max_steps if cpu_sample_steps is None else cpu_sample_steps
        for t in range(1, limit + 1):
            V = O.mu_eg_step(V, O.apply_transform(csr, kind, ell, 1e-6, lam, V), eta)
            if t % eval_every == 0 and max_angle(V, Qu) <= target:
                cpu_steps = t
                break
        cpu_s = time.perf_counter() - t0
        if cpu_sample_steps is not None and cpu_steps is None and gpu_steps:
            # bounded sample: same algorithm, same step count as the GPU run
            cpu_s = cpu_s / limit * gpu_steps
            cpu_steps = gpu_steps
            out["cpu_extrapolated_from_steps"] = limit
        out.update(cpu_steps=cpu_steps, cpu_s=cpu_s, cpu_cores=1,
                   cpu_kind="port (scipy csr @ dense, fp64; the reference path)")
        if gpu_steps and cpu_steps:
            out["speedup"] = out["cpu_s"] / gpu_s
    return out


def stochastic_time_to_angle(target=1e-2, eval_every=100, max_steps=4000, cpu_sample_steps=20,
                             kind="negexp-limit", ell=13, eta=0.1, batch_mult=16):
    """Time to max principal angle <= target in STOCHASTIC mode
    (run_solver(batch_size > 0), solvers.py:150-180,248-249): mu-EG with the
    per-term edge-minibatch oracle (B = 16 m edges per term, device PCG64
    draws, CUDA-graph replay of whole steps) on the config-1 SBM.  The
    stochastic iteration's noise floor sits near 5e-3 at eta = 0.1, so the
    target is 1e-2 (tests/test_gpu_fullsize.py::test_stochastic_run_solver_sbm).
    CPU leg: the restated oracle (the reference's np.add.at estimator per
    term, fp64, one core) on the same graph/seeds, a bounded sample of steps
    scaled to the GPU's step count."""
    import torch
    import oracle as O
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200 import generators as G
    from paper_2207_14589_b200.solvers import _GraphStepper
    spec = G.CONFIGS[1]
    k = spec["k"]
    n, u, v, w = G.config_graph(1)
    g = sp.Graph(n, u.numpy(), v.numpy(), w.numpy())
    U = sp.graph_ground_truth(g, spec["mode"]).bottom(k)
    Qu = np.linalg.qr(U)[0]
    init_seed, _, oracle_seed = O.solver_seeds(2)
    op = sp.make_reversed_operator(g, sp.SpectralTransform(kind, ell), spec["mode"])
    B = batch_mult * g.m
    orc = sp.make_stochastic_oracle(op, B, oracle_seed, estimator="edge-batch")
    V0 = sp.init_state(n, k, init_seed).V
    Qu_d = torch.as_tensor(Qu, dtype=torch.float64, device=V0.device)
    max_angle(V0, Qu_d)
    stepper = _GraphStepper(orc, "mu-eg", eta, op.laplacian.to_internal(V0))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gpu_steps = None
    for t in range(eval_every, max_steps + 1, eval_every):
        stepper.advance(eval_every)
        if max_angle(stepper.V, Qu_d) <= target:
            gpu_steps = t
            break
    gpu_s = time.perf_counter() - t0
    out = {"config": spec["name"] + " stochastic", "estimator": "edge-batch (per-term minibatches)",
           "transform": f"{kind}({ell})", "eta": eta, "k": k, "batch_per_term": B,
           "target_angle": target, "eval_every": eval_every, "gpu_steps": gpu_steps,
           "gpu_s": gpu_s, "gpu_path": "CUDA-graph steps (device PCG64 draws)"}
    # CPU: the same algorithm (restated oracle, identical batches by seed)
    csr = O.laplacian_csr(n, g.u, g.v, g.w, spec["mode"])
    lam = O.choose_lambda_star(kind, O.lambda_upper(n, g.u, g.v, g.w, spec["mode"]))
    rng = np.random.default_rng(oracle_seed)
    nt = len(O.term_schedule(kind, ell, 1e-6, lam)[0])
    V = O.init_state(n, k, init_seed)
    t0 = time.perf_counter()
    for _ in range(cpu_sample_steps):
        bt = O.draw_batches(rng, g.m, B, nt)
        V = O.mu_eg_step(V, O.edge_batch_poly_apply(g.u, g.v, g.w, kind, ell, 1e-6, lam, bt, V), eta)
    per = (time.perf_counter() - t0) / cpu_sample_steps
    del csr
    if gpu_steps:
        out.update(cpu_steps=gpu_steps, cpu_s=per * gpu_steps, cpu_extrapolated_from_steps=cpu_sample_steps,
                   cpu_cores=1, cpu_kind="port (restated edge-batch oracle, np.add.at, fp64)",
                   speedup=per * gpu_steps / gpu_s)
    return out


def exact_step_line(cfg, steps=5, warmup=2):
    """One exact mu-EG step on another BASELINE config (SBM configs 3 / 5:
    natural order, L2-resident gathers; config 5's k = 128 Gram and update
    run on the tensor cores): per-term, apply, Gram+coefficients+update and
    whole-step times (CUDA events), throughput in the headline unit."""
    import torch
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200 import generators as G
    from paper_2207_14589_b200.solvers import StepWorkspace
    spec = G.CONFIGS[cfg]
    dev = torch.device("cuda")
    n, u, v, w = G.config_graph(cfg, device=dev)
    g = sp.Graph.from_canonical(n, u, v, w, validate=False)
    k, ell = spec["k"], spec["ell"]
    t = sp.SpectralTransform("negexp-taylor", ell)
    op = sp.make_reversed_operator(g, t, spec["mode"], device=dev)
    V = torch.randn((n, k), device=dev, generator=torch.Generator(device=dev).manual_seed(cfg))
    V /= torch.linalg.norm(V, dim=0)
    Vn, MV = torch.empty_like(V), torch.empty_like(V)
    ws = StepWorkspace(n, k, dev)
    eta = 0.1
    for _ in range(warmup):
        op.apply_internal(V, out=MV)
        ws.mu_eg(V, MV, eta, Vn)
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for i in range(steps):
        ev[i][0].record()
        op.apply_internal(V, out=MV)
        ev[i][1].record()
        ws.mu_eg(V, MV, eta, Vn)
        ev[i][2].record()
        V, Vn = Vn, V
    torch.cuda.synchronize()
    apply_ms = sum(e[0].elapsed_time(e[1]) for e in ev) / steps
    solve_ms = sum(e[1].elapsed_time(e[2]) for e in ev) / steps
    nt, nnz = op.n_terms, op.laplacian.nnz
    return {"config": spec["name"], "n": n, "nnz": nnz, "k": k,
            "transform": f"negexp-taylor({ell})", "terms": nt,
            "ms_per_step": apply_ms + solve_ms, "ms_per_term": apply_ms / nt,
            "gram_coeffs_update_ms": solve_ms,
            "nnz_k_per_s": nt * nnz * k / ((apply_ms + solve_ms) / 1e3),
            "pLV_nnz_k_per_s": nt * nnz * k / (apply_ms / 1e3)}


def stochastic_line(cfg=3, reps=5):
    """Edge-minibatch apply on a BASELINE stochastic config (3s: B = 1e6 per
    term): device PCG64 draw + per-term histogram/row-sweep kernels, CUDA
    events.  Throughput as sampled-edges*k/s and the compulsory
    bytes B*(4 idx + 8 endpoints + 4 [weighted]) + 8nk (+4nk with an x term)
    per term against the HBM peak."""
    import torch
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200 import generators as G
    spec = G.CONFIGS[cfg]
    dev = torch.device("cuda")
    n, u, v, w = G.config_graph(cfg, device=dev)
    g = sp.Graph.from_canonical(n, u, v, w, validate=False)
    k, B = spec["k"], spec["batch"]
    t = sp.SpectralTransform("negexp-limit", spec["ell"] + 1)  # SURVEY 8d note (i)
    op = sp.make_reversed_operator(g, t, spec["mode"], device=dev)
    orc = sp.make_stochastic_oracle(op, B, seed=7, estimator="edge-batch")
    X = torch.randn((n, k), device=dev)
    nt = op.n_terms
    for _ in range(2):
        orc.apply_internal(X)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    draw_ms = apply_ms = 0.0
    for _ in range(reps):
        ev[0].record()
        batch = orc.draw(nt * B)
        ev[1].record()
        orc.apply_internal(X, batch=batch)
        ev[2].record()
        torch.cuda.synchronize()
        draw_ms += ev[0].elapsed_time(ev[1]) / reps
        apply_ms += ev[1].elapsed_time(ev[2]) / reps
    al = op.schedule[0]
    weighted = not g.is_unit_weight()
    bpt = B * (4 + 8 + (4 if weighted else 0)) + 8 * n * k + (4 * n * k if any(a != 0 for a in al)
                                                              else 0)
    t_term = apply_ms / nt / 1e3
    # the SURVEY 8d formula counts no neighbour rows; every sampled edge also
    # reads its two endpoint rows (4k bytes each, random)
    bpt_rows = bpt + 2 * B * 4 * k
    peak, _ = measured_peak()
    return {"config": f"{spec['name']}s (B={B} per term)", "transform": f"negexp-limit({spec['ell'] + 1})",
            "n": n, "nnz": op.laplacian.nnz, "k": k, "terms": nt,
            "ms_per_term": apply_ms / nt, "draw_ms_per_apply": draw_ms,
            "sampled_edges_k_per_s": nt * B * k / (apply_ms / 1e3),
            "equiv_4Bk_per_s": 4 * nt * B * k / (apply_ms / 1e3),
            "compulsory_bytes_per_term": bpt, "achieved_GBps": bpt / t_term / 1e9,
            "frac_of_peak": bpt / t_term / 1e9 / peak,
            "bytes_per_term_incl_endpoint_rows": bpt_rows,
            "frac_of_peak_incl_endpoint_rows": bpt_rows / t_term / 1e9 / peak}


# ------------------------------------------------------------------------------ sped arm

def run_sped(args):
    import torch
    import torch.distributed as dist
    import paper_2207_14589_b200 as sp
    from paper_2207_14589_b200 import generators as G
    from paper_2207_14589_b200.solvers import StepWorkspace

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # SPED_FORCE_SHARD=1 runs the row-sharded NCCL path even on one rank
    sharded = world > 1 or os.environ.get("SPED_FORCE_SHARD") == "1"
    if sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
    spec = cfg_spec(args.config)
    k, ell, mode = spec["k"], spec["ell"], spec["mode"]
    t_setup = time.perf_counter()
    n, u, v, w = G.config_graph(args.config, device=dev, scale=args.scale)
    t = transform_for(spec)
    if sharded:
        # no whole graph on any rank: each rank keeps a strided slice of the
        # (seeded, identical) generator output, routes it to the row owners
        # and builds only its rows (plan_shard_edges + from_shard_edges)
        from paper_2207_14589_b200.distributed import (ShardedLaplacian, ShardedOperator,
                                                       plan_shard_edges, sharded_mu_eg_step)
        from paper_2207_14589_b200.transforms import choose_lambda_star, term_schedule
        m_all = int(u.numel())
        sel = torch.arange(rank, m_all, world, device=dev)
        se = plan_shard_edges(n, u[sel], v[sel], w[sel], sel, rank, world)
        del u, v, w, sel
        shard = ShardedLaplacian.from_shard_edges(se, mode, device=dev)
        lam_star = choose_lambda_star(t, shard.lambda_upper(mode))
        sop = ShardedOperator(shard, t, lam_star)
        n_loc = shard.n_own
        g = None
        lap = None
        nnz = int(shard.nnz_global)
        m_graph = int(se.m)
        stored = shard.values is not None
        al, be, ga, w0, lf, s = term_schedule(t, lam_star)
        del se
    else:
        g = sp.Graph.from_canonical(n, u, v, w, validate=False)
        op = sp.make_reversed_operator(g, t, mode, device=dev)
        lap = op.laplacian
        nnz = lap.nnz
        m_graph = g.m
        stored = lap.values is not None
        al, be, ga, w0, lf, s = op.schedule
        n_loc = n
    n_terms = len(al)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    V = torch.randn((n_loc, k), device=dev, generator=gen)
    V /= torch.linalg.norm(V, dim=0) * (world ** 0.5)
    Vn = torch.empty_like(V)
    MV = torch.empty_like(V)
    ws = StepWorkspace(n_loc, k, dev)
    eta = 0.1
    stream = torch.cuda.current_stream(dev)

    def step(Vin, Vout, ev=None):
        if ev is not None:
            ev[0].record(stream)
        if sharded:
            sop.apply_local(Vin, out=MV)
        else:
            op.apply_internal(Vin, out=MV)
        if ev is not None:
            ev[1].record(stream)
        if sharded:
            ws.gram(Vin, MV, diag_q=True)
            dist.all_reduce(ws.G)
            lib = sp._lib.load()
            lib.sped_mueg_coeffs(k, ws.G.data_ptr(), eta, ws.A.data_ptr(), ws.scale.data_ptr(),
                                 ws.flag.data_ptr(), stream.cuda_stream)
            ws.update(Vin, ws.A, MV, None, eta, ws.scale, Vout, upper=True)
        else:
            ws.mu_eg(Vin, MV, eta, Vout)
        if ev is not None:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step(V, Vn)
        V, Vn = Vn, V
    torch.cuda.synchronize()
    if sharded:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for i in range(args.steps):
        step(V, Vn, evs[i])
        V, Vn = Vn, V
    end.record(stream)
    torch.cuda.synchronize()
    if sharded:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    total_ms = start.elapsed_time(end)
    apply_ms = sum(e[0].elapsed_time(e[1]) for e in evs)
    solve_ms = sum(e[1].elapsed_time(e[2]) for e in evs)
    if sharded:
        tt = torch.tensor([total_ms, apply_ms, solve_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms, apply_ms, solve_ms = (float(x) for x in tt.tolist())
    ms_per_step = total_ms / args.steps
    work = n_terms * nnz * k
    value = work * args.steps / (total_ms / 1e3)
    t_term_s = apply_ms / 1e3 / (args.steps * n_terms)
    n_b, nnz_b = (n, nnz) if not sharded else (n_loc, shard.nnz_local)
    x_term = any(a != 0 for a in al)
    bpt = bytes_per_term(n_b, nnz_b, k, stored, x_term, lf != 0.0)
    scaled = n_terms >= 2 and (shard.scaled_terms(k) if sharded else lap.row_scale is not None)
    if scaled:
        # terms after the first run on u = D^-1/2 w: no values, + d^-1/2 per row
        b_scaled = bytes_per_term(n_b, nnz_b, k, False, x_term, lf != 0.0) + 4 * n_b
        bpt = (bpt + (n_terms - 1) * b_scaled) / n_terms
    peak, peak_src = measured_peak()
    achieved = bpt / t_term_s / 1e9
    traffic, traffic_src, traffic_ncu = None, None, None
    if not sharded:
        ncu_bytes, ncu_src = measured_traffic(spec["name"])
        traffic_ncu = {"bytes_per_term": ncu_bytes, "source": ncu_src} if ncu_bytes else None
        reps = 4
        xb = torch.randn((n, k), device=dev)
        ob = torch.empty_like(xb)
        op.apply_internal(xb, out=ob)
        for attempt in range(2):  # the range profiler's Stop fails now and then: one retry
            meter = DramMeter(torch.cuda.current_device())
            if not meter.ok:
                break
            try:
                rd, wr = meter.bytes(lambda: [op.apply_internal(xb, out=ob) for _ in range(reps)])
                traffic = (rd + wr) / (reps * n_terms)
                traffic_src = ("in-run CUPTI range profiler (bench_support/libdram_meter.so): "
                               "dram__bytes_read.sum + dram__bytes_write.sum over %d whole "
                               "applies (%.2f + %.2f GB), per term = bytes / (%d x %d terms)"
                               % (reps, rd / 1e9, wr / 1e9, reps, n_terms))
            except RuntimeError as exc:
                meter.err = str(exc)
                traffic = None
            meter.lib.dm_close()
            if traffic is not None:
                break
        del xb, ob
        if traffic is None and traffic_ncu:
            traffic, traffic_src = ncu_bytes, (ncu_src + " (in-run meter unavailable: %s)"
                                               % meter.err)
    # lower bound on a term's DRAM traffic under a PERFECT static L2 (the whole
    # 126 MB holding the most-gathered rows, no streaming pollution): every
    # gather of a row outside that set is a DRAM access of 4k bytes
    l2_bound = None
    if not sharded:
        l2_bound = l2_capacity_bound(lap.rowlen, k, bpt)
    # our kernels per step: per term one launch per row segment (+ the hub
    # chunk launch); Gram (tcgen05 partials + fp64 reduce), coefficients,
    # update.  Sharded: + the halo pack per term (NCCL's own kernels excluded).
    if sharded and shard.split_terms:
        per_term = 1 + sum(int(h.segments(k)[0]) + (1 if h.n_chunks else 0) for h in shard.split)
    else:
        src = shard if sharded else lap
        per_term = int(src.segments(k)[0]) + (1 if src.n_chunks else 0)
    launches_per_step = n_terms * per_term + 4

    e2e = None
    if not args.no_e2e:
        # reference-facing call with HOST buffers: mu_eg_step(EigenState(host V), op, eta)
        Vh = torch.empty((n_loc, k), dtype=torch.float32, pin_memory=True)
        Vh.copy_(V)
        if not sharded:
            # two warm-up calls populate the pinned-host cache (result + input)
            for _ in range(2):
                st = sp.mu_eg_step(sp.EigenState(Vh), op, eta)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.e2e_steps):
                st = sp.mu_eg_step(sp.EigenState(Vh), op, eta)
            torch.cuda.synchronize()
            e2e_s = time.perf_counter() - t0
        else:
            e2e_s = None
            for it in range(args.e2e_steps + 1):
                if it == 1:
                    dist.barrier()
                    t0 = time.perf_counter()
                Vd = Vh.to(dev, non_blocking=True)
                out = torch.empty_like(Vd)
                sharded_mu_eg_step(sop, Vd, eta, ws, out, MV)
                Vh.copy_(out, non_blocking=True)
                torch.cuda.synchronize()
            dist.barrier()
            e2e_s = time.perf_counter() - t0
            tt = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt.item())
        e2e = {"value": work * args.e2e_steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(n * k * 4), "d2h_bytes_per_step": int(n * k * 4),
               "ms_per_step": 1e3 * e2e_s / args.e2e_steps,
               "api": "paper_2207_14589_b200.mu_eg_step(EigenState(pinned host V), op, eta)"}

    cpu = None
    if rank == 0 and not sharded and not args.no_cpu:
        thr = cpu_threads()
        dt, nst, csr_h = cpu_mueg_steps(n, g.u, g.v, g.w, mode, k, ell, eta, 1, 0, thr)
        cpu = {"value": n_terms * csr_h.nnz * k / dt, "unit": UNIT, "cores": thr, "kind": "port",
               "sample": (f"1 whole mu-EG step of the reference algorithm on the same graph: "
                          f"negexp-taylor({ell}) = {n_terms} fp64 scipy csr_matvecs terms over "
                          f"all {n} rows ({csr_h.nnz} nnz), k={k}, {thr} threads, + mu_eg_step"),
               "seconds_per_step": dt}
        del csr_h

    conv = None
    if rank == 0 and not sharded and not args.no_cpu:
        conv = [time_to_angle(1),
                # config 2 (4-room grid, normalized): negexp-limit(17) (covers the
                # spectrum, <= 2), eta = 1.0 (4,500 CPU steps, 92 s);
                # the CPU leg is a 300-step sample scaled to the GPU's step count
                time_to_angle(2, kind="negexp-limit", ell=17, eta=1.0, eval_every=100,
                              cpu_sample_steps=300),
                stochastic_time_to_angle()]
    sto = None
    extra = None
    if rank == 0 and not sharded and not args.no_extra:
        sto = [stochastic_line(3), stochastic_line(5)]
        extra = [exact_step_line(3), exact_step_line(5)]

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded generator, BASELINE shape)",
            "config": workload_config(spec, args.config, n, m_graph, nnz, world, eta),
            "setup_s": setup_s,
            "pLV_nnz_k_per_s": work * args.steps / (apply_ms / 1e3),
            "breakdown_ms_per_step": {"p(L)V": apply_ms / args.steps,
                                      "gram+coeffs+update": solve_ms / args.steps,
                                      "per_term": 1e3 * t_term_s},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "spmm_term_kernel + spmm_chunk_kernel (one fused polynomial term)",
                         "algorithmic_bytes_per_launch": bpt,
                         "algorithmic_bytes_note": ("average over the apply's terms: the first "
                                                    "reads stored values, the rest run on "
                                                    "u = D^-1/2 w without them") if scaled else
                         "stored values every term",
                         "peak_source": peak_src,
                         "traffic_source": traffic_src,
                         "traffic_ncu": traffic_ncu,
                         "dram_frac_actual": (traffic / t_term_s / 1e9 / peak) if traffic else None,
                         "l2_capacity_bound": l2_bound},
            "cpu_baseline": cpu,
            "time_to_angle": conv,
            "stochastic": sto,
            "other_configs_exact": extra,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()


# ------------------------------------------------------------------------- reference arm

def run_reference(args):
    """The reference's own CPU algorithm on the box's host cores: whole mu-EG
    steps (the oracle port of transforms.py:229-262 + solvers.py:121-144,
    fp64, scipy csr_matvecs on all threads) on the SAME graph, k, transform
    and eta as the GPU arm.  A step takes ~10 s at config 4, so at most
    ``REF_MAX_STEPS`` timed steps and one warm-up step run; the line reports
    the steps it actually ran (``steps_requested`` keeps --steps)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch
    from paper_2207_14589_b200 import generators as G
    spec = cfg_spec(args.config)
    k, mode, ell = spec["k"], spec["mode"], spec["ell"]
    eta = 0.1
    device = "cuda" if torch.cuda.is_available() else "cpu"
    # input synthesis only (the same seeded generator as the GPU arm)
    n, u, v, w = G.config_graph(args.config, device=device, scale=args.scale)
    u, v, w = u.cpu().numpy(), v.cpu().numpy(), w.cpu().numpy()
    thr = cpu_threads()
    steps = max(1, min(args.steps, REF_MAX_STEPS))
    warm = min(args.warmup, 1)
    dt, steps, csr = cpu_mueg_steps(n, u, v, w, mode, k, ell, eta, steps, warm, thr)
    rate = ell * csr.nnz * k / dt
    sample = (f"{steps} whole mu-EG steps (+{warm} warm-up): negexp-taylor({ell}) apply = "
              f"{ell} Horner terms of fp64 scipy csr_matvecs over all {n} rows "
              f"({csr.nnz} nnz), k={k}, on {thr} threads, then mu_eg_step (numpy/BLAS)")
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
            "n_gpus": world, "steps": steps, "warmup": warm, "steps_requested": args.steps,
            "warmup_requested": args.warmup, "extrapolated": False,
            "ms_per_step": 1e3 * dt, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, BASELINE shape)",
            "config": workload_config(spec, args.config, n, int(u.size), int(csr.nnz), world, eta),
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": thr, "kind": "port",
                             "sample": sample},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_sped(args)


if __name__ == "__main__":
    main()
