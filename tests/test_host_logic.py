"""Host-side logic of the device package (CPU, no kernel launches) --
transform validation, the fused term schedule,
PCG64 state bookkeeping, generators, solver configuration, distributed
partitioning -- plus the Graph canonicalisation contract (gpu-marked: the
product canonicalises on the device)."""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2207_14589_b200 as sp
from paper_2207_14589_b200 import generators as G
from paper_2207_14589_b200.sampling import pcg64_advance_state
from paper_2207_14589_b200.transforms import term_schedule
from conftest import rel_fro


# --- Graph (graph.py:64-104): canonicalised on the device, so these launch ---------

@pytest.mark.gpu
def test_edges_canonicalized_and_sorted(cuda):
    g = sp.Graph.from_edges(4, [(3, 1), (2, 0), (1, 0)])
    assert g.u.tolist() == [0, 0, 1]
    assert g.v.tolist() == [1, 2, 3]


@pytest.mark.gpu
def test_zero_weight_edges_dropped(cuda):
    assert sp.Graph.from_edges(3, [(0, 1, 1.0), (1, 2, 0.0)]).m == 1


@pytest.mark.parametrize("edges,n,msg", [([(1, 1)], 2, "self-loop"),
                                         ([(0, 1), (1, 0)], 3, "duplicate"),
                                         ([(0, 5)], 2, "out of range"),
                                         ([(0, 1, -1.0)], 2, "nonnegative")])
@pytest.mark.gpu
def test_graph_validation_errors(cuda, edges, n, msg):
    with pytest.raises(ValueError, match=msg):
        sp.Graph.from_edges(n, edges)


@pytest.mark.gpu
def test_graph_matches_oracle_canonicalisation(cuda, golden):
    for name in golden.graph_names():
        n, u, v, w = golden.graph(name)
        g = sp.Graph(n, v, u, w)  # reversed orientation
        np.testing.assert_array_equal(g.u, u)
        np.testing.assert_array_equal(g.v, v)
        np.testing.assert_array_equal(g.degrees(), golden[f"g/{name}/degrees"])


def test_from_canonical_validates():
    u = torch.tensor([0, 0, 1])
    v = torch.tensor([1, 2, 2])
    w = torch.ones(3, dtype=torch.float64)
    g = sp.Graph.from_canonical(3, u, v, w)
    assert g.m == 3 and g.u.tolist() == [0, 0, 1]
    with pytest.raises(ValueError):
        sp.Graph.from_canonical(3, torch.tensor([0, 0]), torch.tensor([2, 1]), torch.ones(2, dtype=torch.float64))
    with pytest.raises(ValueError):
        sp.Graph.from_canonical(3, torch.tensor([1]), torch.tensor([0]), torch.ones(1, dtype=torch.float64))


@pytest.mark.gpu
def test_degree_bounds(cuda):
    g = sp.Graph.from_edges(4, [(0, 1, 2.0), (0, 2), (0, 3)])
    b = sp.degree_bounds(g)
    assert b.deg_star == 3 and b.deg_star_inc == 5 and b.lambda_upper == 8.0


# --- transforms (transforms.py:62-192) -------------------------------------------

def test_transform_validation():
    with pytest.raises(ValueError, match="odd"):
        sp.SpectralTransform("negexp-limit", 10)
    with pytest.raises(ValueError, match="epsilon"):
        sp.SpectralTransform("log", epsilon=0.0)
    with pytest.raises(ValueError, match="unknown transform"):
        sp.SpectralTransform("chebyshev")
    with pytest.raises(ValueError):
        sp.SpectralTransform("negexp-taylor", -1)


def test_lambda_star_rules():
    T = sp.SpectralTransform
    assert sp.choose_lambda_star(T("negexp"), 17.0) == 0.0
    assert sp.choose_lambda_star(T("negexp-limit", 11), 17.0) == 0.0
    assert sp.choose_lambda_star(T("identity"), 4.0) == pytest.approx(4.04)
    assert sp.choose_lambda_star(T("log"), 4.0) == pytest.approx(np.log(4.000001) * 1.01)


def test_coefficients_and_scalar_map_match_oracle():
    lam = np.linspace(0.0, 1.5, 9)
    for kind, ell, eps in [("identity", None, 1e-6), ("negexp-taylor", 6, 1e-6),
                           ("negexp-limit", 5, 1e-6), ("log-taylor", 7, 1e-6)]:
        t = sp.SpectralTransform(kind, ell, eps)
        np.testing.assert_array_equal(sp.polynomial_coefficients(t),
                                      O.polynomial_coefficients(kind, ell, eps))
        np.testing.assert_array_equal(sp.scalar_map(t, lam), O.scalar_map(kind, lam, ell, eps))


def test_product_schedule_equals_oracle_schedule():
    for kind, ell, eps in [("identity", None, 1e-6), ("negexp-limit", 9, 1e-6),
                           ("negexp-taylor", 8, 1e-6), ("negexp-taylor", 0, 1e-6),
                           ("log-taylor", 9, 0.5)]:
        t = sp.SpectralTransform(kind, ell, eps)
        assert term_schedule(t, 1.5) == O.term_schedule(kind, ell, eps, 1.5)


def test_schedule_in_fp32_meets_tolerance(golden):
    """The fused schedule evaluated in fp32 (the kernels' arithmetic) stays
    within the 1e-5 relative Frobenius bar of the fp64 reference on the
    BASELINE-shaped golden cases (SURVEY 8c fp32 feasibility)."""
    for case in sorted({k.rsplit("/", 1)[0] for k in golden.keys("apply/cfg")}):
        _, name, mode, kind, ell, eps, k = case.split("/")
        ell = None if ell == "None" else int(ell)
        n, u, v, w = golden.graph(name)
        csr = O.laplacian_csr(n, u, v, w, mode).astype(np.float32)
        lam = float(golden[case + "/lambda_star"])
        al, be, ga, w0, lf, s = O.term_schedule(kind, ell, float(eps), lam)
        x = golden[case + "/x"].astype(np.float32)
        cur = np.float32(w0) * x
        for t in range(len(al)):
            cur = (np.float32(al[t]) * x + np.float32(be[t]) * (csr @ cur)
                   + np.float32(ga[t]) * cur).astype(np.float32)
        y = np.float32(lf) * x + np.float32(s) * cur
        assert rel_fro(y, golden[case + "/y"]) <= 1e-5, case


# --- PCG64 bookkeeping -------------------------------------------------------------

@pytest.mark.parametrize("m,sizes", [(3, (5, 7, 1)), (1000, (1001, 3)), (9_990_000, (4096, 17))])
def test_pcg64_state_advance_matches_numpy(m, sizes):
    """Host bookkeeping used after a device draw: advancing numpy's PCG64
    state by the reported number of 32-bit draws lands exactly where numpy's
    own ``integers`` call leaves it."""
    mirror = np.random.default_rng(11)
    st = mirror.bit_generator.state
    for s in sizes:
        vals, _, draws = O.pcg64_integers(st, m, s)
        ref = mirror.integers(0, m, size=s)
        np.testing.assert_array_equal(vals, ref)
        new = pcg64_advance_state(st, draws)
        assert new == mirror.bit_generator.state
        st = new


# --- generators -------------------------------------------------------------------

@pytest.mark.parametrize("cfg,scale", [(1, 1.0), (2, 1.0), (3, 0.005), (4, 0.002), (5, 0.005)])
def test_generators_emit_canonical_edges(cfg, scale):
    n, u, v, w = G.config_graph(cfg, scale=scale)
    u, v, w = u.numpy(), v.numpy(), w.numpy()
    assert np.all(u < v) and np.all(u >= 0) and np.all(v < n)
    key = u * n + v
    assert np.all(np.diff(key) > 0)
    assert np.all(w > 0)
    deg = np.bincount(u, minlength=n) + np.bincount(v, minlength=n)
    if G.CONFIGS[cfg]["mode"] == "normalized":
        assert deg.min() >= 1


def test_grid_rooms_connected_and_walled():
    import scipy.sparse as ssp
    import scipy.sparse.csgraph as cg
    n, u, v, w = G.grid_rooms(20)
    A = ssp.coo_matrix((np.ones(len(u)), (u.numpy(), v.numpy())), shape=(n, n))
    assert cg.connected_components(A, directed=False)[0] == 1
    assert len(u) < 2 * 20 * 19  # walls removed edges


# --- solver config -------------------------------------------------------------------

def test_solver_config_validation():
    with pytest.raises(ValueError):
        sp.SolverConfig(solver="lanczos")
    with pytest.raises(ValueError):
        sp.SolverConfig(eta=-0.1)
    with pytest.raises(ValueError):
        sp.SolverConfig(eval_every=0)
    with pytest.raises(ValueError):
        sp.SolverConfig(eta_schedule="cosine")


def test_run_to_csv_format():
    run = sp.SolverRun([sp.MetricRow(0, 0.5, 1, 0), sp.MetricRow(10, 0.25, 2, 0)],
                       sp.EigenState(np.zeros((2, 1))), sp.SolverConfig(), None)
    assert sp.run_to_csv(run) == "step,subspace_error,streak,elapsed_ns\n0,0.5,1,0\n10,0.25,2,0\n"


def test_no_cpu_fallback_without_cuda():
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sp.Graph.from_edges(3, [(0, 1), (1, 2)])  # canonicalisation runs on the device
    g = sp.Graph.from_canonical(3, torch.tensor([0, 1]), torch.tensor([1, 2]),
                                torch.ones(2, dtype=torch.float64))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        sp.build_laplacian(g)


def test_product_does_not_import_oracle():
    import pathlib
    pkg = pathlib.Path(sp.__file__).parent
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f


def test_bench_max_angle_matches_scipy():
    """bench.max_angle (the time-to-angle criterion, truth factored once)
    equals scipy's largest principal angle -- the oracle's definition --
    from 1e-6 rad to pi/2, numpy path."""
    import scipy.linalg as sla
    import bench
    rng = np.random.default_rng(3)
    n, k = 400, 6
    Q = np.linalg.qr(rng.standard_normal((n, k)))[0]
    for eps in (1e-6, 1e-3, 0.1, 1.0, 10.0):
        V = Q @ rng.standard_normal((k, k)) + eps * rng.standard_normal((n, k))
        ref = float(np.max(sla.subspace_angles(V, Q)))
        assert abs(bench.max_angle(V, Q) - ref) <= 1e-9 + 1e-7 * ref


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (the reference's CPU algorithm, host
    cores) prints one JSON line with the driver's keys; runs on CPU."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference",
                        "--scale", "0.01", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
