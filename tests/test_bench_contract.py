"""CPU checks of bench.py helpers (no GPU, no oracle)."""


def test_l2_capacity_bound_model():
    """roofline.l2_capacity_bound: with the N = L2/4k most-gathered rows
    resident, every other gather costs one 4k-byte DRAM access."""
    import numpy as np
    import bench
    k = 32
    n_res = bench.L2_BYTES // (4 * k)
    # n_res hub rows of degree 100 (101 entries with the diagonal), 3 n_res cold rows of degree 1
    rowlen = np.concatenate([np.full(n_res, 101), np.full(3 * n_res, 2)])
    b = bench.l2_capacity_bound(rowlen, k, algorithmic_bytes=1e9)
    total = n_res * 100 + 3 * n_res
    assert b["rows_resident"] == n_res and b["gathers_per_term"] == total
    assert abs(b["hit_share"] - n_res * 100 / total) < 1e-12
    assert abs(b["miss_bytes_per_term"] - 3 * n_res * 4 * k) < 1e-3
    assert abs(b["max_frac"] - 1e9 / (1e9 + 3 * n_res * 4 * k)) < 1e-12
    assert bench.l2_capacity_bound(np.ones(10, dtype=np.int64), k, 1.0) is None  # no off-diagonal entries
