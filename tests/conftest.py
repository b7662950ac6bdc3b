import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running")


class Golden:
    """Lazy view of tests/golden/golden.npz (reference-generated vectors)."""

    def __init__(self, path):
        self.d = np.load(path, allow_pickle=False)
        self.files = set(self.d.files)

    def __getitem__(self, key):
        return self.d[key]

    def __contains__(self, key):
        return key in self.files

    def keys(self, prefix):
        return sorted(k for k in self.files if k.startswith(prefix))

    def graph(self, name):
        n = int(self.d[f"g/{name}/n"])
        return (n, self.d[f"g/{name}/u"].astype(np.int64), self.d[f"g/{name}/v"].astype(np.int64),
                self.d[f"g/{name}/w"])

    def graph_names(self):
        return sorted({k.split("/")[1] for k in self.files if k.startswith("g/")})

    def state(self, key):
        return json.loads(str(self.d[key]))


@pytest.fixture(scope="session")
def golden():
    return Golden(GOLDEN)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test needs CUDA (there is no CPU fallback by design)")
    import paper_2207_14589_b200  # noqa: F401
    from paper_2207_14589_b200 import _lib
    _lib.load()
    return torch.device("cuda", 0)


def rel_fro(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


@pytest.fixture(autouse=True)
def _device_debug_checks(request):
    """With a debug-check build loaded (SPED_LIB=<lib built with
    -DSPED_DEBUG_CHECKS=1>), every GPU test must leave the device-side
    bounds / protocol check bits clear (the stand-in for compute-sanitizer,
    which this pool does not allow)."""
    yield
    if request.node.get_closest_marker("gpu") is None:
        return
    import sys as _sys
    mod = _sys.modules.get("paper_2207_14589_b200._lib")
    if mod is None or mod._lib is None:
        return
    lib = mod._lib
    if int(lib.sped_debug_checks()) != 1:
        return
    bits = int(lib.sped_debug_take())
    assert bits == 0, f"device debug checks failed: bits {bits:#x}"
