"""The C-ABI library loads and exports every entry point include/sped.h
declares (CPU: no kernel launches)."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "sped.h"
LIB = ROOT / "paper_2207_14589_b200" / "libsped.so"


def declared_symbols():
    src = HEADER.read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sped_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for s in ("sped_laplacian_build", "sped_csr_poly_apply", "sped_edge_batch_poly_apply",
              "sped_gram", "sped_mueg_coeffs", "sped_block_update", "sped_pcg64_integers"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    if not LIB.exists():
        pytest.fail(f"{LIB} not built (python -m paper_2207_14589_b200.csrc.build)")
    lib = ctypes.CDLL(str(LIB))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_binding_signatures_cover_header():
    from paper_2207_14589_b200 import _lib
    assert set(declared_symbols()) <= set(_lib.SIGNATURES)


def test_abi_version_callable_without_gpu():
    lib = ctypes.CDLL(str(LIB))
    assert lib.sped_abi_version() == 1
    lib.sped_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.sped_last_error(), bytes)
