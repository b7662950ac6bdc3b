"""ctypes binding of libsped.so — the only way this package reaches the GPU.

The library is built in-tree (``python -m paper_2207_14589_b200.csrc.build``
or ``__graft_entry__.build()``).  There is no CPU fallback: if the library is
missing or CUDA is unavailable, every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import torch

LIB_PATH = Path(__file__).resolve().parent / "libsped.so"

SPED_OK = 0
SPED_ERR_ARG = 1
SPED_ERR_CUDA = 2
SPED_ERR_ZERO_DEGREE = 3
SPED_ERR_UNSUPPORTED = 4

_i32, _i64, _u32, _u64, _f64, _p, _sz = (C.c_int32, C.c_int64, C.c_uint32, C.c_uint64,
                                         C.c_double, C.c_void_p, C.c_size_t)

# name -> (restype, argtypes); mirrors include/sped.h
SIGNATURES = {
    "sped_last_error": (C.c_char_p, []),
    "sped_abi_version": (C.c_int, []),
    "sped_laplacian_build": (C.c_int, [_i64, _i64, _p, _p, _p, C.c_int, C.c_int, _p, _p, _p, _p,
                                       _p, C.POINTER(_i64), _p]),
    "sped_laplacian_build_rows": (C.c_int, [_i64, _i64, _i64, _i64, _p, _p, _p, _p, C.c_int,
                                            C.c_int, _p, _p, _p, _p, _p, C.POINTER(_i64), _p]),
    "sped_canonicalize_edges": (C.c_int, [_i64, _i64, _p, _p, _p, _p, _p, _p, C.POINTER(_i64),
                                          C.POINTER(_i32), _p]),
    "sped_degree_order": (C.c_int, [_i64, _p, _p, _p, _p]),
    "sped_relabel_edges": (C.c_int, [_i64, _i64, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "sped_spmm_plan_max_chunks": (_i64, [_i64, _i64, _i32, _i32]),
    "sped_spmm_plan": (C.c_int, [_i64, _p, _i32, _i32, _p, _i64, C.POINTER(_i64),
                                 C.POINTER(_i64), _p]),
    "sped_csr_poly_apply": (C.c_int, [_i64, _i32, _p, _p, _p, _i32, _i32, _p, _i64, _p, _p, _p,
                                      _i32, _i64, _p, _p, _p, _p, _p, _p, _i32, _p, _p, _p, _f64,
                                      _f64, _f64, _p]),
    "sped_csr_term_split": (C.c_int, [_i64, _i32, _p, _p, _p, _i32, _i32, _p, _i64, _p, _p, _p,
                                      _i32, _p, _p, _p, _i32, _p, _f64, _f64, _f64, _f64, _f64,
                                      _f64, _p]),
    "sped_csr_term_shard": (C.c_int, [_i64, _i32, _p, _p, _p, _i32, _i32, _p, _i64, _p, _p, _p,
                                      _i32, _p, _i32, _i32, _i64, _i64, _p, _p, _p, _i32, _p,
                                      _f64, _f64, _f64, _f64, _f64, _f64, _p]),
    "sped_edge_batch_workspace_bytes": (_i64, [_i64, _i64]),
    "sped_edge_batch_workspace_bytes_terms": (_i64, [_i64, _i64, _i32]),
    "sped_edge_batch_poly_apply": (C.c_int, [_i64, _i32, _i64, _p, _p, _p, _p, _p, _i64, _p, _i64,
                                             _p, _p, _p, _p, _p, _i32, _p, _p, _p, _f64, _f64, _f64,
                                             _p]),
    "sped_edge_batch_poly_apply_scaled": (C.c_int, [_i64, _i32, _i64, _p, _p, _p, _p, _p, _i64,
                                                    _f64, _p, _i64, _p, _p, _p, _p, _p, _i32, _p,
                                                    _p, _p, _f64, _f64, _f64, _p]),
    "sped_gram_workspace_bytes": (_sz, [_i64, _i32]),
    "sped_gram": (C.c_int, [_i64, _i32, _p, _p, _p, _p, _sz, _p]),
    "sped_gram_mueg": (C.c_int, [_i64, _i32, _p, _p, _p, _p, _sz, _p]),
    "sped_mueg_coeffs": (C.c_int, [_i32, _p, _f64, _p, _p, _p, _p]),
    "sped_oja_coeffs": (C.c_int, [_i32, _p, _f64, _i32, _p, _p, _p]),
    "sped_block_update": (C.c_int, [_i64, _i32, _p, _p, _p, _p, _f64, _p, _i32, _p, _p]),
    "sped_persistent_workspace_bytes": (C.c_int, [_i32, _i32, _p]),
    "sped_persistent_mueg": (C.c_int, [_i32, _i32, _i64, _p, _p, _p, _i32, _p, _p, _p, _f64, _f64,
                                       _f64, _f64, _i32, _p, _p, _p, _i64, _p]),
    "sped_persistent_oja": (C.c_int, [_i32, _i32, _i64, _p, _p, _p, _i32, _p, _p, _p, _f64, _f64,
                                      _f64, _f64, _i32, _p, _p, _p, _i64, _p]),
    "sped_walk_index_workspace_bytes": (_i64, [_i64, _i64]),
    "sped_walk_index_build": (C.c_int, [_i64, _i64, _p, _p, _p, _p, _p, _p, _i64, _p]),
    "sped_walk_workspace_bytes": (_i64, [_i64, _i32, _i64]),
    "sped_walk_poly_estimate": (C.c_int, [_i64, _i64, _i32, _p, _p, _p, _p, _p, _p, _i32, _p, _i32,
                                          _i64, _i64, _p, _p, _p, _p, _i64, _p]),
    "sped_axpby": (C.c_int, [_i64, _f64, _p, _f64, _p, _p, _p]),
    "sped_pcg64_workspace_bytes": (_sz, [_i64]),
    "sped_pcg64_integers": (C.c_int, [_u64, _u64, _u64, _u64, _i32, _u32, _u64, _i64, _p,
                                      C.POINTER(_i64), _p, _sz, _p]),
    "sped_pcg64_integers_device": (C.c_int, [_p, _u64, _i64, _p, _p, _p, _sz, _p]),
    "sped_kmeans_assign": (C.c_int, [_i64, _i32, _i32, _p, _p, _p, _p, _p, _p, _p]),
    "sped_row_dist2": (C.c_int, [_i64, _i32, _p, _p, _p, _i32, _p]),
    "sped_gather_rows": (C.c_int, [_i64, _i32, _p, _p, _p, _p]),
    "sped_debug_checks": (C.c_int, []),
    "sped_debug_take": (_u32, []),
}

_lib = None
_lock = threading.Lock()


class SpedError(RuntimeError):
    pass


def load() -> C.CDLL:
    """Load libsped.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("SPED_LIB", str(LIB_PATH))
        if not Path(path).exists():
            raise ImportError(
                f"{path} is missing: build it with `python -m paper_2207_14589_b200.csrc.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == SPED_OK:
        return
    msg = load().sped_last_error().decode(errors="replace")
    if rc in (SPED_ERR_ARG, SPED_ERR_ZERO_DEGREE):
        if rc == SPED_ERR_ZERO_DEGREE:
            msg = "normalized Laplacian requires all degrees > 0"
        raise ValueError(f"{what}: {msg}" if what and rc == SPED_ERR_ARG else msg)
    raise SpedError(f"{what} failed (status {rc}): {msg}")


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2207_14589_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    load()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise ValueError(f"device must be CUDA, got {dev}")
    return dev


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int | None:
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def i64_array(vals):
    return (C.c_int64 * max(1, len(vals)))(*[int(v) for v in vals])


def dbl_array(vals):
    arr = (C.c_double * max(1, len(vals)))(*[float(v) for v in vals])
    return arr
