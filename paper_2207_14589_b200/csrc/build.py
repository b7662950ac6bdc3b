"""Build libsped.so (sm_100a) in-tree with nvcc.

    python -m paper_2207_14589_b200.csrc.build [--force] [-j N]

Every ``*.cu`` in this directory is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` into
``build/<name>.o`` and linked into ``paper_2207_14589_b200/libsped.so``.
Objects are rebuilt when their source, a header or this file changes.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

CSRC = Path(__file__).resolve().parent
PKG = CSRC.parent
ROOT = PKG.parent
BUILD = ROOT / "build" / "sped"
LIB = PKG / "libsped.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xptxas", "-v", "-I", str(ROOT / "include")]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libsped.so")


def _deps_mtime() -> float:
    heads = list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h")) + [Path(__file__)]
    return max(p.stat().st_mtime for p in heads)


def _compile(src: Path, force: bool, defines=(), tag="") -> tuple[Path, str]:
    obj = BUILD / (src.stem + tag + ".o")
    if not force and obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, _deps_mtime()):
        return obj, ""
    cmd = [nvcc(), *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stdout}\n{res.stderr}")
    (BUILD / (src.stem + tag + ".ptxas.txt")).write_text(res.stdout + res.stderr)
    return obj, res.stderr


def build(force: bool = False, jobs: int | None = None, verbose: bool = False,
          defines=(), out: Path | None = None) -> Path:
    """Build libsped.so (or a tuning variant with extra -D defines into
    ``out``; variants are selected at run time with SPED_LIB=<path>)."""
    BUILD.mkdir(parents=True, exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu"))
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)
    lib = LIB if out is None else Path(out)
    tag = "" if not defines else "_" + "_".join(d.replace("=", "") for d in defines)
    with ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(lambda s: _compile(s, force, defines, tag), srcs))
    objs = [r[0] for r in results]
    newest = max(o.stat().st_mtime for o in objs)
    if force or not lib.exists() or lib.stat().st_mtime < newest:
        tmp = lib.with_suffix(".so.tmp")
        cmd = [nvcc(), *ARCH, "-shared", "--cudart", "static", "-o", str(tmp), *map(str, objs)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
        os.replace(tmp, lib)
    if verbose:
        for _, log in results:
            if log:
                print(log, file=sys.stderr)
    return lib


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("-v", action="store_true")
    ap.add_argument("-D", action="append", default=[], help="extra define (tuning variants)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    print(build(force=a.force, jobs=a.j, verbose=a.v, defines=tuple(a.D), out=a.out))


if __name__ == "__main__":
    main()
