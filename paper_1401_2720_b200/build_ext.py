"""Build the in-tree CUDA library ``_lib/libjhsvd_b200.so`` for sm_100a.

The library is plain nvcc output (no torch extension machinery): CUDA
kernels plus the ``extern "C"`` entry points declared in
``include/jhsvd_b200.h``.  Built in-tree so the ``.so`` travels with the repo
snapshot to the GPU box.

    python -m paper_1401_2720_b200.build_ext [--force]
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libjhsvd_b200.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # exactness: never contract a*b+c; only explicit fma() rounds once
    "-fmad=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build jhsvd_b200")


def sources() -> list[Path]:
    return sorted(SRC.glob("*.cu"))


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = sources() + sorted(SRC.glob("*.cuh")) + [ROOT / "include" / "jhsvd_b200.h"]
    return any(p.stat().st_mtime > t for p in deps)


def compile_shared(srcs: list[Path], out: Path, includes: list[Path], obj_dir: Path,
                   verbose: bool = False) -> Path:
    """nvcc -c every source in parallel, then link one shared library."""
    from concurrent.futures import ThreadPoolExecutor

    obj_dir.mkdir(parents=True, exist_ok=True)
    inc = [a for d in includes for a in ("-I", str(d))]
    nvcc = _nvcc()

    def one(src: Path) -> Path:
        obj = obj_dir / (src.stem + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *inc, "-c", "-o", str(obj), str(src)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(one, srcs))
    out.parent.mkdir(parents=True, exist_ok=True)
    tmp = out.with_suffix(".so.tmp")
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp),
           *map(str, objs)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, out)
    return out


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    return compile_shared(sources(), LIB, [ROOT / "include", SRC], ROOT / "build" / "obj",
                          verbose)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
