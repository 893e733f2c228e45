"""Dev-only CUDA library (``tools/dev/_lib/libjhsvd_dev.so``): the probes
that back DESIGN.md's exactness and rate claims -- DMMA rounding vs an
in-order fma chain, DMMA/DFMA issue rates, dependent-op latencies, and the
branch-free division / sqrt fast paths of the inner kernel against the IEEE
operators.  Built from ``tools/dev/csrc`` against the product headers; not
part of the solver library and never loaded by it.

    python tools/dev/devlib.py      # build
"""

from __future__ import annotations

import ctypes
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
LIB = HERE / "_lib" / "libjhsvd_dev.so"

_p, _i32, _i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
SIGNATURES = {
    "jh_probe_dmma": (_i32, [_p, _p, _p, _p, _p, _i32, _p]),
    "jh_probe_rate": (_i32, [_i32, _i32, _i32, _i32, _p, _p]),
    "jh_probe_latency": (_i32, [_p, _p]),
    "jh_probe_fastmath": (_i32, [_p, _p, _i64, _p, _p]),
}
_lib = None


def build(force: bool = False, verbose: bool = False) -> Path:
    sys.path.insert(0, str(ROOT))
    from paper_1401_2720_b200 import build_ext

    srcs = sorted((HERE / "csrc").glob("*.cu"))
    if not force and LIB.exists() and all(p.stat().st_mtime < LIB.stat().st_mtime for p in srcs):
        return LIB
    return build_ext.compile_shared(srcs, LIB, [ROOT / "include", build_ext.SRC],
                                    ROOT / "build" / "obj_dev", verbose)


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        lib = ctypes.CDLL(str(LIB))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


if __name__ == "__main__":
    print(build(force=True, verbose=False))
