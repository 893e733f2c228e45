"""ctypes binding of the in-tree CUDA library ``_lib/libjhsvd_b200.so``.

There is no CPU fallback: importing the solver works anywhere, but the first
call that needs the GPU raises :class:`NativeUnavailable` when the library
or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "_lib" / "libjhsvd_b200.so"
if os.environ.get("JHSVD_LIB"):  # A/B runs against another build of the library
    LIB_PATH = Path(os.environ["JHSVD_LIB"])


class NativeUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is not available."""


_c_i64 = ctypes.c_int64
_c_i32 = ctypes.c_int
_c_d = ctypes.c_double
_c_p = ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/jhsvd_b200.h
SIGNATURES = {
    "jh_sweep_workspace_bytes": (_c_i64, [_c_i64, _c_i32, _c_i64]),
    "jh_cycle_plan_ints": (_c_i64, [_c_i32, _c_i32]),
    "jh_cycle_plan": (_c_i32, [_c_p, _c_i32, _c_i32, _c_p]),
    "jh_block_sweep": (_c_i32, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_i64, _c_i32,
                                _c_p, _c_i32, _c_p, _c_p, _c_i32, _c_i32, _c_i32, _c_i32, _c_p,
                                _c_i64, _c_i32, _c_d, _c_p, _c_i64, _c_p, _c_p]),
    "jh_set_overlap": (_c_i32, [_c_i32]),
    "jh_set_simple_kernels": (_c_i32, [_c_i32]),
    "jh_gram": (_c_i32, [_c_p, _c_i64, _c_i64, _c_i32, _c_p, _c_p]),
    "jh_qr_peeloff": (_c_i32, [_c_p, _c_i64, _c_i64, _c_i32, _c_p, _c_p]),
    "jh_cholesky": (_c_i32, [_c_p, _c_i32, _c_p, _c_p, _c_p]),
    "jh_inner_jacobi": (_c_i32, [_c_p, _c_p, _c_i32, _c_p, _c_p, _c_d, _c_i32, _c_p, _c_p]),
    "jh_gemm": (_c_i32, [_c_p, _c_i64, _c_i64, _c_i32, _c_p, _c_i64, _c_i32, _c_p, _c_i64, _c_p]),
    "jh_back_substitute": (_c_i32, [_c_p, _c_i32, _c_p, _c_i32, _c_p, _c_p]),
    "jh_safe_bounds": (None, [_c_i64, _c_p, _c_p]),
    "jh_column_norms": (_c_i32, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p]),
    "jh_check_scaling": (_c_i32, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p]),
    "jh_sigma_u": (_c_i32, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_p, _c_p]),
    "jh_robust_norms": (_c_i32, [_c_p, _c_i64, _c_i64, _c_i64, _c_i32, _c_i32, _c_p, _c_p, _c_p,
                                 _c_p, _c_p]),
    "jh_common_form": (None, [_c_i64, _c_d, _c_p, _c_p]),
    "jh_add_scaled": (None, [_c_i64, _c_d, _c_i64, _c_d, _c_p, _c_p]),
    "jh_scale_exponent": (_c_i32, [_c_d, _c_d, _c_i32]),
    "jh_rotations": (_c_i32, [_c_p, _c_p, _c_i64, _c_p, _c_p]),
    "jh_gen_workspace_bytes": (_c_i64, [_c_i64, _c_i64, _c_i64, _c_i32]),
    "jh_gen_butterfly": (_c_i32, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, ctypes.c_ulonglong,
                                  _c_i32, _c_d, _c_p, _c_i64, _c_p]),
    "jh_launch_count": (ctypes.c_ulonglong, []),
    "jh_profile_begin": (_c_i32, [_c_i32]),
    "jh_profile_end": (_c_i32, [_c_p, _c_p]),
}

_lib = None


def load_library():
    """Load the shared library (no device needed); raises NativeUnavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeUnavailable(
            f"{LIB_PATH} is missing: run `python -m paper_1401_2720_b200.build_ext` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def require_cuda():
    """The library plus a CUDA device of compute capability 10.x."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: jhsvd_b200 runs on B200 (sm_100a) only")
    major, _ = torch.cuda.get_device_capability()
    if major != 10:
        raise NativeUnavailable(f"sm_{major}x device: jhsvd_b200 is built for sm_100a only")
    return load_library()


def check(rc: int, what: str) -> None:
    if rc != 0:
        if rc in (-1000, -1001):
            raise ValueError(f"{what}: invalid arguments (code {rc})")
        raise RuntimeError(f"{what}: CUDA error {-rc}")


def ptr(t) -> int:
    return t.data_ptr() if t is not None else None


def stream_handle():
    import torch

    return torch.cuda.current_stream().cuda_stream
