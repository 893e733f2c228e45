"""Build a variant of the product library with extra nvcc defines (dev tool),
for A/B runs with tools/ab_pstep.py (JHSVD_LIBS=...):

    python tools/build_variant.py NAME [-DJH_FOO=1 ...]   -> build/variants/NAME.so
"""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1401_2720_b200 import build_ext as B  # noqa: E402


def main():
    name, defines = sys.argv[1], sys.argv[2:]
    saved = list(B.NVCC_FLAGS)
    B.NVCC_FLAGS[:] = saved + defines
    try:
        out = B.compile_shared(B.sources(), ROOT / "build" / "variants" / f"{name}.so",
                               [ROOT / "include", B.SRC], ROOT / "build" / "obj_var" / name)
    finally:
        B.NVCC_FLAGS[:] = saved
    print(out)


if __name__ == "__main__":
    main()
