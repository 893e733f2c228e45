#!/bin/bash
# Build the library with extra nvcc flags into another file, for A/B runs
# through JHSVD_LIB (dev tool):  tools/build_variant.sh OUT.so -DJH_VSLAB=1024 ...
set -e
out=$1; shift
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -Xcompiler -fPIC,-ffp-contract=off -shared -I include "$@" -o "$out" paper_1401_2720_b200/csrc/*.cu
