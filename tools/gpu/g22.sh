# inner variant 6 (warp-0 chain, V warps behind): parity + A/B vs variant 5
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3; echo TESTS_DONE
for v in 0 1 0 1; do echo "I6=$v"; JHSVD_I6=$v timeout 120 python tools/time_sweep.py 16384 32 1 64 2>&1 | grep -E "ms/p|factor_inner"; done
for v in 0 1; do echo "I6=$v n=8192 full sweep"; JHSVD_I6=$v JHSVD_PDL=0 timeout 120 python tools/time_sweep.py 8192 32 1 2>&1 | grep -E "ms/p|factor_inner|gram|update"; done
