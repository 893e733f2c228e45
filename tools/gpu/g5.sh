set -x
JHSVD_CYCLE=1 timeout 300 python -m pytest tests/test_cycle.py -x -q -m gpu 2>&1 | tail -15
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
JHSVD_CYCLE=1 TRACE=1 timeout 300 python tools/time_sweep.py 16384 32 1 64 2>&1 | tail -8
JHSVD_CYCLE=1 TRACE=1 timeout 300 python tools/time_sweep.py 4096 32 1 64 2>&1 | tail -8
JHSVD_CYCLE=1 timeout 300 python tools/time_sweep.py 16384 32 1 2>&1 | tail -3
