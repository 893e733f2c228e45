set -x
timeout 300 python -m pytest tests/test_cycle.py -x -q -m gpu 2>&1 | tail -3
TRACE=1 timeout 300 python tools/time_sweep.py 16384 32 1 64 2>&1 | tail -12
TRACE=1 timeout 300 python tools/time_sweep.py 4096 32 1 64 2>&1 | tail -12
