set -x
timeout 300 python -m pytest tests/test_cycle.py -x -q -m gpu 2>&1 | tail -2
JHSVD_ENGINE=1 timeout 300 python tools/time_sweep.py 16384 32 1 2>&1 | tail -5
JHSVD_ENGINE=1 timeout 300 python tools/time_sweep.py 4096 32 1 2>&1 | tail -5
JHSVD_ENGINE=1 timeout 300 python tools/time_sweep.py 8192 32 1 2>&1 | tail -5
JHSVD_ENGINE=0 timeout 300 python tools/time_sweep.py 8192 32 1 2>&1 | tail -5
