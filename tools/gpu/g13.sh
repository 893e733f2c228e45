set -x
timeout 300 python -m pytest tests/test_cycle.py -x -q -m gpu 2>&1 | tail -3
for e in 0 1; do JHSVD_ENGINE=$e timeout 300 python tools/time_sweep.py 16384 32 1 64 2>&1 | tail -4; done
JHSVD_ENGINE=1 timeout 300 python tools/time_sweep.py 16384 32 1 2>&1 | tail -4
