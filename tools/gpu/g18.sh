set -x
timeout 300 python -m pytest tests/test_cycle.py -x -q -m gpu 2>&1 | tail -2
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for p in 0 1; do JHSVD_PDL=$p timeout 300 python tools/time_sweep.py 16384 32 1 2>&1 | tail -4; done
for p in 0 1; do JHSVD_PDL=$p timeout 300 python tools/time_sweep.py 8192 32 1 2>&1 | tail -4; done
