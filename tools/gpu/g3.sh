set -x
timeout 300 python -m pytest tests/test_cycle.py -x -q -m gpu 2>&1 | tail -15
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for n in 4096 16384; do
  timeout 300 python tools/time_sweep.py $n 32 1 64 2>&1 | tail -3
  JHSVD_CYCLE=0 timeout 300 python tools/time_sweep.py $n 32 1 64 2>&1 | tail -5
done
timeout 300 python tools/time_sweep.py 16384 32 1 2>&1 | tail -3
