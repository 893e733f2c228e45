timeout 300 python -m pytest tests/test_cycle.py -x -q -m gpu 2>&1 | grep -v "^  " | grep -n "Error\|assert\|FAILED\|^E " | head -10
JHSVD_PDL=1 timeout 120 python tools/time_sweep.py 16384 32 1 64 2>&1 | tail -15; echo "exit $?"
