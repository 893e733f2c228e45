timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for r in 1 2; do timeout 120 python tools/time_sweep.py 16384 32 1 128 2>&1 | grep -E "ms/p"; done
JHSVD_PDL=0 timeout 120 python tools/time_sweep.py 16384 32 1 64 2>&1 | grep -E "gram"
timeout 300 python tools/run_configs.py 1 2 4 5 2>&1 | cut -c1-110
