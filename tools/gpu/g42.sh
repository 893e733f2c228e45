timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for r in 1 2; do for v in 0 1; do echo "CHAIN=$v"; JHSVD_PDL_CHAIN=$v timeout 120 python tools/time_sweep.py 16384 32 1 128 2>&1 | grep -E "ms/p"; JHSVD_PDL_CHAIN=$v timeout 120 python tools/time_sweep.py 8192 32 1 2>&1 | grep -E "ms/p"; done; done
for v in 0 1; do JHSVD_PDL_CHAIN=$v timeout 300 python tools/run_configs.py 1 2 4 | cut -c1-80; done
