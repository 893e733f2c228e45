timeout 600 python -m pytest tests/test_cycle.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
for r in 1 2; do for v in 0 1; do echo "SPLIT=$v"; JHSVD_GRAM_SPLIT=$v JHSVD_PDL=0 timeout 120 python tools/time_sweep.py 16384 32 1 64 2>&1 | grep -E "gram"; JHSVD_GRAM_SPLIT=$v timeout 120 python tools/time_sweep.py 16384 32 1 128 2>&1 | grep -E "ms/p"; done; done
