timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
JHSVD_I7=0 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_cycle.py -x -q -m gpu 2>&1 | tail -1
for r in 1 2; do for v in 0 1; do echo "I7=$v"; JHSVD_I7=$v timeout 120 python tools/time_sweep.py 16384 32 1 128 2>&1 | grep -E "ms/p"; JHSVD_I7=$v JHSVD_PDL=0 timeout 120 python tools/time_sweep.py 16384 32 1 64 2>&1 | grep -E "inner"; done; done
for v in 0 1; do echo "I7=$v"; JHSVD_I7=$v timeout 120 python tools/late_probe.py 16384 64 2>&1 | tail -1; JHSVD_I7=$v timeout 120 python tools/time_sweep.py 8192 32 1 2>&1 | grep -E "ms/p"; done
