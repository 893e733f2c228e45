for r in 1 2; do for v in 0 1; do echo "VSCHED=$v"; JHSVD_VSCHED=$v timeout 300 python tools/time_sweep.py 16384 32 2 2>&1 | grep "p-step)"; done; done
JHSVD_VSCHED=0 timeout 300 python -m pytest tests/test_cycle.py -x -q -m gpu 2>&1 | tail -1
