# A/B: Grams of p-step s+1 inside the update launch of p-step s (JHSVD_GMIX)
JHSVD_GMIX=1 timeout 400 python -m pytest tests/test_cycle.py -x -q -m gpu 2>&1 | tail -2; echo TESTS_DONE
for n in 16384 8192 4096; do for v in 0 1 0 1; do echo "GMIX=$v n=$n"; JHSVD_GMIX=$v timeout 120 python tools/time_sweep.py $n 32 1 2>&1 | grep ms/p; done; done
for v in 0 1; do echo "GMIX=$v configs"; JHSVD_GMIX=$v timeout 300 python tools/run_configs.py 2 4 5 2>&1 | tail -3; done
