D=paper_1401_2720_b200/_lib
JHSVD_ENGINE=0 JHSVD_LIB=$D/libjhsvd_b200_e128x3.so timeout 300 python -m pytest tests/test_cycle.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
for r in 1 2; do for L in libjhsvd_b200.so libjhsvd_b200_e128x2.so libjhsvd_b200_e128x3.so libjhsvd_b200_e96x3.so; do echo "$L"; JHSVD_ENGINE=0 JHSVD_LIB=$D/$L timeout 120 python tools/time_sweep.py 16384 32 1 64 2>&1 | grep -E "ms/p"; done; done
for L in libjhsvd_b200.so libjhsvd_b200_e128x2.so libjhsvd_b200_e128x3.so libjhsvd_b200_e96x3.so; do echo "$L"; JHSVD_LIB=$D/$L timeout 120 python tools/run_configs.py 1 2>&1 | cut -c 1-80; done
