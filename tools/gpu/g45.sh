D=paper_1401_2720_b200/_lib
JHSVD_LIB=$D/libjhsvd_b200_s1.so timeout 300 python -m pytest tests/test_cycle.py -x -q -m gpu 2>&1 | tail -1
for r in 1 2; do for L in libjhsvd_b200.so libjhsvd_b200_s1.so libjhsvd_b200_s2.so; do echo "$L"; JHSVD_LIB=$D/$L timeout 120 python tools/time_sweep.py 16384 32 1 128 2>&1 | grep -E "ms/p"; done; done
for L in libjhsvd_b200.so libjhsvd_b200_s1.so libjhsvd_b200_s2.so; do echo "$L"; JHSVD_LIB=$D/$L timeout 120 python tools/time_sweep.py 8192 32 1 2>&1 | grep -E "ms/p"; JHSVD_ENGINE=0 JHSVD_LIB=$D/$L timeout 120 python tools/time_sweep.py 16384 32 1 64 2>&1 | grep -E "ms/p"; done
