D=paper_1401_2720_b200/_lib
for r in 1 2; do for L in libjhsvd_b200_old.so libjhsvd_b200.so; do echo "$L"; JHSVD_LIB=$D/$L timeout 120 python tools/time_sweep.py 16384 32 1 128 2>&1 | grep -E "ms/p"; JHSVD_LIB=$D/$L timeout 120 python tools/time_sweep.py 8192 32 1 2>&1 | grep -E "ms/p"; done; done
