D=paper_1401_2720_b200/_lib
for r in 1 2; do for L in libjhsvd_b200.so libjhsvd_b200_r48s4.so libjhsvd_b200_r32s6.so libjhsvd_b200_r96s2.so libjhsvd_b200_r64s2.so; do echo "$L"; JHSVD_PDL=0 JHSVD_LIB=$D/$L timeout 120 python tools/time_sweep.py 16384 32 1 64 2>&1 | grep -E "gram"; done; done
for L in libjhsvd_b200.so libjhsvd_b200_r48s4.so libjhsvd_b200_r32s6.so; do echo "$L tall"; JHSVD_PDL=0 M=131072 JHSVD_LIB=$D/$L timeout 120 python tools/time_sweep.py 8192 32 1 16 2>&1 | grep -E "gram"; done
