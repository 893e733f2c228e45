D=paper_1401_2720_b200/_lib
for r in 1 2; do for L in libjhsvd_b200.so libjhsvd_b200_u4.so libjhsvd_b200_u8.so libjhsvd_b200_u16.so; do echo "$L"; JHSVD_PDL=0 JHSVD_LIB=$D/$L timeout 120 python tools/time_sweep.py 16384 32 1 64 2>&1 | grep -E "inner"; done; done
