# A/B of two library builds (JHSVD_LIB) on engine-1 sweeps
NEW=paper_1401_2720_b200/_lib/libjhsvd_b200.so
OLD=paper_1401_2720_b200/_lib/libjhsvd_b200_prev.so
for r in 1 2; do for L in $OLD $NEW; do echo "$L"; JHSVD_LIB=$L timeout 120 python tools/time_sweep.py 16384 32 1 128 2>&1 | grep -E "ms/p"; done; done
for L in $OLD $NEW; do echo "$L n=8192"; JHSVD_LIB=$L timeout 120 python tools/time_sweep.py 8192 32 1 2>&1 | grep -E "ms/p"; done
for L in $OLD $NEW; do echo "$L late-sweep-like n=16384 sweep 2"; JHSVD_LIB=$L timeout 200 python tools/time_sweep.py 16384 32 2 256 2>&1 | grep -E "ms/p"; done
