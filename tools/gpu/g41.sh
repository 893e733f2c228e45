D=paper_1401_2720_b200/_lib
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
JHSVD_LIB=$D/libjhsvd_b200_prof.so SWEEPS=1 INNER_PHASES=1 timeout 300 python tools/sweep_profile.py 16384 | grep -v '"tasks": 0' | cut -c1-250
for r in 1 2; do for L in libjhsvd_b200_nosplit.so libjhsvd_b200.so; do echo "$L"; JHSVD_LIB=$D/$L timeout 120 python tools/time_sweep.py 16384 32 1 128 2>&1 | grep -E "ms/p"; JHSVD_PDL=0 JHSVD_LIB=$D/$L timeout 120 python tools/time_sweep.py 16384 32 1 64 2>&1 | grep -E "inner"; done; done
