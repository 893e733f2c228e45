D=paper_1401_2720_b200/_lib
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for L in libjhsvd_b200_old.so libjhsvd_b200.so; do echo "$L engine0"; JHSVD_ENGINE=0 JHSVD_LIB=$D/$L timeout 120 python tools/time_sweep.py 16384 32 1 64 2>&1 | grep -E "ms/p"; done
for L in libjhsvd_b200_old.so libjhsvd_b200.so; do echo "$L configs"; JHSVD_LIB=$D/$L timeout 300 python tools/run_configs.py 2 4 5 2>&1 | cut -c1-120; done
