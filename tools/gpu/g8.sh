set -x
JHSVD_ENGINE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_vpair|k_update_tma|k_gram_tma|k_factor_inner5" --launch-skip 16 -c 8 -o gpurun_out/e1 python tools/time_sweep.py 16384 32 1 16 2>&1 | tail -3
