JHSVD_ENGINE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update5" --launch-skip 8 -c 2 -o gpurun_out/u5 python tools/time_sweep.py 16384 32 1 16 2>&1 | tail -2
