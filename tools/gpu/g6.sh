set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cycle$ --launch-skip 1 -c 1 -o gpurun_out/cy16k python tools/time_sweep.py 16384 32 1 24 2>&1 | tail -5
