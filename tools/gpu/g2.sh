set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dataflow -c 1 -o gpurun_out/df16 python tools/time_sweep.py 16384 32 1 16 2>&1 | tail -5
