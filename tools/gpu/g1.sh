set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for n in 4096 16384; do
  timeout 300 python tools/time_sweep.py $n 32 1 64 2>&1 | tail -8
  JHSVD_DATAFLOW=0 timeout 300 python tools/time_sweep.py $n 32 1 64 2>&1 | tail -8
done
