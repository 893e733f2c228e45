# Round profile captures (run on the GPU box from the repo root):
#  1. launch list of the bench command (our kernels, first 400 launches)
#  2. ncu --set full of one launch of each hot kernel at p-step ~30 of sweep 1
set -x
mkdir -p gpurun_out/prof
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 400 --csv \
  --log-file gpurun_out/prof/launches_bench.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e \
  > gpurun_out/prof/bench_under_ncu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_update_mix|k_gram_tma|k_factor_inner5" --launch-skip 90 -c 3 \
  -o gpurun_out/prof/hot python tools/time_sweep.py 16384 32 1 40 > gpurun_out/prof/hot.log 2>&1
ncu -i gpurun_out/prof/hot.ncu-rep --page raw --csv > gpurun_out/prof/hot_raw.csv 2>/dev/null
ls -la gpurun_out/prof
