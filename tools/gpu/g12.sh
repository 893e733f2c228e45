set -x
timeout 600 python bench.py --n 2048 --warmup 1 --steps 1 --cpu-seconds 2 > gpurun_out/b2048.json 2> gpurun_out/b2048.err; tail -3 gpurun_out/b2048.err; cat gpurun_out/b2048.json
timeout 300 python bench.py --impl reference --n 2048 --warmup 0 --steps 1 --cpu-seconds 2 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
