set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err; tail -3 gpurun_out/bench_r01b.err; cat gpurun_out/bench_r01b.json
