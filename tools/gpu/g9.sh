set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_r01c.json 2> gpurun_out/bench_r01c.err; tail -3 gpurun_out/bench_r01c.err; cat gpurun_out/bench_r01c.json
