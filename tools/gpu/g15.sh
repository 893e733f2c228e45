set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for nw in 2 4; do for n in 4096 16384; do JHSVD_GRAM_NW=$nw timeout 300 python tools/time_sweep.py $n 32 1 64 2>&1 | tail -4 | head -2; done; done
timeout 900 python tools/run_configs.py 5 2>&1 | tail -1
