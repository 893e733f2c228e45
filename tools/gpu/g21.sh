# Gram wave quantization probe: K1 time vs number of tasks at m = 16384
for n in 16384 14208 9472 18944; do echo "n=$n"; OUTER=mm M=16384 JHSVD_PDL=0 timeout 120 python tools/time_sweep.py $n 32 1 32 2>&1 | grep -E "gram|ms/p"; done
