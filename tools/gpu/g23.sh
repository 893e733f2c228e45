# ncu source-level capture of the inner kernels (variant 6 and 5)
mkdir -p gpurun_out
JHSVD_PDL=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_factor_inner6 -s 8 -c 1 -o gpurun_out/inner6 -f python tools/time_sweep.py 8192 32 1 16 > gpurun_out/ncu_i6.log 2>&1
JHSVD_I6=0 JHSVD_PDL=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_factor_inner5 -s 8 -c 1 -o gpurun_out/inner5 -f python tools/time_sweep.py 8192 32 1 16 > gpurun_out/ncu_i5.log 2>&1
tail -3 gpurun_out/ncu_i6.log gpurun_out/ncu_i5.log
