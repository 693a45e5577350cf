mkdir -p gpurun_out
ncu --set full --import-source on -k regex:gemm_swap -s 3 -c 1 -o gpurun_out/swap_o2 python tools/swap_probe.py 64 4096 4096 add 5 > gpurun_out/g32_ncu.log 2>&1
