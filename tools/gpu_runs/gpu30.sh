mkdir -p gpurun_out
python tools/swap_probe.py 64 4096 4096 add > gpurun_out/g30.log 2>&1
python tools/swap_probe.py 64 28672 4096 swiglu >> gpurun_out/g30.log 2>&1
python tools/swap_probe.py 1 4096 4096 add >> gpurun_out/g30.log 2>&1
ncu --set full --import-source on -k regex:gemm_swap -s 3 -c 1 -o gpurun_out/swap_o python tools/swap_probe.py 64 4096 4096 add 5 > gpurun_out/g30_ncu.log 2>&1
