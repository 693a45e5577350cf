mkdir -p gpurun_out
ncu --set full -k regex:gemm_swap -s 3 -c 1 -o gpurun_out/swap_bf16 python tools/swap_probe.py 64 28672 4096 bf16 3 > gpurun_out/g41a.log 2>&1
ncu --set full -k regex:gemm_swap -s 3 -c 1 -o gpurun_out/swap_swiglu python tools/swap_probe.py 64 28672 4096 swiglu 3 > gpurun_out/g41b.log 2>&1
