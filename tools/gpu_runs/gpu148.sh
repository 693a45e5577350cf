mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:gemm_swap -s 2 -c 1 -o gpurun_out/g148_swap256 python tools/gemm_one.py 256 4096 14336 f32 > gpurun_out/g148.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:gemm_swap -s 2 -c 1 -o gpurun_out/g148_swap64 python tools/gemm_one.py 64 4096 14336 f32 >> gpurun_out/g148.log 2>&1
