mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_pair -s 2 -c 1 -o gpurun_out/g74_o1024 python tools/gemm_sweep.py 1024 > gpurun_out/g74.log 2>&1
