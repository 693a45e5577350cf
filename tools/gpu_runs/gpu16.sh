timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "rope or attention" > gpurun_out/kt.log 2>&1; echo "kt exit $?" >> gpurun_out/kt.log
timeout 900 ncu --set full --clock-control none -k regex:gemm_swap -s 8 -c 4 -o gpurun_out/prof_swap python tools/decode_profile.py 64 2048 1 > gpurun_out/ncu_swap.log 2>&1; echo "exit $?" >> gpurun_out/ncu_swap.log
timeout 900 ncu --set full --clock-control none -k regex:decode_tma -s 4 -c 1 -o gpurun_out/prof_dec python tools/decode_profile.py 64 2048 1 > gpurun_out/ncu_dec2.log 2>&1; echo "exit $?" >> gpurun_out/ncu_dec2.log
