timeout 600 python tools/decode_profile.py 64 2048 5 > gpurun_out/dp.log 2>&1
timeout 600 python tools/decode_profile.py 1 2048 5 >> gpurun_out/dp.log 2>&1
timeout 600 python tools/decode_profile.py 256 2048 5 >> gpurun_out/dp.log 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "gemm" > gpurun_out/kt.log 2>&1; echo "kt exit $?" >> gpurun_out/kt.log
