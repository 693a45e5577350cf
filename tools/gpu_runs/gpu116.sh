mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x --tb=short -k "gemm" > gpurun_out/g116t.log 2>&1; echo "exit $?" >> gpurun_out/g116t.log
(echo new_default; timeout 300 python tools/gemm_sweep.py 384 512 768 1024 1536 2048) > gpurun_out/g116.log 2>&1
