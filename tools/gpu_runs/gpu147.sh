mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -q -m gpu -x --tb=short > gpurun_out/g147t.log 2>&1; echo "exit $?" >> gpurun_out/g147t.log
timeout 300 python tools/gemm_sweep.py 512 1024 8192 > gpurun_out/g147.log 2>&1
