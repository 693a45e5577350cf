mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py tests/test_multiproc_gpu.py -q -m gpu -x --tb=short > gpurun_out/g95t.log 2>&1; echo "exit $?" >> gpurun_out/g95t.log
