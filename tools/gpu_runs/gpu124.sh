mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -q -m gpu -x --tb=short -k "rope or head_dim_128 or fused" > gpurun_out/g124t.log 2>&1; echo "exit $?" >> gpurun_out/g124t.log
