mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -q -m gpu -x --tb=short -k "partial_norm or fused_decode_norm or cuda_graph" > gpurun_out/g134t.log 2>&1; echo "exit $?" >> gpurun_out/g134t.log
