timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_kernels_gpu.py tests/test_serving_gpu.py -q -m gpu -x > gpurun_out/gt.log 2>&1; echo "gt exit $?" >> gpurun_out/gt.log
