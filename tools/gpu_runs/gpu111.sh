mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_kernels_gpu.py -q -m gpu -x --tb=short -k "comm or swiftkv or decode_split" > gpurun_out/g111t.log 2>&1; echo "exit $?" >> gpurun_out/g111t.log
