mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fullwidth_gpu.py tests/test_engine_gpu.py -q -m gpu -x --tb=short > gpurun_out/g94t.log 2>&1; echo "exit $?" >> gpurun_out/g94t.log
