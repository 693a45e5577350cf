mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_spec_gpu.py -q -m gpu -x --tb=short > gpurun_out/g98t.log 2>&1; echo "exit $?" >> gpurun_out/g98t.log
