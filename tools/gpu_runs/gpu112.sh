mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multiproc_gpu.py -q -m gpu -x --tb=short > gpurun_out/g112t.log 2>&1; echo "exit $?" >> gpurun_out/g112t.log
