mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_multiproc_gpu.py -q -m gpu -x --tb=long > gpurun_out/g78t.log 2>&1; echo "exit $?" >> gpurun_out/g78t.log
