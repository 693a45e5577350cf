mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_engine_gpu.py -q -m gpu -x --tb=long -k "mixed" > gpurun_out/g77t.log 2>&1; echo "exit $?" >> gpurun_out/g77t.log
