mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -q -m gpu -x --tb=short > gpurun_out/g61t.log 2>&1; echo "exit $?" >> gpurun_out/g61t.log
timeout 1500 python tools/decode_ablation.py 64 2048 > gpurun_out/g61.log 2>&1
