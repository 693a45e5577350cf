timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -q -m gpu -x -k "attention or head_dim_128 or c1 or decode" > gpurun_out/kt.log 2>&1; echo "kt exit $?" >> gpurun_out/kt.log
timeout 300 python tools/kbench.py attn > gpurun_out/kbench.log 2>&1; echo "kb exit $?" >> gpurun_out/kbench.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
