timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu > gpurun_out/kt.log 2>&1; echo "kt exit $?" >> gpurun_out/kt.log
timeout 600 python -m pytest tests/test_engine_gpu.py -q -m gpu -k "head_dim_128 or bitexact" > gpurun_out/et.log 2>&1; echo "et exit $?" >> gpurun_out/et.log
timeout 300 python tools/kbench.py all > gpurun_out/kbench.log 2>&1; echo "kb exit $?" >> gpurun_out/kbench.log
