nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -m gpu > gpurun_out/kt.log 2>&1; echo "kt exit $?" >> gpurun_out/kt.log
timeout 300 python tools/kbench.py all > gpurun_out/kbench.log 2>&1; echo "kb exit $?" >> gpurun_out/kbench.log
