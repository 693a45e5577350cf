timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x > gpurun_out/kt.log 2>&1; echo "kt exit $?" >> gpurun_out/kt.log
timeout 300 python tools/kbench.py gemm > gpurun_out/kbench.log 2>&1; echo "kb exit $?" >> gpurun_out/kbench.log
