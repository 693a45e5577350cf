timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -m gpu -k "attention" > gpurun_out/kt.log 2>&1; echo "kt exit $?" >> gpurun_out/kt.log
timeout 300 python tools/kbench.py attn > gpurun_out/kbench.log 2>&1; echo "kb exit $?" >> gpurun_out/kbench.log
