timeout 300 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "cta_pair" > gpurun_out/kt.log 2>&1; echo "kt exit $?" >> gpurun_out/kt.log
