timeout 1200 python -m pytest tests/test_fullwidth_gpu.py -q -m gpu -x > gpurun_out/fw.log 2>&1; echo "fw exit $?" >> gpurun_out/fw.log
