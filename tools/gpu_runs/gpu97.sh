mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "norm or partial" > gpurun_out/g97t.log 2>&1; echo "exit $?" >> gpurun_out/g97t.log
timeout 600 python tools/decode_ablation.py 64 2048 base > gpurun_out/g97_b64.log 2>&1
timeout 600 python tools/decode_ablation.py 1 2048 base > gpurun_out/g97_b1.log 2>&1
