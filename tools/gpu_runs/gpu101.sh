mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "norm or partial" > gpurun_out/g101t.log 2>&1; echo "exit $?" >> gpurun_out/g101t.log
for v in 1 2 4 8; do echo "cluster $v"; SP_NORM_CLUSTER=$v timeout 300 python tools/decode_ablation.py 64 2048 base 2>&1 | grep TPOT; SP_NORM_CLUSTER=$v timeout 300 python tools/decode_ablation.py 1 2048 base 2>&1 | grep TPOT; done > gpurun_out/g101.log
