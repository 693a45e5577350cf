mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "decode" > gpurun_out/g142t.log 2>&1; echo "exit $?" >> gpurun_out/g142t.log
for b in 1 4 8 16 32 64; do echo "B $b"; timeout 600 python tools/decode_ablation.py $b 2048 base 2>&1 | grep TPOT; done > gpurun_out/g142.log
