mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py tests/test_fullwidth_gpu.py -q -m gpu -x --tb=short > gpurun_out/g107t.log 2>&1; echo "exit $?" >> gpurun_out/g107t.log
for b in 1 16 64; do timeout 600 python tools/decode_ablation.py $b 2048 base 2>&1 | grep TPOT; done > gpurun_out/g107.log
