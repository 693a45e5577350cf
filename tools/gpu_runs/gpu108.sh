mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x --tb=short -k "decode" > gpurun_out/g108k.log 2>&1; echo "exit $?" >> gpurun_out/g108k.log
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_fullwidth_gpu.py tests/test_spec_gpu.py -q -m gpu -x --tb=short > gpurun_out/g108t.log 2>&1; echo "exit $?" >> gpurun_out/g108t.log
for b in 1 16 32 64; do for c in 0 1; do echo "B $b cluster $c"; SP_DECODE_CLUSTER=$c timeout 600 python tools/decode_ablation.py $b 2048 base 2>&1 | grep TPOT; done; done > gpurun_out/g108.log
