mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x --tb=short > gpurun_out/g103t.log 2>&1; echo "exit $?" >> gpurun_out/g103t.log
timeout 900 python tools/decode_ablation.py 256 2048 base > gpurun_out/g103_b256.log 2>&1
timeout 900 python tools/decode_ablation.py 128 2048 base > gpurun_out/g103_b128.log 2>&1
