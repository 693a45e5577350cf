mkdir -p gpurun_out
timeout 1500 python tools/decode_ablation.py 256 2048 > gpurun_out/g102_b256.log 2>&1
