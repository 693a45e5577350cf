mkdir -p gpurun_out
timeout 1500 python tools/decode_ablation.py 1 2048 > gpurun_out/g63.log 2>&1
