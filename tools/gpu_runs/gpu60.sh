mkdir -p gpurun_out
timeout 1500 python tools/decode_ablation.py 64 2048 > gpurun_out/g60.log 2>&1
