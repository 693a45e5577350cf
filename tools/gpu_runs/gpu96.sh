mkdir -p gpurun_out
timeout 1500 python tools/decode_ablation.py 64 2048 > gpurun_out/g96_b64.log 2>&1
timeout 600 python tools/decode_ablation.py 1 2048 > gpurun_out/g96_b1.log 2>&1
