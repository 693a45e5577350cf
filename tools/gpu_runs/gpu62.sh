mkdir -p gpurun_out
for mc in 98 148 120 74 98; do echo "min_ctas $mc" >> gpurun_out/g62.log; SP_SWAP_MIN_CTAS=$mc timeout 600 python tools/decode_ablation.py 64 2048 base >> gpurun_out/g62.log 2>&1; done
for mc in 148 200 296; do echo "B1 min_ctas $mc" >> gpurun_out/g62.log; SP_SWAP_MIN_CTAS=$mc timeout 600 python tools/decode_ablation.py 1 2048 base >> gpurun_out/g62.log 2>&1; done
