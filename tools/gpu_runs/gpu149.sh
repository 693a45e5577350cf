mkdir -p gpurun_out
for v in 0 32 64 96 0 64; do echo "sq $v"; if [ $v = 0 ]; then timeout 600 python tools/decode_ablation.py 64 2048 base 2>&1 | grep TPOT; else SP_SWAP_MIN_CTAS_SQ=$v timeout 600 python tools/decode_ablation.py 64 2048 base 2>&1 | grep TPOT; fi; done > gpurun_out/g149.log
