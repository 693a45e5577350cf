mkdir -p gpurun_out
for b in 128 64; do for v in 118 148 96; do echo "B $b min_ctas $v"; SP_SWAP_MIN_CTAS=$v timeout 600 python tools/decode_ablation.py $b 2048 base 2>&1 | grep TPOT; done; done > gpurun_out/g144.log
