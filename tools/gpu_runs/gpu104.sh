mkdir -p gpurun_out
for v in 32 64 96 148; do echo "min_ctas $v"; SP_SWAP_MIN_CTAS=$v timeout 600 python tools/decode_ablation.py 256 2048 base 2>&1 | grep TPOT; done > gpurun_out/g104.log
