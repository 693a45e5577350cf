mkdir -p gpurun_out
for v in 48 64 96 148; do echo "min_ctas $v"; SP_SWAP_MIN_CTAS=$v timeout 300 python tools/decode_ablation.py 64 2048 base 2>&1 | grep TPOT; done > gpurun_out/g100.log
for v in 256 512; do echo "norm_threads $v"; SP_NORM_THREADS=$v timeout 300 python tools/decode_ablation.py 64 2048 base 2>&1 | grep TPOT; done >> gpurun_out/g100.log
echo "default"; timeout 300 python tools/decode_ablation.py 64 2048 base 2>&1 | grep TPOT >> gpurun_out/g100.log
