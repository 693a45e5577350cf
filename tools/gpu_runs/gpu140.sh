mkdir -p gpurun_out
for b in 1 16; do for v in 0 2 4 6 12; do echo "B $b splits $v"; if [ $v = 0 ]; then timeout 600 python tools/decode_ablation.py $b 2048 base 2>&1 | grep TPOT; else SP_DECODE_SPLITS=$v timeout 600 python tools/decode_ablation.py $b 2048 base 2>&1 | grep TPOT; fi; done; done > gpurun_out/g140.log
