mkdir -p gpurun_out
for b in 4 8 32; do for v in 0 1 2 3 4; do echo "B $b splits $v"; if [ $v = 0 ]; then timeout 600 python tools/decode_ablation.py $b 2048 base 2>&1 | grep TPOT; else SP_DECODE_SPLITS=$v timeout 600 python tools/decode_ablation.py $b 2048 base 2>&1 | grep TPOT; fi; done; done > gpurun_out/g141.log
for v in 0 1 2; do echo "B 16 splits $v"; if [ $v = 0 ]; then timeout 600 python tools/decode_ablation.py 16 2048 base 2>&1 | grep TPOT; else SP_DECODE_SPLITS=$v timeout 600 python tools/decode_ablation.py 16 2048 base 2>&1 | grep TPOT; fi; done >> gpurun_out/g141.log
