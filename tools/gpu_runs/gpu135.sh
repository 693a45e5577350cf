mkdir -p gpurun_out
for b in 1 8; do for f in 1 0 1 0; do echo "B $b fuse_norm $f"; SP_FUSE_NORM=$f timeout 600 python tools/decode_ablation.py $b 2048 base 2>&1 | grep TPOT; done; done > gpurun_out/g135.log
