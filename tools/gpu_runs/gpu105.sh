mkdir -p gpurun_out
for f in 0 1; do for b in 64 256; do echo "fuse $f B $b"; SP_FUSE_SPLITK=$f timeout 600 python tools/decode_ablation.py $b 2048 base 2>&1 | grep TPOT; done; done > gpurun_out/g105.log
