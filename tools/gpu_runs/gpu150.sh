mkdir -p gpurun_out
for v in 1 0; do for b in 1 64; do echo "pdl $v B $b"; SP_PDL=$v timeout 600 python tools/decode_ablation.py $b 2048 base 2>&1 | grep TPOT; done; done > gpurun_out/g150.log
