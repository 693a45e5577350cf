mkdir -p gpurun_out
for s in 0 4 3 6 0; do echo "splits $s" >> gpurun_out/g92.log; if [ $s = 0 ]; then unset SP_DECODE_SPLITS; else export SP_DECODE_SPLITS=$s; fi; timeout 600 python tools/decode_ablation.py 64 2048 base >> gpurun_out/g92.log 2>&1; done
