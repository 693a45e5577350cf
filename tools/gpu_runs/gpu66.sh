mkdir -p gpurun_out
for t in 512 1024 256 512; do echo "threads $t" >> gpurun_out/g66.log; SP_NORM_THREADS=$t timeout 600 python tools/decode_ablation.py 64 2048 base >> gpurun_out/g66.log 2>&1; done
