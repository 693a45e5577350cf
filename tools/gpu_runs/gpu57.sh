mkdir -p gpurun_out
for i in 1 2; do for f in 1 0; do SP_FUSE_SPLITK=$f timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --decode-batch 64 > gpurun_out/g57_f${f}_$i.log 2>&1; done; done
for i in 1 2; do for f in 1 0; do SP_FUSE_SPLITK=$f timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --decode-batch 1 > gpurun_out/g57_b1_f${f}_$i.log 2>&1; done; done
