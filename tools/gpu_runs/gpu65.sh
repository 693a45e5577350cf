mkdir -p gpurun_out
for i in 1 2; do for t in 1024 256 512; do SP_NORM_THREADS=$t timeout 600 python bench.py --steps 5 --warmup 3 --no-decode --no-cpu-baseline > gpurun_out/g65_t${t}_$i.log 2>&1; done; done
