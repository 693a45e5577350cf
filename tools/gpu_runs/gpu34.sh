mkdir -p gpurun_out
for B in 64 1 16; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --decode-batch $B > gpurun_out/g34_b$B.log 2>&1; done
