mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x --tb=short > gpurun_out/g46t.log 2>&1; echo "exit $?" >> gpurun_out/g46t.log
for s in "64 4096 4096 add" "64 28672 4096 swiglu" "64 6144 4096 bf16" "64 4096 14336 add" "1 4096 4096 add" "1 28672 4096 swiglu" "1 6144 4096 bf16" "1 4096 14336 add" "128 4096 14336 add" "64 28672 4096 bf16"; do timeout 60 python tools/swap_probe.py $s >> gpurun_out/g46p.log 2>&1; done
for B in 64 1; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --decode-batch $B > gpurun_out/g46_b$B.log 2>&1; done
