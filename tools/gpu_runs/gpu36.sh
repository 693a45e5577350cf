mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x --tb=short > gpurun_out/g36t.log 2>&1; echo "exit $?" >> gpurun_out/g36t.log
for B in 64 1 16; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --decode-batch $B > gpurun_out/g36_b$B.log 2>&1; done
SP_DECODE_SPLITS=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --decode-batch 64 > gpurun_out/g36_b64s1.log 2>&1
