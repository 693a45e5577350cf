mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x --tb=short > gpurun_out/g52t.log 2>&1; echo "exit $?" >> gpurun_out/g52t.log
for B in 64 1; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --decode-batch $B > gpurun_out/g52_b$B.log 2>&1; done
