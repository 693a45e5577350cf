mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x --tb=short > gpurun_out/g73t.log 2>&1; echo "exit $?" >> gpurun_out/g73t.log
for i in 1 2; do timeout 300 python tools/kbench.py attn 2>&1 | head -1 >> gpurun_out/g73k.log; done
timeout 900 python bench.py > gpurun_out/g73_bench.log 2>&1
