timeout 900 python -m pytest tests/ -q -m gpu > gpurun_out/gt.log 2>&1; echo "gt exit $?" >> gpurun_out/gt.log
timeout 300 python tools/kbench.py gemm > gpurun_out/kbench.log 2>&1; echo "kb exit $?" >> gpurun_out/kbench.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
