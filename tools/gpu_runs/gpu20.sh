timeout 300 python tools/kbench.py gemm > gpurun_out/kbench.log 2>&1; echo "kb exit $?" >> gpurun_out/kbench.log
SP_GEMM_2CTA=0 timeout 300 python tools/kbench.py gemm > gpurun_out/kbench_1cta.log 2>&1
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/gt.log 2>&1; echo "gt exit $?" >> gpurun_out/gt.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
