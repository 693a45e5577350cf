timeout 300 python tools/kbench.py gemm > gpurun_out/kbench.log 2>&1; echo "kb exit $?" >> gpurun_out/kbench.log
timeout 1200 python tools/configs_bench.py all > gpurun_out/configs.log 2>&1; echo "cfg exit $?" >> gpurun_out/configs.log
