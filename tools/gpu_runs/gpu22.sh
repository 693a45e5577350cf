timeout 300 python tools/kbench.py gemm > gpurun_out/kbench.log 2>&1; echo "kb exit $?" >> gpurun_out/kbench.log
