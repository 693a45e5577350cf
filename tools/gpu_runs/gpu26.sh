timeout 1500 python tools/configs_bench.py 70b > gpurun_out/c70.log 2>&1; echo "exit $?" >> gpurun_out/c70.log
