mkdir -p gpurun_out
timeout 300 python tools/symm_probe.py > gpurun_out/g80.log 2>&1; echo "exit $?" >> gpurun_out/g80.log
