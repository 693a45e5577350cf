mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x --tb=short -k attention > gpurun_out/g70t.log 2>&1; echo "exit $?" >> gpurun_out/g70t.log
for i in 1 2; do timeout 300 python tools/kbench.py attn 2>&1 | head -1 >> gpurun_out/g70k.log; done
