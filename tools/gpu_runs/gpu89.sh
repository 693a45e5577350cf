mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x --tb=short -k "attention" > gpurun_out/g89t.log 2>&1; echo "exit $?" >> gpurun_out/g89t.log
for i in 1 2 3; do timeout 120 python tools/kbench.py attn 2>&1 | head -1 >> gpurun_out/g89k.log; done
timeout 300 python tools/attn_sp_shapes.py >> gpurun_out/g89k.log 2>&1
