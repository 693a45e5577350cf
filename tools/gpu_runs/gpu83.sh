mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x --tb=short -k "attention" > gpurun_out/g83t.log 2>&1; echo "exit $?" >> gpurun_out/g83t.log
timeout 300 python tools/attn_sp_shapes.py > gpurun_out/g83.log 2>&1
