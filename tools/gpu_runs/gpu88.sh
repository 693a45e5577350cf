mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x --tb=short > gpurun_out/g88t.log 2>&1; echo "exit $?" >> gpurun_out/g88t.log
echo "== stream-K" >> gpurun_out/g88.log; timeout 300 python tools/gemm_sweep.py 1024 2048 4096 8192 >> gpurun_out/g88.log 2>&1
echo "== whole tiles" >> gpurun_out/g88.log; SP_GEMM_NO_STREAMK=1 timeout 300 python tools/gemm_sweep.py 1024 2048 4096 8192 >> gpurun_out/g88.log 2>&1
