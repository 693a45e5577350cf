mkdir -p gpurun_out
export SP_LIB_PATH=$PWD/paper_2507_11830_b200/libshiftpar_bx.so
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -q -m gpu --tb=line > gpurun_out/g56t.log 2>&1; echo "exit $?" >> gpurun_out/g56t.log
for i in 1 2; do timeout 300 python tools/kbench.py attn 2>&1 | head -1 >> gpurun_out/g56k.log; done
unset SP_LIB_PATH
for i in 1 2; do timeout 300 python tools/kbench.py attn 2>&1 | head -1 >> gpurun_out/g56k.log; done
