mkdir -p gpurun_out
for i in 1 2; do timeout 300 python tools/kbench.py attn 2>&1 | head -1 >> gpurun_out/g58k.log; done
export SP_LIB_PATH=$PWD/paper_2507_11830_b200/libshiftpar_x1.so
for i in 1 2; do timeout 300 python tools/kbench.py attn 2>&1 | head -1 >> gpurun_out/g58k.log; done
