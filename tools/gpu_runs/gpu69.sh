mkdir -p gpurun_out
SP_LIB_PATH=$PWD/paper_2507_11830_b200/libshiftpar_dbg.so ATTN_DBG=1 timeout 120 python tools/attn_probe.py > gpurun_out/g69.log 2>&1
