mkdir -p gpurun_out
timeout 300 python tools/attn_sp_shapes.py > gpurun_out/g82.log 2>&1
