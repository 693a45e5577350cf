mkdir -p gpurun_out
for w in 1 1.5 2 3 4; do echo "waves $w"; SP_ATTN_SPLIT_WAVES=$w timeout 300 python tools/attn_sp_shapes.py 8; done > gpurun_out/g120.log 2>&1
