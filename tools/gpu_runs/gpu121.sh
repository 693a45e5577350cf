mkdir -p gpurun_out
for w in 1 1.5 1.25 1 1.5 1.25 1.75; do echo "waves $w"; SP_ATTN_SPLIT_WAVES=$w timeout 300 python tools/attn_sp_shapes.py 8; done > gpurun_out/g121.log 2>&1
