mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prefill" --csv --log-file gpurun_out/g84.csv python tools/attn_sp_shapes.py 8 > gpurun_out/g84.log 2>&1
