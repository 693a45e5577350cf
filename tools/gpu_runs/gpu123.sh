mkdir -p gpurun_out
for w in 1 1.5 2; do SP_ATTN_SPLIT_WAVES=$w timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"prefill" -c 4 --csv --log-file gpurun_out/g123_$w.csv python tools/attn_sp_shapes.py 8 > /dev/null 2>&1; done
