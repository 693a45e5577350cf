mkdir -p gpurun_out
for mb in 16 24 40; do
SP_GEMM_L2_MB=$mb timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm -c 129 --csv --log-file gpurun_out/g110_l2_$mb.csv python bench.py --steps 1 --warmup 0 --no-decode --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/g110_l2_$mb.csv "L2 $mb" > gpurun_out/g110_l2_$mb.json
done
