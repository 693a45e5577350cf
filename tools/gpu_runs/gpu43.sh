mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/g43_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g43_launches.csv python bench.py --steps 1 --warmup 0 --no-decode --no-cpu-baseline > gpurun_out/g43_l.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm -c 129 --csv --log-file gpurun_out/g43_traffic.csv python bench.py --steps 1 --warmup 0 --no-decode --no-cpu-baseline > gpurun_out/g43_t.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_swap -s 3 -c 1 -o gpurun_out/g43_swap python tools/swap_probe.py 64 28672 4096 swiglu 3 > gpurun_out/g43_s.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_tma -s 40 -c 1 -o gpurun_out/g43_dec python tools/decode_profile.py 64 2048 1 > gpurun_out/g43_d.log 2>&1
