mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g126_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/g126_smoke.log
timeout 900 python bench.py > gpurun_out/g126_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|attn|prefill|rmsnorm|rope|embed|argmax|splitk|combine|peer" -c 300 --csv --log-file gpurun_out/g126_launches.csv python bench.py --steps 1 --warmup 0 --no-decode --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm -c 129 --csv --log-file gpurun_out/g126_traffic.csv python bench.py --steps 1 --warmup 0 --no-decode --no-cpu-baseline > /dev/null 2>&1
