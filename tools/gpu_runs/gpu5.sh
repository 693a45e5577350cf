timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/gt.log 2>&1; echo "gt exit $?" >> gpurun_out/gt.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_kernel|prefill|decode_kernel|rope_kv|add_rmsnorm|embed_kernel|combine|gather_rows|argmax" -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-decode --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_bench.log
