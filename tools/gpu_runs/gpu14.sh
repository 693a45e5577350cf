timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/gt.log 2>&1; echo "gt exit $?" >> gpurun_out/gt.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
SP_PDL=0 timeout 900 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_nopdl.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_nopdl.log
