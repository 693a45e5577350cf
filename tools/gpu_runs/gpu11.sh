timeout 900 python -m pytest tests/test_engine_gpu.py -q -m gpu -x > gpurun_out/et.log 2>&1; echo "et exit $?" >> gpurun_out/et.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 1200 python tools/configs_bench.py decode-sweep > gpurun_out/configs.log 2>&1; echo "cfg exit $?" >> gpurun_out/configs.log
