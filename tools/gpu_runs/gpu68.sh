mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_serving_gpu.py -q -m gpu -x --tb=short > gpurun_out/g68t.log 2>&1; echo "exit $?" >> gpurun_out/g68t.log
timeout 2400 python tools/serve_bench.py --model 70b --kv-gb 26 --max-prefill-tokens 16384 --out gpurun_out/g68_serve70 > gpurun_out/g68_serve70.log 2>&1; echo "exit $?" >> gpurun_out/g68_serve70.log
