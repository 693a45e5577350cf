mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_serving_gpu.py tests/test_spec_gpu.py -q -m gpu -x --tb=short > gpurun_out/g128t.log 2>&1; echo "exit $?" >> gpurun_out/g128t.log
timeout 900 python tools/serve_bench.py --out gpurun_out/g128_serve > gpurun_out/g128_serve.log 2>&1; echo "serve exit $?" >> gpurun_out/g128_serve.log
timeout 900 python tools/serve_bench.py --out gpurun_out/g128_serve_b > gpurun_out/g128_serve_b.log 2>&1; echo "serve exit $?" >> gpurun_out/g128_serve_b.log
