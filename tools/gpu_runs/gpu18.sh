timeout 600 python -m pytest tests/test_serving_gpu.py tests/test_engine_gpu.py -q -m gpu -x > gpurun_out/st.log 2>&1; echo "st exit $?" >> gpurun_out/st.log
timeout 900 python tools/serve_bench.py > gpurun_out/serve.log 2>&1; echo "serve exit $?" >> gpurun_out/serve.log
