mkdir -p gpurun_out
timeout 2400 python tools/serve_bench.py --model 70b --kv-gb 26 --max-prefill-tokens 16384 --out gpurun_out/g130_serve70 > gpurun_out/g130_serve70.log 2>&1; echo "exit $?" >> gpurun_out/g130_serve70.log
