mkdir -p gpurun_out
timeout 900 python tools/serve_bench.py --out gpurun_out/g127_serve > gpurun_out/g127_serve.log 2>&1; echo "serve exit $?" >> gpurun_out/g127_serve.log
timeout 2400 python tools/serve_bench.py --model 70b --kv-gb 26 --max-prefill-tokens 16384 --out gpurun_out/g127_serve70 > gpurun_out/g127_serve70.log 2>&1; echo "exit $?" >> gpurun_out/g127_serve70.log
timeout 1500 python tools/configs_bench.py 70b > gpurun_out/g127_70b.log 2>&1; echo "70b exit $?" >> gpurun_out/g127_70b.log
timeout 1500 python tools/configs_bench.py swiftkv > gpurun_out/g127_skv.log 2>&1; echo "skv exit $?" >> gpurun_out/g127_skv.log
