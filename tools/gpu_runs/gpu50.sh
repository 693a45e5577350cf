mkdir -p gpurun_out
timeout 1800 python tools/configs_bench.py all > gpurun_out/g50_cfg.log 2>&1; echo "cfg exit $?" >> gpurun_out/g50_cfg.log
timeout 1500 python tools/configs_bench.py 70b >> gpurun_out/g50_cfg.log 2>&1; echo "70b exit $?" >> gpurun_out/g50_cfg.log
timeout 900 python tools/serve_bench.py --out gpurun_out/g50_serve > gpurun_out/g50_serve.log 2>&1; echo "serve exit $?" >> gpurun_out/g50_serve.log
