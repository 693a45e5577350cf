mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/g86_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g86_ref.log 2>&1
timeout 2400 python tools/configs_bench.py all > gpurun_out/g86_cfg.log 2>&1; echo "cfg exit $?" >> gpurun_out/g86_cfg.log
timeout 1500 python tools/configs_bench.py 70b >> gpurun_out/g86_cfg.log 2>&1; echo "70b exit $?" >> gpurun_out/g86_cfg.log
timeout 900 python tools/serve_bench.py --out gpurun_out/g86_serve > gpurun_out/g86_serve.log 2>&1; echo "serve exit $?" >> gpurun_out/g86_serve.log
