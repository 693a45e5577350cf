mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x --tb=short > gpurun_out/g64t.log 2>&1; echo "exit $?" >> gpurun_out/g64t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g64_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/g64_smoke.log
timeout 900 python bench.py > gpurun_out/g64_bench.log 2>&1
timeout 1800 python tools/configs_bench.py decode-sweep > gpurun_out/g64_cfg.log 2>&1
