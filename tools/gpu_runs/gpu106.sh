mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g106_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/g106_smoke.log
timeout 900 python bench.py > gpurun_out/g106_bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/g106_ref.log 2>&1
timeout 1500 python tools/configs_bench.py decode-sweep > gpurun_out/g106_cfg.log 2>&1
