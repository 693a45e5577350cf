mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu --tb=short > gpurun_out/g129t.log 2>&1; echo "exit $?" >> gpurun_out/g129t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g129_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/g129_smoke.log
timeout 900 python bench.py > gpurun_out/g129_bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/g129_ref.log 2>&1
timeout 1500 python tools/configs_bench.py decode-sweep > gpurun_out/g129_cfg.log 2>&1
