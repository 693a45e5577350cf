mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu --tb=short > gpurun_out/g138t.log 2>&1; echo "exit $?" >> gpurun_out/g138t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g138_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/g138_smoke.log
timeout 900 python bench.py > gpurun_out/g138_bench.log 2>&1
