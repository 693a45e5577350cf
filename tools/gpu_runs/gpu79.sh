mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x --tb=short > gpurun_out/g79t.log 2>&1; echo "exit $?" >> gpurun_out/g79t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g79_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/g79_smoke.log
