mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x --tb=short > gpurun_out/g118t.log 2>&1; echo "exit $?" >> gpurun_out/g118t.log
