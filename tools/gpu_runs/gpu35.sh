mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x --tb=short > gpurun_out/g35t.log 2>&1; echo "exit $?" >> gpurun_out/g35t.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g35_dec.csv python tools/decode_profile.py 64 2048 1 > gpurun_out/g35_dec.log 2>&1
