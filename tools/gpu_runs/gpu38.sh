mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x --tb=short > gpurun_out/g38t.log 2>&1; echo "exit $?" >> gpurun_out/g38t.log
for mc in 74 98 130 148 200; do
  echo "== min_ctas $mc" >> gpurun_out/g38p.log
  for s in "64 4096 4096 add" "64 28672 4096 swiglu" "64 6144 4096 bf16" "64 4096 14336 add" "1 4096 4096 add" "1 28672 4096 swiglu" "1 6144 4096 bf16" "1 4096 14336 add"; do SP_SWAP_MIN_CTAS=$mc timeout 60 python tools/swap_probe.py $s >> gpurun_out/g38p.log 2>&1; done
done
