mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x --tb=short -k "split_k or bitexact or swiglu" > gpurun_out/g33t.log 2>&1; echo "exit $?" >> gpurun_out/g33t.log
for lib in new old; do
  if [ $lib = old ]; then export SP_LIB_PATH=$PWD/paper_2507_11830_b200/libshiftpar_old.so; fi
  echo "== $lib" >> gpurun_out/g33p.log
  for s in "64 4096 4096 add" "64 28672 4096 swiglu" "64 6144 4096 bf16" "64 4096 14336 add" "1 4096 4096 add" "1 28672 4096 swiglu" "1 6144 4096 bf16" "1 4096 14336 add" "16 6144 4096 bf16" "128 4096 14336 add" "64 128256 4096 f32"; do timeout 60 python tools/swap_probe.py $s >> gpurun_out/g33p.log 2>&1; done
done
unset SP_LIB_PATH
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --decode-batch 64 > gpurun_out/g33_b64.log 2>&1
