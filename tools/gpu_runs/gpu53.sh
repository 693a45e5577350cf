mkdir -p gpurun_out
for lib in main var; do
  if [ $lib = var ]; then export SP_LIB_PATH=$PWD/paper_2507_11830_b200/libshiftpar_var.so; fi
  echo "== $lib" >> gpurun_out/g53p.log
  for s in "64 4096 4096 add" "64 28672 4096 swiglu" "64 6144 4096 bf16" "64 4096 14336 add" "48 28672 4096 swiglu" "64 128256 4096 f32"; do timeout 60 python tools/swap_probe.py $s >> gpurun_out/g53p.log 2>&1; done
done
unset SP_LIB_PATH
SP_LIB_PATH=$PWD/paper_2507_11830_b200/libshiftpar_var.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --decode-batch 64 > gpurun_out/g53_var.log 2>&1
