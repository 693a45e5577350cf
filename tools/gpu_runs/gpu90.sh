mkdir -p gpurun_out
for n in main p0 p6 p8 main; do
  if [ $n = main ]; then unset SP_LIB_PATH; else export SP_LIB_PATH=$PWD/paper_2507_11830_b200/libshiftpar_$n.so; fi
  echo "== $n" >> gpurun_out/g90k.log
  for i in 1 2; do timeout 120 python tools/kbench.py attn 2>&1 | head -1 >> gpurun_out/g90k.log; done
done
