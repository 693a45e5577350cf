mkdir -p gpurun_out
for n in p8 p4 p6 p10 p12 p8; do
  export SP_LIB_PATH=$PWD/paper_2507_11830_b200/libshiftpar_$n.so
  echo "== $n" >> gpurun_out/g72k.log
  for i in 1 2; do timeout 300 python tools/kbench.py attn 2>&1 | head -1 >> gpurun_out/g72k.log; done
done
