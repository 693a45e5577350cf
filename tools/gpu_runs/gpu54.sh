mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x --tb=short -k attention > gpurun_out/g54t.log 2>&1; echo "exit $?" >> gpurun_out/g54t.log
for n in 12 0 8 16 20; do
  if [ $n = 12 ]; then unset SP_LIB_PATH; else export SP_LIB_PATH=$PWD/paper_2507_11830_b200/libshiftpar_p$n.so; fi
  echo "== poly pairs $n" >> gpurun_out/g54k.log
  for i in 1 2; do timeout 300 python tools/kbench.py attn 2>&1 | head -1 >> gpurun_out/g54k.log; done
done
