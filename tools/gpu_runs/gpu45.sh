mkdir -p gpurun_out
for cfg in "40 m" "40 n" "56 n" "64 n" "80 n"; do set -- $cfg; echo "== L2 $1 raster $2" >> gpurun_out/g45k.log; SP_GEMM_L2_MB=$1 SP_GEMM_RASTER=$2 timeout 300 python tools/kbench.py gemm 2>&1 | head -6 >> gpurun_out/g45k.log; done
