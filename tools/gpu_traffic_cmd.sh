set -x
mkdir -p gpurun_out/traffic
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv"
for v in 40 64 80 100; do
  SP_GEMM_L2_MB=$v timeout 300 python tools/gemm_sweep.py 8192 4096 > gpurun_out/traffic/sweep_l2_$v.txt 2>&1
  SP_GEMM_L2_MB=$v timeout 300 ncu $M -k regex:gemm --log-file gpurun_out/traffic/ncu_l2_$v.csv python tools/gemm_traffic.py 8192 > gpurun_out/traffic/alg_l2_$v.txt 2>&1
done
for r in m n; do
  SP_GEMM_RASTER=$r timeout 300 python tools/gemm_sweep.py 8192 > gpurun_out/traffic/sweep_r$r.txt 2>&1
  SP_GEMM_RASTER=$r timeout 300 ncu $M -k regex:gemm --log-file gpurun_out/traffic/ncu_r$r.csv python tools/gemm_traffic.py 8192 > gpurun_out/traffic/alg_r$r.txt 2>&1
done
