mkdir -p gpurun_out
echo "== default" >> gpurun_out/g59.log; timeout 300 python tools/gemm_sweep.py 1024 2048 4096 8192 >> gpurun_out/g59.log 2>&1
echo "== 1cta bn256" >> gpurun_out/g59.log; SP_GEMM_2CTA=0 timeout 300 python tools/gemm_sweep.py 1024 2048 4096 >> gpurun_out/g59.log 2>&1
echo "== bn128" >> gpurun_out/g59.log; SP_GEMM_FORCE_BN=128 SP_GEMM_2CTA=0 timeout 300 python tools/gemm_sweep.py 1024 2048 4096 >> gpurun_out/g59.log 2>&1
