mkdir -p gpurun_out
(echo default; timeout 300 python tools/gemm_sweep.py 1024 2048 4096;
 echo 1cta_bn256; SP_GEMM_2CTA=0 timeout 300 python tools/gemm_sweep.py 1024 2048 4096;
 echo bn128; SP_GEMM_FORCE_BN=128 timeout 300 python tools/gemm_sweep.py 1024 2048 4096;
 echo bn64; SP_GEMM_FORCE_BN=64 timeout 300 python tools/gemm_sweep.py 1024 2048) > gpurun_out/g113.log 2>&1
