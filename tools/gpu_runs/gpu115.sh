mkdir -p gpurun_out
(echo default; timeout 300 python tools/gemm_sweep.py 512 1024 1536;
 echo force256; SP_GEMM_FORCE_BN=256 timeout 300 python tools/gemm_sweep.py 512 1024 1536) > gpurun_out/g115.log 2>&1
