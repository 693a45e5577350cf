# stream-K swap-AB GEMM + decode attention occupancy: parity, kernel bench, decode TPOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x --tb=short > gpurun_out/g29_kt.log 2>&1; echo "kt exit $?" >> gpurun_out/g29_kt.log
timeout 300 python tools/kbench.py gemm > gpurun_out/g29_kbench.log 2>&1
for B in 1 16 64 256; do timeout 400 python tools/decode_profile.py $B 2048 5 >> gpurun_out/g29_dec.log 2>&1; done
for S in 1 2 4; do echo "splits=$S" >> gpurun_out/g29_dec.log; SP_DECODE_SPLITS=$S timeout 400 python tools/decode_profile.py 64 2048 5 >> gpurun_out/g29_dec.log 2>&1; done
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_serving_gpu.py -q -m gpu -x --tb=short > gpurun_out/g29_et.log 2>&1; echo "et exit $?" >> gpurun_out/g29_et.log
