mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x --tb=short -k "split_k or bitexact or swiglu" > gpurun_out/g31t.log 2>&1; echo "exit $?" >> gpurun_out/g31t.log
SP_SWAP_DEBUG=1 timeout 60 python tools/swap_probe.py 64 4096 4096 add 1 > gpurun_out/g31.log 2>&1
SP_SWAP_DEBUG=1 timeout 60 python tools/swap_probe.py 64 28672 4096 swiglu 1 > gpurun_out/g31b.log 2>&1
for s in "64 4096 4096 add" "64 28672 4096 swiglu" "64 6144 4096 bf16" "64 4096 14336 add" "1 4096 4096 add" "1 28672 4096 swiglu" "16 6144 4096 bf16" "128 4096 14336 add" "64 128256 4096 f32"; do timeout 60 python tools/swap_probe.py $s >> gpurun_out/g31p.log 2>&1; done
