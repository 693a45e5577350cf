mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x --tb=short -k "split_k or swiglu or partial or rope" > gpurun_out/g93t.log 2>&1; echo "exit $?" >> gpurun_out/g93t.log
for s in "64 4096 4096 add" "64 28672 4096 swiglu" "64 6144 4096 bf16" "64 4096 14336 add" "1 4096 4096 add" "1 28672 4096 swiglu"; do timeout 60 python tools/swap_probe.py $s >> gpurun_out/g93p.log 2>&1; done
for i in 1 2; do timeout 600 python tools/decode_ablation.py 64 2048 base >> gpurun_out/g93.log 2>&1; timeout 600 python tools/decode_ablation.py 1 2048 base >> gpurun_out/g93.log 2>&1; done
