mkdir -p gpurun_out
for s in "64 28672 4096 bf16" "64 28672 4096 f32" "64 28672 4096 gelu" "64 28672 4096 swiglu" "48 28672 4096 bf16" "32 28672 4096 bf16" "64 6144 4096 bf16" "64 6144 4096 f32" "64 14336 4096 bf16" "64 14336 4096 swiglu"; do timeout 120 python tools/swap_probe.py $s >> gpurun_out/g42p.log 2>&1; done
