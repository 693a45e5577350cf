mkdir -p gpurun_out
for s in "1 28672 4096 bf16" "1 229376 512 bf16" "1 1835008 64 bf16" "64 28672 4096 bf16" "64 229376 512 bf16"; do timeout 120 python tools/swap_probe.py $s >> gpurun_out/g40p.log 2>&1; done
