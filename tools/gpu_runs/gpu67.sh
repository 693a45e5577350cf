mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x --tb=short > gpurun_out/g67t.log 2>&1; echo "exit $?" >> gpurun_out/g67t.log
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g67_$i.log 2>&1; done
timeout 600 python tools/decode_ablation.py 64 2048 base > gpurun_out/g67_abl.log 2>&1
