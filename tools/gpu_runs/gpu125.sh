mkdir -p gpurun_out
for f in 1 0 1 0; do echo "fuse_rope $f"; SP_FUSE_ROPE=$f timeout 600 python bench.py --no-decode --no-cpu-baseline --steps 6 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'], d['gpu_launches'])"; done > gpurun_out/g125.log 2>&1
