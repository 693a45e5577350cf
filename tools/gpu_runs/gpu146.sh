mkdir -p gpurun_out
for t in 256 512 256 512 1024; do echo "norm_threads $t"; SP_NORM_THREADS=$t timeout 600 python bench.py --no-decode --no-cpu-baseline --steps 6 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'])"; done > gpurun_out/g146.log 2>&1
