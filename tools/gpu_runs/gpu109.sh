mkdir -p gpurun_out
for mb in 40 24 64 40; do echo "L2 $mb"; SP_GEMM_L2_MB=$mb timeout 600 python bench.py --no-decode --no-cpu-baseline --steps 6 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"; done > gpurun_out/g109.log 2>&1
