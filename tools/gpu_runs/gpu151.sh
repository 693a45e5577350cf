mkdir -p gpurun_out
for v in base poly base poly; do echo "$v"; if [ $v = poly ]; then export SP_LIB_PATH=$PWD/paper_2507_11830_b200/libshiftpar_poly.so; else unset SP_LIB_PATH; fi; timeout 600 python bench.py --no-decode --no-cpu-baseline --steps 6 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'], d['attention']['achieved_tflops'])"; done > gpurun_out/g151.log 2>&1
