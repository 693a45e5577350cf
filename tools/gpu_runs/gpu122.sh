mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x --tb=short > gpurun_out/g122t.log 2>&1; echo "exit $?" >> gpurun_out/g122t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g122_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/g122_smoke.log
timeout 900 python bench.py > gpurun_out/g122_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|attn|prefill|rmsnorm|rope|embed|argmax|splitk|combine|peer" -c 300 --csv --log-file gpurun_out/g122_launches.csv python bench.py --steps 1 --warmup 0 --no-decode --no-cpu-baseline > /dev/null 2>&1
