mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x --tb=short > gpurun_out/g91t.log 2>&1; echo "exit $?" >> gpurun_out/g91t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g91_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/g91_smoke.log
timeout 900 python bench.py > gpurun_out/g91_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_tc -c 1 -o gpurun_out/g91_attn python tools/attn_probe.py > gpurun_out/g91_ncu.log 2>&1
