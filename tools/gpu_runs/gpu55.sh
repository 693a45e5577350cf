mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_tc -c 1 -o gpurun_out/g55_attn python tools/kbench.py attn > gpurun_out/g55.log 2>&1
