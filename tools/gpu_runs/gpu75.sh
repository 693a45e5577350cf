mkdir -p gpurun_out
timeout 1800 python tools/configs_bench.py swiftkv > gpurun_out/g75_cfg.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:prefill_tc -c 1 -o gpurun_out/g75_attn python tools/attn_probe.py > gpurun_out/g75_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_tma -c 1 -o gpurun_out/g75_dec python tools/kbench.py attn > gpurun_out/g75_ncu2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_swap -s 3 -c 1 -o gpurun_out/g75_swap python tools/swap_probe.py 64 28672 4096 swiglu 3 > gpurun_out/g75_ncu3.log 2>&1
