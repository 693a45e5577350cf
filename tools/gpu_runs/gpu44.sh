mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x --tb=short > gpurun_out/g44t.log 2>&1; echo "exit $?" >> gpurun_out/g44t.log
for mb in 40 64 96; do echo "== L2 $mb" >> gpurun_out/g44k.log; SP_GEMM_L2_MB=$mb timeout 300 python tools/kbench.py gemm 2>&1 | head -6 >> gpurun_out/g44k.log; done
for mb in 40 64; do SP_GEMM_L2_MB=$mb timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm -c 8 --csv --log-file gpurun_out/g44_tr$mb.csv python bench.py --steps 1 --warmup 0 --no-decode --no-cpu-baseline > /dev/null 2>&1; done
