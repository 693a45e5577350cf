mkdir -p gpurun_out
for M in 1024 2048; do
timeout 600 ncu --set full --clock-control none -k regex:gemm -s 2 -c 1 -o gpurun_out/g114_down_$M python tools/gemm_one.py $M 4096 14336 add > /dev/null 2>&1
done
