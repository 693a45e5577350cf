mkdir -p gpurun_out
K='regex:(gemm|prefill|rmsnorm|rope|embed|decode|combine|splitk|argmax|gather_rows|peer|pack|add_f32)'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 300 --csv --log-file gpurun_out/g51_prefill.csv python bench.py --steps 1 --warmup 0 --no-decode --no-cpu-baseline > gpurun_out/g51_p.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/g51_decode.csv python tools/decode_profile.py 64 2048 1 > gpurun_out/g51_d.log 2>&1
