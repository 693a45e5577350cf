timeout 600 python tools/decode_profile.py 64 2048 5 > gpurun_out/dp.log 2>&1
timeout 600 python tools/decode_profile.py 1 2048 5 >> gpurun_out/dp.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"gemm|attn|decode|rope|rmsnorm|embed|combine|gather|argmax|splitk" --csv --log-file gpurun_out/dec_launches.csv python tools/decode_profile.py 64 2048 1 > gpurun_out/ncu_dec.log 2>&1; echo "exit $?" >> gpurun_out/ncu_dec.log
