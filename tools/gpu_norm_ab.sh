mkdir -p gpurun_out; rm -f gpurun_out/norm_ab.txt
for B in 1 8; do for rep in 1 2; do for t in 1024 512 256; do
  echo "threads=$t rep=$rep $(SP_NORM_THREADS=$t timeout 300 python tools/decode_profile.py $B 2048 25 2>&1 | tail -1)" >> gpurun_out/norm_ab.txt
done; done; done
cat gpurun_out/norm_ab.txt
