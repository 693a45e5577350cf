# decode sweeps at HEAD: B=256 swap split target (NT=256), B=16/32 KV splits; interleaved
mkdir -p gpurun_out; rm -f gpurun_out/misc_ab.txt
for rep in 1 2; do for t in 118 104 133 148; do
  echo "B256 min_ctas=$t rep=$rep $(SP_SWAP_MIN_CTAS=$t timeout 300 python tools/decode_profile.py 256 2048 20 2>&1 | tail -1)" >> gpurun_out/misc_ab.txt
done; done
for rep in 1 2; do for t in 2 1 3 4; do
  echo "B16 splits=$t rep=$rep $(SP_DECODE_SPLITS=$t timeout 300 python tools/decode_profile.py 16 2048 25 2>&1 | tail -1)" >> gpurun_out/misc_ab.txt
done; done
for rep in 1 2; do for t in 1 2; do
  echo "B32 splits=$t rep=$rep $(SP_DECODE_SPLITS=$t timeout 300 python tools/decode_profile.py 32 2048 25 2>&1 | tail -1)" >> gpurun_out/misc_ab.txt
done; done
cat gpurun_out/misc_ab.txt
