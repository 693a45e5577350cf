# decode swap-AB split target at one CTA per SM (M > 32): B=64 and B=128, interleaved
mkdir -p gpurun_out; rm -f gpurun_out/swap64_ab.txt
for B in 64 48; do for rep in 1 2; do for t in 118 88 96 104 112; do
  echo "B$B min_ctas=$t rep=$rep $(SP_SWAP_MIN_CTAS=$t timeout 300 python tools/decode_profile.py $B 2048 25 2>&1 | tail -1)" >> gpurun_out/swap64_ab.txt
done; done; done
cat gpurun_out/swap64_ab.txt
