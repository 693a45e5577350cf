# decode swap-AB GEMM split target (SP_SWAP_MIN_CTAS) at B=1 and B=8, interleaved
mkdir -p gpurun_out; rm -f gpurun_out/swap_ab.txt
for B in 1 8 32; do for rep in 1 2; do for t in 148 180 192 224 260; do
  echo "min_ctas=$t rep=$rep $(SP_SWAP_MIN_CTAS=$t timeout 300 python tools/decode_profile.py $B 2048 25 2>&1 | tail -1)" >> gpurun_out/swap_ab.txt
done; done; done
cat gpurun_out/swap_ab.txt
