# decode attention KV splits (SP_DECODE_SPLITS, tuning override) at B=1 and B=8, interleaved
mkdir -p gpurun_out; rm -f gpurun_out/dsplit_ab.txt
for rep in 1 2; do for t in 8 4 6 12 16; do
  echo "B1 splits=$t rep=$rep $(SP_DECODE_SPLITS=$t timeout 300 python tools/decode_profile.py 1 2048 25 2>&1 | tail -1)" >> gpurun_out/dsplit_ab.txt
done; done
for rep in 1 2; do for t in 4 2 3 6 8; do
  echo "B8 splits=$t rep=$rep $(SP_DECODE_SPLITS=$t timeout 300 python tools/decode_profile.py 8 2048 25 2>&1 | tail -1)" >> gpurun_out/dsplit_ab.txt
done; done
cat gpurun_out/dsplit_ab.txt
