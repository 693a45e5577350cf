# swap-AB decode GEMM: two CTAs per SM up to NT=64 (variant build) vs NT=32 (default), interleaved
set -e
mkdir -p gpurun_out; rm -f gpurun_out/cps_ab.txt
SP_NVCC_EXTRA=-DSWAP_CPS_MAX_NT=64 python -m paper_2507_11830_b200.build --force > /dev/null 2>&1
cp paper_2507_11830_b200/libshiftpar.so paper_2507_11830_b200/libshiftpar_cps64.so
python -m paper_2507_11830_b200.build --force > /dev/null 2>&1
for B in 64 48; do for rep in 1 2; do for v in default cps64; do
  if [ $v = cps64 ]; then L=paper_2507_11830_b200/libshiftpar_cps64.so; else L=paper_2507_11830_b200/libshiftpar.so; fi
  echo "$v rep=$rep $(SP_LIB_PATH=$PWD/$L timeout 300 python tools/decode_profile.py $B 2048 25 2>&1 | tail -1)" >> gpurun_out/cps_ab.txt
done; done; done
cat gpurun_out/cps_ab.txt
